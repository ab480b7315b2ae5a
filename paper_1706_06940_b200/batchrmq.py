"""Host-side mirror of the reference ``batchrmq`` operator API over the C-ABI.

Names, argument meaning and error behaviour follow the reference
(/root/reference/proj/core/include/batchrmq/*.hpp and SPEC.md); every call
goes through libbrmq.so into the sm_100a kernels -- nothing here computes an
answer on the CPU.

    reference (C++)                                   here
    ------------------------------------------------  -------------------------------------------
    Query{left,right} (types.hpp:13-23)                QUERY_DTYPE / make_queries()
    collect_endpoints (contraction.hpp:51)             collect_endpoints(batch)
    sort_endpoints(eps, SortKind) (:55)                sort_endpoints(eps, kind)
    build_contracted(values, eps, threads) (:61-64)    build_contracted(values, eps)
    remap_queries_from_sorted(eps, c, q) (:71-73)      remap_queries_from_sorted(eps, c, q)
    floor_log2 (bits.hpp:10-13)                        floor_log2(x)
    build_block_sparse(values, k)        build_block_sparse(values, k)
    solve_batch_bbst(array, batch, [k])  solve_batch_bbst(array, batch, k)
    solve_batch_bbst_con(array, batch, params) (:237)  solve_batch_bbst_con(array, batch, k, sort_kind)

Exceptions mirror the reference's std:: classes: DomainError (domain_error),
OutOfRange (out_of_range), InvalidArgument (invalid_argument), LogicError
(logic_error); CudaError has no reference counterpart.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass

import numpy as np

from . import _lib

# == batchrmq::Query: 16 B, left @0, right @8
QUERY_DTYPE = np.dtype([("left", "<u8"), ("right", "<u8")])
# == batchrmq::Endpoint: 8 B, pos @0, origin @4
ENDPOINT_DTYPE = np.dtype([("pos", "<u4"), ("origin", "<u4")])

PTR_HOST, PTR_DEVICE = 0, 1


class SortKind(enum.IntEnum):  # contraction.hpp:23 (+ BITMAP: device presence-bit sort)
    Radix = 0
    Comparison = 1
    Bitmap = 2


class BrmqError(Exception):
    pass


class DomainError(BrmqError, ArithmeticError):
    pass


class OutOfRange(BrmqError, IndexError):
    pass


class InvalidArgument(BrmqError, ValueError):
    pass


class LogicError(BrmqError, RuntimeError):
    pass


class CudaError(BrmqError, RuntimeError):
    pass


_CODES = {1: DomainError, 2: OutOfRange, 3: InvalidArgument, 4: LogicError, 5: CudaError,
          6: MemoryError, 7: OSError}


def _check(rc: int) -> None:
    if rc != 0:
        msg = _lib.lib().brmq_last_error().decode(errors="replace")
        raise _CODES.get(rc, BrmqError)(msg)


def make_queries(left, right) -> np.ndarray:
    """QueryBatch from endpoint arrays; reversed pairs are swapped (types.hpp:18-20)."""
    left = np.asarray(left, dtype=np.uint64)
    right = np.asarray(right, dtype=np.uint64)
    q = np.empty(left.shape[0], dtype=QUERY_DTYPE)
    q["left"] = np.minimum(left, right)
    q["right"] = np.maximum(left, right)
    return q


def _as_queries(batch) -> np.ndarray:
    a = np.asarray(batch)
    if a.dtype == QUERY_DTYPE:
        return np.ascontiguousarray(a)
    a = np.ascontiguousarray(a, dtype=np.uint64).reshape(-1, 2)
    return a.view(QUERY_DTYPE).reshape(-1)


def _ptr(a) -> int:
    return a.ctypes.data if a.size else 0


def _is_cuda_tensor(x) -> bool:
    return hasattr(x, "is_cuda") and bool(getattr(x, "is_cuda"))


@dataclass
class ContractedArray:  # contraction.hpp:28-34
    aq_values: np.ndarray  # int32, |boundary| - 1
    aq_origin: np.ndarray  # uint64
    boundary: np.ndarray   # uint64

    def size(self) -> int:
        return int(self.aq_values.shape[0])


@dataclass
class ContractedQueryBatch:  # contraction.hpp:39-45 (struct-of-arrays)
    cleft: np.ndarray
    cright: np.ndarray
    degenerate: np.ndarray


class Engine:
    """One device context (stream + grow-only workspace), == brmq_ctx."""

    def __init__(self, device: int = 0):
        self._L = _lib.lib()
        h = C.c_void_p()
        _check(self._L.brmq_ctx_create(C.byref(h), int(device)))
        self._h = h
        self.device = device

    def close(self) -> None:
        if getattr(self, "_h", None):
            self._L.brmq_ctx_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def set_timing(self, level: int = 1) -> None:
        """0 off, 1 every stage, 2 only the roofline kernel (see brmq.h)."""
        _check(self._L.brmq_ctx_set_timing(self._h, int(level)))

    def set_stream(self, stream_ptr: int | None) -> None:
        _check(self._L.brmq_ctx_set_stream(self._h, stream_ptr or None))

    def set_async(self, enable: bool = True) -> None:
        """Device-pointer BbST / [32, k] / BbST_CON solves return once enqueued;
        synchronize() waits and raises what the solve would have raised (brmq.h)."""
        _check(self._L.brmq_ctx_set_async(self._h, int(bool(enable))))

    def synchronize(self) -> None:
        """Wait for the context stream; raises the status of an outstanding async solve."""
        _check(self._L.brmq_synchronize(self._h))

    def set_counters(self, enable: bool = True) -> None:
        """Debug scan-cell counter of BbST (h = 1) solves (solve_info()["scanned_cells"])."""
        _check(self._L.brmq_ctx_set_counters(self._h, int(bool(enable))))

    def stage_times(self) -> list[tuple[str, float, int]]:
        t = _lib.StageTimes()
        _check(self._L.brmq_last_stage_times(self._h, C.byref(t)))
        return [(bytes(t.name[i]).split(b"\0")[0].decode(), float(t.ms[i]), int(t.launches[i]))
                for i in range(t.count)]

    def solve_info(self) -> dict:
        s = _lib.SolveInfo()
        _check(self._L.brmq_last_solve_info(self._h, C.byref(s)))
        return {f: int(getattr(s, f)) for f, _ in _lib.SolveInfo._fields_}

    # ---------------------------------------------------------------- solves
    def solve_batch_bbst(self, array, batch, k: int = 512, out=None):
        """SPEC.md:302-310, BbST with one level."""
        return self._solve(False, array, batch, k, 0, out)

    def solve_batch_bbst_ml(self, array, batch, ks=(32, 512), out=None):
        """SPEC.md:266-310 with LevelConfig ks: any dividing chain k_1 < ... < k_h, h <= 8."""
        return self._solve("ml", array, batch, tuple(int(x) for x in ks), 0, out)

    def solve_batch_bbst_con(self, array, batch, k: int = 512,
                             sort_kind: SortKind = SortKind.Radix, out=None):
        """SPEC.md:237-245, BbST_CON."""
        return self._solve(True, array, batch, k, int(sort_kind), out)

    def _shard(self, fn, shard, batch, offset, n_total, extra, out):
        if _is_cuda_tensor(shard):
            import torch
            ns, q = shard.numel(), batch.numel() // 2
            if out is None:
                out = torch.empty(q, dtype=torch.int64, device=shard.device)
            a, b, o, flags = shard.data_ptr(), batch.data_ptr(), out.data_ptr(), PTR_DEVICE
        else:
            shard = np.ascontiguousarray(shard, dtype=np.int32)
            batch = _as_queries(batch)
            ns, q = shard.shape[0], batch.shape[0]
            if out is None:
                out = np.empty(q, dtype=np.uint64)
            a, b, o, flags = _ptr(shard), _ptr(batch), _ptr(out), PTR_HOST
        _check(fn(self._h, a, ns, int(offset), int(n_total), b, q, *extra, o, flags))
        return out

    def solve_batch_bbst_shard(self, shard, batch, offset: int, n_total: int, k: int = 512,
                               out=None):
        """Packed keys of every query restricted to A[offset, offset + len(shard)) with
        global positions (UINT64_MAX when the query misses the shard); the min over
        shards is the answer's key (include/brmq.h brmq_solve_bbst_shard)."""
        return self._shard(self._L.brmq_solve_bbst_shard, shard, batch, offset, n_total,
                           (int(k),), out)

    def solve_batch_bbst_con_shard(self, shard, batch, offset: int, n_total: int, k: int = 512,
                                   sort_kind: SortKind = SortKind.Radix, out=None):
        """The contraction variant of solve_batch_bbst_shard: the shard is contracted with
        its own endpoints plus the borders of the queries crossing it
        (include/brmq.h brmq_solve_bbst_con_shard)."""
        return self._shard(self._L.brmq_solve_bbst_con_shard, shard, batch, offset, n_total,
                           (int(k), int(sort_kind)), out)

    def solve_batch_naive(self, array, batch, out=None):
        """naive.hpp:13-21 for every query (the harness's "naive"), on the device."""
        return self._solve("naive", array, batch, 1, 0, out)

    def solve_batch_st_rmq_con(self, array, batch, out=None):
        """SPEC.md:331-377, the ST-RMQ_CON baseline (section 2)."""
        return self._solve("st", array, batch, 1, 0, out)

    def _solve(self, con, array, batch, k, sort_kind: int, out):
        if _is_cuda_tensor(array):  # device-resident inputs (torch CUDA tensors)
            import torch
            assert array.dtype == torch.int32 and array.is_contiguous()
            assert batch.dtype in (torch.int64, torch.uint64) and batch.is_contiguous()
            n, q = array.numel(), batch.numel() // 2
            if out is None:
                out = torch.empty(q, dtype=torch.int64, device=array.device)
            a, b, o, flags = array.data_ptr(), batch.data_ptr(), out.data_ptr(), PTR_DEVICE
        else:
            array = np.ascontiguousarray(array, dtype=np.int32)
            batch = _as_queries(batch)
            n, q = array.shape[0], batch.shape[0]
            if out is None:
                out = np.empty(q, dtype=np.uint64)
            a, b, o, flags = _ptr(array), _ptr(batch), _ptr(out), PTR_HOST
        if con == "naive":
            rc = self._L.brmq_solve_naive(self._h, a, n, b, q, o, flags)
        elif con == "st":
            rc = self._L.brmq_solve_st_rmq_con(self._h, a, n, b, q, o, flags)
        elif con == "ml":
            ks = (C.c_uint32 * len(k))(*k)
            rc = self._L.brmq_solve_bbst_ml(self._h, a, n, b, q, ks, len(k), o, flags)
        elif con:
            rc = self._L.brmq_solve_bbst_con(self._h, a, n, b, q, int(k), sort_kind, o, flags)
        else:
            rc = self._L.brmq_solve_bbst(self._h, a, n, b, q, int(k), o, flags)
        _check(rc)
        return out

    # ---------------------------------------------------------------- stages
    def collect_endpoints(self, batch) -> np.ndarray:
        batch = _as_queries(batch)
        eps = np.empty(2 * batch.shape[0], dtype=ENDPOINT_DTYPE)
        _check(self._L.brmq_collect_endpoints(self._h, _ptr(batch), batch.shape[0], _ptr(eps), 0))
        return eps

    def sort_endpoints(self, eps: np.ndarray, kind: SortKind = SortKind.Radix) -> np.ndarray:
        """In place (like the reference), also returned for convenience."""
        assert eps.dtype == ENDPOINT_DTYPE and eps.flags.c_contiguous
        _check(self._L.brmq_sort_endpoints(self._h, _ptr(eps), eps.shape[0], int(kind), 0))
        return eps

    def build_contracted(self, values, sorted_eps: np.ndarray, stats: dict | None = None) -> ContractedArray:
        """contraction.hpp:61-64; `stats` (ContractionStats, :47-49) gets
        stats["array_reads"] += the positions of `values` the device consumed."""
        values = np.ascontiguousarray(values, dtype=np.int32)
        m = sorted_eps.shape[0]
        aqv = np.empty(max(m, 1), dtype=np.int32)
        aqo = np.empty(max(m, 1), dtype=np.uint64)
        bnd = np.empty(max(m, 1), dtype=np.uint64)
        nb = C.c_uint64(0)
        reads = C.c_uint64(0)
        _check(self._L.brmq_build_contracted_stats(self._h, _ptr(values), values.shape[0],
                                                   _ptr(sorted_eps), m, _ptr(aqv), _ptr(aqo), _ptr(bnd),
                                                   C.byref(nb), 0, C.byref(reads)))
        if stats is not None:
            stats["array_reads"] = stats.get("array_reads", 0) + int(reads.value)
        nbv = int(nb.value)
        areas = max(nbv - 1, 0)
        return ContractedArray(aqv[:areas].copy(), aqo[:areas].copy(), bnd[:nbv].copy())

    def remap_queries_from_sorted(self, sorted_eps: np.ndarray, contracted: ContractedArray,
                                  query_count: int) -> ContractedQueryBatch:
        b = np.ascontiguousarray(contracted.boundary, dtype=np.uint64)
        cl = np.zeros(query_count, dtype=np.uint32)
        cr = np.zeros(query_count, dtype=np.uint32)
        dg = np.zeros(query_count, dtype=np.uint8)
        _check(self._L.brmq_remap_from_sorted(self._h, _ptr(sorted_eps), sorted_eps.shape[0],
                                              _ptr(b), b.shape[0], query_count, _ptr(cl), _ptr(cr),
                                              _ptr(dg), 0))
        return ContractedQueryBatch(cl, cr, dg.astype(bool))

    def remap_queries(self, batch, contracted: ContractedArray) -> ContractedQueryBatch:
        """contraction.hpp:67 (contraction.cpp:152-171): binary search of both ends of
        every query in the boundary list; degenerate queries keep cleft = cright = 0."""
        batch = _as_queries(batch)
        b = np.ascontiguousarray(contracted.boundary, dtype=np.uint64)
        q = batch.shape[0]
        cl = np.zeros(q, dtype=np.uint32)
        cr = np.zeros(q, dtype=np.uint32)
        dg = np.zeros(q, dtype=np.uint8)
        _check(self._L.brmq_remap_queries(self._h, _ptr(batch), q, _ptr(b), b.shape[0], _ptr(cl),
                                          _ptr(cr), _ptr(dg), 0))
        return ContractedQueryBatch(cl, cr, dg.astype(bool))

    def build_block_sparse(self, values, k: int):
        """SPEC.md:210-218; returns (table[levels, b] of positions, b, levels)."""
        values = np.ascontiguousarray(values, dtype=np.int32)
        m = values.shape[0]
        b = (m + k - 1) // k if k > 0 else 0
        levels = (b.bit_length() if b else 0)
        table = np.empty(max(levels * b, 1), dtype=np.uint64)
        bo, lo = C.c_uint64(0), C.c_uint32(0)
        _check(self._L.brmq_build_block_sparse(self._h, _ptr(values), m, int(k), _ptr(table),
                                               C.byref(bo), C.byref(lo), 0))
        return table[: lo.value * bo.value].reshape(lo.value, bo.value), int(bo.value), int(lo.value)


def floor_log2(x: int) -> int:
    """bits.hpp:10-13 (DomainError on 0)."""
    out = C.c_uint32()
    _check(_lib.lib().brmq_floor_log2(int(x), C.byref(out)))
    return int(out.value)


_default: Engine | None = None


def default_engine() -> Engine:
    global _default
    if _default is None:
        _default = Engine(0)
    return _default


def solve_batch_bbst(array, batch, k: int = 512):
    return default_engine().solve_batch_bbst(array, batch, k)


def solve_batch_bbst_con(array, batch, k: int = 512, sort_kind: SortKind = SortKind.Radix):
    return default_engine().solve_batch_bbst_con(array, batch, k, sort_kind)


def solve_batch_st_rmq_con(array, batch):
    return default_engine().solve_batch_st_rmq_con(array, batch)


def collect_endpoints(batch):
    return default_engine().collect_endpoints(batch)


def sort_endpoints(eps, kind: SortKind = SortKind.Radix):
    return default_engine().sort_endpoints(eps, kind)


def build_contracted(values, sorted_eps):
    return default_engine().build_contracted(values, sorted_eps)


def remap_queries_from_sorted(sorted_eps, contracted, query_count):
    return default_engine().remap_queries_from_sorted(sorted_eps, contracted, query_count)


def remap_queries(batch, contracted):
    return default_engine().remap_queries(batch, contracted)


def build_block_sparse(values, k):
    return default_engine().build_block_sparse(values, k)
