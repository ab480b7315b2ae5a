"""ctypes access to the CPU checker -- TEST INFRASTRUCTURE ONLY.

* ``port()``  -> oracle/liboracle.so: our C restatement of the reference (oracle.c)
* ``ref()``   -> oracle/_ref/libbrmq_ref.so: the reference's own sources compiled
                 where they lie (oracle/Makefile) + an extern "C" shim.

Only tests/, __graft_entry__.smoke() and bench.py (cpu_baseline leg and
``--impl reference``) may import this module; the product (libbrmq.so and the
paper_1706_06940_b200 package) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
PORT_PATH = HERE / "liboracle.so"
REF_PATH = HERE / "_ref" / "libbrmq_ref.so"

vp, u64p, u32p = C.c_void_p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint32)

_PORT_SIGS = {
    "orc_naive_rmq": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_uint64, u64p]),
    "orc_floor_log2": (C.c_int, [C.c_uint64, u32p]),
    "orc_est_build": (C.c_int, [vp, C.c_uint64, C.POINTER(vp)]),
    "orc_est_arg_min": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, u64p]),
    "orc_est_cell_count": (C.c_uint64, [vp]),
    "orc_est_level_count": (C.c_uint32, [vp]),
    "orc_est_level": (C.c_uint64, [vp, C.c_uint32, vp]),
    "orc_est_free": (None, [vp]),
    "orc_collect_endpoints": (C.c_int, [vp, C.c_uint64, vp]),
    "orc_sort_endpoints": (C.c_int, [vp, C.c_uint64, C.c_int]),
    "orc_build_contracted": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, C.c_uint, vp, vp, vp, u64p,
                                       u64p]),
    "orc_remap_queries": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, vp, vp, vp]),
    "orc_remap_from_sorted": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, C.c_uint64, vp, vp, vp]),
    "orc_solve_oracle": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, C.c_uint, vp]),
    "orc_build_block_sparse": (C.c_int, [vp, C.c_uint64, C.c_uint32, vp, u64p, u32p]),
    "orc_solve_bbst": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, C.c_uint32, vp, u64p, u64p]),
    "orc_solve_bbst_con": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, C.c_uint32, C.c_uint, vp,
                                     u64p]),
}
_REF_SIGS = {
    "ref_floor_log2": (C.c_int, [C.c_uint64, u32p]),
    "ref_naive_rmq": (C.c_int, [vp, C.c_uint64, C.c_uint64, C.c_uint64, u64p]),
    "ref_collect_endpoints": (C.c_int, [vp, C.c_uint64, vp]),
    "ref_sort_endpoints": (C.c_int, [vp, C.c_uint64, C.c_int]),
    "ref_build_contracted": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, C.c_uint, vp, vp, vp, u64p,
                                       u64p]),
    "ref_remap_from_sorted": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, C.c_uint64, vp, vp, vp]),
    "ref_remap_queries": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, vp, vp, vp]),
    "ref_est_build": (vp, [vp, C.c_uint64, C.POINTER(C.c_int)]),
    "ref_est_arg_min": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, u64p]),
    "ref_est_cell_count": (C.c_uint64, [vp]),
    "ref_est_level_count": (C.c_uint64, [vp]),
    "ref_est_level": (C.c_uint64, [vp, C.c_uint64, vp]),
    "ref_est_free": (None, [vp]),
    "ref_solve_oracle": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, C.c_uint, vp,
                                   C.POINTER(C.c_double)]),
}

_port = None
_ref = None


def _load(path: Path, sigs: dict) -> C.CDLL:
    L = C.CDLL(str(path))
    for name, (res, args) in sigs.items():
        f = getattr(L, name)
        f.restype, f.argtypes = res, args
    return L


def build_port() -> None:
    subprocess.run(["make", "-s", "-C", str(HERE), "liboracle.so"], check=True)


def port() -> C.CDLL:
    global _port
    if _port is None:
        if not PORT_PATH.exists():
            build_port()
        _port = _load(PORT_PATH, _PORT_SIGS)
    return _port


def ref_available() -> bool:
    return REF_PATH.exists()


def ref() -> C.CDLL:
    global _ref
    if _ref is None:
        if not REF_PATH.exists():
            raise FileNotFoundError(f"{REF_PATH} not built (make -C oracle ref needs /root/reference)")
        _ref = _load(REF_PATH, _REF_SIGS)
    return _ref


def _p(a: np.ndarray) -> int:
    return a.ctypes.data if a.size else 0


def nthreads() -> int:
    return len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count() or 1


# ------------------------------------------------------------------ numpy helpers
def _queries_u64(Q) -> np.ndarray:
    a = np.asarray(Q)
    if a.dtype.names:
        a = a.view(np.uint64).reshape(-1, 2)
    return np.ascontiguousarray(a, dtype=np.uint64).reshape(-1, 2)


def solve_oracle(A: np.ndarray, Q, threads: int = 0, use_ref: bool | None = None) -> np.ndarray:
    """Leftmost-minimum positions by the SURVEY 8c pipeline (reference code when
    available, else the C restatement)."""
    A = np.ascontiguousarray(A, dtype=np.int32)
    Q = _queries_u64(Q)
    out = np.empty(Q.shape[0], dtype=np.uint64)
    th = threads or nthreads()
    if use_ref is None:
        use_ref = ref_available()
    if use_ref:
        rc = ref().ref_solve_oracle(_p(A), A.shape[0], _p(Q), Q.shape[0], th, _p(out), None)
    else:
        rc = port().orc_solve_oracle(_p(A), A.shape[0], _p(Q), Q.shape[0], th, _p(out))
    if rc:
        raise RuntimeError(f"oracle failed with status {rc}")
    return out


def solve_bbst_port(A, Q, k: int):
    """C restatement of BbST (no contraction): (answers, S, S_early)."""
    A = np.ascontiguousarray(A, dtype=np.int32)
    Q = _queries_u64(Q)
    out = np.empty(Q.shape[0], dtype=np.uint64)
    s, se = C.c_uint64(), C.c_uint64()
    rc = port().orc_solve_bbst(_p(A), A.shape[0], _p(Q), Q.shape[0], k, _p(out), C.byref(s),
                               C.byref(se))
    if rc:
        raise RuntimeError(f"orc_solve_bbst failed with status {rc}")
    return out, int(s.value), int(se.value)


def solve_bbst_con_port(A, Q, k: int, threads: int = 1):
    A = np.ascontiguousarray(A, dtype=np.int32)
    Q = _queries_u64(Q)
    out = np.empty(Q.shape[0], dtype=np.uint64)
    s = C.c_uint64()
    rc = port().orc_solve_bbst_con(_p(A), A.shape[0], _p(Q), Q.shape[0], k, threads, _p(out),
                                   C.byref(s))
    if rc:
        raise RuntimeError(f"orc_solve_bbst_con failed with status {rc}")
    return out, int(s.value)


def naive_answers(A, Q) -> np.ndarray:
    """naive_rmq per query (C restatement); for small cases only."""
    A = np.ascontiguousarray(A, dtype=np.int32)
    Q = _queries_u64(Q)
    out = np.empty(Q.shape[0], dtype=np.uint64)
    L = port()
    r = C.c_uint64()
    for i, (l, rr) in enumerate(Q):
        rc = L.orc_naive_rmq(_p(A), A.shape[0], int(l), int(rr), C.byref(r))
        if rc:
            raise IndexError("naive_rmq: query exceeds array bounds")
        out[i] = r.value
    return out


def naive_numpy(A, Q) -> np.ndarray:
    """Independent pure-numpy leftmost argmin (small cases)."""
    A = np.asarray(A)
    Q = _queries_u64(Q).astype(np.int64)
    lo, hi = np.minimum(Q[:, 0], Q[:, 1]), np.maximum(Q[:, 0], Q[:, 1])  # types.hpp:18-20
    return np.array([l + int(np.argmin(A[l:r + 1])) for l, r in zip(lo, hi)], dtype=np.uint64)
