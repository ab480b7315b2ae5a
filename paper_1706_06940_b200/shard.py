"""Sharded BbST across devices: A in contiguous shards, one per
rank; each rank answers every query on its shard as packed keys with global
positions (brmq_solve_bbst_shard / brmq_solve_bbst_con_shard), and one
min-allreduce of the q keys finishes the batch -- exact, because the unsigned
minimum of packed (value, position) keys is the leftmost minimum.  On
NVLink / NVSwitch the allreduce is a single NCCL call over 8q bytes of device
memory; the keys never leave the GPU.

torch.distributed reduces signed int64, so keys travel order-preserved through
the sign-bit flip k ^ 2^63 (uint64 order == int64 order of the flipped words),
done in place on the tensor (a CUDA tensor under NCCL, a CPU tensor under gloo).

The reference's only parallelism is std::thread chunking inside one process
(/root/reference/proj/core/include/batchrmq/parallel.hpp:14-44); this module is
the device-level counterpart of SURVEY 8e, not a port of it.
"""
from __future__ import annotations

import numpy as np

SIGN = np.uint64(1 << 63)
NO_KEY = np.uint64(0xFFFFFFFFFFFFFFFF)
_INT64_MIN = -(1 << 63)


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """[offset, offset + length) of rank's contiguous shard of an n-array
    (length 0 for trailing ranks when world does not divide n evenly)."""
    per = -(-n // world)
    lo = min(n, rank * per)
    return lo, min(n, lo + per) - lo


def to_signed(keys: np.ndarray) -> np.ndarray:
    return (np.asarray(keys, np.uint64) ^ SIGN).view(np.int64)


def from_signed(x: np.ndarray) -> np.ndarray:
    return np.asarray(x, np.int64).view(np.uint64) ^ SIGN


def _is_tensor(x) -> bool:
    try:
        import torch
    except ImportError:  # pragma: no cover
        return False
    return isinstance(x, torch.Tensor)


def keys_to_answers(keys):
    """Positions from combined keys (low 32 bits); numpy uint64 in -> numpy
    uint64 out, torch int64 (uint64 bit patterns) in -> torch int64 out."""
    if _is_tensor(keys):
        return keys & 0xFFFFFFFF
    return (np.asarray(keys, np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.uint64)


def allreduce_min_keys(keys, group=None):
    """Min-allreduce of packed keys over the process group.

    keys: a torch int64 tensor holding uint64 bit patterns (CUDA under NCCL --
    reduced in place on the device, no host copy) or a numpy uint64 array
    (reduced through a CPU tensor, gloo).  Returns the same kind it was given."""
    import torch
    import torch.distributed as dist
    if _is_tensor(keys):
        t = keys if keys.dtype == torch.int64 else keys.view(torch.int64)
        t.bitwise_xor_(_INT64_MIN)  # order-preserving uint64 -> int64
        dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
        t.bitwise_xor_(_INT64_MIN)
        return t
    t = torch.from_numpy(to_signed(keys).copy())
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return from_signed(t.numpy())


def local_keys(engine, shard, batch, offset: int, n_total: int, k: int = 512,
               contraction: bool = False, sort_kind=None, out=None):
    """Packed keys of every query restricted to this rank's shard.  A rank whose
    shard is empty contributes NO_KEY for every query (it still joins the
    collective, so no rank blocks in the allreduce)."""
    ns = int(shard.shape[0])
    q = int(batch.shape[0])
    if ns == 0 or q == 0:
        if _is_tensor(batch):
            import torch
            t = out if out is not None else torch.empty(q, dtype=torch.int64, device=batch.device)
            return t.fill_(-1)  # all bits set = NO_KEY
        return np.full(q, NO_KEY, np.uint64)
    if contraction:
        from .batchrmq import SortKind
        return engine.solve_batch_bbst_con_shard(shard, batch, offset, n_total, k,
                                                 SortKind.Bitmap if sort_kind is None else sort_kind,
                                                 out=out)
    return engine.solve_batch_bbst_shard(shard, batch, offset, n_total, k, out=out)


def solve_sharded(engine, shard, batch, offset: int, n_total: int, k: int = 512, group=None,
                  contraction: bool = False, sort_kind=None, out=None):
    """This rank's part of a sharded solve plus the combine: answers for all queries.
    With CUDA tensors (shard, batch) the keys stay on the device and the combine is
    one NCCL all_reduce(MIN); contraction=True solves the shard with BbST_CON
    (contraction variant: the shard borders become boundaries)."""
    keys = local_keys(engine, shard, batch, offset, n_total, k, contraction, sort_kind, out)
    if not _is_tensor(keys):
        keys = np.asarray(keys, np.uint64)
    return keys_to_answers(allreduce_min_keys(keys, group))
