"""Sharded BbST across devices: A in contiguous shards, one per
rank; each rank answers every query on its shard as packed keys with global
positions (brmq_solve_bbst_shard), and one min-allreduce of the q keys finishes
the batch -- exact, because the unsigned minimum of packed (value, position)
keys is the leftmost minimum.  On NVLink / NVSwitch the allreduce is a single
NCCL call over 8q bytes.

torch.distributed reduces signed int64, so keys travel order-preserved through
the sign-bit flip k ^ 2^63 (uint64 order == int64 order of the flipped words).
"""
from __future__ import annotations

import numpy as np

SIGN = np.uint64(1 << 63)
NO_KEY = np.uint64(0xFFFFFFFFFFFFFFFF)


def shard_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """[offset, offset + length) of rank's contiguous shard of an n-array."""
    per = -(-n // world)
    lo = min(n, rank * per)
    return lo, min(n, lo + per) - lo


def to_signed(keys: np.ndarray) -> np.ndarray:
    return (np.asarray(keys, np.uint64) ^ SIGN).view(np.int64)


def from_signed(x: np.ndarray) -> np.ndarray:
    return np.asarray(x, np.int64).view(np.uint64) ^ SIGN


def keys_to_answers(keys: np.ndarray) -> np.ndarray:
    """Positions from combined keys (low 32 bits)."""
    return (np.asarray(keys, np.uint64) & np.uint64(0xFFFFFFFF)).astype(np.uint64)


def allreduce_min_keys(keys: np.ndarray, group=None) -> np.ndarray:
    """Min-allreduce of packed keys over the process group (host buffers: gloo;
    CUDA tensors go through the same call with the NCCL backend)."""
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(to_signed(keys).copy())
    dist.all_reduce(t, op=dist.ReduceOp.MIN, group=group)
    return from_signed(t.numpy())


def solve_sharded(engine, shard, batch, offset: int, n_total: int, k: int = 512, group=None,
                  contraction: bool = False, sort_kind=None):
    """This rank's part of a sharded solve plus the combine: answers for all queries.
    contraction=True solves the shard with BbST_CON (contraction variant)."""
    if contraction:
        from .batchrmq import SortKind
        keys = engine.solve_batch_bbst_con_shard(shard, batch, offset, n_total, k,
                                                 SortKind.Bitmap if sort_kind is None else sort_kind)
    else:
        keys = engine.solve_batch_bbst_shard(shard, batch, offset, n_total, k)
    return keys_to_answers(allreduce_min_keys(np.asarray(keys, np.uint64), group))
