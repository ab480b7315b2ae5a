"""Sharded BbST (paper_1706_06940_b200/shard.py).

CPU (gloo, world_size 2): the host side -- shard bounds, key packing, the
order-preserving signed mapping and the min-allreduce -- with each rank's
per-shard keys computed by a numpy stand-in of brmq_solve_bbst_shard.
GPU: the device shard solves (BbST, and BbST_CON with either endpoint sort),
three shards on one device combined with a plain minimum, bit-exact against the
oracle.
"""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import oracle
from paper_1706_06940_b200 import SortKind
from paper_1706_06940_b200 import shard as S


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _pack(v, pos):
    return (np.uint64((int(v) & 0xFFFFFFFF) ^ 0x80000000) << np.uint64(32)) | np.uint64(pos)


def shard_keys_reference(A, Q, off, ns):
    """numpy stand-in for brmq_solve_bbst_shard (host-logic tests only)."""
    keys = np.full(Q.shape[0], S.NO_KEY, np.uint64)
    for i, (l, r) in enumerate(Q):
        l, r = sorted((int(l), int(r)))
        lo, hi = max(l, off), min(r, off + ns - 1)
        if lo <= hi:
            p = lo + int(np.argmin(A[lo:hi + 1]))
            keys[i] = _pack(A[p], p)
    return keys


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    r = np.random.default_rng(5)
    n = 3001
    A = r.integers(-50, 50, n).astype(np.int32)  # signed values, many ties
    Q = r.integers(0, n, (400, 2)).astype(np.uint64)
    off, ns = S.shard_bounds(n, world, rank)
    keys = shard_keys_reference(A, Q, off, ns)
    out[rank] = S.keys_to_answers(S.allreduce_min_keys(keys)).tolist()
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_combine_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    r = np.random.default_rng(5)
    n = 3001
    A = r.integers(-50, 50, n).astype(np.int32)
    Q = r.integers(0, n, (400, 2)).astype(np.uint64)
    want = oracle.naive_numpy(A, Q)
    assert res[0] == res[1] == want.tolist()


def test_signed_mapping_preserves_order():
    r = np.random.default_rng(1)
    k = r.integers(0, 2**63, 1000, dtype=np.uint64) * np.uint64(2) + r.integers(0, 2, 1000).astype(np.uint64)
    k = np.concatenate([k, np.array([0, S.NO_KEY, 1 << 63, (1 << 63) - 1], np.uint64)])
    s = S.to_signed(k)
    assert np.array_equal(np.argsort(s, kind="stable"), np.argsort(k, kind="stable"))
    assert np.array_equal(S.from_signed(s), k)


def test_shard_bounds_cover():
    for n in (1, 7, 1000, 1001):
        for world in (1, 2, 3, 8):
            parts = [S.shard_bounds(n, world, r) for r in range(world)]
            covered = [p for off, ln in parts for p in range(off, off + ln)]
            assert covered == list(range(n))


@pytest.mark.gpu
@pytest.mark.parametrize("variant", ["bbst", "con_bitmap", "con_radix"])
def test_shard_solve_gpu(engine, orc, variant):
    r = np.random.default_rng(8)
    n = 200_003
    A = r.integers(0, 1000, n).astype(np.int32)
    for kind in ("uniform", "short"):
        if kind == "uniform":
            Q = r.integers(0, n, (20_000, 2)).astype(np.uint64)
        else:
            a = r.integers(0, n, 20_000)
            Q = np.stack([np.minimum(a + r.integers(0, 300, 20_000), n - 1), a], 1).astype(np.uint64)
        want = orc.solve_oracle(A, Q)
        world = 3
        keys = np.full(Q.shape[0], S.NO_KEY, np.uint64)
        for rank in range(world):
            off, ns = S.shard_bounds(n, world, rank)
            if variant == "bbst":
                kr = engine.solve_batch_bbst_shard(A[off:off + ns], Q, off, n, 512)
            else:  # SURVEY 8e contraction variant: shard borders become boundaries
                sk = SortKind.Bitmap if variant == "con_bitmap" else SortKind.Radix
                kr = engine.solve_batch_bbst_con_shard(A[off:off + ns], Q, off, n, 512, sk)
            if rank == 1:  # spot-check the per-shard keys against the stand-in
                assert np.array_equal(kr[:300], shard_keys_reference(A, Q[:300], off, ns))
            keys = np.minimum(keys, kr)
        assert np.array_equal(S.keys_to_answers(keys), want), kind
