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


class _StandInEngine:
    """numpy stand-in for the device shard solves (host-logic tests only): the
    same call shapes as Engine.solve_batch_bbst[_con]_shard, CPU tensors in and out."""

    def __init__(self, A):
        self.A = A

    def _keys(self, shard, batch, offset):
        import torch
        Q = batch.numpy().view(np.uint64) if isinstance(batch, torch.Tensor) else batch
        k = shard_keys_reference(self.A, Q, offset, int(shard.shape[0]))
        return torch.from_numpy(k.view(np.int64)) if isinstance(batch, torch.Tensor) else k

    def solve_batch_bbst_shard(self, shard, batch, offset, n_total, k=512, out=None):
        return self._keys(shard, batch, offset)

    def solve_batch_bbst_con_shard(self, shard, batch, offset, n_total, k=512, sort_kind=None, out=None):
        return self._keys(shard, batch, offset)


def _worker_tensor(rank, world, port, out):
    """solve_sharded with tensors (the device path's call sequence, gloo on CPU):
    world 4 over n = 9 leaves rank 3 with an empty shard, which must still join
    the collective with all-NO_KEY keys."""
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    res = {}
    for n in (9, 3001):
        r = np.random.default_rng(n)
        A = r.integers(-5, 5, n).astype(np.int32)
        Q = r.integers(0, n, (300, 2)).astype(np.uint64)
        off, ns = S.shard_bounds(n, world, rank)
        eng = _StandInEngine(A)
        shard = torch.from_numpy(A[off:off + ns].copy())
        tq = torch.from_numpy(Q.view(np.int64).copy())
        ans = S.solve_sharded(eng, shard, tq, off, n, contraction=(n == 9))
        assert isinstance(ans, torch.Tensor) and ans.dtype == torch.int64
        res[n] = (ns, ans.numpy().astype(np.uint64).tolist())
    out[rank] = res
    dist.barrier()
    dist.destroy_process_group()


def test_sharded_tensor_path_gloo_empty_shard():
    world = 4
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker_tensor, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[3][9][0] == 0  # the empty shard
    for n in (9, 3001):
        r = np.random.default_rng(n)
        A = r.integers(-5, 5, n).astype(np.int32)
        Q = r.integers(0, n, (300, 2)).astype(np.uint64)
        want = oracle.naive_numpy(A, Q).tolist()
        for rank in range(world):
            assert res[rank][n][1] == want, (n, rank)


def _worker_nccl(rank, world, port, out):
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world,
                            device_id=torch.device("cuda", rank))
    from paper_1706_06940_b200 import Engine
    r = np.random.default_rng(11)
    n = 1_000_003
    A = r.integers(0, 1 << 20, n).astype(np.int32)
    Q = r.integers(0, n, (50_000, 2)).astype(np.uint64)
    off, ns = S.shard_bounds(n, world, rank)
    eng = Engine(rank)
    dA = torch.from_numpy(A[off:off + ns].copy()).cuda()
    dQ = torch.from_numpy(Q.view(np.int64).copy()).cuda()
    for con in (False, True):
        ans = S.solve_sharded(eng, dA, dQ, off, n, 512, contraction=con)
        assert ans.is_cuda
        out[(rank, con)] = ans.cpu().numpy().astype(np.uint64).tolist()
    eng.close()
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.gpu
def test_sharded_nccl_two_gpus(orc):
    """The device combine: keys stay on each GPU, one NCCL all_reduce(MIN)."""
    import torch
    if torch.cuda.device_count() < 2:
        pytest.skip("needs two GPUs (NCCL min-allreduce across devices)")
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker_nccl, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    r = np.random.default_rng(11)
    n = 1_000_003
    A = r.integers(0, 1 << 20, n).astype(np.int32)
    Q = r.integers(0, n, (50_000, 2)).astype(np.uint64)
    want = orc.solve_oracle(A, Q).tolist()
    for key, got in res.items():
        assert got == want, key


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
        # an empty shard (n_shard = 0) answers NO_KEY for every query
        empty = (engine.solve_batch_bbst_shard(A[:0], Q, n, n, 512) if variant == "bbst" else
                 engine.solve_batch_bbst_con_shard(A[:0], Q, n, n, 512,
                                                   SortKind.Bitmap if variant == "con_bitmap" else SortKind.Radix))
        assert (empty == S.NO_KEY).all()


@pytest.mark.gpu
def test_shard_solve_device_tensors(engine, orc):
    """Device-resident shards and keys (the NCCL path's inputs), one process:
    the combine is done with the same sign-flip the collective uses."""
    import torch
    r = np.random.default_rng(9)
    n = 500_009
    A = r.integers(0, 100, n).astype(np.int32)
    Q = r.integers(0, n, (30_000, 2)).astype(np.uint64)
    want = orc.solve_oracle(A, Q)
    dQ = torch.from_numpy(Q.view(np.int64).copy()).cuda()
    world = 4
    acc = None
    for rank in range(world):
        off, ns = S.shard_bounds(n, world, rank)
        dA = torch.from_numpy(A[off:off + ns].copy()).cuda()
        for con in (False, True):
            k = S.local_keys(engine, dA, dQ, off, n, 512, contraction=con)
            assert k.is_cuda and k.dtype == torch.int64
            kf = k ^ (-(1 << 63))
            if con:
                assert torch.equal(kf, prev)
            prev = kf
        acc = kf if acc is None else torch.minimum(acc, kf)
    got = S.keys_to_answers(acc ^ (-(1 << 63))).cpu().numpy().astype(np.uint64)
    assert np.array_equal(got, want)
