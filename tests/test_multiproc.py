"""Multi-process host logic of bench.py on CPU (gloo, world_size 2).

The engine does not shard on one node ("replicas": every rank solves its own
workload, no data-path collective); what must hold across ranks is the
timing contract: the step time is the MAX over ranks and the reported value
is the whole-job throughput.
"""
import os
import socket

import pytest
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    t_ms = [2.5, 4.0][rank]  # rank 1 is the slow one
    t = bench.max_over_ranks(t_ms, dist, "cpu")
    out[rank] = (t, bench.aggregate_value(100_000, world, t))
    dist.barrier()
    dist.destroy_process_group()


def test_max_over_ranks_gloo():
    world = 2
    port = _free_port()
    with mp.Manager() as m:
        out = m.dict()
        mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
        res = dict(out)
    assert res[0] == res[1] == (4.0, pytest.approx(2 * 100_000 / 4e-3))


def test_single_process_passthrough():
    assert bench.max_over_ranks(3.0) == 3.0
    assert bench.aggregate_value(10, 1, 1.0) == pytest.approx(1e4)
