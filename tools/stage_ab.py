"""Pageable vs pinned host-pointer solve timing (tooling, not the bench):

    BRMQ_STAGE_THREADS=8 BRMQ_STAGE_CHUNK_KB=16384 python tools/stage_ab.py [--config c2] [--steps 8]

Prints wall ms per c2 BbST_CON (bitmap) solve from numpy (pageable) buffers, from
pinned buffers, and a plain pinned / pageable 400 MB cudaMemcpy for scale."""
import argparse
import json
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
from bench import VARIANT_SORT, gen_workload  # noqa: E402
from paper_1706_06940_b200 import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument('--config', default='c2')
ap.add_argument('--steps', type=int, default=8)
a = ap.parse_args()
eng = Engine(0)
A, Q = gen_workload(a.config)
O = np.empty(Q.shape[0], np.uint64)


def timed(f):
    f()
    f()
    ts = []
    for _ in range(a.steps):
        t = time.perf_counter()
        f()
        ts.append((time.perf_counter() - t) * 1e3)
    return round(statistics.median(ts), 3)


res = {'env': {k: v for k, v in os.environ.items() if k.startswith('BRMQ_STAGE')}}
res['pageable_solve_ms'] = timed(lambda: eng.solve_batch_bbst_con(A, Q, 512, VARIANT_SORT["con_bitmap"], out=O))
dA = torch.empty(A.shape[0], dtype=torch.int32, device='cuda')
tA = torch.from_numpy(A)
pA = torch.empty_like(tA).pin_memory()
pA.copy_(tA)
res['pinned_memcpy_ms'] = timed(lambda: (dA.copy_(pA, non_blocking=True), torch.cuda.synchronize()))
res['pageable_memcpy_ms'] = timed(lambda: (dA.copy_(tA), torch.cuda.synchronize()))
pQ = torch.from_numpy(Q.view(np.int64)).pin_memory()
pO = torch.empty(Q.shape[0], dtype=torch.int64).pin_memory()
res['pinned_solve_ms'] = timed(lambda: eng.solve_batch_bbst_con(pA.numpy(), pQ.numpy().view(np.uint64), 512,
                                                                VARIANT_SORT["con_bitmap"], out=pO.numpy().view(np.uint64)))
res['host_memcpy_1t_ms'] = timed(lambda: pA.numpy().__setitem__(slice(None), A))
print(json.dumps(res))
