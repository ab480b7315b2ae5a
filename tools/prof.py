"""Profiling driver: run one workload/variant a few times with device-resident
inputs (used under ncu; never a bench number)."""
import argparse, sys
import numpy as np
sys.path.insert(0, '.')
import torch
from bench import gen_workload, VARIANT_SORT
from paper_1706_06940_b200 import Engine

ap = argparse.ArgumentParser()
ap.add_argument('--config', default='c2')
ap.add_argument('--variant', default='con_radix')
ap.add_argument('--iters', type=int, default=3)
ap.add_argument('--q', type=int, default=None)
a = ap.parse_args()
A, Q = gen_workload(a.config, q=a.q)
eng = Engine(0)
dA = torch.from_numpy(A).cuda()
dQ = torch.from_numpy(Q.view(np.int64)).cuda()
for _ in range(a.iters):
    if a.variant == 'bbst':
        out = eng.solve_batch_bbst(dA, dQ, 512)
    elif a.variant == 'bbst_ml':
        out = eng.solve_batch_bbst_ml(dA, dQ, (32, 512))
    else:
        out = eng.solve_batch_bbst_con(dA, dQ, 512, VARIANT_SORT[a.variant])
torch.cuda.synchronize()
print('ok', a.config, a.variant, int(out[0]))
