import sys, time
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1706_06940_b200 import Engine, SortKind
r = np.random.default_rng(31)
eng = Engine(0)
cases = []
for n, q in [tuple(map(int, a.split('/'))) for a in sys.argv[1:]]:
    A = r.integers(0, 2**31, n, dtype=np.int64).astype(np.int32)
    a, b = r.integers(0, n, q), r.integers(0, n, q)
    Q = np.stack([np.minimum(a, b), np.maximum(a, b)], 1).astype(np.uint64)
    cases.append((n, q, torch.from_numpy(A).cuda(), torch.from_numpy(Q.view(np.int64)).cuda(), torch.empty(q, dtype=torch.int64, device="cuda")))
for rep in range(2):
    for (n, q, dA, dQ, out) in cases:
        eng.solve_batch_bbst_con(dA, dQ, 512, SortKind.Bitmap, out=out)
        torch.cuda.synchronize()
        print(rep, n, q, eng.solve_info()["span_lo"], eng.solve_info()["span_hi"], flush=True)
