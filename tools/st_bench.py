"""Time the block Sparse Table build alone (c4/c5 block counts) for A/B builds."""
import sys, statistics, json
import numpy as np
sys.path.insert(0, '.')
import torch
from paper_1706_06940_b200 import Engine
from bench import time_solves
eng = Engine(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); eng.set_stream(s.cuda_stream)
from bench import L2Flush; flush = L2Flush(torch, 'cuda')
res = {}
for n in (100_000_000, 1_000_000_000, 1 << 30):
    A = torch.randint(0, 2**31 - 1, (n,), dtype=torch.int32, device='cuda')
    Q = torch.zeros(2, dtype=torch.int64, device='cuda')
    f = lambda: eng.solve_batch_bbst(A, Q, 512)
    _, st, _ = time_solves(eng, torch, s, f, 5, 2, flush, timing=1)
    res[n] = {k: round(v[0], 4) for k, v in st.items()}
    del A
print(json.dumps(res))
