"""Solve time at small batches (c1 and q sweeps at n = 1e8) for the query-kernel mode."""
import sys, statistics, json
import numpy as np
sys.path.insert(0, '.')
import torch
from bench import gen_workload, time_solves, SEED0
from paper_1706_06940_b200 import Engine, _lib
eng = Engine(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); eng.set_stream(s.cuda_stream)
from bench import L2Flush; flush = L2Flush(torch, 'cuda')
res = {}
A, Q = gen_workload('c1')
dA = torch.from_numpy(A).cuda(); dQ = torch.from_numpy(Q.view(np.int64)).cuda()
dO = torch.empty(Q.shape[0], dtype=torch.int64, device='cuda')
for v, f in (("c1/bitmap", lambda: eng.solve_batch_bbst_con(dA, dQ, 512, 2, out=dO)), ("c1/bbst", lambda: eng.solve_batch_bbst(dA, dQ, 512, out=dO))):
    ms, _, _ = time_solves(eng, torch, s, f, 30, 3, flush, timing=0)
    _, st, _ = time_solves(eng, torch, s, f, 3, 1, flush, timing=1)
    res[v] = (round(statistics.mean(ms), 4), {k: round(x[0], 4) for k, x in st.items()})
A, _ = gen_workload('c2')
dA = torch.from_numpy(A).cuda()
L = _lib.lib()
for q in (1000, 10000, 100000):
    Q = np.empty((q, 2), np.uint64); L.brmq_workload_queries(0, A.shape[0], q, SEED0 + 2, Q.ctypes.data, 0)
    dQ = torch.from_numpy(Q.view(np.int64)).cuda(); dO = torch.empty(q, dtype=torch.int64, device='cuda')
    for v, f in (("bitmap", lambda: eng.solve_batch_bbst_con(dA, dQ, 512, 2, out=dO)), ("bbst", lambda: eng.solve_batch_bbst(dA, dQ, 512, out=dO))):
        ms, _, _ = time_solves(eng, torch, s, f, 10, 3, flush, timing=0)
        _, st, _ = time_solves(eng, torch, s, f, 3, 1, flush, timing=1)
        res[f"{q}/{v}"] = (round(statistics.mean(ms), 4), {k: round(x[0], 4) for k, x in st.items()})
print(json.dumps(res))
