"""Time the contraction stage for a few q (device-resident, L2 flushed)."""
import sys, statistics, json
import numpy as np
sys.path.insert(0, '.')
import torch
from bench import gen_workload, time_solves
from paper_1706_06940_b200 import Engine
A, _ = gen_workload('c2')
from paper_1706_06940_b200 import _lib
L = _lib.lib()
eng = Engine(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); eng.set_stream(s.cuda_stream); eng.set_timing(True)
dA = torch.from_numpy(A).cuda()
from bench import L2Flush; flush = L2Flush(torch, 'cuda')
res = {}
for q in (1000, 100000, 1000000, 10000000):
    Q = np.empty((q, 2), np.uint64); L.brmq_workload_queries(0, A.shape[0], q, 1706069402, Q.ctypes.data, 0)
    dQ = torch.from_numpy(Q.view(np.int64)).cuda()
    ms, st, _ = time_solves(eng, torch, s, lambda: eng.solve_batch_bbst_con(dA, dQ, 512, 2), 5, 2, flush)
    res[q] = (round(statistics.mean(ms), 4), round(st['contract'][0], 4))
print(json.dumps(res))
