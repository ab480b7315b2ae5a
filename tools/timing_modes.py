"""Step time of the c2 solve under each library timing level, with and without
CUDA-graph replay (BRMQ_GRAPHS), to see what the in-graph event nodes cost."""
import os, sys, statistics, json
import numpy as np
sys.path.insert(0, '.')
import torch
from bench import gen_workload, time_solves
from paper_1706_06940_b200 import Engine
A, Q = gen_workload('c2')
eng = Engine(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); eng.set_stream(s.cuda_stream)
dA = torch.from_numpy(A).cuda(); dQ = torch.from_numpy(Q.view(np.int64)).cuda()
dO = torch.empty(Q.shape[0], dtype=torch.int64, device='cuda')
from bench import L2Flush; flush = L2Flush(torch, 'cuda')
res = {}
for sk in (2, 0):
    for t in (0, 2, 1):
        ms, st, _ = time_solves(eng, torch, s, lambda: eng.solve_batch_bbst_con(dA, dQ, 512, sk, out=dO), 20, 3, flush, timing=t)
        res[f"sort{sk}/timing{t}"] = (round(statistics.mean(ms), 4), {k: round(v[0], 4) for k, v in st.items()})
print(os.environ.get("BRMQ_GRAPHS", "1"), json.dumps(res))
