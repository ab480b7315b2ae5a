"""A/B the contraction stage of several library builds (BRMQ_LIB) on one box.

usage: python tools/ab_contract.py ab/libA.so ab/libB.so ...   (each in a fresh process)
"""
import json, os, subprocess, sys

if len(sys.argv) > 1 and sys.argv[1] != "--child":
    for lib in sys.argv[1:]:
        env = dict(os.environ, BRMQ_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
        print(lib, out.stdout.strip() or out.stderr[-2000:])
    sys.exit(0)

import statistics
import numpy as np
sys.path.insert(0, '.')
import torch
from bench import gen_workload, time_solves
from paper_1706_06940_b200 import Engine, _lib
A, _ = gen_workload('c2')
L = _lib.lib()
eng = Engine(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); eng.set_stream(s.cuda_stream)
dA = torch.from_numpy(A).cuda()
from bench import L2Flush; flush = L2Flush(torch, 'cuda')
res = {}
for q in (1000, 100000, 1000000, 10000000):
    Q = np.empty((q, 2), np.uint64); L.brmq_workload_queries(0, A.shape[0], q, 1706069402, Q.ctypes.data, 0)
    dQ = torch.from_numpy(Q.view(np.int64)).cuda()
    for sk in (0, 2):
        ms, st, _ = time_solves(eng, torch, s, lambda: eng.solve_batch_bbst_con(dA, dQ, 512, sk), 10, 3, flush, timing=2)
        res[f"{q}/{sk}"] = (round(statistics.mean(ms), 4), round(st['contract'][0], 4))
print(json.dumps(res))
