"""Time multi-level BbST chains on a config (device-resident inputs, L2 flushed):
python tools/chain_bench.py [--config c3]"""
import argparse, statistics, sys
sys.path.insert(0, '.')
import numpy as np
import torch
from bench import gen_workload, time_solves, L2Flush
from paper_1706_06940_b200 import Engine

ap = argparse.ArgumentParser()
ap.add_argument('--config', default='c3')
ap.add_argument('--chains', default='')
a = ap.parse_args()
A, Q = gen_workload(a.config)
eng = Engine(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); eng.set_stream(s.cuda_stream)
dA = torch.from_numpy(A).cuda(); dQ = torch.from_numpy(Q.view(np.int64)).cuda()
dO = torch.empty(Q.shape[0], dtype=torch.int64, device='cuda')
flush = L2Flush(torch, 'cuda')
ref = None
for ks in ([tuple(int(v) for v in x.split(',')) for x in a.chains.split(';')] if a.chains else [(512,), (32, 512), (64, 512), (16, 512), (128, 4096), (8, 64, 512), (4, 32, 512), (32, 256, 4096)]):
    f = lambda: eng.solve_batch_bbst_ml(dA, dQ, ks, out=dO)
    ms, st, _ = time_solves(eng, torch, s, f, 5, 3, flush, timing=1)
    got = dO.cpu().numpy()
    ref = got if ref is None else ref
    print(a.config, ks, round(statistics.mean(ms), 4), {k: round(v[0], 4) for k, v in st.items()},
          'same' if np.array_equal(got, ref) else 'DIFF', flush=True)
