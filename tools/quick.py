"""Quick A/B timing of solves on the GPU box (tooling, not the bench):

    python tools/quick.py --configs c2,c3 --variants con_bitmap,bbst [--check] [--steps 10]

Per (config, variant): mean ms per solve with no stage events (graph replay,
PDL on), the per-stage breakdown from a second pass with stage events, and with
--check the answers of the last timed replay (output poisoned before each step)
against the reference pipeline (oracle/_ref)."""
import argparse
import json
import statistics
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
from bench import L2Flush, VARIANT_SORT, gen_workload, time_solves  # noqa: E402
from paper_1706_06940_b200 import Engine  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument('--configs', default='c2')
ap.add_argument('--variants', default='con_bitmap')
ap.add_argument('--steps', type=int, default=10)
ap.add_argument('--check', action='store_true')
ap.add_argument('--q', type=int, default=None)
a = ap.parse_args()

eng = Engine(0)
eng.set_async(True)  # as bench.py: the window is the device time of the solve
s = torch.cuda.Stream()
torch.cuda.set_stream(s)
eng.set_stream(s.cuda_stream)
flush = L2Flush(torch, 'cuda')
res = {}
for cfg in a.configs.split(','):
    A, Q = gen_workload(cfg, q=a.q)
    want = None
    if a.check:
        import oracle
        want = oracle.solve_oracle(A, Q)
    dA = torch.from_numpy(A).cuda()
    dQ = torch.from_numpy(Q.view(np.int64)).cuda()
    dO = torch.empty(Q.shape[0], dtype=torch.int64, device='cuda')
    for v in a.variants.split(','):
        def f(v=v):
            if v == 'bbst':
                eng.solve_batch_bbst(dA, dQ, 512, out=dO)
            elif v == 'bbst_ml':
                eng.solve_batch_bbst_ml(dA, dQ, (32, 512), out=dO)
            elif v == 'st_rmq_con':
                eng.solve_batch_st_rmq_con(dA, dQ, out=dO)
            else:
                eng.solve_batch_bbst_con(dA, dQ, 512, VARIANT_SORT[v], out=dO)
        ms, _, nl = time_solves(eng, torch, s, f, a.steps, 3, flush, timing=0,
                                poison=lambda: dO.fill_(-1))
        ok = None if want is None else bool(np.array_equal(dO.cpu().numpy().view(np.uint64), want))
        _, st, _ = time_solves(eng, torch, s, f, 3, 1, flush, timing=1)
        res[f'{cfg}/{v}'] = {'ms': round(statistics.mean(ms), 4), 'min_ms': round(min(ms), 4),
                             'launches': nl // a.steps, 'ok': ok,
                             **{k: round(x[0], 4) for k, x in st.items()}}
        print(json.dumps({f'{cfg}/{v}': res[f'{cfg}/{v}']}), flush=True)
    del dA, dQ, dO
    torch.cuda.empty_cache()
eng.close()
