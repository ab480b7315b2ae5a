import sys, numpy as np, torch
sys.path.insert(0, '.')
from bench import gen_workload
from paper_1706_06940_b200 import Engine
A, Q = gen_workload('c2')
eng = Engine(0)
s = torch.cuda.Stream(); torch.cuda.set_stream(s); eng.set_stream(s.cuda_stream)
dA = torch.from_numpy(A).cuda(); dQ = torch.from_numpy(Q.view(np.int64)).cuda(); out = torch.empty(Q.shape[0], dtype=torch.int64, device='cuda')
for timing in (False, True):
    eng.set_timing(timing)
    for v in (0, 2):
        for it in range(3):
            eng.solve_batch_bbst_con(dA, dQ, 512, v, out=out)
            print('timing', timing, 'kind', v, 'iter', it, 'graph', eng.solve_info()['graph'], eng.stage_times()[:2])
    for it in range(2):
        eng.solve_batch_bbst(dA, dQ, 512, out=out); print('bbst graph', eng.solve_info()['graph'])
