import sys, numpy as np, torch
sys.path.insert(0, '.')
from bench import gen_workload
from paper_1706_06940_b200 import Engine
A, Q = gen_workload('c3')
eng = Engine(0)
dA = torch.from_numpy(A).cuda(); dQ = torch.from_numpy(Q.view(np.int64)).cuda()
for _ in range(2):
    eng.solve_batch_bbst_ml(dA, dQ, (32, 512)); eng.solve_batch_bbst(dA, dQ, 512)
torch.cuda.synchronize(); print('ok')
