import sys, statistics, json, numpy as np, torch
sys.path.insert(0, '.')
from bench import gen_workload, time_solves
from paper_1706_06940_b200 import Engine
res = {}
for cfg in ('c3', 'c4', 'c5'):
    A, Q = gen_workload(cfg)
    eng = Engine(0)
    s = torch.cuda.Stream(); torch.cuda.set_stream(s); eng.set_stream(s.cuda_stream)
    dA = torch.from_numpy(A).cuda(); dQ = torch.from_numpy(Q.view(np.int64)).cuda()
    from bench import L2Flush; flush = L2Flush(torch, 'cuda')
    for name, f in (('h1', lambda: eng.solve_batch_bbst(dA, dQ, 512)), ('ml', lambda: eng.solve_batch_bbst_ml(dA, dQ, (32, 512)))):
        ms, _, _ = time_solves(eng, torch, s, f, 5, 2, flush, timing=0)
        _, st, _ = time_solves(eng, torch, s, f, 3, 1, flush, timing=1)
        res[cfg + '/' + name] = {'ms': round(statistics.mean(ms), 4), 'qps': Q.shape[0] / statistics.mean(ms) * 1e3, **{k: round(v[0], 4) for k, v in st.items()}}
    del dA, dQ, A, Q; eng.close(); torch.cuda.empty_cache()
print(json.dumps(res, indent=0))
