"""Debug helper: replay the bench sweep call sequence with per-call checks."""
import sys, time
import numpy as np
sys.path.insert(0, '.')
import torch
import oracle
from paper_1706_06940_b200 import Engine, _lib, SortKind
L = _lib.lib()
n = int(sys.argv[1]) if len(sys.argv) > 1 else 100_000_000
A = np.empty(n, np.int32); L.brmq_workload_array(0, n, 1706069402, A.ctypes.data, 0)
eng = Engine(0)
dA = torch.from_numpy(A).cuda()
for q in (1_000, 10_000, 100_000, 1_000_000, 10_000_000):
    Q = np.empty((q, 2), np.uint64); L.brmq_workload_queries(0, n, q, 1706069402, Q.ctypes.data, 0)
    want = oracle.solve_oracle(A, Q)
    dQ = torch.from_numpy(Q.view(np.int64)).cuda()
    for v in ("con_radix", "con_bitmap", "bbst"):
        print("run", q, v, flush=True)
        if v == "bbst":
            o = eng.solve_batch_bbst(dA, dQ, 512)
        else:
            o = eng.solve_batch_bbst_con(dA, dQ, 512, SortKind.Radix if v == "con_radix" else SortKind.Bitmap)
        got = o.cpu().numpy().view(np.uint64)
        print(q, v, "ok" if np.array_equal(got, want) else f"MISMATCH {np.sum(got != want)}", eng.solve_info(), flush=True)
