"""Contraction tail diagnostics (A/B build with -DBRMQ_CONTRACT_STAMPS): per-warp
start / loop-end / stitch-end %globaltimer stamps of one c2 solve.

    BRMQ_LIB=ab/stamps.so python tools/contract_tail.py [--config c2] [--variant con_bitmap]
"""
import argparse, ctypes as C, sys
import numpy as np
import torch
sys.path.insert(0, '.')
from bench import gen_workload, VARIANT_SORT, L2Flush  # noqa: E402
from paper_1706_06940_b200 import Engine, _lib  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument('--config', default='c2')
ap.add_argument('--variant', default='con_bitmap')
a = ap.parse_args()
A, Q = gen_workload(a.config)
eng = Engine(0)
dA = torch.from_numpy(A).cuda()
dQ = torch.from_numpy(Q.view(np.int64)).cuda()
L = _lib.lib()
f = L.brmq_debug_contract_stamps
f.argtypes = [C.c_void_p, C.c_int]
W = 2048 * 8
buf = np.zeros((W, 3), np.uint64)
flush = L2Flush(torch, 'cuda')
for it in range(4):
    flush()
    torch.cuda.synchronize()
    eng.solve_batch_bbst_con(dA, dQ, 512, VARIANT_SORT[a.variant])
    torch.cuda.synchronize()
    f(buf.ctypes.data, W)
    if hasattr(L, 'brmq_debug_contract_stamps2'):
        buf2 = np.zeros((W, 3), np.uint64)
        L.brmq_debug_contract_stamps2(C.c_void_p(buf2.ctypes.data), C.c_int(W))
live = buf[(buf[:, 0] > 0) & (buf[:, 1] > 0)]
t0 = live[:, 0].min()
s, e1, e2 = (live[:, 0] - t0) / 1e3, (live[:, 1] - t0) / 1e3, (live[:, 2] - t0) / 1e3
print(f"warps {len(live)}; start: min 0 max {s.max():.2f} us; loop end: min {e1.min():.2f} "
      f"p10 {np.percentile(e1, 10):.2f} p50 {np.median(e1):.2f} p90 {np.percentile(e1, 90):.2f} max {e1.max():.2f}; "
      f"stitch end max {e2.max():.2f}")
# lost warp-time: sum over warps of (kernel end - loop end) / (warps * kernel span)
span = e2.max()
print(f"idle fraction after the loop: {np.mean(span - e1) / span:.3f}; mean loop time {np.mean(e1 - s):.2f} us")
hist, edges = np.histogram(e1, bins=12)
print("loop-end histogram:", " ".join(f"{edges[i]:.0f}:{hist[i]}" for i in range(len(hist))))
# within-CTA vs across-CTA spread (8 warps per CTA)
ends = {}
for w in range(W):
    if buf[w, 0] > 0 and buf[w, 1] > 0:
        ends.setdefault(w // 8, []).append((buf[w, 1] - t0) / 1e3)
cta_max = np.array([max(v) for v in ends.values() if len(v) == 8])
cta_min = np.array([min(v) for v in ends.values() if len(v) == 8])
cta_mean = np.array([np.mean(v) for v in ends.values() if len(v) == 8])
print(f"CTAs {len(cta_max)}: within-CTA spread (max-min) mean {np.mean(cta_max - cta_min):.2f} us p90 "
      f"{np.percentile(cta_max - cta_min, 90):.2f}; CTA mean loop end p10 {np.percentile(cta_mean, 10):.2f} "
      f"p50 {np.median(cta_mean):.2f} p90 {np.percentile(cta_mean, 90):.2f} max {cta_mean.max():.2f}")
# SM pairing: CTAs b and b + 148 likely share an SM? print correlation of neighbours
st_minus_loop = (live[:, 2] - live[:, 1]) / 1e3
print(f"stitch time per warp: p50 {np.median(st_minus_loop):.2f} p90 {np.percentile(st_minus_loop, 90):.2f} max {st_minus_loop.max():.2f}")
if 'buf2' in dir():
    ok = (buf2[:, 0] > 0) & (buf[:, 0] > 0)
    e0 = buf2[ok, 0].astype(np.int64); t00 = e0.min()
    ent, bas, lps = (e0 - t00) / 1e3, (buf2[ok, 1].astype(np.int64) - t00) / 1e3, (buf[ok, 0].astype(np.int64) - t00) / 1e3
    ends_all = (buf[ok, 2].astype(np.int64) - t00) / 1e3
    print(f"from the first warp's entry: entry p50 {np.median(ent):.2f} max {ent.max():.2f}; rank bases known "
          f"p10 {np.percentile(bas, 10):.2f} p50 {np.median(bas):.2f} p90 {np.percentile(bas, 90):.2f} max {bas.max():.2f}; "
          f"loop start p50 {np.median(lps):.2f} max {lps.max():.2f}; kernel end {ends_all.max():.2f}")
    wr = (buf2[ok, 2].astype(np.int64) - t00) / 1e3
    print(f"wait released p10 {np.percentile(wr, 10):.2f} p50 {np.median(wr):.2f} max {wr.max():.2f}; "
          f"bases - release p10 {np.percentile(bas - wr, 10):.2f} p50 {np.median(bas - wr):.2f} max {(bas - wr).max():.2f}")
late = np.argsort(-(buf[:, 2].astype(np.int64) - int(t0)))[:5]
for w in late:
    print(f"  warp {w} (cta {w // 8}): start {(buf[w,0]-t0)/1e3:.2f} loop end {(buf[w,1]-t0)/1e3:.2f} stitch end {(buf[w,2]-t0)/1e3:.2f}")
# what explains a warp's loop time: its boundaries, its warp slot, its CTA?
n = A.shape[0]
pos = np.unique(np.concatenate([np.minimum(Q[:, 0], Q[:, 1]), np.maximum(Q[:, 0], Q[:, 1])]).astype(np.int64))
b0, blast = int(pos[0]), int(pos[-1])
tiles = (n + 4095) // 4096
G = (W // 8) if False else int(np.max(np.nonzero(buf[:, 0])[0]) // 8 + 1)
R = (tiles + G - 1) // G
cnts, times, slots = [], [], []
for cta in range(G):
    ta, tb = max(cta * R, b0 // 4096), min(cta * R + R - 1, blast // 4096)
    if ta > tb:
        continue
    w0, w1 = max(ta * 4, b0 // 1024), min(tb * 4 + 3, blast // 1024)
    per = (w1 - w0 + 8) // 8
    for w in range(8):
        wa = w0 + w * per
        wb = min(wa + per - 1, w1)
        if wa > wb or buf[cta * 8 + w, 0] == 0:
            continue
        c = np.searchsorted(pos, (wb + 1) * 1024) - np.searchsorted(pos, wa * 1024)
        cnts.append(c)
        times.append((buf[cta * 8 + w, 1] - buf[cta * 8 + w, 0]) / 1e3)
        slots.append(w)
cnts, times, slots = np.array(cnts), np.array(times), np.array(slots)
m = times > 20
print(f"pieces {m.sum()}: boundaries mean {cnts[m].mean():.1f} sd {cnts[m].std():.1f}; loop time sd {times[m].std():.2f} us; "
      f"corr(boundaries, time) {np.corrcoef(cnts[m], times[m])[0, 1]:.3f}")
print("mean loop time by warp slot:", " ".join(f"{w}:{times[m & (slots == w)].mean():.2f}" for w in range(8)))
