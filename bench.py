#!/usr/bin/env python
"""Benchmark of the batched-RMQ hot path on B200 (one JSON line on rank 0).

Headline workload (BASELINE.json configs[1], "c2"): n = 1e8 int32 values uniform in
[0, 2^31), q = 1e5 queries with uniform endpoints, BbST_CON (endpoint sort +
segmented-argmin contraction + block Sparse Table over A_Q, k = 512).  The
headline variant sorts the endpoints as a presence-bitmap counting sort
(BRMQ_SORT_BITMAP: one digit of log2(n) bits, duplicates merged); the LSD radix
sort of the reference's SortKind::Radix is timed beside it
("variants_queries_per_s") -- both return identical answers.  One step =
one complete batched solve (preprocessing included) with A and the queries
resident in HBM; the L2 is flushed (256 MiB write, then a 256 MiB read that
drains the write's dirty lines) before every step, outside the per-step
CUDA-event window.

    python bench.py [--gpus N --steps K --warmup W] [--impl ours|reference]
                    [--config c2] [--variant con_radix|con_bitmap|bbst] [--no-sweep]

N > 1 (torchrun): every rank solves its own replica of the workload on its own
GPU (the path does not shard on one node here: "replicas", weak scaling), the
step time is the max over ranks, value = N*q / time.

``--impl reference`` times the reference's own CPU pipeline (oracle/_ref, the
reference sources compiled unmodified: collect -> radix sort ->
build_contracted(threads = all cores) -> remap -> ElementSparseTable -> arg_min)
on the same workload; under torchrun only rank 0 runs it.
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (array kind, n, query kind, q, seed offset, default variant, description)
    "c1": (0, 1 << 20, 0, 1000, 1, "con_bitmap", "n=2^20 uniform [0,2^31), q=1e3 uniform endpoints"),
    "c2": (0, 100_000_000, 0, 100_000, 2, "con_bitmap",
           "n=1e8 int32 uniform [0,2^31), q=1e5 uniform endpoints, BbST_CON k=512"),
    "c3": (0, 100_000_000, 1, 10_000_000, 3, "bbst",
           "n=1e8 uniform [0,2^31), q=1e7 log-uniform lengths, BbST (no contraction) k=512"),
    "c4": (1, 1_000_000_000, 2, 1_000_000, 4, "bbst",
           "n=1e9 values in [0,16), q=1e6 half short [1,256] half long, k=512"),
    "c5": (2, 1 << 30, 0, 10_000_000, 5, "bbst",
           "n=2^30 +-1 random walk, q=1e7 uniform endpoints, k=512"),
}
VARIANT_SORT = {"con_radix": 0, "con_bitmap": 2}
SEED0 = 1706069400


def peaks() -> dict:
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return {"hbm_gbs": float(d["hbm_gbs"]), "src": "measured"}
    return {"hbm_gbs": 6650.0, "src": "fallback"}


def gen_workload(name: str, n: int | None = None, q: int | None = None, L=None):
    """The seeded workload of config `name` (include/brmq_workload.h).  L is the
    library exporting brmq_workload_*: libbrmq.so by default; the reference arm
    passes oracle/_ref/libbrmq_ref.so (the same generator source compiled into the
    reference build, oracle/Makefile) so that its process never loads libbrmq.so."""
    ak, n0, qk, q0, c, _, _ = CONFIGS[name]
    n, q = n or n0, q or q0
    if L is None:
        from paper_1706_06940_b200 import _lib
        L = _lib.lib()
    for f in (L.brmq_workload_array, L.brmq_workload_queries):
        f.restype = C.c_int
    L.brmq_workload_array.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_void_p, C.c_uint]
    L.brmq_workload_queries.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_void_p,
                                        C.c_uint]
    A = np.empty(n, np.int32)
    Q = np.empty((q, 2), np.uint64)
    assert L.brmq_workload_array(ak, n, SEED0 + c, A.ctypes.data, 0) == 0
    assert L.brmq_workload_queries(qk, n, q, SEED0 + c, Q.ctypes.data, 0) == 0
    return A, Q


class Clocks:
    """nvidia-smi sampler running during the timed region."""
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu: int):
        self.gpu = gpu
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except FileNotFoundError:
            self.p = None
        return self

    def __exit__(self, *a):
        self.out = ""
        if self.p:
            time.sleep(0.25)
            self.p.terminate()
            try:
                self.out = self.p.communicate(timeout=5)[0]
            except Exception:
                self.p.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in (self.out or "").strip().splitlines():
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ------------------------------------------------------------------ reference arm
def loaded_libraries() -> list[str]:
    """Shared objects mapped into this process (Linux /proc/self/maps)."""
    try:
        with open("/proc/self/maps") as f:
            return sorted({ln.split()[-1] for ln in f if ".so" in ln.split()[-1]})
    except OSError:
        return []


def run_reference(args) -> dict:
    import oracle
    name = args.config
    A, Q = gen_workload(name, L=oracle.ref())
    own = [p for p in loaded_libraries() if p.endswith("libbrmq.so")]
    assert not own, f"reference arm must not load the engine library: {own}"
    q = Q.shape[0]
    th = oracle.nthreads()
    L = oracle.ref()
    out = np.empty(q, np.uint64)
    stage = (C.c_double * 5)()
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        rc = L.ref_solve_oracle(A.ctypes.data, A.shape[0], Q.ctypes.data, q, th, out.ctypes.data, stage)
        dt = time.perf_counter() - t0
        assert rc == 0, rc
        if i >= args.warmup:
            times.append(dt)
    t = statistics.mean(times)
    v = q / t
    return {
        "impl": "reference", "metric": metric_name(), "value": v, "unit": "queries/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": config_dict(name),
        "variant": "reference CPU pipeline: collect -> radix sort -> build_contracted -> remap "
                   "-> ElementSparseTable",
        "cpu_baseline": {"value": v, "unit": "queries/s", "cores": th, "kind": "reference",
                         "sample": f"full {name} workload per step (reference sources compiled "
                                   f"unmodified, build_contracted threads={th})",
                         "stage_ms_last": [x * 1e3 for x in stage]},
        "e2e": {"value": v, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def max_over_ranks(x: float, dist=None, device=None) -> float:
    """Max of a per-rank scalar over all ranks (NCCL on GPU, gloo on CPU)."""
    if dist is None or not dist.is_initialized() or dist.get_world_size() == 1:
        return x
    import torch
    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def aggregate_value(q_per_rank: int, world: int, t_step_ms: float) -> float:
    """Whole-job queries/s: every rank solves q queries; the step ends with the slowest rank."""
    return world * q_per_rank / (t_step_ms * 1e-3)


def metric_name() -> str:
    return "batched RMQ queries/s incl. preprocess (n=1e8 int32); scan GB/s vs HBM peak"


def config_dict(name: str) -> dict:
    """The workload, identical in both arms (the algorithm each arm runs is the
    line's top-level "variant")."""
    ak, n, qk, q, c, _, desc = CONFIGS[name]
    return {"workload": f"{name}: {desc}", "n": n, "q": q, "k": 512,
            "seed": SEED0 + c, "l2": "flushed before every step, outside the timed window: 256 MiB write, then a 256 MiB read (the write's dirty lines drain before the window)",
            "parallelism": "replicas (one independent solve per GPU)"}


# ------------------------------------------------------------------ our arm
def cpu_baseline(A, Q, name) -> dict:
    import oracle
    th = oracle.nthreads()
    out = np.empty(Q.shape[0], np.uint64)
    ts = []
    budget = time.perf_counter() + 20.0
    for _ in range(5):
        t0 = time.perf_counter()
        rc = oracle.ref().ref_solve_oracle(A.ctypes.data, A.shape[0], Q.ctypes.data, Q.shape[0], th,
                                           out.ctypes.data, None)
        ts.append(time.perf_counter() - t0)
        assert rc == 0
        if time.perf_counter() > budget:
            break
    t = statistics.median(ts)
    return {"value": Q.shape[0] / t, "unit": "queries/s", "cores": th, "kind": "reference",
            "sample": f"full {name} workload (n={A.shape[0]}, q={Q.shape[0]}), median of {len(ts)}, "
                      "reference sources compiled unmodified (oracle/_ref)"}, out


class L2Flush:
    """The L2 flush between steps: write a 256 MiB buffer (> the 126 MB L2), then
    read another 256 MiB one, so the write's dirty lines are written back here and
    not inside the next timed window (measured: they cost the c2 solve ~4 us)."""

    def __init__(self, torch, dev):
        self.torch = torch
        self.w = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
        self.r = torch.ones(64 << 20, dtype=torch.int32, device=dev)

    def __call__(self):
        self.w.fill_(1)
        self.torch.max(self.r)


def time_solves(eng, torch, stream, fn, steps, warmup, flush, timing=2, poison=None):
    """Per-step CUDA-event windows on the library stream; L2 flushed between steps.
    timing: library stage events (0 off, 1 every stage, 2 only the roofline kernel).
    poison: called before every step, outside the window (fills the answer buffer
    with 0xFF so a replay that wrote nothing cannot pass the check that follows).
    Async device solves (Engine.set_async) are settled after each window closes."""
    eng.set_timing(timing)
    for _ in range(warmup):
        flush()
        fn()
    torch.cuda.synchronize()
    ms, stage_acc, launches = [], {}, 0
    for _ in range(steps):
        if poison is not None:
            poison()
        flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record(stream)
        fn()
        e.record(stream)
        e.synchronize()
        eng.synchronize()  # (async device solves) the solve's status, outside the window
        ms.append(s.elapsed_time(e))
        for nm, t, nl in eng.stage_times():
            a = stage_acc.setdefault(nm, [0.0, 0])
            a[0] += t
            a[1] += nl
        launches += eng.solve_info()["kernel_launches"]
    return ms, {k: (v[0] / steps, v[1] // steps) for k, v in stage_acc.items()}, launches


def run_ours(args) -> dict:
    import torch
    from paper_1706_06940_b200 import Engine, _lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    if world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    else:
        torch.cuda.set_device(local)
    dev = torch.device("cuda", local)

    name = args.config
    variant = args.variant or CONFIGS[name][5]
    A, Q = gen_workload(name)
    n, q = A.shape[0], Q.shape[0]
    eng = Engine(local)
    # one explicit (non-default) stream shared by torch and the library, so the
    # CUDA events, the L2 flush and the kernels are ordered on the same queue
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    eng.set_stream(stream.cuda_stream)
    # device-pointer solves return once enqueued: the timed window is the device
    # time of the solve, not the host's wake-up after a blocking call (~10 us at
    # c2); time_solves settles each solve's status after its window closes
    eng.set_async(True)
    dA = torch.from_numpy(A).to(dev)
    dQ = torch.from_numpy(Q.view(np.int64)).to(dev)
    dAns = torch.empty(q, dtype=torch.int64, device=dev)
    flush = L2Flush(torch, dev)

    def solve(a=dA, qq=dQ, out=dAns, v=variant):
        if v == "bbst":
            eng.solve_batch_bbst(a, qq, 512, out=out)
        else:
            eng.solve_batch_bbst_con(a, qq, 512, VARIANT_SORT[v], out=out)

    # correctness gate on the bench workload itself (oracle on rank 0 host cores)
    base, want = (None, None)
    if rank == 0 and not args.no_cpu:
        base, want = cpu_baseline(A, Q, name)
    solve()
    torch.cuda.synchronize()
    if want is not None:
        got = dAns.cpu().numpy().view(np.uint64)
        assert np.array_equal(got, want), "bench answers differ from the reference oracle"

    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    # Timed region: K solves with no stage events inside the replayed graph (an event
    # node costs ~5-7 us of serialisation each on this part, measured with
    # tools/timing_modes.py).  The roofline kernel is then timed by CUDA events
    # around it in a second K-step pass of the same workload (timing level 2).
    poison = lambda: dAns.fill_(-1)  # noqa: E731

    def check(tag, buf=None):
        if want is None:
            return None
        got = (dAns if buf is None else buf).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, want), f"{tag}: answers of the last replay differ from the oracle"
        return True

    with Clocks(local) as clk:
        ms, _, launches = time_solves(eng, torch, stream, solve, args.steps, args.warmup, flush,
                                      timing=0, poison=poison)
        checks = {"timed": check("timed region")}
        ms_roof, stages, _ = time_solves(eng, torch, stream, solve, args.steps, 1, flush, timing=2,
                                         poison=poison)
        checks["roofline_pass"] = check("roofline pass")
    torch.cuda.synchronize()
    # per-stage breakdown (every stage bracketed by events; informative, not the headline)
    _, breakdown, _ = time_solves(eng, torch, stream, solve, 5, 1, flush, timing=1, poison=poison)
    checks["stage_pass"] = check("per-stage pass")
    # preprocess vs query (timing level 3: one event pair around everything before
    # the query kernel, one around the query -- 4 event nodes instead of 2 per stage)
    _, phases, _ = time_solves(eng, torch, stream, solve, args.steps, 1, flush, timing=3, poison=poison)
    checks["phase_pass"] = check("two-phase pass")
    # the other endpoint-sort pipeline on the same workload (same answers)
    variants = {variant: aggregate_value(q, 1, statistics.mean(ms))}
    if variant != "bbst":
        alt = "con_bitmap" if variant == "con_radix" else "con_radix"
        ms_alt, _, _ = time_solves(eng, torch, stream, lambda: solve(v=alt), args.steps, 2, flush,
                                   timing=0, poison=poison)
        checks[alt] = check(alt)
        variants[alt] = aggregate_value(q, 1, statistics.mean(ms_alt))
    t_step = max_over_ranks(statistics.mean(ms), dist, dev)
    if dist:
        dist.barrier()
    info = eng.solve_info()

    # e2e: the public C-ABI with pinned HOST buffers, copies inside the window
    L = _lib.lib()
    hp = C.c_void_p()
    nbytes_a, nbytes_q, nbytes_o = n * 4, q * 16, q * 8
    assert L.brmq_host_alloc(C.byref(hp), nbytes_a + nbytes_q + nbytes_o) == 0
    base_ptr = hp.value
    C.memmove(base_ptr, A.ctypes.data, nbytes_a)
    C.memmove(base_ptr + nbytes_a, Q.ctypes.data, nbytes_q)
    hA = np.ctypeslib.as_array((C.c_int32 * n).from_address(base_ptr))
    hQ = np.ctypeslib.as_array((C.c_uint64 * (2 * q)).from_address(base_ptr + nbytes_a)).reshape(q, 2)
    hO = np.ctypeslib.as_array((C.c_uint64 * q).from_address(base_ptr + nbytes_a + nbytes_q))

    def solve_host():
        if variant == "bbst":
            eng.solve_batch_bbst(hA, hQ, 512, out=hO)
        else:
            eng.solve_batch_bbst_con(hA, hQ, 512, VARIANT_SORT[variant], out=hO)

    e2e_ms, _, _ = time_solves(eng, torch, stream, solve_host, max(3, args.steps // 2), 2, flush,
                               timing=0, poison=lambda: hO.fill(np.uint64(0xFFFFFFFFFFFFFFFF)))
    e2e_t = statistics.mean(e2e_ms)
    if want is not None:
        assert np.array_equal(hO, want), "e2e answers differ from the reference oracle"
        checks["e2e"] = True
    # the link's own rate for the same bytes (pinned H2D copy, nothing else): the
    # denominator of e2e's roofline
    dcopy = torch.empty(nbytes_a + nbytes_q, dtype=torch.uint8, device=dev)
    hcopy = torch.from_numpy(np.ctypeslib.as_array((C.c_uint8 * (nbytes_a + nbytes_q)).from_address(base_ptr)))
    pcie = []
    for it in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            e0.record(stream)
            dcopy.copy_(hcopy, non_blocking=True)
            e1.record(stream)
        e1.synchronize()
        if it:
            pcie.append(e0.elapsed_time(e1))
    h2d_peak = (nbytes_a + nbytes_q) / (min(pcie) * 1e-3) / 1e9
    del dcopy
    L.brmq_host_free(hp)
    e2e_t = max_over_ranks(e2e_t, dist, dev)

    # the same through PAGEABLE host buffers (numpy arrays, as the reference's
    # std::vector callers pass them): the library stages them through a pinned
    # double-buffered ring (csrc/staging.h) instead of the driver's bounce buffer
    pA, pQ = np.ascontiguousarray(A), np.ascontiguousarray(Q)
    pO = np.empty(q, np.uint64)

    def solve_pageable():
        if variant == "bbst":
            eng.solve_batch_bbst(pA, pQ, 512, out=pO)
        else:
            eng.solve_batch_bbst_con(pA, pQ, 512, VARIANT_SORT[variant], out=pO)

    pg_ms, _, _ = time_solves(eng, torch, stream, solve_pageable, max(3, args.steps // 2), 2, flush,
                              timing=0, poison=lambda: pO.fill(np.uint64(0xFFFFFFFFFFFFFFFF)))
    pg_t = max_over_ranks(statistics.mean(pg_ms), dist, dev)
    if want is not None:
        assert np.array_equal(pO, want), "pageable e2e answers differ from the reference oracle"
        checks["e2e_pageable"] = True

    # roofline of the dominant kernel
    pk = peaks()
    dom = max(breakdown.items(), key=lambda kv: kv[1][0])[0]
    if variant == "bbst":
        alg_bytes = 4 * n  # block_argmin reads A once
        dom_for_roof = "block_argmin"
    else:
        span = info["span_hi"] - info["span_lo"] + 1
        aq = max(info["boundary"] - 1, 0)
        alg_bytes = 4 * span + 8 * aq  # A span read + packed A_Q written
        dom_for_roof = "contract"
    kt = stages.get(dom_for_roof, (float("nan"), 0))[0]
    achieved = alg_bytes / (kt * 1e-3) / 1e9 if kt > 0 else None
    traffic = None
    tp = ROOT / "profiles" / "traffic.json"
    if tp.exists():
        traffic = json.loads(tp.read_text()).get(f"{name}/{variant}/{dom_for_roof}")
    pre_ms = phases.get("preprocess", (float("nan"),))[0]
    pre_bytes = 4 * n if variant == "bbst" else 4 * (info["span_hi"] - info["span_lo"] + 1) + 16 * q + 8 * max(info["boundary"] - 1, 0)

    rec = {
        "metric": metric_name(), "value": aggregate_value(q, world, t_step), "unit": "queries/s",
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic", "config": config_dict(name), "variant": variant,
        "e2e": {"value": aggregate_value(q, world, e2e_t), "unit": "queries/s",
                "h2d_bytes_per_step": nbytes_a + nbytes_q, "d2h_bytes_per_step": nbytes_o,
                "ms_per_step": e2e_t,
                "roofline": {"bound": "pcie", "achieved": (nbytes_a + nbytes_q + nbytes_o) / (e2e_t * 1e-3) / 1e9,
                             "peak": h2d_peak, "unit": "GB/s",
                             "frac": (nbytes_a + nbytes_q + nbytes_o) / (e2e_t * 1e-3) / 1e9 / h2d_peak,
                             "peak_src": "measured live: one pinned cudaMemcpyAsync H2D of the step's input "
                                         "bytes (best of 4)"}},
        "e2e_pageable": {"value": aggregate_value(q, world, pg_t), "unit": "queries/s",
                         "h2d_bytes_per_step": nbytes_a + nbytes_q, "d2h_bytes_per_step": nbytes_o,
                         "ms_per_step": pg_t,
                         "note": "numpy (pageable) host buffers, staged through a pinned ring"},
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": dom_for_roof, "achieved": achieved,
                     "peak": pk["hbm_gbs"], "peak_src": pk["src"], "unit": "GB/s",
                     "frac": (achieved / pk["hbm_gbs"]) if achieved else None,
                     "traffic": traffic, "alg_bytes_per_launch": alg_bytes,
                     "avg_launch_ms": kt, "launches_timed": args.steps,
                     "method": "CUDA events on the library stream around the kernel, second "
                               "K-step pass (step time with those events: "
                               f"{statistics.mean(ms_roof):.4f} ms)"},
        "preprocess": {"ms": pre_ms, "alg_bytes": pre_bytes,
                       "gbs": pre_bytes / (pre_ms * 1e-3) / 1e9 if pre_ms > 0 else None,
                       "frac": pre_bytes / (pre_ms * 1e-3) / 1e9 / pk["hbm_gbs"] if pre_ms > 0 else None,
                       "query_ms": phases.get("query", (float("nan"),))[0],
                       "method": "timing level 3: a CUDA event on the stream before the solve's graph launch "
                                 "and an event node before the query kernel; every kernel of the solve up to "
                                 "the query (query_ms: event nodes around the query kernel)"},
        "stages_ms": {k: round(v[0], 5) for k, v in breakdown.items()},
        "dominant_stage": dom,
        "variants_queries_per_s": variants,
        "bit_exact_vs_reference": checks,
        "clocks": clk.summary(),
        "info": info,
    }
    if base is not None:
        rec["cpu_baseline"] = base
    if rank == 0 and args.sweep and world == 1:
        rec["sweep"] = run_sweep(eng, torch, stream, flush, dA, A, args)
        # BbST_CON vs the ST-RMQ_CON baseline, per q (time ratio)
        ms = {(p["q"], p["variant"]): p["ms"] for p in rec["sweep"]}
        rec["baseline_relation"] = {
            str(q): {"st_rmq_con_ms": ms[(q, "st_rmq_con")],
                     "speedup_con_radix": ms[(q, "st_rmq_con")] / ms[(q, "con_radix")],
                     "speedup_con_bitmap": ms[(q, "st_rmq_con")] / ms[(q, "con_bitmap")]}
            for q in sorted({p["q"] for p in rec["sweep"]})}
        del dA, dQ, dAns
        torch.cuda.empty_cache()
        rec["configs"] = run_configs(eng, torch, stream, flush, args)
    eng.close()
    if dist:
        dist.destroy_process_group()
    return rec if rank == 0 else None


def run_shard(args) -> dict | None:
    """--shard: one array split over the ranks.  Rank g holds the
    contiguous shard g of an array of N x n(config) elements (weak scaling: the
    shard per GPU is the config's n, the batch is N x q(config) queries over the
    whole array); every step is one sharded BbST_CON solve per rank
    (brmq_solve_bbst_con_shard on device buffers) plus ONE NCCL all_reduce(MIN)
    of the q packed keys (8q bytes), which leaves the answers on every rank."""
    import torch
    from paper_1706_06940_b200 import Engine, SortKind, _lib
    from paper_1706_06940_b200 import shard as S

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    import torch.distributed as dist
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29531")
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)

    name = args.config
    ak, n0, qk, q0, c, _, desc = CONFIGS[name]
    if ak not in (0, 1):
        raise SystemExit(f"--shard: config {name}'s array is not slice-generated")
    n_total, q = n0 * world, q0 * world
    off, ns = S.shard_bounds(n_total, world, rank)
    L = _lib.lib()
    A = np.empty(ns, np.int32)
    assert L.brmq_workload_array_range(ak, n_total, SEED0 + c, off, ns, A.ctypes.data, 0) == 0
    Q = np.empty((q, 2), np.uint64)
    assert L.brmq_workload_queries(qk, n_total, q, SEED0 + c, Q.ctypes.data, 0) == 0
    eng = Engine(local)
    stream = torch.cuda.Stream(dev)
    torch.cuda.set_stream(stream)
    eng.set_stream(stream.cuda_stream)
    dA = torch.from_numpy(A).to(dev)
    dQ = torch.from_numpy(Q.view(np.int64)).to(dev)
    dK = torch.empty(q, dtype=torch.int64, device=dev)
    flush = L2Flush(torch, dev)

    def step():
        return S.solve_sharded(eng, dA, dQ, off, n_total, 512, contraction=True,
                               sort_kind=SortKind.Bitmap, out=dK)

    want = None
    if rank == 0 and not args.no_cpu and n_total * 4 <= (4 << 30):
        import oracle
        Afull = np.empty(n_total, np.int32)
        assert L.brmq_workload_array(ak, n_total, SEED0 + c, Afull.ctypes.data, 0) == 0
        want = oracle.solve_oracle(Afull, Q)
        del Afull
    for _ in range(max(args.warmup, 3)):
        flush()
        step()
    torch.cuda.synchronize()
    dist.barrier()
    ms = []
    for _ in range(args.steps):
        dK.fill_(-1)
        flush()
        s_, e_ = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s_.record(stream)
        ans = step()
        e_.record(stream)
        e_.synchronize()
        ms.append(s_.elapsed_time(e_))
    torch.cuda.synchronize()
    ok = None
    if want is not None:
        ok = bool(np.array_equal(ans.cpu().numpy().view(np.uint64), want))
        assert ok, "sharded answers differ from the reference oracle"
    t = max_over_ranks(statistics.mean(ms), dist, dev)
    dist.barrier()
    backend = dist.get_backend()
    eng.close()
    dist.destroy_process_group()
    if rank != 0:
        return None
    return {
        "metric": metric_name(), "value": q / (t * 1e-3), "unit": "queries/s", "n_gpus": world,
        "steps": args.steps, "warmup": max(args.warmup, 3), "ms_per_step": t,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic",
        "config": {"workload": f"{name} sharded: {desc}; array of N x n elements split in N "
                               f"contiguous shards, N x q queries over the whole array",
                   "n_total": n_total, "n_per_gpu": n0, "q": q, "k": 512, "seed": SEED0 + c,
                   "l2": "flushed before every step, outside the timed window",
                   "parallelism": f"shard{world} (SURVEY 8e: per-shard BbST_CON + one NCCL "
                                  "all_reduce(MIN) of packed keys)"},
        "variant": "con_bitmap_shard",
        "comm": {"collective": "all_reduce(MIN) int64", "bytes_per_step": 8 * q,
                 "backend": backend},
        "bit_exact_vs_reference": ok,
    }


def run_sweep(eng, torch, stream, flush, dA, A, args) -> list:
    """North-star sweep: end-to-end queries/s at n = 1e8 for q = 1e3 .. 1e7, every
    variant (device-resident inputs).  The answer buffer is poisoned before every
    step and the last replay of each point is checked against the reference
    pipeline (oracle/_ref) on the host."""
    import oracle
    from paper_1706_06940_b200 import _lib
    L = _lib.lib()
    n = A.shape[0]
    out = []
    for q in (1_000, 10_000, 100_000, 1_000_000, 10_000_000):
        Q = np.empty((q, 2), np.uint64)
        L.brmq_workload_queries(0, n, q, SEED0 + 2, Q.ctypes.data, 0)
        want = None if args.no_cpu else oracle.solve_oracle(A, Q)
        dQ = torch.from_numpy(Q.view(np.int64)).to(dA.device)
        dO = torch.empty(q, dtype=torch.int64, device=dA.device)
        for v in ("con_radix", "con_bitmap", "bbst", "st_rmq_con"):
            def f(v=v):
                if v == "bbst":
                    eng.solve_batch_bbst(dA, dQ, 512, out=dO)
                elif v == "st_rmq_con":  # the paper's baseline (SPEC "baseline" module)
                    eng.solve_batch_st_rmq_con(dA, dQ, out=dO)
                else:
                    eng.solve_batch_bbst_con(dA, dQ, 512, VARIANT_SORT[v], out=dO)
            pz = lambda: dO.fill_(-1)  # noqa: E731
            ms, _, _ = time_solves(eng, torch, stream, f, 5, 2, flush, timing=0, poison=pz)
            ok = None if want is None else bool(np.array_equal(dO.cpu().numpy().view(np.uint64), want))
            _, stages, _ = time_solves(eng, torch, stream, f, 2, 0, flush, timing=1)
            t = statistics.mean(ms)
            out.append({"q": q, "variant": v, "queries_per_s": q / (t * 1e-3), "ms": t,
                        "bit_exact_vs_reference": ok,
                        "stages_ms": {k: round(x[0], 5) for k, x in stages.items()}})
    return out


def run_configs(eng, torch, stream, flush, args) -> dict:
    """Every BASELINE.json configuration at full size, every engine variant, each
    answer set checked against the reference pipeline (oracle/_ref) on the host."""
    import oracle
    out = {}
    for name in ("c1", "c3", "c4", "c5"):
        A, Q = gen_workload(name)
        q = Q.shape[0]
        t0 = time.perf_counter()
        want = None if args.no_cpu else oracle.solve_oracle(A, Q)
        t_cpu = time.perf_counter() - t0
        dA = torch.from_numpy(A).to("cuda")
        dQ = torch.from_numpy(Q.view(np.int64)).to("cuda")
        dO = torch.empty(q, dtype=torch.int64, device="cuda")
        res = {"n": int(A.shape[0]), "q": q}
        if want is not None:
            res["cpu_reference_queries_per_s"] = q / t_cpu
        variants = {
            "bbst": lambda: eng.solve_batch_bbst(dA, dQ, 512, out=dO),
            "bbst_ml_32_512": lambda: eng.solve_batch_bbst_ml(dA, dQ, (32, 512), out=dO),
            "con_radix": lambda: eng.solve_batch_bbst_con(dA, dQ, 512, 0, out=dO),
            "con_bitmap": lambda: eng.solve_batch_bbst_con(dA, dQ, 512, 2, out=dO),
            "st_rmq_con": lambda: eng.solve_batch_st_rmq_con(dA, dQ, out=dO),
        }
        for v, f in variants.items():
            pz = lambda: dO.fill_(-1)  # noqa: E731
            ms, _, _ = time_solves(eng, torch, stream, f, 5, 3, flush, timing=0, poison=pz)
            ok = None if want is None else bool(np.array_equal(dO.cpu().numpy().view(np.uint64), want))
            _, stages, _ = time_solves(eng, torch, stream, f, 2, 0, flush, timing=1)
            t = statistics.mean(ms)
            res[v] = {"queries_per_s": q / (t * 1e-3), "ms": t, "bit_exact_vs_reference": ok,
                      "stages_ms": {k: round(x[0], 5) for k, x in stages.items()}}
            if v == "bbst" and "query" in stages:
                # query-phase roofline: algorithmic bytes 24 q + 4 S, S =
                # cells the speculation rule scans, from the kernel's debug counter
                # (one extra, untimed solve)
                eng.set_counters(True)
                f()
                S = eng.solve_info()["scanned_cells"]
                eng.set_counters(False)
                qb = 24 * q + 4 * S
                qms = stages["query"][0]
                pk = peaks()["hbm_gbs"]
                res[v]["query_roofline"] = {
                    "scanned_cells": int(S), "scanned_per_query": S / q, "alg_bytes": int(qb),
                    "query_ms": qms, "achieved_gbs": qb / (qms * 1e-3) / 1e9,
                    "frac": qb / (qms * 1e-3) / 1e9 / pk, "peak_gbs": pk}
        out[name] = res
        del dA, dQ, dO, A, Q, want
        torch.cuda.empty_cache()
    return out


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--config", choices=sorted(CONFIGS), default="c2")
    ap.add_argument("--variant", choices=["con_radix", "con_bitmap", "bbst"], default=None)
    ap.add_argument("--no-sweep", dest="sweep", action="store_false")
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline / oracle gate")
    ap.add_argument("--shard", action="store_true",
                    help="one array split over the ranks + one NCCL min-allreduce per step (SURVEY 8e)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "ours" else args.warmup
    if args.impl == "reference":
        if int(os.environ.get("RANK", "0")) != 0:
            return
        print(json.dumps(run_reference(args)))
        return
    rec = run_shard(args) if args.shard else run_ours(args)
    if rec is not None:
        print(json.dumps(rec))


if __name__ == "__main__":
    main()
