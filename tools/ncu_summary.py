"""Summaries of ncu output for profiles/ (tooling, not shipped).

  python tools/ncu_summary.py launches <launch list .csv>      per-kernel count / avg / share
  python tools/ncu_summary.py full <report .ncu-rep> [top]     speed-of-light, occupancy,
                                                               stalls, DRAM bytes, hot lines
"""
import csv
import io
import subprocess
import sys
from collections import defaultdict


def launches(path):
    rows = [r for r in csv.reader(l for l in open(path) if not l.startswith("=="))]
    h = rows[0]
    ki, vi, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name")
    agg = defaultdict(list)
    for r in rows[1:]:
        if r[mi] == "gpu__time_duration.sum":
            agg[r[ki].split("(")[0].replace("brmq::<unnamed>::", "")[:44]].append(float(r[vi]) / 1e3)
    tot = sum(sum(v) for v in agg.values())
    print(f"{'kernel':44s} {'count':>6s} {'avg_us':>10s} {'share_%':>9s}")
    for k, v in agg.items():
        print(f"{k:44s} {len(v):6d} {sum(v) / len(v):10.2f} {100 * sum(v) / tot:9.1f}")
    print(f"total launches {sum(len(v) for v in agg.values())}, total {tot:.1f} us")


def _ncu(rep, *args):
    return subprocess.run(["ncu", "-i", rep, *args], capture_output=True, text=True).stdout


def full(rep, top=12):
    want = ("Duration", "DRAM Throughput", "Memory Throughput", "L2 Hit Rate", "Executed Ipc Active",
            "Issue Slots Busy", "Registers Per Thread", "Theoretical Occupancy", "Achieved Occupancy",
            "Grid Size", "Block Size")
    for r in csv.reader(io.StringIO(_ncu(rep, "--page", "details", "--csv"))):
        if len(r) > 14 and r[12] in want:
            print(f"{r[11]} | {r[12]} | {r[14]} {r[13]}")
    rows = list(csv.reader(io.StringIO(_ncu(rep, "--page", "raw", "--csv"))))
    h, v = rows[0], rows[2]
    for k in ("dram__bytes_read.sum", "dram__bytes_write.sum", "smsp__inst_executed.sum",
              "smsp__thread_inst_executed_per_inst_executed.ratio"):
        if k in h:
            print(k, v[h.index(k)], rows[1][h.index(k)])
    st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v[i]) for i, k in enumerate(h)
          if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
          and v[i].replace(".", "").isdigit()}
    tot = sum(st.values()) or 1
    print("stall samples:", ", ".join(f"{k} {100 * x / tot:.0f}%" for k, x in
                                      sorted(st.items(), key=lambda t: -t[1])[:6]))
    out, f = [], None
    for r in csv.reader(io.StringIO(_ncu(rep, "--page", "source", "--csv", "--print-source", "sass,cuda"))):
        if len(r) == 2 and r[0] == "File Path":
            f = r[1].split("/")[-1]
        elif len(r) > 8 and r[0].isdigit():
            try:
                out.append((int(r[7]), int(r[4]), f, r[0], r[1].strip()[:70]))
            except ValueError:
                pass
    ti, ts = sum(o[0] for o in out) or 1, sum(o[1] for o in out) or 1
    print(f"hot source lines (inst %, warp-sample %) of {ti} warp instructions:")
    for o in sorted(out, key=lambda t: -t[1])[:top]:
        print(f"  {100 * o[0] / ti:5.1f} {100 * o[1] / ts:5.1f}  {o[2]}:{o[3]}  {o[4]}")


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2])
    else:
        full(sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 12)
