"""bench.py's reference arm on CPU (no GPU needed): the JSON line the driver parses.

`--impl reference` times the reference's own CPU pipeline (oracle/_ref, or the
oracle port) on the host; rank 0 alone prints one JSON line, other ranks exit 0.
"""
import json
import os
import subprocess
import sys

from conftest import ROOT


def _run(*args, env=None):
    return subprocess.run([sys.executable, str(ROOT / "bench.py"), *args], capture_output=True,
                          text=True, env={**os.environ, **(env or {})}, timeout=600, cwd=ROOT)


def test_reference_arm_json_line():
    p = _run("--impl", "reference", "--config", "c1", "--steps", "2", "--warmup", "1")
    assert p.returncode == 0, p.stderr[-2000:]
    lines = [l for l in p.stdout.splitlines() if l.strip()]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    assert rec["impl"] == "reference" and rec["unit"] == "queries/s" and rec["value"] > 0
    assert rec["steps"] == 2 and rec["warmup"] == 1 and rec["n_gpus"] == 1
    assert rec["higher_is_better"] is True and rec["config"]["workload"].startswith("c1")
    cb = rec["cpu_baseline"]
    assert cb["kind"] in ("reference", "port") and cb["cores"] >= 1 and cb["value"] == rec["value"]
    assert isinstance(cb["sample"], str) and cb["sample"]
    e2e = rec["e2e"]
    assert e2e["value"] == rec["value"] and e2e["unit"] == rec["unit"]
    assert e2e["h2d_bytes_per_step"] == 0 and e2e["d2h_bytes_per_step"] == 0


def test_reference_arm_other_ranks_silent():
    p = _run("--impl", "reference", "--config", "c1", "--steps", "1", "--warmup", "0",
             env={"RANK": "1", "WORLD_SIZE": "2", "LOCAL_RANK": "1"})
    assert p.returncode == 0 and p.stdout.strip() == ""


def test_reference_arm_never_loads_engine():
    """The reference arm builds its workload with the generator compiled into
    oracle/_ref (oracle/Makefile), so libbrmq.so is never mapped in its process."""
    code = ("import sys, bench, oracle; sys.argv=['bench.py']; "
            "A, Q = bench.gen_workload('c1', L=oracle.ref()); "
            "assert not [p for p in bench.loaded_libraries() if p.endswith('libbrmq.so')]; "
            "from paper_1706_06940_b200 import _lib; _lib.lib(); "
            "B, R = bench.gen_workload('c1'); "
            "assert (A == B).all() and (Q == R).all(); "
            "assert [p for p in bench.loaded_libraries() if p.endswith('libbrmq.so')]; print('ok')")
    p = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, cwd=ROOT,
                       timeout=300)
    assert p.returncode == 0 and p.stdout.strip().endswith("ok"), p.stderr[-2000:]
