"""Register-spill budget of the built kernels (CPU: reads libbrmq.so with
cuobjdump -res-usage; no GPU).  A spill that slips into a hot instance shows up
as a slower kernel and nothing else: the round-2 control-header publication,
inlined into the BbST h = 1 query, cost it 16 bytes of stack per thread and
0.538 -> 0.578 ms at c3 before this test existed.  Kernels not listed must not
use any stack; the listed ones may not exceed their measured budget."""
import re
import shutil
import subprocess
from pathlib import Path

import pytest

LIB = Path(__file__).resolve().parents[1] / "paper_1706_06940_b200" / "libbrmq.so"

# substring of the mangled name -> max stack bytes (measured, each an A/B'd trade-off)
BUDGET = {
    "k_query_flatINS0_6RowKeyENS0_15QueryContractedELi128": 32,
    "k_query_flatINS0_6RowKeyENS0_17QueryContractedWIELi128": 24,
    "k_query_flatINS0_6RowI32ILb1EEENS0_11QueryDirectELi128": 8,
    "k_query_flatINS0_6RowI32ILb0EEENS0_11QueryDirectELi128": 8,  # unaligned A only
    "k_query_budgetINS0_7ElemKey": 8,
    "k_rs_pass": 16,
}


def _usage():
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not Path(exe).exists() or not LIB.exists():
        pytest.skip("cuobjdump or libbrmq.so missing")
    out = subprocess.run([exe, "-res-usage", str(LIB)], capture_output=True, text=True, check=True).stdout
    names = re.findall(r"Function (\S+):\s*\n\s*REG:(\d+) STACK:(\d+)", out)
    assert names, "no kernels found in libbrmq.so"
    return [(n, int(r), int(s)) for n, r, s in names]


def test_stack_budget():
    bad = []
    for name, _, stack in _usage():
        cap = next((v for k, v in BUDGET.items() if k in name), 0)
        if stack > cap:
            bad.append((name, stack, cap))
    assert not bad, bad


def test_hot_instances_spill_free():
    usage = {n: (r, s) for n, r, s in _usage()}
    hot = ["k_query_budgetINS0_8ElemI32T", "k_contract", "k_msd_partition",
           "k_bucket_mark", "k_block_argmin_i32_vec", "k_st_tile", "k_collect"]
    for h in hot:
        hits = [(n, rs) for n, rs in usage.items() if h in n]
        assert hits, h
        for n, (_, s) in hits:
            assert s == 0, (n, s)
