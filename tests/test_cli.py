"""The harness command line: gen-array / gen-queries / verify on the
host, `run` for every algorithm on the GPU (cross-algorithm checksum agreement,
SPEC.md:468 acceptance criterion 2)."""
import csv
import subprocess

import numpy as np
import pytest

import oracle
from paper_1706_06940_b200 import _lib
from paper_1706_06940_b200 import harness as H
from paper_1706_06940_b200.build import CLI, build_cli

ALGOS = ["naive", "sparse", "st-rmq-con", "bbst-con", "bbst", "bbst-ml"]


@pytest.fixture(scope="module")
def cli():
    build_cli()
    return str(CLI)


def _run(cli, *args):
    return subprocess.run([cli, *map(str, args)], capture_output=True, text=True)


def test_gen_and_verify(cli, tmp_path):
    a, q, r = tmp_path / "a.rmqa", tmp_path / "q.rmqq", tmp_path / "r.rmqr"
    assert _run(cli, "gen-array", "--n", 20000, "--seed", 5, "--out", a).returncode == 0
    assert _run(cli, "gen-queries", "--n", 20000, "--q", 3000, "--seed", 6, "--out", q).returncode == 0
    A, Q = H.read_array(a), H.read_queries(q)
    # gen-array default = SPEC gen_permutation; gen-queries = uniform endpoints
    want_a = np.empty(20000, np.int32)
    _lib.lib().brmq_workload_array(3, 20000, 5, want_a.ctypes.data, 0)
    assert np.array_equal(A, want_a)
    assert np.array_equal(np.sort(A), np.arange(1, 20001))
    assert (Q[:, 0] <= Q[:, 1]).all() and Q.shape == (3000, 2)
    ans = oracle.naive_numpy(A, Q)
    H.write_answers(r, ans)
    p = _run(cli, "verify", "--array", a, "--queries", q, "--answers", r)
    assert p.returncode == 0, p.stderr
    ans[17] = (ans[17] + 1) % 20000
    H.write_answers(r, ans)
    p = _run(cli, "verify", "--array", a, "--queries", q, "--answers", r)
    assert p.returncode == 2 and "first at query 17" in p.stderr


def test_usage_errors(cli, tmp_path):
    assert _run(cli).returncode == 1
    assert _run(cli, "frobnicate").returncode == 1
    assert _run(cli, "gen-array", "--n", 10).returncode == 1  # missing --seed/--out
    p = _run(cli, "verify", "--array", tmp_path / "nope", "--queries", tmp_path / "nope",
             "--answers", tmp_path / "nope")
    assert p.returncode == 1 and "cannot open" in p.stderr


@pytest.mark.gpu
def test_run_all_algorithms(cli, tmp_path):
    n, q = 100_000, 10_000  # SPEC.md:468 criterion 2 workload size
    a, qf = tmp_path / "a.rmqa", tmp_path / "q.rmqq"
    assert _run(cli, "gen-array", "--n", n, "--seed", 11, "--out", a).returncode == 0
    assert _run(cli, "gen-queries", "--n", n, "--q", q, "--seed", 12, "--out", qf).returncode == 0
    A, Q = H.read_array(a), H.read_queries(qf)
    want = oracle.solve_oracle(A, Q)
    table = tmp_path / "runs.csv"
    for algo in ALGOS:
        extra = ["--chain", "32,512"] if algo == "bbst-ml" else ["--k", "512"]
        r = tmp_path / f"{algo}.rmqr"
        p = _run(cli, "run", "--algo", algo, "--array", a, "--queries", qf, *extra, "--runs", 3,
                 "--csv", table, "--answers", r)
        assert p.returncode == 0, (algo, p.stderr)
        assert np.array_equal(H.read_answers(r), want), algo
        p = _run(cli, "verify", "--array", a, "--queries", qf, "--answers", r)
        assert p.returncode == 0, (algo, p.stderr)
    rows = list(csv.DictReader(open(table)))
    assert [row["algo"] for row in rows] == ALGOS
    assert len({row["answers_checksum"] for row in rows}) == 1  # value-level agreement
    assert int(rows[0]["answers_checksum"]) == H.answers_checksum(A, want)
    for row in rows:
        assert int(row["runs"]) == 3 and float(row["t_total_ns"]) > 0
    by = {row["algo"]: row for row in rows}
    assert int(by["bbst-con"]["extra_bytes"]) == H.account_memory("bbst-con", n, q, (512,))[0]
    assert float(by["bbst-con"]["t_sort_ns"]) > 0 and float(by["bbst-con"]["t_contract_ns"]) > 0
    # a three-level chain through the CLI (query_chain.cu), recorded as k_chain "8;64;512"
    r = tmp_path / "ml3.rmqr"
    p = _run(cli, "run", "--algo", "bbst-ml", "--array", a, "--queries", qf, "--chain", "8,64,512",
             "--runs", 1, "--csv", table, "--answers", r)
    assert p.returncode == 0, p.stderr
    assert np.array_equal(H.read_answers(r), want)
    assert list(csv.DictReader(open(table)))[-1]["k_chain"] == "8;64;512"
    p = _run(cli, "run", "--algo", "bbst-ml", "--array", a, "--queries", qf, "--chain", "8,60",
             "--runs", 1, "--csv", table)
    assert p.returncode != 0  # not a dividing chain
