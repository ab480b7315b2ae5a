"""CPU tests: pin the oracle (oracle/oracle.c) to the reference.

1. SPEC.md worked examples (tests/golden/spec_examples.json).
2. Golden fixtures produced by the reference's own compiled code
   (tests/golden/ref_cases.npz, generator tests/golden/make_golden.py):
   every stage output must be reproduced bit-exactly.
3. Fresh seeded instances: oracle/oracle.c vs the compiled reference
   (oracle/_ref) when it is present, and vs a pure-numpy argmin.
No GPU needed.
"""
import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

import oracle

GOLD = Path(__file__).parent / "golden"
P = oracle._p


def port():
    return oracle.port()


@pytest.fixture(scope="module")
def spec():
    return json.loads((GOLD / "spec_examples.json").read_text())


@pytest.fixture(scope="module")
def cases():
    return np.load(GOLD / "ref_cases.npz")


def _q(pairs):
    return np.array(pairs, np.uint64).reshape(-1, 2)


# ---------------------------------------------------------------- SPEC examples
def test_spec_naive_and_est(spec):
    L = port()
    for ex in spec["naive_rmq"] + spec["element_st_rmq"]:
        A = np.array(ex["A"], np.int32)
        out = C.c_uint64()
        assert L.orc_naive_rmq(P(A), A.shape[0], ex["q"][0], ex["q"][1], C.byref(out)) == 0
        assert out.value == ex["answer"], ex
    for ex in spec["element_st_rmq"]:
        A = np.array(ex["A"], np.int32)
        h = C.c_void_p()
        assert L.orc_est_build(P(A), A.shape[0], C.byref(h)) == 0
        out = C.c_uint64()
        assert L.orc_est_arg_min(h, P(A), A.shape[0], ex["q"][0], ex["q"][1], C.byref(out)) == 0
        assert out.value == ex["answer"]
        L.orc_est_free(h)
    for ex in spec["element_sparse_table"]:
        A = np.array(ex["A"], np.int32)
        h = C.c_void_p()
        assert L.orc_est_build(P(A), A.shape[0], C.byref(h)) == 0
        rows = []
        for e in range(L.orc_est_level_count(h)):
            buf = np.empty(A.shape[0], np.uint32)
            rows.append(list(buf[: L.orc_est_level(h, e, P(buf))]))
        if "levels" in ex:
            assert rows == ex["levels"]
        else:
            e, j = ex["entry"]
            assert rows[e][j] == ex["value"]
        L.orc_est_free(h)
    # empty input -> invalid_argument (element_sparse_table.cpp:11)
    assert L.orc_est_build(None, 0, C.byref(C.c_void_p())) == 3


def test_spec_floor_log2(spec):
    L = port()
    for ex in spec["floor_log2"]:
        out = C.c_uint32()
        rc = L.orc_floor_log2(ex["x"], C.byref(out))
        if "error" in ex:
            assert rc == 1  # domain_error
        else:
            assert rc == 0 and out.value == ex["out"]


def test_spec_contraction(spec):
    L = port()
    for ex in spec["collect_endpoints"]:
        Q = _q(ex["Q"])
        eps = np.empty(2 * 2 * Q.shape[0], np.uint32)
        assert L.orc_collect_endpoints(P(Q), Q.shape[0], P(eps)) == 0
        assert list(eps[0::2]) == ex["positions"]
    for ex in spec["sort_endpoints"]:
        eps = np.zeros(2 * len(ex["positions"]), np.uint32)
        eps[0::2] = ex["positions"]
        for kind in (0, 1):
            e = eps.copy()
            assert L.orc_sort_endpoints(P(e), len(ex["positions"]), kind) == 0
            assert list(e[0::2]) == ex["sorted"]
    for ex in spec["build_contracted"]:
        A = np.array(ex["A"], np.int32)
        Q = _q(ex["Q"])
        m = 2 * Q.shape[0]
        eps = np.empty(2 * m, np.uint32)
        L.orc_collect_endpoints(P(Q), Q.shape[0], P(eps))
        L.orc_sort_endpoints(P(eps), m, 0)
        aqv, aqo, bnd = np.empty(m, np.int32), np.empty(m, np.uint64), np.empty(m, np.uint64)
        nb = C.c_uint64()
        assert L.orc_build_contracted(P(A), A.shape[0], P(eps), m, 1, P(aqv), P(aqo), P(bnd),
                                      C.byref(nb), None) == 0
        areas = max(nb.value - 1, 0)
        assert list(bnd[: nb.value]) == ex["boundary"]
        assert list(aqv[:areas]) == ex["aq_values"]
        assert list(aqo[:areas]) == ex["aq_origin"]
    for ex in spec["remap_queries"]:
        A = np.array(ex["A"], np.int32)
        Q = _q(ex["Q"])
        q, m = Q.shape[0], 2 * Q.shape[0]
        eps = np.empty(2 * m, np.uint32)
        L.orc_collect_endpoints(P(Q), q, P(eps))
        L.orc_sort_endpoints(P(eps), m, 0)
        aqv, aqo, bnd = np.empty(m, np.int32), np.empty(m, np.uint64), np.empty(m, np.uint64)
        nb = C.c_uint64()
        L.orc_build_contracted(P(A), A.shape[0], P(eps), m, 1, P(aqv), P(aqo), P(bnd), C.byref(nb), None)
        cl, cr, dg = np.empty(q, np.uint32), np.empty(q, np.uint32), np.empty(q, np.uint8)
        assert L.orc_remap_from_sorted(P(eps), m, P(bnd), nb.value, q, P(cl), P(cr), P(dg)) == 0
        assert list(cl[dg == 0]) == [x for x, d in zip(ex["cleft"], ex["degenerate"]) if not d]
        assert list(cr[dg == 0]) == [x for x, d in zip(ex["cright"], ex["degenerate"]) if not d]
        assert list(dg) == ex["degenerate"]


def test_spec_block_sparse_and_solve(spec):
    L = port()
    for ex in spec["build_block_sparse"]:
        v = np.array(ex["values"], np.int32)
        b = (v.shape[0] + ex["k"] - 1) // ex["k"]
        table = np.empty(max(b * ex["levels"], 1), np.uint64)
        bb, lv = C.c_uint64(), C.c_uint32()
        assert L.orc_build_block_sparse(P(v), v.shape[0], ex["k"], P(table), C.byref(bb), C.byref(lv)) == 0
        assert (bb.value, lv.value) == (ex["b"], ex["levels"])
        assert list(table[:b]) == ex["level0"]
        if "entry_1_0" in ex:
            assert table[b] == ex["entry_1_0"]
    for ex in spec["solve"]:
        A = np.array(ex["A"], np.int32)
        Q = _q(ex["Q"])
        for k in ([ex["k"]] if "k" in ex else [1, 2, 3, 512]):
            assert list(oracle.solve_bbst_port(A, Q, k)[0]) == ex["answers"]
            assert list(oracle.solve_bbst_con_port(A, Q, k)[0]) == ex["answers"]
        assert list(oracle.solve_oracle(A, Q, use_ref=False)) == ex["answers"]


# ---------------------------------------------------------------- golden fixtures
def test_golden_fixtures_reproduced(cases):
    """The C restatement reproduces every stage the compiled reference produced."""
    L = port()
    names = [str(c).split(":")[0] for c in cases["cases"]]
    for c in names:
        A, Q = cases[f"{c}_A"], cases[f"{c}_Q"]
        n, q = A.shape[0], Q.shape[0]
        m = 2 * q
        eps = np.empty(2 * m, np.uint32)
        assert L.orc_collect_endpoints(P(Q), q, P(eps)) == 0
        assert np.array_equal(eps, cases[f"{c}_collected"]), c
        assert L.orc_sort_endpoints(P(eps), m, 0) == 0
        ref_sorted = cases[f"{c}_sorted"]
        if m >= 64:  # the reference radix sort is stable; below 64 it calls std::sort
            assert np.array_equal(eps, ref_sorted), c
        else:
            assert np.array_equal(eps[0::2], ref_sorted[0::2]), c
            eps = ref_sorted.copy()
        aqv, aqo, bnd = np.empty(m, np.int32), np.empty(m, np.uint64), np.empty(m, np.uint64)
        nb, reads = C.c_uint64(), C.c_uint64()
        assert L.orc_build_contracted(P(A), n, P(eps), m, 1, P(aqv), P(aqo), P(bnd), C.byref(nb),
                                      C.byref(reads)) == 0
        nbv = nb.value
        assert np.array_equal(bnd[:nbv], cases[f"{c}_boundary"]), c
        assert np.array_equal(aqv[: max(nbv - 1, 0)], cases[f"{c}_aq_values"]), c
        assert np.array_equal(aqo[: max(nbv - 1, 0)], cases[f"{c}_aq_origin"]), c
        assert reads.value == int(cases[f"{c}_array_reads"][0]), c  # ContractionStats (serial)
        cl, cr, dg = np.empty(q, np.uint32), np.empty(q, np.uint32), np.empty(q, np.uint8)
        assert L.orc_remap_from_sorted(P(eps), m, P(bnd), nbv, q, P(cl), P(cr), P(dg)) == 0
        assert np.array_equal(cl, cases[f"{c}_cleft"]) and np.array_equal(cr, cases[f"{c}_cright"]), c
        assert np.array_equal(dg, cases[f"{c}_degenerate"]), c
        want = cases[f"{c}_answers"]
        assert np.array_equal(oracle.solve_oracle(A, Q, use_ref=False), want), c
        for k in (1, 2, 7, 64, 512):
            assert np.array_equal(oracle.solve_bbst_port(A, Q, k)[0], want), (c, k)
            assert np.array_equal(oracle.solve_bbst_con_port(A, Q, k)[0], want), (c, k)
        assert np.array_equal(oracle.naive_numpy(A, Q), want), c
        if f"{c}_est_levels" in cases:
            h = C.c_void_p()
            assert L.orc_est_build(P(A), n, C.byref(h)) == 0
            rows = []
            for e in range(L.orc_est_level_count(h)):
                buf = np.empty(n, np.uint32)
                rows.append(buf[: L.orc_est_level(h, e, P(buf))])
            assert np.array_equal(np.concatenate(rows), cases[f"{c}_est_levels"]), c
            assert L.orc_est_cell_count(h) == int(cases[f"{c}_est_cells"][0])
            L.orc_est_free(h)


@pytest.mark.skipif(not oracle.ref_available(), reason="compiled reference (oracle/_ref) absent")
def test_port_vs_compiled_reference_random():
    r = np.random.default_rng(424242)
    for trial in range(40):
        n = int(r.integers(1, 20000))
        q = int(r.integers(1, 3000))
        kind = trial % 4
        A = [r.integers(0, 2**31, n), r.integers(0, 2, n), r.integers(0, 16, n),
             r.integers(-(2**31), 2**31, n)][kind].astype(np.int32)
        a, b = r.integers(0, n, q), r.integers(0, n, q)
        Q = np.stack([a, b], 1).astype(np.uint64)  # unnormalised pairs: the Query ctor swaps
        want = oracle.solve_oracle(A, Q, threads=3, use_ref=True)
        assert np.array_equal(oracle.solve_oracle(A, Q, threads=3, use_ref=False), want)
        assert np.array_equal(oracle.solve_bbst_port(A, Q, 512)[0], want)
        assert np.array_equal(oracle.solve_bbst_con_port(A, Q, 64, threads=2)[0], want)


def test_bbst_speculation_counter():
    """S (cells scanned) is zero when every query is covered by stored block minima
     and grows with k for random queries."""
    A = np.arange(4096, dtype=np.int32)[::-1].copy()  # strictly decreasing: min at the right end
    Q = np.array([[i * 512, i * 512 + 1023] for i in range(6)], np.uint64)
    ans, S, _ = oracle.solve_bbst_port(A, Q, 512)
    assert np.array_equal(ans, Q[:, 1]) and S == 0
    r = np.random.default_rng(5)
    A = r.integers(0, 2**31, 100_000).astype(np.int32)
    a, b = r.integers(0, 100_000, 20_000), r.integers(0, 100_000, 20_000)
    Q = np.stack([np.minimum(a, b), np.maximum(a, b)], 1).astype(np.uint64)
    s = [oracle.solve_bbst_port(A, Q, k)[1] for k in (16, 128, 1024)]
    assert s[0] < s[1] < s[2]


def test_error_codes():
    L = port()
    A = np.arange(10, dtype=np.int32)
    out = C.c_uint64()
    assert L.orc_naive_rmq(P(A), 10, 0, 10, C.byref(out)) == 2  # out_of_range
    eps = np.array([5, 0, 3, 1], np.uint32)  # unsorted
    aqv, aqo, bnd = np.empty(2, np.int32), np.empty(2, np.uint64), np.empty(2, np.uint64)
    nb = C.c_uint64()
    assert L.orc_build_contracted(P(A), 10, P(eps), 2, 1, P(aqv), P(aqo), P(bnd), C.byref(nb), None) == 3
    sorted_eps = np.array([3, 0, 5, 1], np.uint32)
    bad_boundary = np.array([3], np.uint64)
    cl, cr, dg = np.empty(1, np.uint32), np.empty(1, np.uint32), np.empty(1, np.uint8)
    assert L.orc_remap_from_sorted(P(sorted_eps), 2, P(bad_boundary), 1, 1, P(cl), P(cr), P(dg)) == 4


def test_remap_queries_binary_search():
    """contraction.cpp:152-171 remap_queries: SPEC worked instance, agreement with the
    merge walk (remap_queries_from_sorted) on non-degenerate queries of the golden
    fixtures, a missing end -> logic_error, and the compiled reference when present."""
    L = port()
    bnd = np.array([1, 3, 4, 6], np.uint64)
    Q = _q([[1, 4], [6, 3], [2, 2]])
    cl, cr, dg = np.empty(3, np.uint32), np.empty(3, np.uint32), np.empty(3, np.uint8)
    assert L.orc_remap_queries(P(Q), 3, P(bnd), 4, P(cl), P(cr), P(dg)) == 0
    assert list(cl) == [0, 1, 0] and list(cr) == [1, 2, 0] and list(dg) == [0, 0, 1]
    assert L.orc_remap_queries(P(_q([[0, 4]])), 1, P(bnd), 4, P(cl), P(cr), P(dg)) == 4
    cases = np.load(GOLD / "ref_cases.npz")
    for c in [str(x).split(":")[0] for x in cases["cases"]]:
        Q, b = cases[f"{c}_Q"], cases[f"{c}_boundary"]
        q = Q.shape[0]
        cl, cr, dg = np.empty(q, np.uint32), np.empty(q, np.uint32), np.empty(q, np.uint8)
        assert L.orc_remap_queries(P(Q), q, P(b), b.shape[0], P(cl), P(cr), P(dg)) == 0
        keep = cases[f"{c}_degenerate"] == 0
        assert np.array_equal(dg, cases[f"{c}_degenerate"]), c
        assert np.array_equal(cl[keep], cases[f"{c}_cleft"][keep]), c
        assert np.array_equal(cr[keep], cases[f"{c}_cright"][keep]), c
        assert not cl[~keep].any() and not cr[~keep].any(), c
        if oracle.ref_available():
            rl, rr, rd = np.empty(q, np.uint32), np.empty(q, np.uint32), np.empty(q, np.uint8)
            assert oracle.ref().ref_remap_queries(P(Q), q, P(b), b.shape[0], P(rl), P(rr), P(rd)) == 0
            assert np.array_equal(rl, cl) and np.array_equal(rr, cr) and np.array_equal(rd, dg), c

