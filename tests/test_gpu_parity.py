"""Parity of the CUDA path (through the C-ABI) against the CPU oracle.

Bar: bit-exact leftmost-minimum positions (integer work).  The oracle is the
reference's own code compiled under oracle/_ref when present (it travels with
the gpurun snapshot) and the C restatement oracle/liboracle.so otherwise; for
small cases a pure-numpy argmin is checked too.
"""
import numpy as np
import pytest

from paper_1706_06940_b200 import (ENDPOINT_DTYPE, InvalidArgument, LogicError, OutOfRange,
                                   SortKind, make_queries)

pytestmark = pytest.mark.gpu

KS = [1, 2, 3, 7, 8, 64, 128, 256, 512, 1024, 2048, 4096]
VARIANTS = ["bbst", "bbst_ml", "con_radix", "con_bitmap", "st_rmq_con"]


def _values(r, n, kind):
    if kind == "uniform":
        return r.integers(0, 2**31, n, dtype=np.int64).astype(np.int32)
    if kind == "binary":
        return r.integers(0, 2, n).astype(np.int32)
    if kind == "ties16":
        return r.integers(0, 16, n).astype(np.int32)
    if kind == "signed":
        v = r.integers(-(2**31), 2**31, n, dtype=np.int64).astype(np.int32)
        v[r.integers(0, n, max(1, n // 50))] = np.iinfo(np.int32).min
        v[r.integers(0, n, max(1, n // 50))] = np.iinfo(np.int32).max
        return v
    if kind == "const_max":
        return np.full(n, np.iinfo(np.int32).max, np.int32)
    if kind == "walk":
        s = np.cumsum(np.where(r.integers(0, 2, n) == 1, 1, -1)).astype(np.int64)
        return (s - s.min()).astype(np.int32)
    raise ValueError(kind)


def _queries(r, n, q, kind):
    if kind == "uniform":
        a, b = r.integers(0, n, q), r.integers(0, n, q)
    elif kind == "short":
        a = r.integers(0, n, q)
        b = np.minimum(a + r.integers(0, 40, q), n - 1)
    elif kind == "mixed":
        a = r.integers(0, n, q)
        ln = np.where(r.random(q) < 0.5, r.integers(1, 700, q), r.integers(1, n + 1, q))
        b = np.minimum(a + ln - 1, n - 1)
    elif kind == "degenerate":
        a = r.integers(0, n, q)
        b = a.copy()
    elif kind == "reversed":
        a, b = r.integers(0, n, q), r.integers(0, n, q)
        Q = np.empty((q, 2), np.uint64)
        Q[:, 0], Q[:, 1] = np.maximum(a, b), np.minimum(a, b)  # left > right: normalised
        return Q
    else:
        raise ValueError(kind)
    return np.stack([np.minimum(a, b), np.maximum(a, b)], 1).astype(np.uint64)


def _solve(engine, variant, A, Q, k):
    if variant == "bbst":
        return engine.solve_batch_bbst(A, Q, k)
    if variant == "bbst_ml":  # multi-level [32, k]; k must be a multiple of 32 above 32
        if k == 0:
            return engine.solve_batch_bbst_ml(A, Q, (32, 0))
        return engine.solve_batch_bbst_ml(A, Q, (32, k if k % 32 == 0 and k > 32 else 512))
    if variant == "st_rmq_con":  # the baseline has no block size
        return engine.solve_batch_st_rmq_con(A, Q)
    kind = SortKind.Radix if variant == "con_radix" else SortKind.Bitmap
    return engine.solve_batch_bbst_con(A, Q, k, kind)


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("vkind", ["uniform", "binary", "ties16", "signed", "const_max", "walk"])
def test_random_small_all_k(engine, orc, variant, vkind):
    r = np.random.default_rng(hash((variant, vkind)) % 2**32)
    for trial in range(6):
        n = int(r.integers(1, 6000))
        q = int(r.integers(1, 1500))
        A = _values(r, n, vkind)
        qk = ["uniform", "short", "mixed", "degenerate", "reversed", "uniform"][trial]
        Q = _queries(r, n, q, qk)
        want = orc.naive_numpy(A, Q)
        for k in KS:
            got = _solve(engine, variant, A, Q, k)
            bad = np.nonzero(got != want)[0]
            assert bad.size == 0, (variant, vkind, qk, n, q, k, bad[:5], got[bad[:5]], want[bad[:5]])


@pytest.mark.parametrize("variant", VARIANTS)
def test_spec_worked_instance(engine, variant):
    # A=[5,3,8,2,7,6,9,1], queries (1,4),(3,6) -> [3,3]
    A = np.array([5, 3, 8, 2, 7, 6, 9, 1], np.int32)
    Q = make_queries([1, 3], [4, 6])
    for k in (1, 2, 3, 512):
        assert list(_solve(engine, variant, A, Q, k)) == [3, 3]
    # SPEC.md:64-66, 82-84
    assert list(_solve(engine, variant, np.array([7], np.int32), make_queries([0], [0]), 512)) == [0]
    assert list(_solve(engine, variant, np.array([2, 2, 2], np.int32), make_queries([0], [2]), 2)) == [0]
    assert list(_solve(engine, variant, A, make_queries([0, 4], [7, 4]), 2)) == [7, 4]


@pytest.mark.parametrize("variant", VARIANTS)
def test_edge_cases(engine, orc, variant):
    A = np.arange(100, 0, -1, dtype=np.int32)
    # empty batch -> empty answers
    assert _solve(engine, variant, A, np.zeros((0, 2), np.uint64), 512).shape == (0,)
    # all queries identical
    Q = np.tile(np.array([[10, 90]], np.uint64), (777, 1))
    assert (_solve(engine, variant, A, Q, 8) == 90).all()
    # full-range and single-element arrays
    assert list(_solve(engine, variant, np.array([5], np.int32), make_queries([0], [0]), 1)) == [0]
    # out of range -> std::out_of_range
    with pytest.raises(OutOfRange):
        _solve(engine, variant, A, make_queries([0], [100]), 512)
    # k = 0 -> invalid_argument (BbstConParams invariant k >= 1)
    if variant != "st_rmq_con":  # no block size
        with pytest.raises(InvalidArgument):
            _solve(engine, variant, A, make_queries([0], [5]), 0)
    # the engine is still healthy after an error
    assert list(_solve(engine, variant, A, make_queries([3], [9]), 4)) == [9]


def test_multilevel_configs(engine, orc):
    r = np.random.default_rng(31)
    A = _values(r, 70_001, "ties16")
    Q = _queries(r, 70_001, 20_000, "mixed")
    want = orc.naive_numpy(A, Q)
    for ks in [(512,), (32, 64), (32, 96), (32, 128), (32, 512), (32, 1024), (32, 4096)]:
        assert np.array_equal(engine.solve_batch_bbst_ml(A, Q, ks), want), ks
    # short ranges over sorted runs with ties: most queries descend to rows
    A2 = np.sort(_values(r, 70_010, "ties16").reshape(10, 7001), axis=1)
    A2[1::2] = A2[1::2, ::-1]  # ascending and descending runs
    A2 = np.ascontiguousarray(A2).ravel()
    for kind in ("short", "uniform"):
        Q2 = _queries(r, A2.shape[0], 20_000, kind)
        want2 = orc.naive_numpy(A2, Q2)
        for ks in [(32, 64), (32, 512)]:
            assert np.array_equal(engine.solve_batch_bbst_ml(A2, Q2, ks), want2), (kind, ks)
    # short ranges straddling a block boundary: both sides descend, each to one
    # partial row (the right side's row lies in its first sub-block)
    A3 = _values(r, 50_000, "uniform")
    for k in (64, 128, 256, 512):
        edge = (r.integers(1, 50_000 // k, 5000) * k).astype(np.int64)
        Q3 = np.stack([edge - r.integers(1, 40, 5000), edge + r.integers(0, 40, 5000)], 1)
        Q3 = np.clip(Q3, 0, 49_999).astype(np.uint64)
        assert np.array_equal(engine.solve_batch_bbst_ml(A3, Q3, (32, k)), orc.naive_numpy(A3, Q3)), k
    # BbST_CON's sub-block level over A_Q (power-of-two k in [64, 512]): many short
    # queries make A_Q long and the contracted ranges short -- sides and rows in
    # A_Q index space, inside-tests on original positions (ties16: equal keys)
    A4 = _values(r, 200_000, "ties16")
    for kind in ("short", "mixed"):
        Q4 = _queries(r, 200_000, 60_000, kind)
        want4 = orc.naive_numpy(A4, Q4)
        for k in (64, 256, 512):
            for sk in (SortKind.Bitmap, SortKind.Radix):
                assert np.array_equal(engine.solve_batch_bbst_con(A4, Q4, k, sk), want4), (kind, k, sk)
    for bad in [(32, 48), (32, 16), (7, 7), (0, 4), (2, 4, 6), tuple(2 ** i for i in range(1, 10))]:
        with pytest.raises(InvalidArgument):
            engine.solve_batch_bbst_ml(A, Q, bad)
    # unaligned device pointer (scalar fallbacks)
    torch = pytest.importorskip("torch")
    dA = torch.from_numpy(np.concatenate([[0], A]).astype(np.int32)).cuda()[1:]
    dQ = torch.from_numpy(Q.view(np.int64)).cuda()
    assert np.array_equal(engine.solve_batch_bbst_ml(dA, dQ, (32, 512)).cpu().numpy().view(np.uint64), want)
    assert np.array_equal(engine.solve_batch_bbst(dA, dQ, 512).cpu().numpy().view(np.uint64), want)


def test_multilevel_general_chains(engine, orc):
    """oracle equality for cfg in {[1],[2],[7],[k],[k1,k2],[k1,k2,k3]}
    with randomized dividing chains, n <= 1e5 (query_chain.cu for every chain
    other than [k] and [32, k])."""
    A = np.array([5, 3, 8, 2, 7, 6, 9, 1], np.int32)  # SPEC.md:287-298 worked instance
    assert list(engine.solve_batch_bbst_ml(A, np.array([[0, 7]], np.uint64), (2, 4))) == [7]
    assert list(engine.solve_batch_bbst_ml(A, np.array([[1, 4], [3, 6]], np.uint64), (2, 4))) == [3, 3]
    r = np.random.default_rng(2024)
    fixed = [(1, 2), (2, 4), (1, 4, 64), (2, 4, 8), (3, 6, 24), (7, 14), (16, 512), (64, 512),
             (32, 64, 512), (4, 16, 64, 256, 1024), (1, 2, 4, 8, 16, 32, 64, 128), (5, 25, 125, 625)]
    chains = list(fixed)
    for _ in range(10):  # randomized dividing chains
        h = int(r.integers(2, 5))
        ks = [int(r.integers(1, 9))]
        for _ in range(h - 1):
            ks.append(ks[-1] * int(r.integers(2, 6)))
        chains.append(tuple(ks))
    for trial, ks in enumerate(chains):
        n = int(r.integers(1, 100_000))
        vkind = ["uniform", "ties16", "walk", "binary"][trial % 4]
        qk = ["uniform", "short", "mixed", "degenerate"][trial % 4]
        A = _values(r, n, vkind)
        Q = _queries(r, n, int(r.integers(1, 5000)), qk)
        got = engine.solve_batch_bbst_ml(A, Q, ks)
        want = orc.naive_numpy(A, Q)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (ks, n, vkind, qk, bad[:5], got[bad[:5]], want[bad[:5]])
    # range errors and empty batches behave as on the other paths
    with pytest.raises(Exception):
        engine.solve_batch_bbst_ml(A, np.array([[0, A.shape[0]]], np.uint64), (2, 4))
    assert engine.solve_batch_bbst_ml(A, np.zeros((0, 2), np.uint64), (2, 4)).shape[0] == 0


def test_device_pointers(engine, orc):
    torch = pytest.importorskip("torch")
    r = np.random.default_rng(7)
    A = _values(r, 200_000, "ties16")
    Q = _queries(r, 200_000, 50_000, "mixed")
    want = orc.solve_oracle(A, Q)
    dA = torch.from_numpy(A).cuda()
    dQ = torch.from_numpy(Q.view(np.int64)).cuda()
    for variant in VARIANTS:
        if variant == "bbst":
            out = engine.solve_batch_bbst(dA, dQ, 512)
        elif variant == "bbst_ml":
            out = engine.solve_batch_bbst_ml(dA, dQ, (32, 512))
        else:
            out = engine.solve_batch_bbst_con(dA, dQ, 512,
                                              SortKind.Radix if variant == "con_radix" else SortKind.Bitmap)
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want), variant


def _solve_into(engine, variant, dA, dQ, out):
    if variant == "bbst":
        return engine.solve_batch_bbst(dA, dQ, 512, out=out)
    if variant == "bbst_ml":
        return engine.solve_batch_bbst_ml(dA, dQ, (32, 512), out=out)
    if variant == "bbst_ml3":
        return engine.solve_batch_bbst_ml(dA, dQ, (8, 64, 512), out=out)
    if variant == "st_rmq_con":
        return engine.solve_batch_st_rmq_con(dA, dQ, out=out)
    kind = SortKind.Radix if variant == "con_radix" else SortKind.Bitmap
    return engine.solve_batch_bbst_con(dA, dQ, 512, kind, out=out)


def test_graph_replays_poisoned(engine, orc):
    """Device-pointer solves are captured once into a CUDA graph and replayed
    (api.cu run_solve): every replay must rewrite every answer.  The output is
    filled with 0xFF before each call, shapes and q are interleaved so that the
    look-back epochs, the persistent bitmap and the control header are reused
    across graphs, and every replay is checked (naive.hpp:13-21, leftmost)."""
    torch = pytest.importorskip("torch")
    r = np.random.default_rng(31)
    cases = []
    for n, q, vk, qk in ((300_000, 40_000, "ties16", "mixed"), (1_000_003, 100_000, "uniform", "uniform"),
                         (70_001, 5_000, "walk", "short"), (1_000_003, 7, "binary", "uniform")):
        A = _values(r, n, vk)
        Q = _queries(r, n, q, qk)
        cases.append((torch.from_numpy(A).cuda(), torch.from_numpy(Q.view(np.int64)).cuda(),
                      torch.empty(q, dtype=torch.int64, device="cuda"), orc.solve_oracle(A, Q)))
    variants = VARIANTS + ["bbst_ml3"]
    for rep in range(3):
        for ci, (dA, dQ, out, want) in enumerate(cases):
            for variant in variants:
                out.fill_(-1)
                _solve_into(engine, variant, dA, dQ, out)
                got = out.cpu().numpy().view(np.uint64)
                bad = np.nonzero(got != want)[0]
                assert bad.size == 0, (rep, ci, variant, bad[:5])


def test_async_device_solves(engine, orc):
    """brmq_ctx_set_async (brmq.h): device-pointer solves return once enqueued and
    brmq_synchronize returns their status -- the answers, the exceptions the
    synchronous call raises (naive.hpp:14-15 range check) and the solve info
    must be the same; a call with an async solve outstanding settles it first."""
    torch = pytest.importorskip("torch")
    r = np.random.default_rng(77)
    n, q = 500_000, 60_000
    A = _values(r, n, "ties16")
    Q = _queries(r, n, q, "mixed")
    want = orc.solve_oracle(A, Q)
    dA = torch.from_numpy(A).cuda()
    dQ = torch.from_numpy(Q.view(np.int64)).cuda()
    variants = ["bbst", "bbst_ml", "bbst_ml3", "con_radix", "con_bitmap"]
    outs = {v: torch.empty(q, dtype=torch.int64, device="cuda") for v in variants}
    bad = torch.from_numpy(make_queries([0, 5], [n - 1, n]).view(np.int64)).cuda()
    engine.set_async(True)
    try:
        for rep in range(2):
            for v in variants:  # one at a time
                outs[v].fill_(-1)
                torch.cuda.synchronize()
                _solve_into(engine, v, dA, dQ, outs[v])
                engine.synchronize()
                assert np.array_equal(outs[v].cpu().numpy().view(np.uint64), want), (rep, v)
            for v in variants:  # back to back: each call settles the one before
                outs[v].fill_(-1)
            torch.cuda.synchronize()
            for v in variants:
                _solve_into(engine, v, dA, dQ, outs[v])
            engine.synchronize()
            for v in variants:
                assert np.array_equal(outs[v].cpu().numpy().view(np.uint64), want), (rep, v, "b2b")
            info = engine.solve_info()  # of the last (BbST_CON) solve
            assert info["boundary"] > 0 and info["blocks"] > 0
            # a failing solve reports at synchronize(), and the next one is clean
            engine.solve_batch_bbst_con(dA, bad, 512, SortKind.Bitmap,
                                        out=torch.empty(2, dtype=torch.int64, device="cuda"))
            with pytest.raises(OutOfRange):
                engine.synchronize()
            engine.solve_batch_bbst(dA, bad, 512, out=torch.empty(2, dtype=torch.int64, device="cuda"))
            with pytest.raises(OutOfRange):  # settled by the next call
                _solve_into(engine, "con_bitmap", dA, dQ, outs["con_bitmap"])
            _solve_into(engine, "con_bitmap", dA, dQ, outs["con_bitmap"])
            engine.synchronize()
            assert np.array_equal(outs["con_bitmap"].cpu().numpy().view(np.uint64), want)
            # switching the context's stream settles the outstanding solve first
            outs["bbst"].fill_(-1)
            torch.cuda.synchronize()
            _solve_into(engine, "bbst", dA, dQ, outs["bbst"])
            other = torch.cuda.Stream()
            engine.set_stream(other.cuda_stream)
            assert np.array_equal(outs["bbst"].cpu().numpy().view(np.uint64), want)
            engine.set_stream(None)
    finally:
        engine.set_async(False)


@pytest.mark.slow
def test_positions_above_2_31(engine, orc):
    """n = 2^31 + 4099 (the reference allows n up to 2^32 - 1,
    element_sparse_table.cpp:12-13; Endpoint.pos is uint32, contraction.hpp:13):
    the top half of the 32-bit position range through every vectorised / flat
    query path, both endpoint sorts and the multi-level [32, 512] solve."""
    torch = pytest.importorskip("torch")
    from paper_1706_06940_b200 import _lib
    L = _lib.lib()
    n = (1 << 31) + 4099
    A = np.empty(n, np.int32)
    assert L.brmq_workload_array(1, n, 1706069499, A.ctypes.data, 0) == 0  # ties: values in [0, 16)
    # a planted unique minimum above 2^31 and one exactly at 2^31
    A[(1 << 31) + 1000] = -5
    A[1 << 31] = -3
    r = np.random.default_rng(2 ** 31)
    top = 1 << 31
    qs = [
        r.integers(0, n, (2000, 2)),                                     # uniform
        top - 600 + r.integers(0, 1200, (1000, 2)),                      # straddle 2^31
        n - 1 - r.integers(0, 3000, (1000, 2)),                          # the last blocks
        np.stack([r.integers(top, n, 1000), r.integers(top, n, 1000)], 1),  # top half only
    ]
    sh = r.integers(top, n - 600, 1000)                                  # short, in-block
    qs.append(np.stack([sh, sh + r.integers(0, 600, 1000)], 1))
    Q = np.concatenate(qs).astype(np.uint64)
    Q = np.stack([Q.min(1), Q.max(1)], 1).astype(np.uint64)
    want = orc.solve_oracle(A, Q)
    dA = torch.from_numpy(A).cuda()
    del A
    dQ = torch.from_numpy(Q.view(np.int64)).cuda()
    out = torch.empty(Q.shape[0], dtype=torch.int64, device="cuda")
    for variant in ("bbst", "bbst_ml", "con_bitmap", "con_radix"):
        out.fill_(-1)
        _solve_into(engine, variant, dA, dQ, out)
        got = out.cpu().numpy().view(np.uint64)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (variant, bad[:5], Q[bad[:5]])
    assert (want[(Q[:, 0] <= top + 1000) & (Q[:, 1] >= top + 1000)] == top + 1000).all()
    del dA
    torch.cuda.empty_cache()


# ------------------------------------------------------------------ stage parity
def test_stage_collect_sort(engine, orc):
    import ctypes as C
    r = np.random.default_rng(11)
    for q in (0, 1, 5, 31, 32, 33, 1000, 100_000):
        n = 1_000_003
        Q = _queries(r, n, q, "uniform")
        eps = engine.collect_endpoints(Q)
        want = np.empty(2 * q, ENDPOINT_DTYPE)
        orc.port().orc_collect_endpoints(orc._p(Q), q, orc._p(want))
        assert np.array_equal(eps, want)
        # device radix sort is stable: identical to the reference Radix order
        got = engine.sort_endpoints(eps.copy())
        ref = want.copy()
        if orc.ref_available():
            orc.ref().ref_sort_endpoints(orc._p(ref), 2 * q, 0)
        else:
            orc.port().orc_sort_endpoints(orc._p(ref), 2 * q, 0)
        if 2 * q >= 64:
            assert np.array_equal(got, ref), q
        else:  # reference uses std::sort below 64 endpoints: order of equal pos unspecified
            assert np.array_equal(got["pos"], ref["pos"])
            assert np.array_equal(np.sort(got.view(np.uint64)), np.sort(ref.view(np.uint64)))
    # full 32-bit keys
    e = np.empty(50_000, ENDPOINT_DTYPE)
    e["pos"] = r.integers(0, 2**32, e.shape[0], dtype=np.uint64).astype(np.uint32)
    e["origin"] = np.arange(e.shape[0], dtype=np.uint32)
    got = engine.sort_endpoints(e.copy())
    order = np.argsort(e["pos"], kind="stable")
    assert np.array_equal(got, e[order])


def test_stage_contract_remap(engine, orc):
    r = np.random.default_rng(12)
    for n, q, vk in [(1, 1, "uniform"), (50, 3, "binary"), (10_000, 100, "ties16"),
                     (300_000, 20_000, "uniform"), (100_000, 70_000, "walk"), (9000, 5, "signed")]:
        A = _values(r, n, vk)
        Q = _queries(r, n, q, "uniform")
        eps = np.empty(2 * q, ENDPOINT_DTYPE)
        orc.port().orc_collect_endpoints(orc._p(Q), q, orc._p(eps))
        orc.port().orc_sort_endpoints(orc._p(eps), 2 * q, 0)
        stats = {}
        con = engine.build_contracted(A, eps, stats)
        m = 2 * q
        aqv = np.empty(m, np.int32)
        aqo = np.empty(m, np.uint64)
        bnd = np.empty(m, np.uint64)
        import ctypes as C
        nb = C.c_uint64()
        reads = C.c_uint64()
        orc.port().orc_build_contracted(orc._p(A), n, orc._p(eps), m, 1, orc._p(aqv), orc._p(aqo),
                                        orc._p(bnd), C.byref(nb), C.byref(reads))
        nbv = nb.value
        # ContractionStats.array_reads (contraction.hpp:47-49): the device counter
        # equals the reference's serial count
        assert stats["array_reads"] == reads.value, (n, q, stats, reads.value)
        assert np.array_equal(con.boundary, bnd[:nbv])
        assert np.array_equal(con.aq_values, aqv[:max(nbv - 1, 0)])
        assert np.array_equal(con.aq_origin, aqo[:max(nbv - 1, 0)])
        cq = engine.remap_queries_from_sorted(eps, con, q)
        cl = np.empty(q, np.uint32)
        cr = np.empty(q, np.uint32)
        dg = np.empty(q, np.uint8)
        orc.port().orc_remap_from_sorted(orc._p(eps), m, orc._p(bnd), nbv, q, orc._p(cl), orc._p(cr),
                                         orc._p(dg))
        assert np.array_equal(cq.cleft, cl)
        assert np.array_equal(cq.cright, cr)
        assert np.array_equal(cq.degenerate, dg.astype(bool))
        # remap_queries: binary search per query (contraction.cpp:152-171)
        bq = engine.remap_queries(Q, con)
        orc.port().orc_remap_queries(orc._p(Q), q, orc._p(bnd), nbv, orc._p(cl), orc._p(cr),
                                     orc._p(dg))
        assert np.array_equal(bq.cleft, cl) and np.array_equal(bq.cright, cr)
        assert np.array_equal(bq.degenerate, dg.astype(bool))


def test_stage_contract_errors(engine):
    A = np.arange(10, dtype=np.int32)
    e = np.zeros(2, ENDPOINT_DTYPE)
    e["pos"] = [5, 3]  # unsorted -> invalid_argument (contraction.cpp:123)
    with pytest.raises(InvalidArgument):
        engine.build_contracted(A, e)
    # the bitmap was cleared: a valid call afterwards is exact
    e["pos"] = [3, 5]
    con = engine.build_contracted(A, e)
    assert list(con.boundary) == [3, 5] and list(con.aq_origin) == [3]
    # endpoint missing from boundary -> logic_error (contraction.cpp:182-183)
    from paper_1706_06940_b200 import ContractedArray
    bad = ContractedArray(np.zeros(0, np.int32), np.zeros(0, np.uint64), np.array([3], np.uint64))
    with pytest.raises(LogicError):
        engine.remap_queries_from_sorted(e, bad, 1)
    with pytest.raises(LogicError):  # contraction.cpp:157-158
        engine.remap_queries(make_queries([3], [5]), bad)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 8, 16, 32, 64, 128, 512])
def test_stage_block_sparse(engine, orc, k):
    import ctypes as C
    r = np.random.default_rng(k)
    # k <= 2 at 2^21 + 777 keys: 22 levels, all three tiled launches (bases 0, 10, 17)
    for m in (1, 2, 5, 1000, 100_000) + (((1 << 21) + 777,) if k <= 2 else ()):
        v = _values(r, m, "ties16")
        table, b, levels = engine.build_block_sparse(v, k)
        ref = np.empty(max(levels * b, 1), np.uint64)
        bb, ll = C.c_uint64(), C.c_uint32()
        orc.port().orc_build_block_sparse(orc._p(v), m, k, orc._p(ref), C.byref(bb), C.byref(ll))
        assert (b, levels) == (bb.value, ll.value)
        assert np.array_equal(table.reshape(-1), ref[: levels * b])
    # values=[2,2,6], k=2 -> level0 [0,2], (1,0) = 0
    t, b, lv = engine.build_block_sparse(np.array([2, 2, 6], np.int32), 2)
    assert (b, lv) == (2, 2) and list(t[0]) == [0, 2] and t[1][0] == 0


# ------------------------------------------------------------------ BASELINE configs
from conftest import ROOT  # noqa: E402

CONFIGS = {
    # name: (array kind, n, query kind, q, seed offset)
    "c1": (0, 1 << 20, 0, 1000, 1),
    "c2": (0, 100_000_000, 0, 100_000, 2),
    "c3": (0, 100_000_000, 1, 10_000_000, 3),
    "c4": (1, 1_000_000_000, 2, 1_000_000, 4),
    "c5": (2, 1 << 30, 0, 10_000_000, 5),
}


def _workload(name, n=None, q=None):
    import ctypes as C
    from paper_1706_06940_b200 import _lib
    ak, n0, qk, q0, c = CONFIGS[name]
    n = n or n0
    q = q or q0
    L = _lib.lib()
    A = np.empty(n, np.int32)
    Q = np.empty((q, 2), np.uint64)
    assert L.brmq_workload_array(ak, n, 1706069400 + c, A.ctypes.data, 0) == 0
    assert L.brmq_workload_queries(qk, n, q, 1706069400 + c, Q.ctypes.data, 0) == 0
    return A, Q


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_configs_reduced(engine, orc, name):
    """Every config's generators and variants at sizes the oracle finishes in seconds."""
    sizes = {"c1": (None, None), "c2": (2_000_000, 20_000), "c3": (2_000_000, 400_000),
             "c4": (4_000_000, 100_000), "c5": (1 << 22, 400_000)}
    A, Q = _workload(name, *sizes[name])
    want = orc.solve_oracle(A, Q)
    for variant in VARIANTS:
        got = _solve(engine, variant, A, Q, 512)
        assert np.array_equal(got, want), (name, variant, np.nonzero(got != want)[0][:5])


@pytest.mark.slow
@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_configs_full(engine, orc, name):
    """BASELINE.json full sizes: bit-exact against the reference pipeline
    (collect -> radix sort -> build_contracted -> ElementSparseTable), plus
    size-independent properties (range membership, value = A[answer])."""
    A, Q = _workload(name)
    want = orc.solve_oracle(A, Q)
    for variant in VARIANTS:
        got = _solve(engine, variant, A, Q, 512)
        assert np.array_equal(got, want), (name, variant, np.nonzero(got != want)[0][:5])
    assert ((got >= Q[:, 0]) & (got <= Q[:, 1])).all()


def test_workspace_reuse_sequence(engine, orc):
    """Solves of different shapes back to back on one context: the grow-only
    workspace holds stale data from earlier calls, which must never be read as
    live look-back status (regression: status words now live in their own arena)."""
    r = np.random.default_rng(99)
    n = 3_000_000
    A = _values(r, n, "uniform")
    Qbig = _queries(r, n, 300_000, "uniform")
    assert np.array_equal(engine.solve_batch_bbst_con(A, Qbig, 512, SortKind.Radix),
                          orc.solve_oracle(A, Qbig))
    for q in (1_000, 100_000, 10, 250_000, 3_000, 600_000, 1):
        Q = _queries(r, n, q, "uniform" if q % 2 else "mixed")
        want = orc.solve_oracle(A, Q)
        for variant in VARIANTS:
            got = _solve(engine, variant, A, Q, 512)
            assert np.array_equal(got, want), (q, variant, np.nonzero(got != want)[0][:5])


def test_control_block_protocol(engine, orc):
    """Solves leave the device control header zeroed for the next solve (no memset
    in their graphs); stage calls and failed solves leave it dirty and the next
    solve must re-zero it.  Interleave them all and check every answer."""
    r = np.random.default_rng(2024)
    n = 400_000
    A = _values(r, n, "ties16")
    Qs = [_queries(r, n, q, kind) for q, kind in ((5000, "uniform"), (70_000, "mixed"), (300, "short"))]
    wants = [orc.solve_oracle(A, Q) for Q in Qs]
    eps = engine.collect_endpoints(Qs[0])
    for rep in range(2):
        for Q, want in zip(Qs, wants):
            for variant in VARIANTS:
                assert np.array_equal(_solve(engine, variant, A, Q, 512), want), (rep, variant)
            engine.sort_endpoints(eps.copy())  # stage call: header dirty
            assert np.array_equal(_solve(engine, "con_bitmap", A, Q, 512), want)
            with pytest.raises(OutOfRange):  # failed solve
                engine.solve_batch_bbst_con(A, make_queries([0], [n]), 512, SortKind.Bitmap)
            assert np.array_equal(_solve(engine, "con_radix", A, Q, 512), want)
            engine.build_block_sparse(A[:1000], 8)  # stage call
            assert np.array_equal(_solve(engine, "bbst", A, Q, 512), want)


def test_pageable_host_buffers_staged(engine, orc):
    """Host-pointer solves with pageable (numpy) buffers larger than the staging
    ring's 16 MiB chunks (csrc/staging.h): A of 80 MB + 3 bytes' worth of odd
    tail, answers of 24 MB (two D2H chunks), every variant against the oracle;
    and a pinned buffer through the direct path."""
    r = np.random.default_rng(4242)
    n = 20_000_003
    A = _values(r, n, "ties16")
    Q = _queries(r, n, 3_000_001, "mixed")
    want = orc.solve_oracle(A, Q)
    for variant in ("bbst", "con_bitmap", "con_radix", "bbst_ml"):
        got = _solve(engine, variant, A, Q, 512)
        bad = np.nonzero(got != want)[0]
        assert bad.size == 0, (variant, bad[:5])


def test_scan_counter_matches_oracle(engine, orc):
    """The debug scan-cell counter of the BbST (h = 1) query kernel (SPEC.md:249,
    :472 instrumented counter) equals the C restatement's S on the same inputs:
    both apply the same leftmost-exact speculation rule."""
    r = np.random.default_rng(77)
    for n, q, vk, qk in ((1_000_000, 100_000, "uniform", "mixed"), (300_007, 50_000, "ties16", "short"),
                         (2_000_000, 20_000, "walk", "uniform")):
        A = _values(r, n, vk)
        Q = _queries(r, n, q, qk)
        want, S, _ = orc.solve_bbst_port(A, Q, 512)
        engine.set_counters(True)
        try:
            got = engine.solve_batch_bbst(A, Q, 512)
            info = engine.solve_info()
        finally:
            engine.set_counters(False)
        assert np.array_equal(got, want)
        # a degenerate query (l == r) is answered directly on the device; the
        # restatement walks answer_one for it and scans the one cell unless the
        # block minimum sits there
        lo = np.minimum(Q[:, 0], Q[:, 1]).astype(np.int64)
        deg = lo[Q[:, 0] == Q[:, 1]]
        blk = deg // 512
        bmin = np.array([b * 512 + int(np.argmin(A[b * 512:min(n, b * 512 + 512)])) for b in blk], np.int64)
        S_dev = S - int(np.count_nonzero(bmin != deg))
        assert info["scanned_cells"] == S_dev, (n, q, info["scanned_cells"], S, S_dev)
    engine.solve_batch_bbst(A, Q, 512)
    assert engine.solve_info()["scanned_cells"] == 0  # off again


@pytest.mark.parametrize("n", [130, 1000, 4097, 65_541, (1 << 20) + 3, 3_000_001])
def test_radix_msd_partition(engine, orc, n):
    """The radix pipeline's two-level sort + dedup (radix_sort.cu
    launch_radix_partition_mark: an MSD partition by the top digit, then a
    counting digit per bucket in shared memory), used from 2^14 endpoints: key
    widths 8..22 bits, n just above a power of two (the last bucket runs past
    the bitmap), every endpoint inside one bucket, heavy duplicates, and the
    out-of-range error -- against the oracle and the bitmap pipeline."""
    r = np.random.default_rng(n)
    A = _values(r, n, "ties16" if n % 2 else "uniform")
    q = 12_000
    cases = [_queries(r, n, q, "uniform"), _queries(r, n, q, "short")]
    lo = n // 3
    a = r.integers(lo, min(n, lo + 100), q)  # one bucket (or two) holds every endpoint
    b = np.minimum(a + r.integers(0, 60, q), n - 1)
    cases.append(np.stack([np.minimum(a, b), np.maximum(a, b)], 1).astype(np.uint64))
    cases.append(np.tile(np.array([[lo, n - 1]], np.uint64), (q, 1)))  # 2q copies of two keys
    for Q in cases:
        want = orc.solve_oracle(A, Q)
        for kind in (SortKind.Radix, SortKind.Bitmap):
            for k in (8, 512):
                got = engine.solve_batch_bbst_con(A, Q, k, kind)
                bad = np.nonzero(got != want)[0]
                assert bad.size == 0, (n, kind, k, bad[:5])
    Q = _queries(r, n, q, "uniform")
    Q[q // 2, 1] = n  # out of range -> std::out_of_range (naive.hpp:14-15)
    with pytest.raises(OutOfRange):
        engine.solve_batch_bbst_con(A, Q, 512, SortKind.Radix)
    assert list(engine.solve_batch_bbst_con(A, make_queries([0], [n - 1]), 512, SortKind.Radix)) == \
        list(orc.solve_oracle(A, make_queries([0], [n - 1])))
