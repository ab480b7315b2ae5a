"""Generate the golden fixtures from the REFERENCE's own compiled code.

    make -C oracle ref && python tests/golden/make_golden.py

Writes tests/golden/ref_cases.npz: seeded small instances (arrays, query
batches) together with every stage output of the reference pipeline, produced
by oracle/_ref/libbrmq_ref.so (the reference sources compiled unmodified):
collect_endpoints, sort_endpoints(Radix), build_contracted (+ array_reads),
remap_queries_from_sorted, ElementSparseTable levels, and the final answers
(SURVEY 8c pipeline).  The fixtures pin oracle/oracle.c and the CUDA path on
machines without /root/reference.
"""
from __future__ import annotations

import ctypes as C
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
import oracle  # noqa: E402


def _p(a):
    return a.ctypes.data if a.size else 0


def values(r, n, kind):
    if kind == "uniform":
        return r.integers(0, 2**31, n, dtype=np.int64).astype(np.int32)
    if kind == "binary":
        return r.integers(0, 2, n).astype(np.int32)
    if kind == "ties16":
        return r.integers(0, 16, n).astype(np.int32)
    if kind == "signed":
        v = r.integers(-(2**31), 2**31, n, dtype=np.int64).astype(np.int32)
        v[r.integers(0, n, max(1, n // 40))] = np.iinfo(np.int32).min
        v[r.integers(0, n, max(1, n // 40))] = np.iinfo(np.int32).max
        return v
    if kind == "walk":
        s = np.cumsum(np.where(r.integers(0, 2, n) == 1, 1, -1)).astype(np.int64)
        return (s - s.min()).astype(np.int32)
    raise ValueError(kind)


def queries(r, n, q, kind):
    if kind == "uniform":
        a, b = r.integers(0, n, q), r.integers(0, n, q)
    elif kind == "short":
        a = r.integers(0, n, q)
        b = np.minimum(a + r.integers(0, 40, q), n - 1)
    elif kind == "degenerate_mix":
        a = r.integers(0, n, q)
        b = np.where(r.random(q) < 0.3, a, r.integers(0, n, q))
    else:
        raise ValueError(kind)
    return np.stack([np.minimum(a, b), np.maximum(a, b)], 1).astype(np.uint64)


def ref_case(A, Q):
    L = oracle.ref()
    n, q = A.shape[0], Q.shape[0]
    m = 2 * q
    eps = np.empty(2 * m, np.uint32)
    assert L.ref_collect_endpoints(_p(Q), q, _p(eps)) == 0
    collected = eps.copy()
    assert L.ref_sort_endpoints(_p(eps), m, 0) == 0
    aqv = np.empty(max(m, 1), np.int32)
    aqo = np.empty(max(m, 1), np.uint64)
    bnd = np.empty(max(m, 1), np.uint64)
    nb, reads = C.c_uint64(), C.c_uint64()
    assert L.ref_build_contracted(_p(A), n, _p(eps), m, 1, _p(aqv), _p(aqo), _p(bnd), C.byref(nb),
                                  C.byref(reads)) == 0
    nbv = nb.value
    areas = max(nbv - 1, 0)
    cl = np.empty(q, np.uint32)
    cr = np.empty(q, np.uint32)
    dg = np.empty(q, np.uint8)
    assert L.ref_remap_from_sorted(_p(eps), m, _p(bnd), nbv, q, _p(cl), _p(cr), _p(dg)) == 0
    ans = np.empty(q, np.uint64)
    assert L.ref_solve_oracle(_p(A), n, _p(Q), q, 1, _p(ans), None) == 0
    return {
        "collected": collected, "sorted": eps, "boundary": bnd[:nbv].copy(),
        "aq_values": aqv[:areas].copy(), "aq_origin": aqo[:areas].copy(),
        "array_reads": np.array([reads.value], np.uint64),
        "cleft": cl, "cright": cr, "degenerate": dg, "answers": ans,
    }


def est_levels(values_):
    """ElementSparseTable rows of the reference (jagged, concatenated)."""
    L = oracle.ref()
    rc = C.c_int()
    h = L.ref_est_build(_p(values_), values_.shape[0], C.byref(rc))
    assert rc.value == 0 and h
    rows = []
    for e in range(L.ref_est_level_count(h)):
        out = np.empty(values_.shape[0], np.uint32)
        cnt = L.ref_est_level(h, e, _p(out))
        rows.append(out[:cnt].copy())
    cells = L.ref_est_cell_count(h)
    L.ref_est_free(h)
    return np.concatenate(rows), np.array([len(r) for r in rows], np.uint64), cells


def main():
    if not oracle.ref_available():
        raise SystemExit("build the reference first: make -C oracle ref")
    r = np.random.default_rng(1706069400)
    out = {}
    cases = []
    plan = [(1, 1, "uniform", "uniform"), (2, 3, "binary", "uniform"), (8, 2, "uniform", "uniform"),
            (63, 40, "ties16", "short"), (64, 33, "signed", "degenerate_mix"),
            (1000, 500, "uniform", "uniform"), (1000, 500, "binary", "short"),
            (3000, 2000, "ties16", "degenerate_mix"), (4096, 1500, "walk", "uniform"),
            (5000, 100, "signed", "uniform"), (777, 2048, "uniform", "short")]
    for i, (n, q, vk, qk) in enumerate(plan):
        A = values(r, n, vk)
        Q = queries(r, n, q, qk)
        res = ref_case(A, Q)
        out[f"c{i}_A"] = A
        out[f"c{i}_Q"] = Q
        for k, v in res.items():
            out[f"c{i}_{k}"] = v
        if n <= 1000:
            lv, lens, cells = est_levels(A)
            out[f"c{i}_est_levels"] = lv
            out[f"c{i}_est_lens"] = lens
            out[f"c{i}_est_cells"] = np.array([cells], np.uint64)
        cases.append(f"c{i}:{n}:{q}:{vk}:{qk}")
    out["cases"] = np.array(cases)
    path = Path(__file__).with_name("ref_cases.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path} ({path.stat().st_size} bytes, {len(cases)} cases)")


if __name__ == "__main__":
    main()
