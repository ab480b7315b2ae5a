"""CPU tests of the C-ABI boundary and the host-side logic (no GPU needed).

* libbrmq.so loads and exports every function include/*.h declares;
* the reference-facing types have the reference's layouts;
* the host-only entry points behave like the reference (floor_log2);
* without a GPU the compute path fails loudly (no CPU fallback);
* the workload generators are deterministic and match a numpy restatement.
"""
import ctypes as C
import re
from pathlib import Path

import numpy as np
import pytest

import paper_1706_06940_b200 as brmq
from paper_1706_06940_b200 import _lib

ROOT = Path(__file__).resolve().parents[1]


def declared_functions():
    names = []
    for h in (ROOT / "include").glob("*.h"):
        text = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        names += re.findall(r"\b(brmq_\w+)\s*\(", text)
    return sorted(set(names))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    decl = declared_functions()
    assert len(decl) >= 25
    missing = [n for n in decl if not hasattr(L, n)]
    assert not missing, missing
    # and the Python binding covers exactly the declared surface
    assert sorted(_lib.SIGNATURES) == decl


def test_nm_exports():
    import shutil
    import subprocess
    if not shutil.which("nm"):
        pytest.skip("nm not available")
    out = subprocess.run(["nm", "-D", "--defined-only", str(_lib.LIB_PATH)], capture_output=True,
                         text=True, check=True).stdout
    syms = set(re.findall(r"\bT (brmq_\w+)", out))
    assert set(declared_functions()) <= syms


def test_reference_layouts():
    # batchrmq::Query is 16 B with left@0 right@8 (types.hpp:13-23, SURVEY probe);
    # batchrmq::Endpoint is 8 B with pos@0 origin@4 (contraction.hpp:12-21)
    assert brmq.QUERY_DTYPE.itemsize == 16 and brmq.QUERY_DTYPE.fields["right"][1] == 8
    assert brmq.ENDPOINT_DTYPE.itemsize == 8 and brmq.ENDPOINT_DTYPE.fields["origin"][1] == 4
    q = brmq.make_queries([5, 1], [2, 9])  # normalising constructor (types.hpp:18-20)
    assert q.tolist() == [(2, 5), (1, 9)]


def test_floor_log2_host():
    assert [brmq.floor_log2(x) for x in (1, 2, 3, 48829, 2**63)] == [0, 1, 1, 15, 63]
    with pytest.raises(brmq.DomainError):
        brmq.floor_log2(0)  # bits.hpp:11


def test_fails_loudly_without_gpu_or_library(monkeypatch):
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(brmq.CudaError):
        brmq.Engine(0)
    # a missing shared object is an ImportError, never a silent fallback
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", ROOT / "does-not-exist.so")
    with pytest.raises(ImportError):
        _lib.lib()


# ---------------------------------------------------------------- workloads
MASK = (1 << 64) - 1


def mix64(z):
    z ^= z >> 30
    z = (z * 0xBF58476D1CE4E5B9) & MASK
    z ^= z >> 27
    z = (z * 0x94D049BB133111EB) & MASK
    z ^= z >> 31
    return z


def draw(seed, stream, i):
    base = mix64(seed ^ ((0xA0761D6478BD642F * (stream + 1)) & MASK))
    return mix64((base + (i + 1) * 0x9E3779B97F4A7C15) & MASK)


def test_workload_generators_match_restatement():
    L = _lib.lib()
    assert L.brmq_workload_mix64(12345) == mix64(12345)
    n, seed = 5000, 1706069401
    for kind, f in ((0, lambda x: x >> 33), (1, lambda x: x >> 60)):
        A = np.empty(n, np.int32)
        assert L.brmq_workload_array(kind, n, seed, A.ctypes.data, 3) == 0
        assert [int(v) for v in A[:200]] == [f(draw(seed, 0, i)) for i in range(200)]
    # random walk: +-1 steps from 0, shifted so the minimum is 0
    A = np.empty(n, np.int32)
    assert L.brmq_workload_array(2, n, seed, A.ctypes.data, 4) == 0
    steps = [0] + [1 if draw(seed, 0, i) & 1 else -1 for i in range(1, n)]
    walk = np.cumsum(steps)
    assert np.array_equal(A, walk - walk.min())
    # uniform queries: mulhi(x, n), swapped so left <= right
    Q = np.empty((300, 2), np.uint64)
    assert L.brmq_workload_queries(0, n, 300, seed, Q.ctypes.data, 2) == 0
    for i in range(300):
        a = (draw(seed, 1, 2 * i) * n) >> 64
        b = (draw(seed, 1, 2 * i + 1) * n) >> 64
        assert (int(Q[i, 0]), int(Q[i, 1])) == (min(a, b), max(a, b))
    # log-uniform and mixed lengths stay inside the array
    for kind in (1, 2):
        Q = np.empty((20000, 2), np.uint64)
        assert L.brmq_workload_queries(kind, n, 20000, seed, Q.ctypes.data, 0) == 0
        assert (Q[:, 0] <= Q[:, 1]).all() and (Q[:, 1] < n).all()
    lens = Q[:, 1] - Q[:, 0] + 1
    assert lens[0::2].max() <= 256  # mixed: even queries are short


def test_workload_threads_deterministic():
    L = _lib.lib()
    a1 = np.empty(1 << 20, np.int32)
    a2 = np.empty(1 << 20, np.int32)
    L.brmq_workload_array(2, a1.shape[0], 7, a1.ctypes.data, 1)
    L.brmq_workload_array(2, a2.shape[0], 7, a2.ctypes.data, 8)
    assert np.array_equal(a1, a2)


def test_workload_array_range_is_a_slice():
    """brmq_workload_array_range (sharded runs generate only their shard) equals
    the same slice of the whole array; kinds without slice locality are refused."""
    L = _lib.lib()
    n, seed = 300_001, 1706069402
    for kind in (0, 1):
        full = np.empty(n, np.int32)
        assert L.brmq_workload_array(kind, n, seed, full.ctypes.data, 0) == 0
        for first, count in ((0, n), (0, 1), (12345, 100_000), (n - 7, 7)):
            part = np.empty(count, np.int32)
            assert L.brmq_workload_array_range(kind, n, seed, first, count, part.ctypes.data, 3) == 0
            assert np.array_equal(part, full[first:first + count])
    part = np.empty(10, np.int32)
    assert L.brmq_workload_array_range(2, n, seed, 0, 10, part.ctypes.data, 0) != 0
    assert L.brmq_workload_array_range(0, n, seed, n - 5, 10, part.ctypes.data, 0) != 0
