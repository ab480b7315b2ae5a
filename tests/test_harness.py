"""Bench-harness contract (SPEC.md "bench-harness", :379-456), host side, no GPU:
Table 2 memory model, RMQA/RMQQ/RMQR files, the value checksum, the verifier
and the workload generators' SPEC examples."""
import os

import numpy as np
import pytest

import oracle
from paper_1706_06940_b200 import harness as H
from paper_1706_06940_b200 import _lib
from paper_1706_06940_b200.batchrmq import InvalidArgument

# PAPER.md:622-637 Table 2 / SPEC.md:468 acceptance criterion 3: every value to +-0.01
# (q ~ sqrt(n), 32 sqrt(n), 1024 sqrt(n): 1e4 / 3.2e5 / 1.024e7 at n = 1e8 and
# 3.2e4 / 1.024e6 / 3.2768e7 at n = 1e9)
TABLE2 = [
    ("bbst-con", 10**8, 10_000, 512, 0.10), ("bbst-con", 10**9, 32_000, 512, 0.03),
    ("bbst-con", 10**8, 320_000, 512, 3.23), ("bbst-con", 10**9, 1_024_000, 512, 1.03),
    ("bbst-con", 10**8, 10_240_000, 512, 103.68), ("bbst-con", 10**9, 32_768_000, 512, 33.20),
    ("bbst", 10**8, 0, 2048, 1.56), ("bbst", 10**9, 0, 2048, 1.86),
    ("bbst", 10**8, 0, 4096, 0.73), ("bbst", 10**9, 0, 4096, 0.88),
    ("bbst", 10**8, 0, 8192, 0.34), ("bbst", 10**9, 0, 8192, 0.42),
    ("bbst", 10**8, 0, 16384, 0.16), ("bbst", 10**9, 0, 16384, 0.20),
    ("bbst", 10**8, 0, 32768, 0.07), ("bbst", 10**9, 0, 32768, 0.09),
]


@pytest.mark.parametrize("algo,n,q,k,want", TABLE2)
def test_table2(algo, n, q, k, want):
    _, pct = H.account_memory(algo, n, q, (k,))
    assert abs(round(pct, 2) - want) <= 0.01 + 1e-9


def test_memory_model_examples():
    # SPEC.md:417-420 worked numbers
    assert H.account_memory("bbst", 10**8, 0, (2048,))[0] == 48829 * 16 * 8 == 6_250_112
    assert H.account_memory("bbst-con", 10**8, 10_240_000, (512,))[0] == 409_600_000 + 5_120_000
    assert H.account_memory("naive", 1000)[0] == 0
    # element table over A: jagged uint32 rows (element_sparse_table.cpp:16-31)
    n = 1000
    cells = sum(n - (1 << e) + 1 for e in range(n.bit_length()))
    assert H.account_memory("sparse", n)[0] == 4 * cells
    # bbst-ml [32, 512]: level-1 keys + block ST over 512-blocks
    b512 = -(-10**6 // 512)
    assert H.account_memory("bbst-ml", 10**6, 0, (32, 512))[0] == \
        8 * b512 * (b512.bit_length()) + 8 * (10**6 // 32)
    with pytest.raises(InvalidArgument):
        H.account_memory("bbst", 100, 0, (0,))


def _fnv(values):
    h = 0xcbf29ce484222325
    for v in values:
        v &= 0xFFFFFFFF
        for b in range(4):
            h ^= (v >> (8 * b)) & 0xFF
            h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return h


def test_checksum_values_not_positions():
    A = np.array([5, 3, 8, 3, 7, -2], np.int32)
    assert H.answers_checksum(A, np.array([1, 5, 0], np.uint64)) == _fnv([3, -2, 5])
    # tie positions with equal values fold identically
    assert H.answers_checksum(A, np.array([1], np.uint64)) == H.answers_checksum(A, np.array([3], np.uint64))
    # out-of-range answer folds 0xFFFFFFFF
    assert H.answers_checksum(A, np.array([99], np.uint64)) == _fnv([0xFFFFFFFF])
    assert H.answers_checksum(A, np.array([], np.uint64)) == 0xcbf29ce484222325


def test_files_roundtrip(tmp_path):
    rng = np.random.default_rng(7)
    A = rng.integers(-2**31, 2**31, 1000, dtype=np.int64).astype(np.int32)
    Q = np.sort(rng.integers(0, 1000, (300, 2), dtype=np.uint64), axis=1)
    ans = rng.integers(0, 1000, 300, dtype=np.uint64)
    H.write_array(tmp_path / "a", A)
    H.write_queries(tmp_path / "q", Q)
    H.write_answers(tmp_path / "r", ans)
    assert np.array_equal(H.read_array(tmp_path / "a"), A)
    assert np.array_equal(H.read_queries(tmp_path / "q"), Q)
    assert np.array_equal(H.read_answers(tmp_path / "r"), ans)
    raw = (tmp_path / "q").read_bytes()  # SPEC.md:455 layout, little-endian
    assert raw[:5] == b"RMQQ\x01" and int.from_bytes(raw[5:13], "little") == 300
    assert len(raw) == 13 + 300 * 16
    assert int.from_bytes(raw[13:21], "little") == int(Q[0, 0])
    raw = (tmp_path / "a").read_bytes()
    assert raw[:5] == b"RMQA\x01" and len(raw) == 13 + 4000
    # empty files
    H.write_array(tmp_path / "e", np.zeros(0, np.int32))
    assert H.read_array(tmp_path / "e").shape == (0,)


def test_file_errors(tmp_path):
    H.write_array(tmp_path / "a", np.arange(10, dtype=np.int32))
    with pytest.raises(InvalidArgument):  # wrong magic: an array file read as queries
        H.read_queries(tmp_path / "a")
    raw = bytearray((tmp_path / "a").read_bytes())
    raw[4] = 2
    (tmp_path / "v").write_bytes(bytes(raw))
    with pytest.raises(InvalidArgument):  # unsupported version
        H.read_array(tmp_path / "v")
    (tmp_path / "t").write_bytes((tmp_path / "a").read_bytes()[:-3])
    with pytest.raises(InvalidArgument):  # truncated body
        H.read_array(tmp_path / "t")
    with pytest.raises(OSError):
        H.read_array(tmp_path / "missing")


def test_verify():
    rng = np.random.default_rng(3)
    n = 5000
    A = rng.integers(0, 50, n, dtype=np.int64).astype(np.int32)  # heavy ties
    Q = rng.integers(0, n, (2000, 2), dtype=np.uint64)
    want = oracle.naive_numpy(A, Q)
    assert H.verify(A, Q, want) == (0, 2000)
    bad = want.copy()
    # a tie further right (same value, not leftmost) must be rejected
    for i in range(len(Q)):
        l, r = sorted(map(int, Q[i]))
        ties = np.nonzero(A[l:r + 1] == A[want[i]])[0] + l
        if len(ties) > 1:
            bad[i] = ties[-1]
            break
    nb, first = H.verify(A, Q, bad)
    assert nb == 1 and first == i
    bad = want.copy()
    bad[7] = n + 5  # outside the array
    assert H.verify(A, Q, bad) == (1, 7)


def test_gen_permutation_spec():
    # [1..n] then floor(n/2) swaps -> a permutation of 1..n
    L = _lib.lib()
    out = np.empty(1, np.int32)
    assert L.brmq_workload_array(3, 1, 5, out.ctypes.data, 0) == 0 and out[0] == 1
    n = 10_000
    a = np.empty(n, np.int32)
    b = np.empty(n, np.int32)
    L.brmq_workload_array(3, n, 11, a.ctypes.data, 0)
    L.brmq_workload_array(3, n, 12, b.ctypes.data, 0)
    assert np.array_equal(np.sort(a), np.arange(1, n + 1))
    assert not np.array_equal(a, b)


def test_gen_queries_spec():
    # left <= right, mean(right - left) ~ n/3 within 2% at q = 1e6
    L = _lib.lib()
    n, q = 10**6, 10**6
    Q = np.empty((q, 2), np.uint64)
    assert L.brmq_workload_queries(0, n, q, 99, Q.ctypes.data, 0) == 0
    assert (Q[:, 0] <= Q[:, 1]).all() and (Q[:, 1] < n).all()
    m = float((Q[:, 1] - Q[:, 0]).mean())
    assert abs(m - n / 3) <= 0.02 * n / 3


def test_memory_model_multilevel_counts_every_level():
    """bbst-ml with h >= 3: the keys of every lower level are counted (the
    chain solve allocates M_j for every j < h - 1, api.cu solve_chain)."""
    from paper_1706_06940_b200 import harness as H
    n = 10**8
    b2, _ = H.account_memory("bbst-ml", n, 0, (32, 512))
    b3, _ = H.account_memory("bbst-ml", n, 0, (8, 64, 512))
    b1, _ = H.account_memory("bbst", n, 0, (512,))
    assert b2 == b1 + 8 * (-(-n // 32))
    assert b3 == b1 + 8 * (-(-n // 8)) + 8 * (-(-n // 64))


def test_emit_plot(tmp_path):
    """emit_plot: one series per algorithm, deterministic,
    empty input is a no-op, mixed n is refused."""
    from paper_1706_06940_b200 import InvalidArgument
    from paper_1706_06940_b200 import harness as H
    hdr = ("algo,n,q,k_chain,threads,runs,t_sort_ns,t_contract_ns,t_build_ns,t_answer_ns,"
           "t_total_ns,extra_bytes,extra_pct,answers_checksum\n")
    rows = []
    for algo, k in (("bbst", "512"), ("bbst-con", "512"), ("st-rmq-con", "")):
        for t in range(11):
            q = int(10**4 * 2**t)
            rows.append(f"{algo},100000000,{q},{k},1,7,0,0,0,0,{1000 * (t + 1) * (2 if k else 5)},0,0.0,1\n")
    csv = tmp_path / "r.csv"
    csv.write_text(hdr + "".join(rows))
    svg1, svg2 = tmp_path / "a.svg", tmp_path / "b.svg"
    H.emit_plot(csv, svg1)
    H.emit_plot(csv, svg2)
    text = svg1.read_text()
    assert text.startswith("<svg") and text.rstrip().endswith("</svg>")
    assert text.count('class="series"') == 3 and text.count("<circle") == 33
    assert svg1.read_bytes() == svg2.read_bytes()
    empty = tmp_path / "e.csv"
    empty.write_text(hdr)
    H.emit_plot(empty, tmp_path / "none.svg")
    assert not (tmp_path / "none.svg").exists()
    mixed = tmp_path / "m.csv"
    mixed.write_text(hdr + rows[0] + rows[1].replace("100000000", "1000"))
    with pytest.raises(InvalidArgument):
        H.emit_plot(mixed, tmp_path / "m.svg")
