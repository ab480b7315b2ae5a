"""Python view of the bench-harness contract (include/brmq_harness.h,
SPEC.md:379-456): RMQA / RMQQ / RMQR files, the Table 2 memory model, the
answer-value checksum and the verifier.  Host-only (no GPU needed); errors are
the reference's exception classes, as in batchrmq.py.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import numpy as np

from . import _lib
from .batchrmq import _check

ALGOS = {"naive": 0, "sparse": 1, "st-rmq-con": 2, "bbst-con": 3, "bbst": 4, "bbst-ml": 5}


def _p(a: np.ndarray) -> int:
    return a.ctypes.data


def account_memory(algo: str, n: int, q: int = 0, ks=(512,)) -> tuple[int, float]:
    """Extra bytes and their percentage of 4n (Table 2)."""
    L = _lib.lib()
    arr = (C.c_uint32 * max(1, len(ks)))(*ks)
    b, pct = C.c_uint64(), C.c_double()
    _check(L.brmq_account_memory(ALGOS[algo], n, q, arr, len(ks), C.byref(b), C.byref(pct)))
    return b.value, pct.value


def answers_checksum(A: np.ndarray, answers: np.ndarray) -> int:
    """64-bit FNV-1a fold over the answer values A[answer]."""
    A = np.ascontiguousarray(A, dtype=np.int32)
    ans = np.ascontiguousarray(answers, dtype=np.uint64)
    out = C.c_uint64()
    _check(_lib.lib().brmq_answers_checksum(_p(A), A.shape[0], _p(ans), ans.shape[0], C.byref(out)))
    return out.value


def write_array(path, A: np.ndarray) -> None:
    A = np.ascontiguousarray(A, dtype=np.int32)
    _check(_lib.lib().brmq_write_array_file(str(path).encode(), _p(A), A.shape[0]))


def read_array(path) -> np.ndarray:
    L, n = _lib.lib(), C.c_uint64()
    _check(L.brmq_read_array_file(str(path).encode(), None, 0, C.byref(n)))
    A = np.empty(n.value, dtype=np.int32)
    _check(L.brmq_read_array_file(str(path).encode(), _p(A), A.shape[0], C.byref(n)))
    return A


def write_queries(path, Q: np.ndarray) -> None:
    Q = np.ascontiguousarray(Q, dtype=np.uint64).reshape(-1, 2)
    _check(_lib.lib().brmq_write_query_file(str(path).encode(), _p(Q), Q.shape[0]))


def read_queries(path) -> np.ndarray:
    L, q = _lib.lib(), C.c_uint64()
    _check(L.brmq_read_query_file(str(path).encode(), None, 0, C.byref(q)))
    Q = np.empty((q.value, 2), dtype=np.uint64)
    _check(L.brmq_read_query_file(str(path).encode(), _p(Q), Q.shape[0], C.byref(q)))
    return Q


def write_answers(path, answers: np.ndarray) -> None:
    a = np.ascontiguousarray(answers, dtype=np.uint64)
    _check(_lib.lib().brmq_write_answer_file(str(path).encode(), _p(a), a.shape[0]))


def read_answers(path) -> np.ndarray:
    L, q = _lib.lib(), C.c_uint64()
    _check(L.brmq_read_answer_file(str(path).encode(), None, 0, C.byref(q)))
    a = np.empty(q.value, dtype=np.uint64)
    _check(L.brmq_read_answer_file(str(path).encode(), _p(a), a.shape[0], C.byref(q)))
    return a


def verify(A: np.ndarray, Q: np.ndarray, answers: np.ndarray, threads: int = 0) -> tuple[int, int]:
    """(#wrong answers, index of the first wrong one or q): leftmost-minimum check."""
    A = np.ascontiguousarray(A, dtype=np.int32)
    Q = np.ascontiguousarray(Q, dtype=np.uint64).reshape(-1, 2)
    a = np.ascontiguousarray(answers, dtype=np.uint64)
    bad, first = C.c_uint64(), C.c_uint64()
    _check(_lib.lib().brmq_verify_answers(_p(A), A.shape[0], _p(Q), Q.shape[0], _p(a), threads,
                                          C.byref(bad), C.byref(first)))
    return bad.value, first.value


def emit_plot(csv_path, svg_path) -> None:
    """SVG time-vs-q chart, one series per algorithm, from a harness CSV
    (include/brmq_harness.h brmq_emit_plot)."""
    _check(_lib.lib().brmq_emit_plot(str(csv_path).encode(), str(svg_path).encode()))
