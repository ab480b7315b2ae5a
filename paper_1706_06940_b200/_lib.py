"""ctypes binding of libbrmq.so (include/brmq.h, include/brmq_workload.h).

The library is built in-tree (``python -m paper_1706_06940_b200.build``).  There
is no fallback: if the shared object is missing, importing the compute API
raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

# BRMQ_LIB overrides the in-tree library (A/B builds in tools/; never a fallback)
LIB_PATH = Path(os.environ.get("BRMQ_LIB") or Path(__file__).resolve().parent / "libbrmq.so")

u8p = C.POINTER(C.c_uint8)
u32p = C.POINTER(C.c_uint32)
u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)
vp = C.c_void_p

BRMQ_MAX_STAGES = 16


class StageTimes(C.Structure):
    _fields_ = [("count", C.c_int),
                ("name", (C.c_char * 24) * BRMQ_MAX_STAGES),
                ("ms", C.c_float * BRMQ_MAX_STAGES),
                ("launches", C.c_uint32 * BRMQ_MAX_STAGES)]


class SolveInfo(C.Structure):
    _fields_ = [("n", C.c_uint64), ("q", C.c_uint64), ("k", C.c_uint64),
                ("blocks", C.c_uint64), ("levels", C.c_uint32),
                ("boundary", C.c_uint64), ("span_lo", C.c_uint64), ("span_hi", C.c_uint64),
                ("kernel_launches", C.c_uint32), ("graph", C.c_uint32),
                ("scanned_cells", C.c_uint64)]


# name -> (restype, argtypes): exactly the declarations of include/brmq*.h
SIGNATURES = {
    "brmq_ctx_create": (C.c_int, [C.POINTER(vp), C.c_int]),
    "brmq_ctx_destroy": (None, [vp]),
    "brmq_ctx_set_stream": (C.c_int, [vp, vp]),
    "brmq_ctx_stream": (vp, [vp]),
    "brmq_last_error": (C.c_char_p, []),
    "brmq_solve_bbst": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, C.c_uint32, vp, C.c_uint32]),
    "brmq_solve_bbst_ml": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp, C.c_uint32, vp,
                                     C.c_uint32]),
    "brmq_solve_bbst_con": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, C.c_uint32, C.c_int, vp,
                                      C.c_uint32]),
    "brmq_solve_bbst_shard": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, vp, C.c_uint64,
                                        C.c_uint32, vp, C.c_uint32]),
    "brmq_solve_bbst_con_shard": (C.c_int, [vp, vp, C.c_uint64, C.c_uint64, C.c_uint64, vp,
                                            C.c_uint64, C.c_uint32, C.c_int, vp, C.c_uint32]),
    "brmq_solve_naive": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp, C.c_uint32]),
    "brmq_solve_st_rmq_con": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp, C.c_uint32]),
    "brmq_collect_endpoints": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint32]),
    "brmq_sort_endpoints": (C.c_int, [vp, vp, C.c_uint64, C.c_int, C.c_uint32]),
    "brmq_build_contracted": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp, vp, vp, u64p,
                                        C.c_uint32]),
    "brmq_build_contracted_stats": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp, vp, vp, u64p,
                                              C.c_uint32, u64p]),
    "brmq_remap_queries": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, vp, vp, vp, C.c_uint32]),
    "brmq_remap_from_sorted": (C.c_int, [vp, vp, C.c_uint64, vp, C.c_uint64, C.c_uint64, vp, vp,
                                         vp, C.c_uint32]),
    "brmq_build_block_sparse": (C.c_int, [vp, vp, C.c_uint64, C.c_uint32, vp, u64p,
                                          u32p, C.c_uint32]),
    "brmq_floor_log2": (C.c_int, [C.c_uint64, u32p]),
    "brmq_ctx_set_timing": (C.c_int, [vp, C.c_int]),
    "brmq_ctx_set_counters": (C.c_int, [vp, C.c_int]),
    "brmq_ctx_set_async": (C.c_int, [vp, C.c_int]),
    "brmq_last_stage_times": (C.c_int, [vp, C.POINTER(StageTimes)]),
    "brmq_last_solve_info": (C.c_int, [vp, C.POINTER(SolveInfo)]),
    "brmq_host_alloc": (C.c_int, [C.POINTER(vp), C.c_size_t]),
    "brmq_host_free": (C.c_int, [vp]),
    "brmq_device_alloc": (C.c_int, [vp, C.POINTER(vp), C.c_size_t]),
    "brmq_device_free": (C.c_int, [vp, vp]),
    "brmq_memcpy": (C.c_int, [vp, vp, vp, C.c_size_t, C.c_int]),
    "brmq_synchronize": (C.c_int, [vp]),
    "brmq_workload_array": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, vp, C.c_uint]),
    "brmq_workload_array_range": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, C.c_uint64, vp,
                                            C.c_uint]),
    "brmq_workload_queries": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, C.c_uint64, vp, C.c_uint]),
    "brmq_workload_mix64": (C.c_uint64, [C.c_uint64]),
    # include/brmq_harness.h
    "brmq_account_memory": (C.c_int, [C.c_int, C.c_uint64, C.c_uint64, u32p, C.c_uint32, u64p,
                                      C.POINTER(C.c_double)]),
    "brmq_answers_checksum": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, u64p]),
    "brmq_write_array_file": (C.c_int, [C.c_char_p, vp, C.c_uint64]),
    "brmq_read_array_file": (C.c_int, [C.c_char_p, vp, C.c_uint64, u64p]),
    "brmq_write_query_file": (C.c_int, [C.c_char_p, vp, C.c_uint64]),
    "brmq_read_query_file": (C.c_int, [C.c_char_p, vp, C.c_uint64, u64p]),
    "brmq_write_answer_file": (C.c_int, [C.c_char_p, vp, C.c_uint64]),
    "brmq_read_answer_file": (C.c_int, [C.c_char_p, vp, C.c_uint64, u64p]),
    "brmq_emit_plot": (C.c_int, [C.c_char_p, C.c_char_p]),
    "brmq_verify_answers": (C.c_int, [vp, C.c_uint64, vp, C.c_uint64, vp, C.c_uint, u64p, u64p]),
}

_lib = None


def lib() -> C.CDLL:
    """Load libbrmq.so (fails loudly when it has not been built)."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise ImportError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1706_06940_b200.build` "
                "(there is no CPU fallback)")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib
