"""B200-native batched range-minimum queries (arXiv 1706.06940: BbST / BbST_CON).

The product is libbrmq.so: a C-ABI (include/brmq.h) over hand-written sm_100a
kernels.  This package holds the kernels' sources (csrc/), the in-tree build
(build.py), the ctypes binding (_lib.py) and a host-side mirror of the
reference operator API (batchrmq.py).
"""
from .batchrmq import (  # noqa: F401
    ENDPOINT_DTYPE, QUERY_DTYPE, ContractedArray, ContractedQueryBatch, CudaError, DomainError,
    Engine, InvalidArgument, LogicError, OutOfRange, SortKind, build_block_sparse,
    build_contracted, collect_endpoints, floor_log2, make_queries, remap_queries,
    remap_queries_from_sorted,
    solve_batch_bbst, solve_batch_bbst_con, sort_endpoints)
