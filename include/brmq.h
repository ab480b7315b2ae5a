/*
 * brmq.h -- C-ABI of the B200-native batched range-minimum-query engine
 * (arXiv 1706.06940, BbST / BbST_CON) -- the drop-in boundary.
 *
 * The reference exposes C++ free functions in namespace `batchrmq`
 * (/root/reference/proj/core/include/batchrmq/*.hpp) plus the SPEC-level
 * solves.  Each entry point below replaces one of
 * them; the cited file:line is the interface it stands in for.  Plain
 * pointers and sizes only; no C++ or torch types cross this boundary.
 *
 * Semantics shared by every entry point:
 *   - Positions are 0-based, queries inclusive [left, right]; a query with
 *     left > right is normalised by swapping, exactly as the
 *     batchrmq::Query constructor does (types.hpp:18-20).
 *   - Every answer is the LEFTMOST position of the minimum of A[left..right],
 *     bit-identical to naive_rmq (naive.hpp:13-21).  Answers are emitted in
 *     input order (types.hpp:25-29).
 *   - Errors are status codes that map 1:1 onto the reference's exception
 *     classes (BRMQ_EDOMAIN = std::domain_error, ...); brmq_last_error()
 *     returns the thread-local message.  include/batchrmq_b200.hpp rethrows
 *     them as the same std:: types.
 *   - A context owns one CUDA stream and a grow-only device workspace.  One
 *     context must not be used by two threads at once; distinct contexts may
 *     run concurrently.
 *   - BRMQ_PTR_DEVICE in `flags` says A / Q / answers are device pointers
 *     (resident in HBM); otherwise they are host pointers and the call copies
 *     them in and out on the context stream.  Every call returns after the
 *     answers are complete (host or device).
 *
 * The only limits are the reference's: n <= 2^32 - 1 (32-bit positions,
 * element_sparse_table.cpp:12-13, contraction.hpp:13) and q <= 2^31
 * (contraction.cpp:14-15).
 */
#ifndef BRMQ_H
#define BRMQ_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* == batchrmq::Query (types.hpp:13-23): 16 B, left @0, right @8. */
typedef struct brmq_query {
    uint64_t left;
    uint64_t right;
} brmq_query;

/* == batchrmq::Endpoint (contraction.hpp:12-21): origin = (qi << 1) | is_right. */
typedef struct brmq_endpoint {
    uint32_t pos;
    uint32_t origin;
} brmq_endpoint;

typedef struct brmq_ctx brmq_ctx;

enum brmq_status {
    BRMQ_OK = 0,
    BRMQ_EDOMAIN = 1, /* std::domain_error    (bits.hpp:11)                          */
    BRMQ_ERANGE = 2,  /* std::out_of_range    (naive.hpp:15, element_sparse_table.cpp:37) */
    BRMQ_EINVAL = 3,  /* std::invalid_argument (contraction.cpp:15,123; est.cpp:11,13,36) */
    BRMQ_ELOGIC = 4,  /* std::logic_error     (contraction.cpp:159,183)                */
    BRMQ_ECUDA = 5,   /* CUDA runtime failure (no reference equivalent)               */
    BRMQ_ENOMEM = 6,  /* std::bad_alloc / cudaErrorMemoryAllocation                   */
    BRMQ_EIO = 7      /* harness file I/O (brmq_harness.h; no reference equivalent)   */
};

enum brmq_flags {
    BRMQ_PTR_HOST = 0,
    BRMQ_PTR_DEVICE = 1 /* A, Q, answers (and stage buffers) are device pointers */
};

enum brmq_sort_kind { /* == batchrmq::SortKind (contraction.hpp:23) */
    BRMQ_SORT_RADIX = 0,
    BRMQ_SORT_COMPARISON = 1,
    BRMQ_SORT_BITMAP = 2 /* device presence-bitmap (1-bit counting) sort; no reference counterpart */
};

/* ------------------------------------------------------------ context */
int brmq_ctx_create(brmq_ctx** out, int device);
void brmq_ctx_destroy(brmq_ctx* ctx);
/* Use a caller-owned cudaStream_t (NULL restores the context's own stream). */
int brmq_ctx_set_stream(brmq_ctx* ctx, void* cuda_stream);
void* brmq_ctx_stream(brmq_ctx* ctx);
/* Thread-local message of the last failing call on this thread. */
const char* brmq_last_error(void);

/* ------------------------------------------------------------- solves */

/* SPEC.md:302-310 solve_batch_bbst(array, batch, LevelConfig{[k]}) -- BbST with
 * no contraction: block-argmin scan over A, block Sparse
 * Table over the n/k block minima, speculative query answering. */
int brmq_solve_bbst(brmq_ctx* ctx, const int32_t* A, uint64_t n, const brmq_query* Q,
                    uint64_t q, uint32_t k, uint64_t* answers, uint32_t flags);

/* SPEC.md:266-310 solve_batch_bbst(array, batch, LevelConfig{k_1 < ... < k_h})
 * -- multi-level BbST.  Any dividing chain, 1 <= h <= 8:
 * h = 1 is brmq_solve_bbst; [32, k] (32 | k) has the specialised path (one pass
 * over A stores the 32-element sub-block minima next to the k-block minima); any
 * other chain builds the k_i-block minima level by level from the one below and
 * answers with one warp per query descending the levels (query_chain.cu).  A
 * chain that is not strictly ascending with k_i | k_{i+1}, or has h = 0 or h > 8
 * -> BRMQ_EINVAL ("non-dividing chain -> configuration error"). */
int brmq_solve_bbst_ml(brmq_ctx* ctx, const int32_t* A, uint64_t n, const brmq_query* Q,
                       uint64_t q, const uint32_t* ks, uint32_t h, uint64_t* answers,
                       uint32_t flags);

/* SPEC.md:237-245 solve_batch_bbst_con(array, batch, BbstConParams{k, sort_kind})
 * -- BbST_CON: endpoint sort, contraction of A into A_Q,
 * block Sparse Table over A_Q, speculative answering. */
int brmq_solve_bbst_con(brmq_ctx* ctx, const int32_t* A, uint64_t n, const brmq_query* Q,
                        uint64_t q, uint32_t k, int sort_kind, uint64_t* answers,
                        uint32_t flags);

/* Sharded BbST: this device holds A[offset, offset + n_shard) of an
 * array of n_total.  keys[i] = packed key (((uint32)v ^ 0x80000000) << 32 | pos)
 * of the leftmost minimum of query i restricted to the shard, with pos GLOBAL,
 * or UINT64_MAX when the query misses the shard.  The answer of query i over
 * the whole array is (uint32)(min over shards of keys[i]) -- one min-allreduce
 * of q uint64 (NCCL over NVLink) combines the devices exactly.  Query bounds
 * are checked against n_total (BRMQ_ERANGE).  n_shard may be 0 (a rank left
 * without elements when the world size does not divide n_total): every key is
 * then UINT64_MAX, so that rank still joins the collective. */
int brmq_solve_bbst_shard(brmq_ctx* ctx, const int32_t* A, uint64_t n_shard, uint64_t offset,
                          uint64_t n_total, const brmq_query* Q, uint64_t q, uint32_t k,
                          uint64_t* keys, uint32_t flags);

/* Sharded BbST_CON (contraction variant): as brmq_solve_bbst_shard,
 * with the shard solved by brmq_solve_bbst_con -- the shard is contracted with
 * the endpoints that fall inside it plus the shard borders of the queries that
 * cross them (the clipped queries' endpoints). */
int brmq_solve_bbst_con_shard(brmq_ctx* ctx, const int32_t* A, uint64_t n_shard, uint64_t offset,
                              uint64_t n_total, const brmq_query* Q, uint64_t q, uint32_t k,
                              int sort_kind, uint64_t* keys, uint32_t flags);

/* naive.hpp:13-21 for every query, on the device (one warp per query): the
 * harness's "naive" algorithm. */
int brmq_solve_naive(brmq_ctx* ctx, const int32_t* A, uint64_t n, const brmq_query* Q,
                     uint64_t q, uint64_t* answers, uint32_t flags);

/* SPEC.md:331-377 solve_batch_st_rmq_con(array, batch) -- the comparison baseline
 * ST-RMQ_CON of Alzamel et al. (section 2): marked contraction of A
 * into <= 4q + 1 entries, element Sparse Table over them, two probes per query.
 * The endpoint sort is the LSD radix sort. */
int brmq_solve_st_rmq_con(brmq_ctx* ctx, const int32_t* A, uint64_t n, const brmq_query* Q,
                          uint64_t q, uint64_t* answers, uint32_t flags);

/* ------------------------------------------------ stage-level entry points */

/* contraction.hpp:51 collect_endpoints (contraction.cpp:13-23): eps gets 2q
 * endpoints in collect order (left, right per query). */
int brmq_collect_endpoints(brmq_ctx* ctx, const brmq_query* Q, uint64_t q, brmq_endpoint* eps,
                           uint32_t flags);

/* contraction.hpp:55 sort_endpoints (contraction.cpp:27-74): in place, by pos,
 * non-decreasing.  The device sort is a stable LSD radix sort for both kinds,
 * so the order equals the reference Radix sort's exactly. */
int brmq_sort_endpoints(brmq_ctx* ctx, brmq_endpoint* eps, uint64_t m, int sort_kind,
                        uint32_t flags);

/* contraction.hpp:61-64 build_contracted (contraction.cpp:112-151): boundary
 * (>= m entries) gets the deduplicated sorted positions, *nb their count;
 * aq_values / aq_origin (>= m entries) get the nb-1 inclusive area minima and
 * their leftmost positions. */
int brmq_build_contracted(brmq_ctx* ctx, const int32_t* A, uint64_t n,
                          const brmq_endpoint* sorted_eps, uint64_t m, int32_t* aq_values,
                          uint64_t* aq_origin, uint64_t* boundary, uint64_t* nb,
                          uint32_t flags);
/* The same with ContractionStats (contraction.hpp:47-49, contraction.cpp:84-107):
 * *array_reads (nullable) += the positions of A the device contraction consumed,
 * counted by the kernel (each warp adds its tiles clipped to [b_0, b_last]; each
 * position is read once: b_last - b_0 + 1 with one area or more, 0 otherwise --
 * the reference's serial count; its threaded path adds a re-read per seam). */
int brmq_build_contracted_stats(brmq_ctx* ctx, const int32_t* A, uint64_t n,
                                const brmq_endpoint* sorted_eps, uint64_t m, int32_t* aq_values,
                                uint64_t* aq_origin, uint64_t* boundary, uint64_t* nb,
                                uint32_t flags, uint64_t* array_reads);

/* contraction.hpp:71-73 remap_queries_from_sorted (contraction.cpp:174-199). */
int brmq_remap_from_sorted(brmq_ctx* ctx, const brmq_endpoint* sorted_eps, uint64_t m,
                           const uint64_t* boundary, uint64_t nb, uint64_t q, uint32_t* cleft,
                           uint32_t* cright, uint8_t* degenerate, uint32_t flags);

/* contraction.hpp:67 remap_queries (contraction.cpp:152-171): per query, the
 * boundary index of each end by binary search (cleft = index(left), cright =
 * index(right) - 1); a degenerate query (left == right) keeps cleft = cright = 0.
 * An end missing from the boundary list -> BRMQ_ELOGIC. */
int brmq_remap_queries(brmq_ctx* ctx, const brmq_query* Q, uint64_t q, const uint64_t* boundary,
                       uint64_t nb, uint32_t* cleft, uint32_t* cright, uint8_t* degenerate,
                       uint32_t flags);

/* SPEC.md:210-218 build_block_sparse(values, k): table[e*b + j] (b = ceil(m/k),
 * levels = floor_log2(b)+1, table sized levels*b) = position of the leftmost
 * minimum over blocks j .. j+2^e-1; cells whose span does not fit are
 * UINT64_MAX.  *b_out / *levels_out receive b and levels. */
int brmq_build_block_sparse(brmq_ctx* ctx, const int32_t* values, uint64_t m, uint32_t k,
                            uint64_t* table, uint64_t* b_out, uint32_t* levels_out,
                            uint32_t flags);

/* bits.hpp:10-13 floor_log2 (host; BRMQ_EDOMAIN on 0). */
int brmq_floor_log2(uint64_t x, uint32_t* out);

/* --------------------------------------------------------- instrumentation */

/* Per-stage device times of the last solve on this context, measured with
 * CUDA events on the context stream (no synchronisation is added).
 * brmq_ctx_set_timing: 0 off, 1 every stage, 2 only the HBM-bound kernel
 * the roofline is quoted on (the contraction scan, or the block-argmin scan
 * of BbST) -- two event nodes instead of two per stage inside a CUDA graph. */
#define BRMQ_MAX_STAGES 16
typedef struct brmq_stage_times {
    int count;
    char name[BRMQ_MAX_STAGES][24];
    float ms[BRMQ_MAX_STAGES];
    uint32_t launches[BRMQ_MAX_STAGES]; /* kernel launches inside the stage */
} brmq_stage_times;

int brmq_ctx_set_timing(brmq_ctx* ctx, int enable);
/* Debug instrumentation: 1 = BbST (h = 1) solves count the
 * array cells their partial-block scans cover (brmq_solve_info.scanned_cells;
 * one reduction per warp).  0 (default) = off. */
int brmq_ctx_set_counters(brmq_ctx* ctx, int enable);
int brmq_last_stage_times(brmq_ctx* ctx, brmq_stage_times* out);

/* Facts about the last solve: sizes of the intermediate structures and the
 * number of kernel launches it issued. */
typedef struct brmq_solve_info {
    uint64_t n, q, k;
    uint64_t blocks;        /* b = ceil(len/k) of the block Sparse Table   */
    uint32_t levels;        /* floor_log2(b) + 1                          */
    uint64_t boundary;      /* contraction: |boundary| (0 for BbST)       */
    uint64_t span_lo;       /* contraction: boundary[0]                   */
    uint64_t span_hi;       /* contraction: boundary[last]                */
    uint32_t kernel_launches;
    uint32_t graph;         /* 1: the solve ran as a replayed CUDA graph     */
    uint64_t scanned_cells; /* BbST (h = 1) with counters on: cells of A inside
                               the partial-block ranges the speculation rule had
                               to scan (SPEC.md:249, :472 instrumented counter) */
} brmq_solve_info;

int brmq_last_solve_info(brmq_ctx* ctx, brmq_solve_info* out);

/* Host pinned memory helpers (cudaHostAlloc / cudaFreeHost) so callers can
 * keep H2D/D2H at full PCIe rate without linking the CUDA runtime. */
int brmq_host_alloc(void** out, size_t bytes);
int brmq_host_free(void* p);
int brmq_device_alloc(brmq_ctx* ctx, void** out, size_t bytes);
int brmq_device_free(brmq_ctx* ctx, void* p);
int brmq_memcpy(brmq_ctx* ctx, void* dst, const void* src, size_t bytes, int kind /* cudaMemcpyKind */);
int brmq_synchronize(brmq_ctx* ctx);
/* Async device solves: with enable = 1, brmq_solve_bbst / _bbst_ml / _bbst_con on
 * DEVICE pointers (BRMQ_PTR_DEVICE, no stage timing) return once the solve is
 * enqueued on the context stream instead of waiting for it.  brmq_synchronize
 * then waits, fills brmq_last_solve_info and returns that solve's status (the
 * exceptions the synchronous call would have raised); any other call on the
 * context settles an outstanding async solve first, so no status is dropped.
 * Host-pointer solves stay synchronous (their answers land in host memory). */
int brmq_ctx_set_async(brmq_ctx* ctx, int enable);

#ifdef __cplusplus
}
#endif
#endif /* BRMQ_H */
