/*
 * oracle.h -- CPU restatement of the reference batched-RMQ algorithm.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the CUDA path is compared
 * against; it is never linked into, called by, or shipped with the product
 * library (paper_1706_06940_b200/libbrmq.so).  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference legs may load it.
 *
 * Every function cites the reference file:line it restates
 * (paths relative to the reference tree, proj/core/...).
 *
 * Parity pin: the restatement is checked (tests/test_oracle.py) against
 *   (1) the SPEC.md worked examples (tests/golden/spec_examples.json), and
 *   (2) the reference's own code compiled from its sources into
 *       oracle/_ref/libbrmq_ref.so (oracle/Makefile), on seeded inputs, and
 *   (3) golden vectors produced by that compiled reference
 *       (binary fixtures under tests/golden, generator tests/golden/make_golden.py).
 *
 * Conventions: positions are 0-based, queries are inclusive [left, right]
 * (types.hpp:11-23).  Query arrays are `uint64_t[2*q]` = {left, right} pairs,
 * byte-identical to batchrmq::Query (16 B, left@0, right@8).  Endpoints are
 * `uint32_t[2*m]` = {pos, origin} pairs, identical to batchrmq::Endpoint.
 *
 * Return codes follow the C-ABI (include/brmq.h): 0 ok, 1 domain_error,
 * 2 out_of_range, 3 invalid_argument, 4 logic_error, 6 out of memory.
 */
#ifndef BRMQ_ORACLE_H
#define BRMQ_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* naive.hpp:13-21 -- leftmost minimum by linear scan.  Returns 0 / 2 (range). */
int orc_naive_rmq(const int32_t* A, uint64_t n, uint64_t left, uint64_t right, uint64_t* out);

/* bits.hpp:10-13 */
int orc_floor_log2(uint64_t x, uint32_t* out);

/* element_sparse_table.{hpp,cpp}: jagged doubling table of uint32 positions.
 * Opaque handle; build is element_sparse_table.cpp:10-32, arg_min :34-44. */
typedef struct orc_est orc_est;
int orc_est_build(const int32_t* values, uint64_t n, orc_est** out);
int orc_est_arg_min(const orc_est* t, const int32_t* values, uint64_t n,
                    uint64_t left, uint64_t right, uint64_t* out);
uint64_t orc_est_cell_count(const orc_est* t);
uint32_t orc_est_level_count(const orc_est* t);
/* copies row e (n - 2^e + 1 entries) into out; returns the entry count */
uint64_t orc_est_level(const orc_est* t, uint32_t e, uint32_t* out);
void orc_est_free(orc_est* t);

/* contraction.cpp:13-23 */
int orc_collect_endpoints(const uint64_t* Q, uint64_t q, uint32_t* eps);
/* contraction.cpp:27-63 (radix) / :71-72 (comparison); in place, m endpoints.
 * kind 0 = Radix (LSD bytes, constant-byte skip), 1 = Comparison. Both are
 * stable here; the reference's comparison sort is not (order of equal pos
 * is unspecified there, and irrelevant to every downstream output). */
int orc_sort_endpoints(uint32_t* eps, uint64_t m, int kind);
/* contraction.cpp:112-151 (+ scan_areas :81-108).  Outputs are sized by the
 * caller: boundary >= m entries, aq_* >= m entries.  *nb = |boundary|,
 * areas = nb - 1 (0 if nb <= 1).  reads (may be NULL) += array reads. */
int orc_build_contracted(const int32_t* A, uint64_t n, const uint32_t* sorted_eps, uint64_t m,
                         unsigned threads, int32_t* aq_values, uint64_t* aq_origin,
                         uint64_t* boundary, uint64_t* nb, uint64_t* reads);
/* contraction.cpp:174-199 */
int orc_remap_queries(const uint64_t* Q, uint64_t q, const uint64_t* boundary, uint64_t nb,
                      uint32_t* cleft, uint32_t* cright, uint8_t* degenerate);
int orc_remap_from_sorted(const uint32_t* sorted_eps, uint64_t m, const uint64_t* boundary,
                          uint64_t nb, uint64_t q, uint32_t* cleft, uint32_t* cright,
                          uint8_t* degenerate);

/* The oracle pipeline: collect -> sort(Radix) -> build_contracted
 * -> remap_from_sorted -> ElementSparseTable(aq_values) -> arg_min -> aq_origin;
 * degenerate queries answer `left`.  Equals naive_rmq (leftmost). */
int orc_solve_oracle(const int32_t* A, uint64_t n, const uint64_t* Q, uint64_t q,
                     unsigned threads, uint64_t* answers);

/* SPEC.md:198-218 build_block_sparse over int32 values: b = ceil(m/k) blocks,
 * levels = floor_log2(b)+1; table[e*b + j] = position of leftmost min over
 * blocks j .. j+2^e-1 (only j <= b-2^e written; rest set to UINT64_MAX). */
int orc_build_block_sparse(const int32_t* values, uint64_t m, uint32_t k, uint64_t* table,
                           uint64_t* b_out, uint32_t* levels_out);

/* SPEC.md:266-310 solve_batch_bbst, h = 1 (no contraction), with the
 * leftmost-exact speculative rule.  scanned (may be NULL)
 * receives S = array cells inside the partial ranges the rule had to scan
 * (whole partial range, no early exit -- the device reads a partial range
 * in one pass); scanned_early receives the same with the sequential
 * early-exit at the stored block minimum (SURVEY 8a probe figure). */
int orc_solve_bbst(const int32_t* A, uint64_t n, const uint64_t* Q, uint64_t q, uint32_t k,
                   uint64_t* answers, uint64_t* scanned, uint64_t* scanned_early);

/* SPEC.md:193-245 solve_batch_bbst_con: stages 1-2 as above, block ST over
 * A_Q (k), speculative answering over A_Q, translate through aq_origin. */
int orc_solve_bbst_con(const int32_t* A, uint64_t n, const uint64_t* Q, uint64_t q, uint32_t k,
                       unsigned threads, uint64_t* answers, uint64_t* scanned);

#ifdef __cplusplus
}
#endif
#endif
