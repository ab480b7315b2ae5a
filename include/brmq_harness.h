/*
 * brmq_harness.h -- the reference's bench-harness contract (SPEC.md "bench-harness"
 * module), host side: workload / answer files, the Table 2
 * memory model, the value checksum and an answer verifier.  Exported by
 * libbrmq.so next to the solver ABI (include/brmq.h); no GPU is needed for any
 * of these.  The `brmq` command-line tool (paper_1706_06940_b200/csrc/cli.cpp)
 * is built on them and on the solvers.
 *
 * File formats, all little-endian:
 *   array   : "RMQA", u8 version = 1, u64 n, n x i32
 *   queries : "RMQQ", u8 version = 1, u64 q, q x (u64 left, u64 right), 0-based inclusive
 *   answers : "RMQR", u8 version = 1, u64 q, q x u64 position   (SPEC leaves the
 *             --answers format open; this one mirrors the other two)
 */
#ifndef BRMQ_HARNESS_H
#define BRMQ_HARNESS_H

#include <stddef.h>
#include <stdint.h>

#include "brmq.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Algorithm ids of the harness CLI `run --algo`. */
enum brmq_algo {
    BRMQ_ALGO_NAIVE = 0,      /* "naive": linear scan per query              */
    BRMQ_ALGO_SPARSE = 1,     /* "sparse": element Sparse Table over A        */
    BRMQ_ALGO_ST_RMQ_CON = 2, /* "st-rmq-con": Alzamel et al. baseline        */
    BRMQ_ALGO_BBST_CON = 3,   /* "bbst-con"                                   */
    BRMQ_ALGO_BBST = 4,       /* "bbst" (h = 1)                               */
    BRMQ_ALGO_BBST_ML = 5     /* "bbst-ml" (chain k_1 < ... < k_h)            */
};

/* Table 2 byte model: extra bytes beyond the
 * input and their share of 4n bytes in percent.
 *   bbst      : 8 * cells(n, k),  cells(m, k) = ceil(m/k) * (floor_log2(ceil(m/k)) + 1)
 *   bbst-con  : 20 * 2q + 8 * cells(2q, k)   (8 B endpoint pair + 4 B A_Q value + 8 B origin per endpoint)
 *   bbst-ml   : 8 * sum_{j < h-1} ceil(n / k_j) (the keys of every lower level) + 8 * cells(n, k_h)
 *   sparse    : 4 * sum_e (n - 2^e + 1)      (element_sparse_table.cpp:16-31 jagged uint32 rows)
 *   st-rmq-con: n/8 (mark bits) + 12 * M + 4 * sum_e (M - 2^e + 1), M = 4q + 1
 *   naive     : 0
 * ks/h: the block size (h = 1) or chain; ignored where not used. */
int brmq_account_memory(int algo, uint64_t n, uint64_t q, const uint32_t* ks, uint32_t h,
                        uint64_t* extra_bytes, double* extra_pct);

/* 64-bit FNV-1a fold over the answer VALUES A[answer] (4 little-endian bytes
 * each; an answer >= n folds 0xFFFFFFFF), so algorithms agreeing on values agree
 * on the checksum even where tie positions could differ. */
int brmq_answers_checksum(const int32_t* A, uint64_t n, const uint64_t* answers, uint64_t q,
                          uint64_t* out);

/* emit_plot: reads the records of a harness CSV (the emit_csv
 * columns) and writes a self-contained SVG with one time-vs-q line per
 * algorithm series (algo + k_chain), q on a log scale, t_total_ns on a log
 * scale.  Deterministic for fixed records.  Records must share n (BRMQ_EINVAL
 * otherwise); an empty record set writes nothing and returns BRMQ_OK with a
 * warning on stderr.  BRMQ_EIO when a file cannot be read or written. */
int brmq_emit_plot(const char* csv_path, const char* svg_path);

/* File I/O.  Readers with a NULL buffer only report the count. BRMQ_EIO on I/O
 * failure, BRMQ_EINVAL on a bad magic / version / truncated body or when the
 * count exceeds `cap`. */
int brmq_write_array_file(const char* path, const int32_t* A, uint64_t n);
int brmq_read_array_file(const char* path, int32_t* A, uint64_t cap, uint64_t* n);
int brmq_write_query_file(const char* path, const brmq_query* Q, uint64_t q);
int brmq_read_query_file(const char* path, brmq_query* Q, uint64_t cap, uint64_t* q);
int brmq_write_answer_file(const char* path, const uint64_t* answers, uint64_t q);
int brmq_read_answer_file(const char* path, uint64_t* answers, uint64_t cap, uint64_t* q);

/* The harness's `verify`: every answer must be the LEFTMOST
 * position of the minimum of A[left..right] (naive.hpp:13-21).  Host checker
 * (a block-minimum sparse table plus partial-block scans, `threads` workers, 0 =
 * all).  *bad = number of wrong answers, *first_bad = index of the first one
 * (q if none). */
int brmq_verify_answers(const int32_t* A, uint64_t n, const brmq_query* Q, uint64_t q,
                        const uint64_t* answers, unsigned threads, uint64_t* bad,
                        uint64_t* first_bad);

#ifdef __cplusplus
}
#endif
#endif /* BRMQ_HARNESS_H */
