/*
 * brmq_workload.h -- deterministic synthetic workloads of BASELINE.json's five
 * configurations (measurement infrastructure, exported by libbrmq.so; host-only,
 * multi-threaded, no GPU needed).
 *
 * Generator (SPEC.md:397,448 ask for a documented splitmix-style PRNG):
 *   mix64(z): z ^= z >> 30; z *= 0xBF58476D1CE4E5B9; z ^= z >> 27;
 *             z *= 0x94D049BB133111EB; z ^= z >> 31
 *   stream base  B(seed, s) = mix64(seed ^ (0xA0761D6478BD642F * (s + 1)))
 *   draw i       x_i = mix64(B + (i + 1) * 0x9E3779B97F4A7C15)
 * Stream 0 draws the array, stream 1 the queries.  Config c uses
 * seed = 1706069400 + c.  mulhi(x, m) = floor(x * m / 2^64).
 */
#ifndef BRMQ_WORKLOAD_H
#define BRMQ_WORKLOAD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum brmq_array_kind {
    BRMQ_ARRAY_UNIFORM31 = 0, /* v = x >> 33, uniform in [0, 2^31)          (c1, c2, c3) */
    BRMQ_ARRAY_TIES16 = 1,    /* v = x >> 60, uniform in [0, 16)            (c4)         */
    BRMQ_ARRAY_WALK = 2,      /* A[0]=0, A[i]=A[i-1]+(x_i&1 ? +1 : -1), then minus min (c5) */
    BRMQ_ARRAY_PERMUTATION = 3/* SPEC.md:394-402 gen_permutation: [1..n], floor(n/2) swaps  */
};

enum brmq_query_kind {
    BRMQ_QUERIES_UNIFORM = 0,    /* l = mulhi(x_2i, n), r = mulhi(x_2i+1, n), swap     (c1, c2, c5) */
    BRMQ_QUERIES_LOGUNIFORM = 1, /* len = clamp(floor(exp(u ln n)), 1, n), u = (x_2i >> 11) 2^-53,
                                    l = mulhi(x_2i+1, n - len + 1), r = l + len - 1  (c3)          */
    BRMQ_QUERIES_MIXED = 2       /* even i: len = 1 + mulhi(x_2i, 256) (clamped to n),
                                    odd i: len = 1 + mulhi(x_2i, n); start as above      (c4)     */
};

/* out: n int32 values.  threads = 0 -> all hardware threads. */
int brmq_workload_array(int kind, uint64_t n, uint64_t seed, int32_t* out, unsigned threads);
/* out: elements [first, first + count) of the array above (kinds UNIFORM31 and
 * TIES16 only; a sharded run generates just its own shard). */
int brmq_workload_array_range(int kind, uint64_t n, uint64_t seed, uint64_t first, uint64_t count,
                              int32_t* out, unsigned threads);
/* out: q {left, right} uint64 pairs (== brmq_query). */
int brmq_workload_queries(int kind, uint64_t n, uint64_t q, uint64_t seed, uint64_t* out,
                          unsigned threads);
uint64_t brmq_workload_mix64(uint64_t z);

#ifdef __cplusplus
}
#endif
#endif
