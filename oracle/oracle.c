/*
 * oracle.c -- CPU restatement of the reference batched-RMQ algorithm.
 *
 * TEST INFRASTRUCTURE ONLY (see oracle.h): the checker, never the product.
 * Reference paths are relative to /root/reference/proj/core unless noted.
 * Plain C11 + pthreads; no code is copied from the reference, each routine
 * restates the cited behaviour.
 */
#define _GNU_SOURCE
#include "oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

enum { OK = 0, EDOMAIN_ = 1, ERANGE_ = 2, EINVAL_ = 3, ELOGIC_ = 4, ENOMEM_ = 6 };

/* ---------------------------------------------------------------- bits.hpp */

/* bits.hpp:10-13: largest e with 2^e <= x; domain error on 0. */
int orc_floor_log2(uint64_t x, uint32_t* out) {
    if (x == 0) return EDOMAIN_;
    *out = 63u - (uint32_t)__builtin_clzll(x);
    return OK;
}

static inline uint32_t flog2(uint64_t x) { return 63u - (uint32_t)__builtin_clzll(x); }

/* --------------------------------------------------------------- naive.hpp */

/* naive.hpp:13-21: strict '<' keeps the first (leftmost) minimum. */
int orc_naive_rmq(const int32_t* A, uint64_t n, uint64_t left, uint64_t right, uint64_t* out) {
    if (left > right) { uint64_t t = left; left = right; right = t; } /* types.hpp:18-20 */
    if (right >= n) return ERANGE_;                                   /* naive.hpp:14-15 */
    uint64_t best = left;
    for (uint64_t i = left + 1; i <= right; ++i)
        if (A[i] < A[best]) best = i;
    *out = best;
    return OK;
}

/* ------------------------------------------------ element_sparse_table.cpp */

struct orc_est {
    uint64_t n;
    uint32_t levels;
    uint32_t** rows; /* row e has n - 2^e + 1 entries */
};

/* element_sparse_table.cpp:10-32 */
int orc_est_build(const int32_t* values, uint64_t n, orc_est** out) {
    if (n == 0) return EINVAL_;                 /* :11 */
    if (n > 0xFFFFFFFFull) return EINVAL_;      /* :12-13 */
    orc_est* t = (orc_est*)calloc(1, sizeof(*t));
    if (!t) return ENOMEM_;
    t->n = n;
    t->levels = flog2(n) + 1;                   /* :15 */
    t->rows = (uint32_t**)calloc(t->levels, sizeof(uint32_t*));
    if (!t->rows) { free(t); return ENOMEM_; }
    t->rows[0] = (uint32_t*)malloc(n * sizeof(uint32_t));
    if (!t->rows[0]) { orc_est_free(t); return ENOMEM_; }
    for (uint64_t j = 0; j < n; ++j) t->rows[0][j] = (uint32_t)j; /* :18 identity */
    for (uint32_t e = 1; e < t->levels; ++e) {  /* :20-31 */
        const uint64_t half = 1ull << (e - 1);
        const uint64_t count = n - (1ull << e) + 1;
        const uint32_t* prev = t->rows[e - 1];
        uint32_t* cur = (uint32_t*)malloc(count * sizeof(uint32_t));
        if (!cur) { orc_est_free(t); return ENOMEM_; }
        for (uint64_t j = 0; j < count; ++j) {
            const uint32_t a = prev[j], b = prev[j + half];
            cur[j] = values[b] < values[a] ? b : a; /* :29 leftmost on ties */
        }
        t->rows[e] = cur;
    }
    *out = t;
    return OK;
}

/* element_sparse_table.cpp:34-44 */
int orc_est_arg_min(const orc_est* t, const int32_t* values, uint64_t n, uint64_t left,
                    uint64_t right, uint64_t* out) {
    if (left > right) { uint64_t s = left; left = right; right = s; }
    if (n != t->n) return EINVAL_;       /* :35-36 */
    if (right >= t->n) return ERANGE_;   /* :37 */
    if (left == right) { *out = left; return OK; } /* :38 */
    const uint32_t e = flog2(right - left);        /* :40 */
    const uint32_t a = t->rows[e][left];
    const uint32_t b = t->rows[e][right - (1ull << e) + 1];
    *out = values[b] < values[a] ? b : a;          /* :43 */
    return OK;
}

uint64_t orc_est_cell_count(const orc_est* t) { /* element_sparse_table.cpp:46-50 */
    uint64_t total = 0;
    for (uint32_t e = 0; e < t->levels; ++e) total += t->n - (1ull << e) + 1;
    return total;
}

uint32_t orc_est_level_count(const orc_est* t) { return t->levels; }

uint64_t orc_est_level(const orc_est* t, uint32_t e, uint32_t* out) {
    if (e >= t->levels) return 0;
    const uint64_t count = t->n - (1ull << e) + 1;
    memcpy(out, t->rows[e], count * sizeof(uint32_t));
    return count;
}

void orc_est_free(orc_est* t) {
    if (!t) return;
    if (t->rows)
        for (uint32_t e = 0; e < t->levels; ++e) free(t->rows[e]);
    free(t->rows);
    free(t);
}

/* ------------------------------------------------------- parallel.hpp */

/* parallel.hpp:13-44: static contiguous chunking, ceil(total/parts) per chunk,
 * worker 0 runs on the calling thread. */
typedef void (*chunk_fn)(uint64_t begin, uint64_t end, unsigned worker, void* ctx);
typedef struct { chunk_fn fn; void* ctx; uint64_t begin, end; unsigned w; } chunk_job;

static void* chunk_tramp(void* p) {
    chunk_job* j = (chunk_job*)p;
    j->fn(j->begin, j->end, j->w, j->ctx);
    return NULL;
}

static void parallel_chunks(uint64_t total, unsigned threads, chunk_fn fn, void* ctx) {
    if (total == 0) return;
    uint64_t parts = threads == 0 ? 1 : threads;
    if (parts > total) parts = total;
    if (parts <= 1) { fn(0, total, 0, ctx); return; }
    const uint64_t chunk = (total + parts - 1) / parts;
    chunk_job* jobs = (chunk_job*)calloc(parts, sizeof(chunk_job));
    pthread_t* tid = (pthread_t*)calloc(parts, sizeof(pthread_t));
    for (unsigned w = 0; w < parts; ++w) {
        uint64_t b = (uint64_t)w * chunk, e = b + chunk < total ? b + chunk : total;
        jobs[w] = (chunk_job){fn, ctx, b, e, w};
    }
    for (unsigned w = 1; w < parts; ++w)
        if (jobs[w].begin < jobs[w].end) pthread_create(&tid[w], NULL, chunk_tramp, &jobs[w]);
    if (jobs[0].begin < jobs[0].end) chunk_tramp(&jobs[0]);
    for (unsigned w = 1; w < parts; ++w)
        if (jobs[w].begin < jobs[w].end) pthread_join(tid[w], NULL);
    free(jobs);
    free(tid);
}

/* ------------------------------------------------------- contraction.cpp */

/* contraction.cpp:13-23: 2q endpoints, origin = (qi << 1) | is_right. */
int orc_collect_endpoints(const uint64_t* Q, uint64_t q, uint32_t* eps) {
    if (q > (1ull << 31)) return EINVAL_; /* :14-15 */
    for (uint64_t i = 0; i < q; ++i) {
        uint64_t l = Q[2 * i], r = Q[2 * i + 1];
        if (l > r) { uint64_t t = l; l = r; r = t; } /* Query ctor normalisation */
        eps[4 * i + 0] = (uint32_t)l;                 /* :19 truncation to 32 bits */
        eps[4 * i + 1] = (uint32_t)(i << 1);
        eps[4 * i + 2] = (uint32_t)r;                 /* :20 */
        eps[4 * i + 3] = (uint32_t)((i << 1) | 1u);
    }
    return OK;
}

static void insertion_sort_eps(uint64_t* e, uint64_t m) { /* stable, by pos (low word) */
    for (uint64_t i = 1; i < m; ++i) {
        uint64_t x = e[i];
        uint32_t k = (uint32_t)x;
        uint64_t j = i;
        while (j > 0 && (uint32_t)e[j - 1] > k) { e[j] = e[j - 1]; --j; }
        e[j] = x;
    }
}

/* Each endpoint is read as one uint64 = pos | (origin << 32) (little endian). */
static int radix_sort_by_pos(uint64_t* e, uint64_t m) { /* contraction.cpp:27-63 */
    if (m < 64) { insertion_sort_eps(e, m); return OK; } /* :29-33 */
    uint64_t (*hist)[256] = (uint64_t(*)[256])calloc(4 * 256, sizeof(uint64_t));
    uint64_t* buf = (uint64_t*)malloc(m * sizeof(uint64_t));
    if (!hist || !buf) { free(hist); free(buf); return ENOMEM_; }
    for (uint64_t i = 0; i < m; ++i) {            /* :35-41 one up-front histogram */
        const uint32_t p = (uint32_t)e[i];
        hist[0][p & 0xFF]++; hist[1][(p >> 8) & 0xFF]++;
        hist[2][(p >> 16) & 0xFF]++; hist[3][(p >> 24) & 0xFF]++;
    }
    uint64_t* src = e;
    uint64_t* dst = buf;
    for (unsigned pass = 0; pass < 4; ++pass) {   /* :46-60 */
        int constant = 0;
        for (unsigned b = 0; b < 256; ++b) if (hist[pass][b] == m) constant = 1; /* :49-50 */
        if (constant) continue;
        uint64_t start[256], off = 0;
        for (unsigned b = 0; b < 256; ++b) { start[b] = off; off += hist[pass][b]; }
        const unsigned shift = pass * 8;
        for (uint64_t i = 0; i < m; ++i) dst[start[((uint32_t)src[i] >> shift) & 0xFF]++] = src[i];
        uint64_t* t = src; src = dst; dst = t;
    }
    if (src != e) memcpy(e, src, m * sizeof(uint64_t)); /* :61-62 */
    free(hist);
    free(buf);
    return OK;
}

static int cmp_pos(const void* a, const void* b) {
    const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
    const uint32_t px = (uint32_t)x, py = (uint32_t)y;
    if (px != py) return px < py ? -1 : 1;
    /* tie-break on origin keeps the result deterministic (stable for collect order) */
    const uint32_t ox = (uint32_t)(x >> 32), oy = (uint32_t)(y >> 32);
    return ox < oy ? -1 : (ox > oy);
}

/* contraction.cpp:67-74 */
int orc_sort_endpoints(uint32_t* eps, uint64_t m, int kind) {
    uint64_t* e = (uint64_t*)eps;
    if (kind == 0) return radix_sort_by_pos(e, m);
    if (kind != 1) return EINVAL_;
    qsort(e, m, sizeof(uint64_t), cmp_pos);  /* :71-72 (comparison sort by pos) */
    return OK;
}

typedef struct {
    const int32_t* A;
    const uint64_t* boundary;
    int32_t* aq_values;
    uint64_t* aq_origin;
    uint64_t* reads; /* per worker */
} scan_ctx;

/* contraction.cpp:81-108: one pass over A[boundary[first]..boundary[last+1]];
 * the boundary element closes area t and opens area t+1 (read once). */
static void scan_areas(uint64_t first_area, uint64_t end_area, unsigned w, void* vctx) {
    scan_ctx* c = (scan_ctx*)vctx;
    const uint64_t last_area = end_area - 1;
    uint64_t area = first_area;
    int32_t cur_min = c->A[c->boundary[first_area]];
    uint64_t cur_pos = c->boundary[first_area];
    uint64_t reads = 1;
    for (uint64_t pos = c->boundary[first_area] + 1; pos <= c->boundary[last_area + 1]; ++pos) {
        const int32_t v = c->A[pos];
        ++reads;
        if (v < cur_min) { cur_min = v; cur_pos = pos; }   /* :93-96 strict => leftmost */
        if (pos == c->boundary[area + 1]) {                 /* :97-105 */
            c->aq_values[area] = cur_min;
            c->aq_origin[area] = cur_pos;
            ++area;
            if (area > last_area) break;
            cur_min = v;
            cur_pos = pos;
        }
    }
    if (c->reads) c->reads[w] += reads;
}

/* contraction.cpp:112-151 */
int orc_build_contracted(const int32_t* A, uint64_t n, const uint32_t* sorted_eps, uint64_t m,
                         unsigned threads, int32_t* aq_values, uint64_t* aq_origin,
                         uint64_t* boundary, uint64_t* nb, uint64_t* reads) {
    *nb = 0;
    if (m == 0) return OK;                                  /* :116 */
    uint32_t prev = sorted_eps[0];
    uint64_t cnt = 0;
    boundary[cnt++] = prev;                                 /* :119-120 */
    for (uint64_t i = 0; i < m; ++i) {                      /* :121-127 dedup */
        const uint32_t p = sorted_eps[2 * i];
        if (p != prev) {
            if (p < prev) return EINVAL_;                   /* :123 */
            boundary[cnt++] = p;
            prev = p;
        }
    }
    *nb = cnt;
    if (boundary[cnt - 1] >= n) return ERANGE_; /* guard: the reference would read past A */
    const uint64_t areas = cnt - 1;
    if (areas == 0) return OK;                              /* :130 */
    unsigned parts = threads <= 1 ? 1 : threads;
    uint64_t* wr = (uint64_t*)calloc(parts, sizeof(uint64_t));
    scan_ctx c = {A, boundary, aq_values, aq_origin, wr};
    parallel_chunks(areas, parts, scan_areas, &c);          /* :134-149 */
    if (reads) for (unsigned w = 0; w < parts; ++w) *reads += wr[w];
    free(wr);
    return OK;
}

/* contraction.cpp:174-199: merge walk of sorted endpoints against boundary. */
int orc_remap_from_sorted(const uint32_t* sorted_eps, uint64_t m, const uint64_t* boundary,
                          uint64_t nb, uint64_t q, uint32_t* cleft, uint32_t* cright,
                          uint8_t* degenerate) {
    memset(cleft, 0, q * sizeof(uint32_t));
    memset(cright, 0, q * sizeof(uint32_t));
    memset(degenerate, 0, q);
    uint64_t b = 0;
    for (uint64_t i = 0; i < m; ++i) {
        const uint32_t pos = sorted_eps[2 * i], origin = sorted_eps[2 * i + 1];
        while (b + 1 < nb && boundary[b] < pos) ++b;                    /* :181 */
        if (b >= nb || boundary[b] != pos) return ELOGIC_;              /* :182-183 */
        const uint64_t qi = origin >> 1;
        if (qi >= q) return ELOGIC_;
        if (origin & 1u) cright[qi] = (uint32_t)b; else cleft[qi] = (uint32_t)b; /* :185-189 */
    }
    for (uint64_t i = 0; i < q; ++i) {                                  /* :191-197 */
        if (cright[i] == cleft[i]) degenerate[i] = 1;
        else --cright[i];
    }
    return OK;
}

/* contraction.cpp:152-171 remap_queries: lower_bound of each end of every query
 * in the boundary list (queries normalised left <= right, types.hpp:18-20); a
 * degenerate query keeps cleft = cright = 0 (:163-166); a missing end is a
 * logic_error (:157-158). */
int orc_remap_queries(const uint64_t* Q, uint64_t q, const uint64_t* boundary, uint64_t nb,
                      uint32_t* cleft, uint32_t* cright, uint8_t* degenerate) {
    for (uint64_t i = 0; i < q; ++i) {
        const uint64_t a = Q[2 * i], b = Q[2 * i + 1];
        const uint64_t l = a < b ? a : b, r = a < b ? b : a;
        cleft[i] = cright[i] = 0;
        degenerate[i] = 0;
        if (l == r) { degenerate[i] = 1; continue; }
        uint64_t idx[2];
        for (int e = 0; e < 2; ++e) {
            const uint64_t p = e ? r : l;
            uint64_t lo = 0, hi = nb;
            while (lo < hi) {
                const uint64_t mid = (lo + hi) / 2;
                if (boundary[mid] < p) lo = mid + 1; else hi = mid;
            }
            if (lo >= nb || boundary[lo] != p) return ELOGIC_;
            idx[e] = lo;
        }
        cleft[i] = (uint32_t)idx[0];
        cright[i] = (uint32_t)(idx[1] - 1);
    }
    return OK;
}

/* SURVEY 8c oracle pipeline, made of the restated reference stages. */
int orc_solve_oracle(const int32_t* A, uint64_t n, const uint64_t* Q, uint64_t q,
                     unsigned threads, uint64_t* answers) {
    if (q == 0) return OK;
    for (uint64_t i = 0; i < q; ++i) {
        uint64_t l = Q[2 * i], r = Q[2 * i + 1];
        if ((l > r ? l : r) >= n) return ERANGE_;
    }
    const uint64_t m = 2 * q;
    int rc = OK;
    uint32_t* eps = (uint32_t*)malloc(m * 2 * sizeof(uint32_t));
    uint64_t* boundary = (uint64_t*)malloc(m * sizeof(uint64_t));
    int32_t* aqv = (int32_t*)malloc(m * sizeof(int32_t));
    uint64_t* aqo = (uint64_t*)malloc(m * sizeof(uint64_t));
    uint32_t* cl = (uint32_t*)malloc(q * sizeof(uint32_t));
    uint32_t* cr = (uint32_t*)malloc(q * sizeof(uint32_t));
    uint8_t* dg = (uint8_t*)malloc(q);
    orc_est* est = NULL;
    if (!eps || !boundary || !aqv || !aqo || !cl || !cr || !dg) { rc = ENOMEM_; goto done; }
    if ((rc = orc_collect_endpoints(Q, q, eps))) goto done;
    if ((rc = orc_sort_endpoints(eps, m, 0))) goto done;
    uint64_t nb = 0;
    if ((rc = orc_build_contracted(A, n, eps, m, threads, aqv, aqo, boundary, &nb, NULL))) goto done;
    if ((rc = orc_remap_from_sorted(eps, m, boundary, nb, q, cl, cr, dg))) goto done;
    const uint64_t areas = nb > 0 ? nb - 1 : 0;
    if (areas > 0 && (rc = orc_est_build(aqv, areas, &est))) goto done;
    for (uint64_t i = 0; i < q; ++i) {
        uint64_t l = Q[2 * i], r = Q[2 * i + 1];
        if (l > r) l = r;
        if (dg[i] || areas == 0) { answers[i] = l; continue; }
        uint64_t t;
        if ((rc = orc_est_arg_min(est, aqv, areas, cl[i], cr[i], &t))) goto done;
        answers[i] = aqo[t];
    }
done:
    orc_est_free(est);
    free(eps); free(boundary); free(aqv); free(aqo); free(cl); free(cr); free(dg);
    return rc;
}

/* ------------------------------------------- SPEC-level block sparse table */

/* level 0 = leftmost argmin per block (trailing block clipped,
 * SPEC.md:213,253); level e entry j = arg-smaller of (e-1, j), (e-1, j+2^(e-1)). */
int orc_build_block_sparse(const int32_t* values, uint64_t m, uint32_t k, uint64_t* table,
                           uint64_t* b_out, uint32_t* levels_out) {
    if (k == 0) return EINVAL_;
    const uint64_t b = (m + k - 1) / k;
    *b_out = b;
    *levels_out = b ? flog2(b) + 1 : 0;
    if (b == 0) return OK;
    for (uint64_t j = 0; j < b; ++j) {
        const uint64_t lo = j * k, hi = (lo + k < m ? lo + k : m);
        uint64_t best = lo;
        for (uint64_t i = lo + 1; i < hi; ++i) if (values[i] < values[best]) best = i;
        table[j] = best;
    }
    for (uint32_t e = 1; e < *levels_out; ++e) {
        const uint64_t half = 1ull << (e - 1);
        uint64_t* cur = table + (uint64_t)e * b;
        const uint64_t* prev = cur - b;
        for (uint64_t j = 0; j < b; ++j) {
            if (j + (1ull << e) <= b) {
                const uint64_t x = prev[j], y = prev[j + half];
                cur[j] = values[y] < values[x] ? y : x;
            } else {
                cur[j] = UINT64_MAX;
            }
        }
    }
    return OK;
}

/* --------------------------------------------- speculative answering (SPEC) */

/* Leftmost argmin over values[lo..hi]; *early counts cells up to and
 * including the first element equal to stop_val (the stored block minimum,
 * which nothing in the block can undercut). */
static uint64_t scan_range(const int32_t* v, uint64_t lo, uint64_t hi, int use_stop,
                           int32_t stop_val, uint64_t* early) {
    uint64_t best = lo, cells = hi - lo + 1;
    for (uint64_t i = lo; i <= hi; ++i) {
        if (v[i] < v[best]) best = i;
        if (use_stop && v[i] == stop_val) { cells = i - lo + 1; break; }
    }
    if (early) *early += cells;
    return best;
}

/* SPEC.md:219-236 inner_span_min + answer_one with the leftmost-exact rule
 * (SURVEY 0.5/7): decisions use only O(1) information (inner span min and
 * the two stored block minima), as the device kernel does.
 *   right endpoint block: scan iff (no best || v[R] <  v[best]) and R > r
 *   left  endpoint block: scan iff (no best || v[L] <= v[best]) and L < l
 *   single block: stored min if l <= p <= r, else scan [l, r].            */
static uint64_t answer_one(const int32_t* v, const uint64_t* table, uint64_t b, uint32_t k,
                           uint64_t l, uint64_t r, uint64_t* S, uint64_t* Se) {
    const uint64_t bl = l / k, br = r / k;
    if (bl == br) {
        const uint64_t p = table[bl];
        if (p >= l && p <= r) return p;
        if (S) *S += r - l + 1;
        return scan_range(v, l, r, p < l, v[p], Se);
    }
    int have = 0;
    uint64_t best = 0;
    if (br - bl >= 2) {                                 /* inner_span_min SPEC.md:222 */
        const uint32_t e = flog2(br - bl - 1);
        const uint64_t a = table[(uint64_t)e * b + bl + 1];
        const uint64_t c = table[(uint64_t)e * b + br - (1ull << e)];
        best = v[c] < v[a] ? c : a;
        have = 1;
    }
    const uint64_t R = table[br], L = table[bl];
    int scan_right = 0, scan_left = 0;
    if (!have || v[R] < v[best]) {
        if (R <= r) { best = R; have = 1; }             /* stored min inside range */
        else scan_right = 1;
    }
    if (!have || v[L] <= v[best]) {
        if (L >= l) { best = L; have = 1; }
        else scan_left = 1;
    }
    if (scan_right) {
        const uint64_t lo = br * (uint64_t)k;
        if (S) *S += r - lo + 1;
        const uint64_t c = scan_range(v, lo, r, 0, 0, Se);
        if (!have || v[c] < v[best]) { best = c; have = 1; }
    }
    if (scan_left) {
        const uint64_t hi = bl * (uint64_t)k + k - 1;
        if (S) *S += hi - l + 1;
        const uint64_t c = scan_range(v, l, hi, 1, v[L], Se);
        if (!have || v[c] <= v[best]) { best = c; have = 1; }
    }
    return best;
}

int orc_solve_bbst(const int32_t* A, uint64_t n, const uint64_t* Q, uint64_t q, uint32_t k,
                   uint64_t* answers, uint64_t* scanned, uint64_t* scanned_early) {
    if (k == 0) return EINVAL_;
    if (q == 0) return OK;
    for (uint64_t i = 0; i < q; ++i) {
        uint64_t l = Q[2 * i], r = Q[2 * i + 1];
        if ((l > r ? l : r) >= n) return ERANGE_;
    }
    const uint64_t b = (n + k - 1) / k;
    const uint32_t levels = flog2(b) + 1;
    uint64_t* table = (uint64_t*)malloc((uint64_t)levels * b * sizeof(uint64_t));
    if (!table) return ENOMEM_;
    uint64_t bb; uint32_t lv;
    orc_build_block_sparse(A, n, k, table, &bb, &lv);
    uint64_t S = 0, Se = 0;
    for (uint64_t i = 0; i < q; ++i) {
        uint64_t l = Q[2 * i], r = Q[2 * i + 1];
        if (l > r) { uint64_t t = l; l = r; r = t; }
        answers[i] = answer_one(A, table, b, k, l, r, &S, &Se);
    }
    if (scanned) *scanned = S;
    if (scanned_early) *scanned_early = Se;
    free(table);
    return OK;
}

int orc_solve_bbst_con(const int32_t* A, uint64_t n, const uint64_t* Q, uint64_t q, uint32_t k,
                       unsigned threads, uint64_t* answers, uint64_t* scanned) {
    if (k == 0) return EINVAL_;
    if (q == 0) return OK;
    for (uint64_t i = 0; i < q; ++i) {
        uint64_t l = Q[2 * i], r = Q[2 * i + 1];
        if ((l > r ? l : r) >= n) return ERANGE_;
    }
    const uint64_t m = 2 * q;
    int rc = OK;
    uint32_t* eps = (uint32_t*)malloc(m * 2 * sizeof(uint32_t));
    uint64_t* boundary = (uint64_t*)malloc(m * sizeof(uint64_t));
    int32_t* aqv = (int32_t*)malloc(m * sizeof(int32_t));
    uint64_t* aqo = (uint64_t*)malloc(m * sizeof(uint64_t));
    uint32_t* cl = (uint32_t*)malloc(q * sizeof(uint32_t));
    uint32_t* cr = (uint32_t*)malloc(q * sizeof(uint32_t));
    uint8_t* dg = (uint8_t*)malloc(q);
    uint64_t* table = NULL;
    uint64_t S = 0;
    if (!eps || !boundary || !aqv || !aqo || !cl || !cr || !dg) { rc = ENOMEM_; goto done; }
    if ((rc = orc_collect_endpoints(Q, q, eps))) goto done;               /* stage 1 */
    if ((rc = orc_sort_endpoints(eps, m, 0))) goto done;
    uint64_t nb = 0;
    if ((rc = orc_build_contracted(A, n, eps, m, threads, aqv, aqo, boundary, &nb, NULL)))
        goto done;                                                        /* stage 2 */
    if ((rc = orc_remap_from_sorted(eps, m, boundary, nb, q, cl, cr, dg))) goto done;
    const uint64_t areas = nb > 0 ? nb - 1 : 0;
    uint64_t b = 0;
    uint32_t levels = 0;
    if (areas > 0) {                                                      /* stage 3 */
        const uint64_t bb = (areas + k - 1) / k;
        table = (uint64_t*)malloc((uint64_t)(flog2(bb) + 1) * bb * sizeof(uint64_t));
        if (!table) { rc = ENOMEM_; goto done; }
        orc_build_block_sparse(aqv, areas, k, table, &b, &levels);
    }
    for (uint64_t i = 0; i < q; ++i) {                                    /* stage 4 */
        uint64_t l = Q[2 * i], r = Q[2 * i + 1];
        if (l > r) l = r;
        if (dg[i] || areas == 0) { answers[i] = l; continue; }
        answers[i] = aqo[answer_one(aqv, table, b, k, cl[i], cr[i], &S, NULL)];
    }
    if (scanned) *scanned = S;
done:
    free(table);
    free(eps); free(boundary); free(aqv); free(aqo); free(cl); free(cr); free(dg);
    return rc;
}
