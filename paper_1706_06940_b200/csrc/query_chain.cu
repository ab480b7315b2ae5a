// query_chain.cu -- multi-level BbST for an arbitrary dividing chain
// k_1 < k_2 < ... < k_h (h >= 2).
//
// Levels: M_j (j = 0 .. h-2) holds the leftmost-min key of every k_{j+1}-block
// of A (trailing block clipped); the top level is the block Sparse
// Table over the k_h-blocks, built from M_{h-2} ("h = 2 build uses
// level-1 minima to compute level-2 minima").  The [32, k] chain keeps its
// specialised kernels (query.cu k_query_ml_flat); every other chain answers here.
//
// Answering (answer_one_ml): the top level is BbST's -- inner
// span by two ST probes, endpoint blocks by the leftmost-exact speculative rule
// (a left partial is descended iff its stored minimum lies outside the range and
// v(stored) <= v(best), a right partial iff v(stored) < v(best), an in-block
// range iff its stored minimum lies outside).  A partial range inside one
// k_{j+1}-block is resolved from its k_j-children: the full children by one
// warp-strided read of M_{j-1}, each partial child by its stored key when that
// lies inside, else (rule permitting) one level down; at the bottom raw A is
// scanned inside one k_1-block.  Each edge descends one chain of partial
// children, so per query at most 2(k_h/k_{h-1} + ... + k_2/k_1 + k_1) cells are
// read (SPEC.md:317 read-counter bound).
//
// B200 mapping: one lane per query, lane-private fixed-shape descents (no work
// list: an in-block range descends while it stays inside one child, then splits
// into one left and one right chain, each a loop over the levels with <= 1
// partial child per level).  All lanes' loads overlap; a warp-per-query version
// with cooperative reads was latency-bound (c3, [64, 512]: 6.9 ms of queries).
#include "common.cuh"
#include "kernels.h"

namespace brmq {
namespace {

constexpr int kThreads = 128;

struct ChainArgs {
    const int32_t* A;
    uint64_t n;
    const uint64_t* M[kMaxChain];  // M[j]: k_{j+1}-block minima, j < h - 1
    uint64_t mlen[kMaxChain];
    uint32_t ks[kMaxChain];
    uint32_t h;
    const uint64_t* ST;
    uint64_t stride;
    const uint64_t* Q;
    uint64_t q;
    uint64_t* ans;
    uint32_t* err;
};

__device__ __forceinline__ uint64_t keys_min(const uint64_t* M, uint64_t a, uint64_t b, uint64_t best) {
#pragma unroll 4
    for (uint64_t c = a; c <= b; ++c) best = kmin(best, __ldg(M + c));
    return best;
}

__device__ __forceinline__ uint64_t cells_min(const int32_t* A, uint64_t a, uint64_t b, uint64_t best) {
#pragma unroll 4
    for (uint64_t i = a; i <= b; ++i) best = kmin(best, pack_key(__ldg(A + i), uint32_t(i)));
    return best;
}

// Left edge: [lo, end of its k_{lev+1}-block]; descend while the partial child's
// stored minimum lies left of lo and v(stored) <= v(best) (leftmost ties).
__device__ __forceinline__ uint64_t left_chain(const ChainArgs& c, uint64_t lo, uint32_t lev, uint64_t best) {
    for (;;) {
        const uint64_t bs = c.ks[lev];
        const uint64_t end = (lo / bs) * bs + bs - 1 < c.n - 1 ? (lo / bs) * bs + bs - 1 : c.n - 1;
        if (lev == 0) return cells_min(c.A, lo, end, best);
        const uint64_t cs = c.ks[lev - 1];
        const uint64_t* M = c.M[lev - 1];
        const uint64_t cl = lo / cs, cr = end / cs;
        const bool lfull = lo % cs == 0;
        best = keys_min(M, lfull ? cl : cl + 1, cr, best);  // full children
        if (lfull) return best;
        const uint64_t K = __ldg(M + cl);
        if (key_pos(K) >= lo) return kmin(best, K);
        if (best != kNoKey && key_hi(K) > key_hi(best)) return best;
        --lev;
    }
}

// Right edge: [start of its k_{lev+1}-block, hi]; descend iff v(stored) < v(best).
__device__ __forceinline__ uint64_t right_chain(const ChainArgs& c, uint64_t hi, uint32_t lev, uint64_t best) {
    for (;;) {
        const uint64_t bs = c.ks[lev];
        const uint64_t start = (hi / bs) * bs;
        if (lev == 0) return cells_min(c.A, start, hi, best);
        const uint64_t cs = c.ks[lev - 1];
        const uint64_t* M = c.M[lev - 1];
        const uint64_t cl = start / cs, cr = hi / cs;
        const bool rfull = (hi + 1) % cs == 0 || hi == c.n - 1;
        if (rfull) return keys_min(M, cl, cr, best);
        if (cr > cl) best = keys_min(M, cl, cr - 1, best);  // full children
        const uint64_t K = __ldg(M + cr);
        if (key_pos(K) <= hi) return kmin(best, K);
        if (best != kNoKey && key_hi(K) >= key_hi(best)) return best;
        --lev;
    }
}

__device__ __forceinline__ uint64_t answer_chain(const ChainArgs& c, uint64_t l, uint64_t r) {
    const uint32_t top = c.h - 1;  // the ST level: blocks of k_h
    const uint64_t kh = c.ks[top];
    const uint64_t bl = l / kh, br = r / kh;
    const uint64_t Lk = __ldg(c.ST + bl);
    if (bl == br) {
        if (key_pos(Lk) >= l && key_pos(Lk) <= r) return Lk;
        // in-block: descend while [l, r] stays inside one child, then split
        uint32_t lev = top;
        for (;;) {
            if (lev == 0) return cells_min(c.A, l, r, kNoKey);
            const uint64_t cs = c.ks[lev - 1];
            const uint64_t* M = c.M[lev - 1];
            const uint64_t cl = l / cs, cr = r / cs;
            const bool lfull = l % cs == 0;
            const bool rfull = (r + 1) % cs == 0 || r == c.n - 1;
            if (cl == cr) {
                const uint64_t K = __ldg(M + cl);
                if ((lfull && rfull) || (key_pos(K) >= l && key_pos(K) <= r)) return K;
                --lev;
                continue;
            }
            uint64_t best = kNoKey;
            const uint64_t f0 = lfull ? cl : cl + 1, f1 = rfull ? cr : cr - 1;
            if (f0 <= f1) best = keys_min(M, f0, f1, best);
            if (!rfull) {
                const uint64_t K = __ldg(M + cr);
                if (key_pos(K) <= r) best = kmin(best, K);
                else if (best == kNoKey || key_hi(K) < key_hi(best)) best = right_chain(c, r, lev - 1, best);
            }
            if (!lfull) {
                const uint64_t K = __ldg(M + cl);
                if (key_pos(K) >= l) best = kmin(best, K);
                else if (best == kNoKey || key_hi(K) <= key_hi(best)) best = left_chain(c, l, lev - 1, best);
            }
            return best;
        }
    }
    uint64_t best = kNoKey;
    if (br - bl >= 2) {  // inner_span_min
        const uint32_t e = floor_log2_u64(br - bl - 1);
        const uint64_t* row = c.ST + uint64_t(e) * c.stride;
        best = kmin(__ldg(row + bl + 1), __ldg(row + br - (1ull << e)));
    }
    const uint64_t Rk = __ldg(c.ST + br);
    if (key_pos(Rk) <= r) best = kmin(best, Rk);
    else if (best == kNoKey || key_hi(Rk) < key_hi(best)) best = right_chain(c, r, top, best);
    if (key_pos(Lk) >= l) best = kmin(best, Lk);
    else if (best == kNoKey || key_hi(Lk) <= key_hi(best)) best = left_chain(c, l, top, best);
    return best;
}

__global__ void __launch_bounds__(kThreads) k_query_chain(const __grid_constant__ ChainArgs c,
                                                          const CtlPublish pub) {
    brmq::pdl_wait();
    const uint64_t qi = uint64_t(blockIdx.x) * kThreads + threadIdx.x;
    if (qi < c.q) {
        const ulonglong2 x = __ldcs(reinterpret_cast<const ulonglong2*>(c.Q) + qi);  // streamed
        uint64_t l = x.x, r = x.y;
        if (l > r) { const uint64_t t = l; l = r; r = t; }  // types.hpp:18-20
        uint64_t out;
        if (r >= c.n) {  // naive.hpp:14-15
            atomicOr(c.err, 1u);
            out = ~0ull;
        } else if (l == r) {
            out = l;
        } else {
            out = key_pos(answer_chain(c, l, r));
        }
        __stcs(reinterpret_cast<unsigned long long*>(c.ans + qi), (unsigned long long)out);
    }
}

}  // namespace

int launch_query_chain(const int32_t* A, uint64_t n, const uint32_t* ks, uint32_t h,
                       const uint64_t* const* M, const uint64_t* ST, uint64_t stride,
                       const uint64_t* Q, uint64_t q, uint64_t* answers, uint32_t* err,
                       cudaStream_t stream, const CtlPublish& pub) {
    ChainArgs a{};
    a.A = A;
    a.n = n;
    a.h = h;
    for (uint32_t j = 0; j < h; ++j) {
        a.ks[j] = ks[j];
        if (j + 1 < h) {
            a.M[j] = M[j];
            a.mlen[j] = (n + ks[j] - 1) / ks[j];
        }
    }
    a.ST = ST;
    a.stride = stride;
    a.Q = Q;
    a.q = q;
    a.ans = answers;
    a.err = err;
    brmq::launch_k(k_query_chain, dim3(unsigned((q + kThreads - 1) / kThreads)), dim3(kThreads), 0, stream, a, pub);
    return 1;
}

}  // namespace brmq
