// query.cu -- speculative query answering over the block Sparse Table (K3).
//
// SPEC.md:219-236 (inner_span_min + answer_one), PAPER.md:242-255 (BbST_CON
// stage 4) and PAPER.md:301-327 (BbST), with the leftmost-exact speculation
// rule of SURVEY 0.5/7 (SPEC's literal "scan only if stored min < best" is
// value-exact but not position-exact under ties):
//   inner span  : blocks bl+1..br-1 via two ST probes at e = floor_log2(br-bl-1)
//   right block : scan iff (no best || v(R) <  v(best)) and the stored min R lies right of r
//   left block  : scan iff (no best || v(L) <= v(best)) and the stored min L lies left of l
//   single block: stored min if it lies in [l, r], else scan [l, r]
// All candidates are packed keys, so combining them is an unsigned min.
//
// B200 design (k_query): one lane per query does the O(1) part (4 random 8-byte
// ST reads, L2-resident for n = 1e8).  Lanes that need a partial-block scan
// publish it with __ballot_sync and the whole warp scans the pending ranges, TPR
// per round: each lane issues VPL predicated 128-bit loads per range (only for
// vectors that overlap it), folds them into a 32-bit (value, position)
// accumulator, and a redux.sync pair reduces the range to its leftmost-min key,
// which goes back to the owning lane.  No lane idles on the queries that need
// no scan.  With a 32-element sub-block level (multi-level BbST [32, k], and
// BbST_CON over A_Q for power-of-two k in [64, 512]) k_query_flat answers
// instead: fixed-shape lane-private descents through the sub-block keys and
// pooled half-warp row scans (see the comment above ml_flat_group).
//
// Two element policies share the kernel: int32 A (key = pack(A[i], i)) for
// BbST, and packed keys A_Q (key carries the original position, "aq_origin")
// for BbST_CON.  For A_Q, "stored min lies inside the range" is decided on
// original positions: aq_origin is non-decreasing, so a block-min
// key whose origin is >= l (resp. <= r) is present in the partial range.
#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace brmq {
namespace {

constexpr int kThreads = 256;
// k_query's register budget for the k = 512 batch instance (4 vectors per lane):
// 48 resident warps per SM (<= 40 registers, no spills with the round-2 scans;
// c3 / c4 / c5 query phases 0.574 / 0.249 / 0.193 -> 0.538 / 0.241 / 0.187 ms
// against 40 warps, 0.610 / 0.255 / 0.200 at 32).  (Round 1, per-element
// accumulators: 40 warps, 48 registers; 48 warps spilled.)
// k_query_flat's register budget: the 128-thread instances for 56 resident warps
// per SM (32 registers, a few spilled words), the 32-thread (small-batch)
// instances for 64 registers as before.  c3 [32, 512] query 0.471 -> 0.428 ms, c3-con
// 0.533 -> 0.486 ms, c5-con 0.411 -> 0.405 ms (48 warps: 0.442 / 0.505 / 0.407).
// (An explicit minimum of 1 CTA lets ptxas take up to 255 registers: 0.90 ms.)
#ifndef BRMQ_FLAT_WARPS
#define BRMQ_FLAT_WARPS 56
#endif
#ifndef BRMQ_QUERY_WARPS
#define BRMQ_QUERY_WARPS 48
#endif

// WHOLE: len is a multiple of 4, so every vector a scan touches lies inside the
// array and load_vec is one unchecked 128-bit load (c3: the per-vector tail test
// was ~8% of the h = 1 query kernel's instructions).
template <bool WHOLE>
struct ElemI32T {
    using vec_t = int4;
    static constexpr int EPV = 4;
    static constexpr bool kI32 = true;
    const int32_t* data;
    uint64_t len;
    unsigned long long* scanned = nullptr;  // debug counter (launch_query_direct)
    __device__ __forceinline__ uint64_t key_at(uint64_t i) const {
        return pack_key(__ldg(data + i), uint32_t(i));
    }
    // 128-bit load when the vector lies inside the array, scalar tail otherwise
    // (never touches memory past `len`; out-of-range lanes are masked later).
    __device__ __forceinline__ vec_t load_vec(uint64_t v) const {
        if (WHOLE || v * 4 + 3 < len) return ld_stream_v4(reinterpret_cast<const int4*>(data) + v);
        int4 x = make_int4(0, 0, 0, 0);
        if (v * 4 + 0 < len) x.x = __ldg(data + v * 4 + 0);
        if (v * 4 + 1 < len) x.y = __ldg(data + v * 4 + 1);
        if (v * 4 + 2 < len) x.z = __ldg(data + v * 4 + 2);
        return x;
    }
    // Lane accumulator over the lane's vectors in increasing position order: a
    // value and its position in 32-bit registers (strict '<' keeps the leftmost),
    // one packed key at the end.  Positions fit 32 bits (n <= 2^32 - 1).
    struct Acc {
        int32_t bv = 0x7FFFFFFF;
        uint32_t bi = 0xFFFFFFFFu;  // none yet
        __device__ __forceinline__ void add(const vec_t& x, uint32_t v, uint32_t lo, uint32_t span) {
            const uint32_t p = v * 4;
            const int32_t e[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (p + t - lo <= span && (e[t] < bv || bi == 0xFFFFFFFFu)) {  // p + t in [lo, lo + span]
                    bv = e[t];
                    bi = p + t;
                }
        }
        __device__ __forceinline__ uint64_t key() const { return bi == 0xFFFFFFFFu ? kNoKey : pack_key(bv, bi); }
    };
};
using ElemI32 = ElemI32T<false>;

struct ElemKey {
    using vec_t = uint4;
    static constexpr int EPV = 2;
    static constexpr bool kI32 = false;
    const uint64_t* data;  // allocation padded to a multiple of 2 keys by the caller
    __device__ __forceinline__ uint64_t key_at(uint64_t i) const { return __ldg(data + i); }
    __device__ __forceinline__ vec_t load_vec(uint64_t v) const {
        return ld_stream_u4(reinterpret_cast<const uint4*>(data) + v);
    }
    __device__ __forceinline__ uint64_t vec_min(const vec_t& x, uint64_t v, uint64_t lo,
                                                uint64_t hi) const {
        const uint64_t p = v * 2;
        uint64_t b = kNoKey;
        if (p + 0 >= lo && p + 0 <= hi) b = kmin(b, (uint64_t(x.y) << 32) | x.x);
        if (p + 1 >= lo && p + 1 <= hi) b = kmin(b, (uint64_t(x.w) << 32) | x.z);
        return b;
    }
    struct Acc {
        uint64_t b = kNoKey;
        __device__ __forceinline__ void add(const vec_t& x, uint32_t v, uint32_t lo, uint32_t span) {
            const uint32_t p = v * 2;
            if (p - lo <= span) b = kmin(b, (uint64_t(x.y) << 32) | x.x);
            if (p + 1 - lo <= span) b = kmin(b, (uint64_t(x.w) << 32) | x.z);
        }
        __device__ __forceinline__ uint64_t key() const { return b; }
    };
};

// A query resolved to index coordinates [il, ir] of the scanned array and
// original-position coordinates [pl, pr] of A (equal for BbST).
struct Resolved {
    uint64_t il, ir, pl, pr;
    uint64_t direct;  // final answer when `done` (degenerate query / range error)
    bool done;
};

struct QueryDirect {
    const uint64_t* Q;
    uint64_t n;
    uint32_t* err;
    __device__ __forceinline__ Resolved resolve(uint64_t i) const {
        const ulonglong2 x = __ldcs(reinterpret_cast<const ulonglong2*>(Q) + i);  // streamed
        uint64_t l = x.x, r = x.y;
        if (l > r) { const uint64_t t = l; l = r; r = t; }  // types.hpp:18-20
        Resolved o{l, r, l, r, 0, false};
        if (r >= n) {                                        // naive.hpp:14-15
            atomicOr(err, 1u);
            o.direct = ~0ull;
            o.done = true;
        } else if (l == r) {
            o.direct = l;
            o.done = true;
        }
        return o;
    }
};

struct QueryContracted {
    const uint64_t* Q;
    const uint32_t* cleft;
    const uint32_t* cright_raw;
    __device__ __forceinline__ Resolved resolve(uint64_t i) const {
        const ulonglong2 x = __ldcs(reinterpret_cast<const ulonglong2*>(Q) + i);  // streamed
        uint64_t l = x.x, r = x.y;
        if (l > r) { const uint64_t t = l; l = r; r = t; }
        const uint32_t cl = __ldg(cleft + i), cr = __ldg(cright_raw + i);
        Resolved o{cl, uint64_t(cr) - 1, l, r, l, cl == cr};  // degenerate: answer = left
                                                               // (contraction.cpp:192-193)
        return o;
    }
};

// Bitmap pipeline: the contracted coordinates come straight from the per-word
// (rank prefix, bits) the contraction emitted -- remap_queries_from_sorted
// (contraction.cpp:174-199) folded into the query kernel.
struct QueryContractedWI {
    const uint64_t* Q;
    const uint2* word_info;
    uint64_t n;
    __device__ __forceinline__ Resolved resolve(uint64_t i) const {
        const ulonglong2 x = __ldcs(reinterpret_cast<const ulonglong2*>(Q) + i);  // streamed
        uint64_t l = x.x, r = x.y;
        if (l > r) { const uint64_t t = l; l = r; r = t; }
        if (r >= n) { r = n - 1; if (l > r) l = r; }  // already reported by the endpoint stage
        const uint2 wl = __ldg(word_info + (l >> 5)), wr = __ldg(word_info + (r >> 5));
        const uint32_t cl = wl.x + __popc(wl.y & ((1u << (l & 31)) - 1u));
        const uint32_t cr = wr.x + __popc(wr.y & ((1u << (r & 31)) - 1u));
        Resolved o{cl, uint64_t(cr) - 1, l, r, l, cl == cr};
        return o;
    }
};

// L2 prefetch of the 16-byte vectors [v0, v0 + nv) of A (one bulk request per
// range, issued by the lane that owns the query as soon as it knows the range
// must be scanned): the warp's serial scan rounds then hit L2 (~250 cycles)
// instead of DRAM, and all of a warp's ranges are fetched concurrently.
__device__ __forceinline__ void prefetch_vecs_l2(const int32_t* A, uint64_t v0, uint32_t nv) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(A + 4 * v0), "r"(nv * 16u)
                 : "memory");
}

// Masked minimum of one 16-byte vector: elements t in [a, b] only (a vector of
// the range always holds at least one of them).
__device__ __forceinline__ int32_t vec_min_masked(const int4& x, uint32_t a, uint32_t b) {
    const int32_t m0 = a == 0u ? x.x : 0x7FFFFFFF;
    const int32_t m1 = (a <= 1u && b >= 1u) ? x.y : 0x7FFFFFFF;
    const int32_t m2 = (a <= 2u && b >= 2u) ? x.z : 0x7FFFFFFF;
    const int32_t m3 = b == 3u ? x.w : 0x7FFFFFFF;
    return __vimin3_s32(m0, m1, min(m2, m3));
}
// First element t in [a, b] of the vector equal to wv (one exists).
__device__ __forceinline__ uint32_t vec_first_eq(const int4& x, uint32_t a, uint32_t b, int32_t wv) {
    return (a == 0u && x.x == wv) ? 0u : (a <= 1u && b >= 1u && x.y == wv) ? 1u
                                       : (a <= 2u && b >= 2u && x.z == wv) ? 2u : 3u;
}

// Leftmost-min key of A[lo..hi] (within one block, 16-byte aligned A), by the
// whole warp.  Value pass: lane j takes the range's vectors j, j + 32, ...
// (NJ per lane, coalesced), masked 3-way mins, one redux.min; position pass:
// each lane's first vector holding the minimum gives its first element equal to
// it, and one redux.min over the element offsets is the leftmost position.
// ~30 instructions per lane for a range of <= 32 vectors (NJ = 1), against ~90
// for the per-element (value, position) accumulator it replaces (ncu: the c3
// h = 1 query kernel was issue-bound, 69% of issue slots busy).
template <int NJ, class E>
__device__ __forceinline__ uint64_t scan_i32_vecs(const E& e, uint64_t v0, uint32_t nv,
                                                  uint32_t lo_t, uint32_t hi_t) {
    const uint32_t lane = lane_id();
    int4 x[NJ];
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const uint32_t vi = lane + 32u * j;
        x[j] = vi < nv ? e.load_vec(v0 + vi) : make_int4(0, 0, 0, 0);
    }
    int32_t m[NJ];
    int32_t lm = 0x7FFFFFFF;
#pragma unroll
    for (int j = 0; j < NJ; ++j) {
        const uint32_t vi = lane + 32u * j;
        const uint32_t a = vi == 0u ? lo_t : 0u, b = vi == nv - 1u ? hi_t : 3u;
        m[j] = vi < nv ? vec_min_masked(x[j], a, b) : 0x7FFFFFFF;
        lm = min(lm, m[j]);
    }
    const int32_t wv = __reduce_min_sync(kFull, lm);
    uint32_t cand = 0xFFFFFFFFu;
#pragma unroll
    for (int j = NJ - 1; j >= 0; --j) {  // the lane's first vector holding wv wins
        const uint32_t vi = lane + 32u * j;
        if (vi < nv && m[j] == wv) {
            const uint32_t a = vi == 0u ? lo_t : 0u, b = vi == nv - 1u ? hi_t : 3u;
            cand = 4u * vi + vec_first_eq(x[j], a, b, wv);
        }
    }
    const uint32_t off = __reduce_min_sync(kFull, cand);
    return pack_key(wv, uint32_t(4 * v0) + off);
}

template <int VPL, class E>
__device__ __forceinline__ uint64_t scan_i32(const E& e, uint32_t lo, uint32_t hi) {
    const uint64_t v0 = lo >> 2;
    const uint32_t nv = (hi >> 2) - (lo >> 2) + 1u;
    if (VPL <= 1 || nv <= 32u) return scan_i32_vecs<1, E>(e, v0, nv, lo & 3u, hi & 3u);
    return scan_i32_vecs<(VPL > 1 ? VPL : 1), E>(e, v0, nv, lo & 3u, hi & 3u);
}

template <class E>
__device__ __forceinline__ uint64_t scan_generic(const E& e, uint64_t lo, uint64_t hi) {
    uint64_t b = kNoKey;
    for (uint64_t i = lo + lane_id(); i <= hi; i += 32) b = kmin(b, e.key_at(i));
    return warp_min_key(b);
}

// VPL vectors per lane cover one block (k = 32 * EPV * VPL); TPR ranges per round.
// WPQ: one warp per query (small batches: the per-warp rounds of partial scans
// are the latency chain, so spread the queries over 32x more warps).
template <class E, class QP, int VPL, int TPR, bool WPQ = false, int NT = kThreads>
__device__ __forceinline__ void query_body(E elem, QP qp, uint32_t k_rt,
                                              const uint64_t* __restrict__ ST,
                                              uint64_t stride, uint64_t q,
                                              uint64_t* __restrict__ answers,
                                              const CtlPublish pub) {
    // BbST_CON only: the BbST (QueryDirect) instances publish from a tail kernel.
    // Compiled out of them: inlined there, it cost the c3 / c5 h = 1 query 16 bytes
    // of spills per thread and 0.538 -> 0.578 / 0.188 -> 0.233 ms.
    if constexpr (!std::is_same<QP, QueryDirect>::value) publish_early(pub);
    // the vectorised instances know k at compile time (k = 32 * EPV * VPL): block
    // indices by shifts, not 64-bit divisions
    const uint32_t k = VPL > 0 ? uint32_t(32 * E::EPV * (VPL > 0 ? VPL : 1)) : k_rt;
    const unsigned lane = lane_id();
    const uint64_t i = WPQ ? (uint64_t(blockIdx.x) * NT + threadIdx.x) >> 5
                           : (uint64_t(blockIdx.x) * NT + threadIdx.x);
    const bool active = i < q && (!WPQ || lane == 0);

    uint64_t best = kNoKey, direct = 0;
    bool done = false, t0 = false, t1 = false;
    uint64_t lo0 = 0, hi0 = 0, lo1 = 0, hi1 = 0;
    if (active) {
        const Resolved rq = qp.resolve(i);
        direct = rq.direct;
        done = rq.done;
        if (!done) {
            const uint64_t bl = rq.il / k, br = rq.ir / k;
            const uint64_t L = __ldg(ST + bl);
            if (bl == br) {
                if (key_pos(L) >= rq.pl && key_pos(L) <= rq.pr) best = L;
                else { t0 = true; lo0 = rq.il; hi0 = rq.ir; }
            } else {
                if (br - bl >= 2) {  // inner_span_min
                    const uint32_t e = floor_log2_u64(br - bl - 1);
                    const uint64_t* row = ST + uint64_t(e) * stride;
                    best = kmin(__ldg(row + bl + 1), __ldg(row + br - (1ull << e)));
                }
                const uint64_t R = __ldg(ST + br);
                if (best == kNoKey || key_hi(R) < key_hi(best)) {
                    if (key_pos(R) <= rq.pr) best = kmin(best, R);
                    else { t1 = true; lo1 = br * k; hi1 = rq.ir; }
                }
                if (best == kNoKey || key_hi(L) <= key_hi(best)) {
                    if (key_pos(L) >= rq.pl) best = kmin(best, L);
                    else { t0 = true; lo0 = rq.il; hi0 = bl * k + k - 1; }
                }
            }
        }
    }

    if constexpr (E::kI32 && VPL > 0) {
        // a range inside at most two 16-byte vectors (<= 8 cells) is scanned by its
        // own lane at once: no warp round for it (c3: ~1 in 10 queries)
        auto tiny = [&](bool& t, uint64_t lo, uint64_t hi) {
            if (!t || (hi >> 2) - (lo >> 2) > 1) return;
            t = false;
            // masked 3-way minima of the one or two vectors, then the first element
            // equal to the minimum (leftmost: the first vector wins ties)
            const uint32_t lo32 = uint32_t(lo), hi32 = uint32_t(hi);
            const bool two = (hi32 >> 2) != (lo32 >> 2);
            const int4 x0 = elem.load_vec(lo >> 2);
            const int4 x1 = two ? elem.load_vec((lo >> 2) + 1) : x0;
            const uint32_t a0 = lo32 & 3u, b0 = two ? 3u : (hi32 & 3u), b1 = hi32 & 3u;
            const int32_t m0 = vec_min_masked(x0, a0, b0);
            const int32_t m1 = two ? vec_min_masked(x1, 0u, b1) : 0x7FFFFFFF;
            const int32_t wv = min(m0, m1);
            const uint32_t pos = m0 == wv ? (lo32 & ~3u) + vec_first_eq(x0, a0, b0, wv)
                                          : (lo32 & ~3u) + 4u + vec_first_eq(x1, 0u, b1, wv);
            best = kmin(best, pack_key(wv, pos));
        };
#ifndef BRMQ_NO_SCAN_COUNT
        if (elem.scanned) {  // instrumented: cells of every range the rule scans
            uint64_t cells = (t0 ? hi0 - lo0 + 1 : 0) + (t1 ? hi1 - lo1 + 1 : 0);
            cells = __reduce_add_sync(kFull, uint32_t(cells));
            if (lane == 0 && cells) atomicAdd(elem.scanned, (unsigned long long)cells);
        }
#endif
        tiny(t0, lo0, hi0);
        tiny(t1, lo1, hi1);
    }
    // Warp-cooperative partial-block scans.
    unsigned m0 = __ballot_sync(kFull, t0), m1 = __ballot_sync(kFull, t1);
    if constexpr (E::kI32 && VPL > 0) {
        // int32 A (BbST): ranges prefetched into L2 at once, then one range per
        // round by the value-then-position scan (positions < 2^32: 32-bit shuffles)
        // (whole vectors inside the array only: the last partial vector is not prefetched)
        if (t0 && (hi0 | 3) < elem.len) prefetch_vecs_l2(elem.data, lo0 >> 2, uint32_t((hi0 >> 2) - (lo0 >> 2)) + 1u);
        if (t1 && (hi1 | 3) < elem.len) prefetch_vecs_l2(elem.data, lo1 >> 2, uint32_t((hi1 >> 2) - (lo1 >> 2)) + 1u);
        // ranges within 16 vectors (<= 64 cells) go two per round, one per half warp
        unsigned s0 = __ballot_sync(kFull, t0 && (hi0 >> 2) - (lo0 >> 2) < 16);
        unsigned s1 = __ballot_sync(kFull, t1 && (hi1 >> 2) - (lo1 >> 2) < 16);
        m0 &= ~s0;
        m1 &= ~s1;
        const bool upper = lane >= 16;
        const uint32_t j = lane & 15u;
        while (s0 | s1) {
            int sa = -1, sb = -1;
            uint32_t la = 0, ha = 0, lb = 0, hb = 0;
            auto take = [&](int& sl, uint32_t& lo, uint32_t& hi) {
                if (s0) {
                    sl = __ffs(s0) - 1;
                    s0 &= s0 - 1;
                    lo = __shfl_sync(kFull, uint32_t(lo0), sl);
                    hi = __shfl_sync(kFull, uint32_t(hi0), sl);
                } else if (s1) {
                    sl = __ffs(s1) - 1;
                    s1 &= s1 - 1;
                    lo = __shfl_sync(kFull, uint32_t(lo1), sl);
                    hi = __shfl_sync(kFull, uint32_t(hi1), sl);
                }
            };
            take(sa, la, ha);
            take(sb, lb, hb);
            const uint32_t lo = upper ? lb : la, hi = upper ? hb : ha;
            const bool live = upper ? sb >= 0 : true;
            const uint32_t nv = (hi >> 2) - (lo >> 2) + 1u;
            const bool in = live && j < nv;
            const int4 x = in ? elem.load_vec((lo >> 2) + j) : make_int4(0, 0, 0, 0);
            const uint32_t a = j == 0u ? (lo & 3u) : 0u, b = j == nv - 1u ? (hi & 3u) : 3u;
            const int32_t mv = in ? vec_min_masked(x, a, b) : 0x7FFFFFFF;
            const int32_t wa = __reduce_min_sync(kFull, upper ? 0x7FFFFFFF : mv);
            const int32_t wb = __reduce_min_sync(kFull, upper ? mv : 0x7FFFFFFF);
            const int32_t wv = upper ? wb : wa;
            const uint32_t cand = (in && mv == wv) ? 4u * j + vec_first_eq(x, a, b, wv) : 0xFFFFFFFFu;
            const uint32_t oa = __reduce_min_sync(kFull, upper ? 0xFFFFFFFFu : cand);
            const uint32_t ob = __reduce_min_sync(kFull, upper ? cand : 0xFFFFFFFFu);
            if (int(lane) == sa) best = kmin(best, pack_key(wa, (la & ~3u) + oa));
            if (sb >= 0 && int(lane) == sb) best = kmin(best, pack_key(wb, (lb & ~3u) + ob));
        }
        while (m0 | m1) {
            int sl;
            uint32_t lo, hi;
            if (m0) {
                sl = __ffs(m0) - 1;
                m0 &= m0 - 1;
                lo = __shfl_sync(kFull, uint32_t(lo0), sl);
                hi = __shfl_sync(kFull, uint32_t(hi0), sl);
            } else {
                sl = __ffs(m1) - 1;
                m1 &= m1 - 1;
                lo = __shfl_sync(kFull, uint32_t(lo1), sl);
                hi = __shfl_sync(kFull, uint32_t(hi1), sl);
            }
            const uint64_t kb = scan_i32<VPL, E>(elem, lo, hi);
            if (int(lane) == sl) best = kmin(best, kb);
        }
        m0 = m1 = 0;
    }
    while (m0 | m1) {
        uint64_t tlo[TPR > 0 ? TPR : 1], thi[TPR > 0 ? TPR : 1];
        int src[TPR > 0 ? TPR : 1];
#pragma unroll
        for (int u = 0; u < (TPR > 0 ? TPR : 1); ++u) {
            src[u] = -1;
            tlo[u] = 0;
            thi[u] = 0;
            if (m0) {
                const int s = __ffs(m0) - 1;
                m0 &= m0 - 1;
                src[u] = s;
                tlo[u] = __shfl_sync(kFull, lo0, s);
                thi[u] = __shfl_sync(kFull, hi0, s);
            } else if (m1) {
                const int s = __ffs(m1) - 1;
                m1 &= m1 - 1;
                src[u] = s;
                tlo[u] = __shfl_sync(kFull, lo1, s);
                thi[u] = __shfl_sync(kFull, hi1, s);
            }
        }
        if constexpr (VPL == 0) {
            const uint64_t kk = scan_generic(elem, tlo[0], thi[0]);
            if (int(lane) == src[0]) best = kmin(best, kk);
        } else {
            typename E::vec_t x[TPR][VPL];
            constexpr int EPV = E::EPV;
#pragma unroll
            for (int u = 0; u < TPR; ++u) {
                const uint64_t vb = (tlo[u] / k) * (k / EPV);  // first vector of the block
#pragma unroll
                for (int j = 0; j < VPL; ++j) {
                    const uint64_t v = vb + lane + 32 * j;
                    if (src[u] >= 0 && v * EPV + (EPV - 1) >= tlo[u] && v * EPV <= thi[u])
                        x[u][j] = elem.load_vec(v);
                }
            }
#pragma unroll
            for (int u = 0; u < TPR; ++u) {
                if (src[u] < 0) break;  // warp-uniform
                const uint32_t vb = uint32_t((tlo[u] / k) * (k / EPV));
                const uint32_t lo32 = uint32_t(tlo[u]), span = uint32_t(thi[u] - tlo[u]);
                typename E::Acc acc;
#pragma unroll
                for (int j = 0; j < VPL; ++j) {
                    const uint32_t v = vb + lane + 32 * j;
                    // 32-bit: the dispatch keeps arrays within 2^32 - 4096 positions
                    // on this path, so no vector of a block wraps
                    if (v * EPV + (EPV - 1) >= lo32 && v * EPV <= lo32 + span) acc.add(x[u][j], v, lo32, span);
                }
                const uint64_t kb = warp_min_key(acc.key());
                if (int(lane) == src[u]) best = kmin(best, kb);
            }
        }
    }
    if (active) __stcs(reinterpret_cast<unsigned long long*>(answers + i), (unsigned long long)(done ? direct : uint64_t(key_pos(best))));
}

template <class E, class QP, int VPL, int TPR, bool WPQ = false, int NT = kThreads>
__global__ void __launch_bounds__(NT) k_query(E elem, QP qp, uint32_t k_rt, const uint64_t* __restrict__ ST,
                                              uint64_t stride, uint64_t q, uint64_t* __restrict__ answers,
                                              const CtlPublish pub) {
    brmq::pdl_wait();
    query_body<E, QP, VPL, TPR, WPQ, NT>(elem, qp, k_rt, ST, stride, q, answers, pub);
}
// the k = 512 batch instance with its register budget (BRMQ_QUERY_WARPS)
template <class E, class QP, int VPL, int TPR>
__global__ void __launch_bounds__(128, BRMQ_QUERY_WARPS / 4) k_query_budget(E elem, QP qp, uint32_t k_rt,
                                                                            const uint64_t* __restrict__ ST,
                                                                            uint64_t stride, uint64_t q,
                                                                            uint64_t* __restrict__ answers,
                                                                            const CtlPublish pub) {
    brmq::pdl_wait();
    query_body<E, QP, VPL, TPR, false, 128>(elem, qp, k_rt, ST, stride, q, answers, pub);
}

constexpr uint64_t kWarpPerQueryMax = 16384;  // batches up to this size: one warp per query

template <class E, class QP, int VPL, int TPR>
void launch_q(E e, QP qp, uint32_t k, const uint64_t* ST, uint64_t stride, uint64_t q,
              uint64_t* ans, cudaStream_t s, const CtlPublish& pub) {
    if (q <= kWarpPerQueryMax) {
        const unsigned grid = unsigned((q * 32 + kThreads - 1) / kThreads);
        brmq::launch_k(k_query<E, QP, VPL, TPR, true>, dim3(grid), dim3(kThreads), 0, s, e, qp, k, ST, stride, q, ans, pub);
        return;
    }
    // 128-thread CTAs: a CTA holds its SM slot until its slowest warp is done
    // (c3 h = 1: 256 -> 128 threads 1.15 -> 1.04 ms; 64 is slower on c5)
    if constexpr (VPL == 4 && TPR == 1) {
        brmq::launch_k(k_query_budget<E, QP, VPL, TPR>, dim3(unsigned((q + 127) / 128)), dim3(128), 0, s, e, qp, k, ST, stride, q,
                                                                                 ans, pub);
        return;
    }
    brmq::launch_k(k_query<E, QP, VPL, TPR, false, 128>, dim3(unsigned((q + 127) / 128)), dim3(128), 0, s, e, qp, k, ST, stride,
                                                                                  q, ans, pub);
}

template <class QP>
void dispatch_i32(ElemI32 e, QP qp, uint32_t k, const uint64_t* ST, uint64_t stride, uint64_t q,
                  uint64_t* ans, cudaStream_t s, const CtlPublish& pub) {
    // (the vectorised instances do 32-bit position arithmetic inside a block)
    const bool aligned = (reinterpret_cast<uintptr_t>(e.data) & 15u) == 0 && e.len <= 0xFFFFFFFFull - 4096;
    // one pending range per round: fewer registers -> more resident warps, which
    // beats batching ranges per round on this latency-bound kernel (measured)
    if (aligned && k == 512) {
        if ((e.len & 3u) == 0)  // whole vectors: no tail test per load (ElemI32T)
            return launch_q<ElemI32T<true>, QP, 4, 1>(ElemI32T<true>{e.data, e.len, e.scanned}, qp, k, ST, stride,
                                                        q, ans, s, pub);
        return launch_q<ElemI32, QP, 4, 1>(e, qp, k, ST, stride, q, ans, s, pub);
    }
    if (aligned && k == 256) return launch_q<ElemI32, QP, 2, 1>(e, qp, k, ST, stride, q, ans, s, pub);
    if (aligned && k == 1024) return launch_q<ElemI32, QP, 8, 1>(e, qp, k, ST, stride, q, ans, s, pub);
    if (aligned && k == 2048) return launch_q<ElemI32, QP, 16, 1>(e, qp, k, ST, stride, q, ans, s, pub);
    if (aligned && k == 128) return launch_q<ElemI32, QP, 1, 1>(e, qp, k, ST, stride, q, ans, s, pub);
    return launch_q<ElemI32, QP, 0, 0>(e, qp, k, ST, stride, q, ans, s, pub);
}

template <class QP>
void dispatch_key(ElemKey e, QP qp, uint32_t k, const uint64_t* ST, uint64_t stride, uint64_t q,
                  uint64_t* ans, cudaStream_t s, const CtlPublish& pub) {
    // |A_Q| < 2q: the vectorised instances' 32-bit index arithmetic needs 2q + k < 2^32
    if (2 * q + 4096 > 0xFFFFFFFFull) return launch_q<ElemKey, QP, 0, 0>(e, qp, k, ST, stride, q, ans, s, pub);
    if (k == 512) return launch_q<ElemKey, QP, 8, 1>(e, qp, k, ST, stride, q, ans, s, pub);
    if (k == 256) return launch_q<ElemKey, QP, 4, 1>(e, qp, k, ST, stride, q, ans, s, pub);
    if (k == 1024) return launch_q<ElemKey, QP, 16, 1>(e, qp, k, ST, stride, q, ans, s, pub);
    if (k == 128) return launch_q<ElemKey, QP, 2, 2>(e, qp, k, ST, stride, q, ans, s, pub);
    return launch_q<ElemKey, QP, 0, 0>(e, qp, k, ST, stride, q, ans, s, pub);
}

// The harness's "naive" algorithm (naive.hpp:13-21 on the device): one warp per
// query scans A[l..r]; lanes take strided elements, a redux pair keeps the
// leftmost minimum.
__device__ __forceinline__ void naive_one(const int32_t* __restrict__ A, uint64_t n,
                                          const ulonglong2* __restrict__ Q, uint64_t i,
                                          uint64_t* __restrict__ answers, uint32_t* __restrict__ err) {
    const ulonglong2 x = __ldg(Q + i);
    uint64_t l = x.x, r = x.y;
    if (l > r) { const uint64_t t = l; l = r; r = t; }  // types.hpp:18-20
    if (r >= n) {                                        // naive.hpp:14-15
        if (lane_id() == 0) {
            atomicOr(err, 1u);
            answers[i] = ~0ull;
        }
        return;
    }
    uint64_t b = kNoKey;
    for (uint64_t p = l + lane_id(); p <= r; p += 32) b = kmin(b, pack_key(__ldg(A + p), uint32_t(p)));
    b = warp_min_key(b);
    if (lane_id() == 0) answers[i] = key_pos(b);
}

__global__ void __launch_bounds__(kThreads) k_naive(const int32_t* __restrict__ A, uint64_t n,
                                                    const ulonglong2* __restrict__ Q, uint64_t q,
                                                    uint64_t* __restrict__ answers,
                                                    uint32_t* __restrict__ err, const CtlPublish pub) {
    brmq::pdl_wait();
    const uint64_t i = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    if (i < q) naive_one(A, n, Q, i, answers, err);
}

}  // namespace

int launch_naive(const int32_t* A, uint64_t n, const uint64_t* Q, uint64_t q, uint64_t* answers,
                 uint32_t* err, cudaStream_t stream, const CtlPublish& pub) {
    if (q == 0) return 0;
    brmq::launch_k(k_naive, dim3(unsigned((q * 32 + kThreads - 1) / kThreads)), dim3(kThreads), 0, stream, 
        A, n, reinterpret_cast<const ulonglong2*>(Q), q, answers, err, pub);
    return 1;
}

int launch_query_direct(const int32_t* A, uint64_t n, uint32_t k, const uint64_t* ST, uint64_t b,
                        const uint64_t* Q, uint64_t q, uint64_t* answers, uint32_t* err,
                        cudaStream_t stream, const CtlPublish& pub, uint64_t* scanned) {
    if (q == 0) return 0;
    dispatch_i32(ElemI32{A, n, reinterpret_cast<unsigned long long*>(scanned)}, QueryDirect{Q, n, err}, k,
                 ST, b, q, answers, stream, pub);
    return 1;
}

int launch_query_contracted_wi(const uint64_t* AQ, uint32_t k, const uint64_t* ST, uint64_t b_max,
                               const uint64_t* Q, const uint2* word_info, uint64_t n, uint64_t q,
                               uint64_t* answers, cudaStream_t stream, const CtlPublish& pub) {
    if (q == 0) return 0;
    dispatch_key(ElemKey{AQ}, QueryContractedWI{Q, word_info, n}, k, ST, b_max, q, answers, stream,
                 pub);
    return 1;
}

int launch_query_contracted(const uint64_t* AQ, const uint64_t* /*aq_len_dev*/, uint32_t k,
                            const uint64_t* ST, uint64_t b_max, const uint64_t* Q,
                            const uint32_t* cleft, const uint32_t* cright_raw, uint64_t q,
                            uint64_t* answers, cudaStream_t stream, const CtlPublish& pub) {
    if (q == 0) return 0;
    dispatch_key(ElemKey{AQ}, QueryContracted{Q, cleft, cright_raw}, k, ST, b_max, q, answers,
                 stream, pub);
    return 1;
}

}  // namespace brmq

// ---------------------------------------------------------------------------
// Multi-level BbST [k1 = 32, k] (SPEC.md:293-296 answer_one_ml).
// The O(1) part is the same as above; an endpoint block that must be resolved
// descends to its 32-element sub-blocks: full sub-blocks inside the range come
// from their stored keys (one 128-byte line per block for k = 512), and raw A
// is read only for a partial sub-block whose stored minimum lies outside the
// range -- with the same leftmost-exact speculation (<= on the left, < on the
// right) one level down.  Each lane resolves its own query: per lane at most
// two sub-block-key lines and four 128-byte rows, all lanes in parallel, so the
// warp never serialises on other lanes' scans.
namespace brmq {
namespace {

// leftmost-min key of A[lo..hi] inside one 32-aligned row (one 128-byte line)
// Out of line on purpose: one shared copy keeps the kernel inside the
// instruction cache (the inlined variants thrashed it: "no_instructions" stalls).
template <bool VEC>
__device__ __noinline__ uint64_t row_scan(const int32_t* __restrict__ A, uint64_t n, uint64_t lo,
                                             uint64_t hi) {
    const uint64_t r0 = lo & ~uint64_t(31);
    uint64_t best = kNoKey;
    if (VEC && r0 + 32 <= n) {
        const int4* v = reinterpret_cast<const int4*>(A + r0);
        const uint32_t c0 = uint32_t(lo - r0) >> 2, c1 = uint32_t(hi - r0) >> 2;
#pragma unroll
        for (uint32_t c = 0; c < 8; ++c) {
            if (c < c0 || c > c1) continue;
            const int4 x = __ldg(v + c);
            const uint64_t p = r0 + 4 * c;
            if (p + 0 >= lo && p + 0 <= hi) best = kmin(best, pack_key(x.x, uint32_t(p + 0)));
            if (p + 1 >= lo && p + 1 <= hi) best = kmin(best, pack_key(x.y, uint32_t(p + 1)));
            if (p + 2 >= lo && p + 2 <= hi) best = kmin(best, pack_key(x.z, uint32_t(p + 2)));
            if (p + 3 >= lo && p + 3 <= hi) best = kmin(best, pack_key(x.w, uint32_t(p + 3)));
        }
        return best;
    }
    for (uint64_t i = lo; i <= hi; ++i) best = kmin(best, pack_key(__ldg(A + i), uint32_t(i)));
    return best;
}

// Resolve A[lo..hi] (inside one k-block) against the running best, through the
// sub-block keys.  A partial sub-block [a, b] whose stored minimum S lies outside
// it can hold no key below pack(value(S), a), so it is scanned iff that bound is
// below the running best -- the exact form of the leftmost rule, valid whatever
// side of the partial range the current best comes from.
template <bool VEC>
__device__ __noinline__ uint64_t resolve_sub(const int32_t* __restrict__ A, uint64_t n,
                                                const uint64_t* __restrict__ sub, uint64_t lo,
                                                uint64_t hi, uint64_t best) {
    const uint64_t sl = lo >> 5, sr = hi >> 5;
    if (sl == sr) {
        const uint64_t S = __ldg(sub + sl);
        if (key_pos(S) >= lo && key_pos(S) <= hi) return kmin(best, S);
        if ((S & ~0xFFFFFFFFull) + lo >= best) return best;  // bound pack(v(S), lo) not below best
        return kmin(best, row_scan<VEC>(A, n, lo, hi));
    }
    uint64_t inner = kNoKey;
    for (uint64_t s = sl + 1; s < sr; ++s) inner = kmin(inner, __ldg(sub + s));
    best = kmin(best, inner);
    const uint64_t Rk = __ldg(sub + sr), Lk = __ldg(sub + sl);
    bool scan_r = false, scan_l = false;
    if (key_pos(Rk) <= hi) best = kmin(best, Rk);
    else scan_r = true;
    if (key_pos(Lk) >= lo) best = kmin(best, Lk);
    else scan_l = true;
    if (scan_r && (Rk & ~0xFFFFFFFFull) + (sr << 5) < best)
        best = kmin(best, row_scan<VEC>(A, n, sr << 5, hi));
    if (scan_l && (Lk & ~0xFFFFFFFFull) + lo < best)
        best = kmin(best, row_scan<VEC>(A, n, lo, (sl << 5) + 31));
    return best;
}

template <bool VEC>
__device__ __forceinline__ void ml_one(const int32_t* __restrict__ A, uint64_t n, uint32_t k,
                                       const uint64_t* __restrict__ ST, uint64_t stride,
                                       const uint64_t* __restrict__ sub,
                                       const uint64_t* __restrict__ Q, uint64_t i,
                                       uint64_t* __restrict__ answers, uint32_t* __restrict__ err) {
    const ulonglong2 x = __ldg(reinterpret_cast<const ulonglong2*>(Q) + i);
    uint64_t l = x.x, r = x.y;
    if (l > r) { const uint64_t t = l; l = r; r = t; }  // types.hpp:18-20
    if (r >= n) {                                        // naive.hpp:14-15
        atomicOr(err, 1u);
        answers[i] = ~0ull;
        return;
    }
    if (l == r) {
        answers[i] = l;
        return;
    }
    const uint64_t bl = l / k, br = r / k;
    const uint64_t L = __ldg(ST + bl);
    uint64_t best = kNoKey;
    if (bl == br) {
        best = (key_pos(L) >= l && key_pos(L) <= r) ? L : resolve_sub<VEC>(A, n, sub, l, r, kNoKey);
    } else {
        if (br - bl >= 2) {  // inner_span_min
            const uint32_t e = floor_log2_u64(br - bl - 1);
            const uint64_t* row = ST + uint64_t(e) * stride;
            best = kmin(__ldg(row + bl + 1), __ldg(row + br - (1ull << e)));
        }
        const uint64_t R = __ldg(ST + br);
        bool res_r = false, res_l = false;
        if (best == kNoKey || key_hi(R) < key_hi(best)) {
            if (key_pos(R) <= r) best = kmin(best, R);
            else res_r = true;
        }
        if (best == kNoKey || key_hi(L) <= key_hi(best)) {
            if (key_pos(L) >= l) best = kmin(best, L);
            else res_l = true;
        }
        if (res_r) best = resolve_sub<VEC>(A, n, sub, br * k, r, best);
        if (res_l) best = resolve_sub<VEC>(A, n, sub, l, bl * k + k - 1, best);
    }
    answers[i] = key_pos(best);
}

template <bool VEC>
__global__ void __launch_bounds__(kThreads) k_query_ml(const int32_t* __restrict__ A, uint64_t n,
                                                       uint32_t k, const uint64_t* __restrict__ ST,
                                                       uint64_t stride,
                                                       const uint64_t* __restrict__ sub,
                                                       const uint64_t* __restrict__ Q, uint64_t q,
                                                       uint64_t* __restrict__ answers,
                                                       uint32_t* __restrict__ err,
                                                       const CtlPublish pub) {
    brmq::pdl_wait();
    const uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x;
    if (i < q) ml_one<VEC>(A, n, k, ST, stride, sub, Q, i, answers, err);
}

// ---- flat variant: power-of-two k <= 512 (<= 16 sub-blocks per block) --------
// ncu on c3 showed the lane-private resolution above at 4.9 active threads per
// issued instruction: the lanes that must descend (a third of the queries) run
// their variable-length sub-key loops and row scans one after another while
// the rest idle.  Here the descent has a FIXED shape, so a warp issues it once
// for all its lanes:
//   - a side [lo, hi] (inside one k-block) is resolved lane-privately from the
//     block's sub-block keys -- one 128-byte line for k = 512, loaded as 8
//     predicated 16-byte vectors -- plus its two edge keys;
//   - the partial edge rows that survive (their exact bound is below the
//     running best) are pooled per warp and scanned by HALF-warps, one
//     coalesced 8-byte load per lane per row, a batch of rows in flight at once.
// Same speculation and bounds as ml_one / resolve_sub; all shifts, no division.
constexpr int kMlBatch = 4;  // rows per half-warp per batch

// minimum key over the calling lane's half-warp (both halves at once)
__device__ __forceinline__ uint64_t half_min_key(uint64_t k, bool upper) {
    const uint32_t hi = key_hi(k), lo = key_pos(k);
    const uint32_t h0 = __reduce_min_sync(kFull, upper ? 0xFFFFFFFFu : hi);
    const uint32_t h1 = __reduce_min_sync(kFull, upper ? hi : 0xFFFFFFFFu);
    const uint32_t mh = upper ? h1 : h0;
    const uint32_t p0 = __reduce_min_sync(kFull, (!upper && hi == mh) ? lo : 0xFFFFFFFFu);
    const uint32_t p1 = __reduce_min_sync(kFull, (upper && hi == mh) ? lo : 0xFFFFFFFFu);
    return (uint64_t(mh) << 32) | (upper ? p1 : p0);
}

__device__ __forceinline__ uint64_t shfl_u64(uint64_t v, int src) {
    const uint32_t a = __shfl_sync(kFull, uint32_t(v), src);
    const uint32_t b = __shfl_sync(kFull, uint32_t(v >> 32), src);
    return (uint64_t(b) << 32) | a;
}

// One partial edge row: elements [lo..hi] of one 32-aligned row, scanned only
// if pack(v, a) -- v the stored minimum of its sub-block, which lies outside the
// row part, a a lower bound on the positions in the row part -- is below the
// owner's best.
struct RowTask {
    uint32_t lo, hi, v, a;
    bool need;
};

// Row loaders: min key of elements p, p + 1 (p even) that lie in [lo, hi].
template <bool VEC>
struct RowI32 {  // A itself: positions are indices
    const int32_t* A;
    uint64_t n;
    static constexpr bool kDirect = true;
    __device__ __forceinline__ uint64_t pair(uint64_t p, uint32_t lo, uint32_t hi) const {
        int32_t v0, v1;
        if (VEC && p + 1 < n) {
            const int2 v = __ldcs(reinterpret_cast<const int2*>(A + p));
            v0 = v.x;
            v1 = v.y;
        } else {
            v0 = p < n ? __ldg(A + p) : 0;
            v1 = p + 1 < n ? __ldg(A + p + 1) : 0;
        }
        uint64_t k = kNoKey;
        if (p >= lo && p <= hi) k = pack_key(v0, uint32_t(p));
        if (p + 1 >= lo && p + 1 <= hi) k = kmin(k, pack_key(v1, uint32_t(p + 1)));
        return k;
    }
};
struct RowKey {  // A_Q: packed keys carrying original positions (16-byte aligned, even-padded)
    const uint64_t* K;
    static constexpr bool kDirect = false;
    __device__ __forceinline__ uint64_t pair(uint64_t p, uint32_t lo, uint32_t hi) const {
        if (p > hi || p + 1 < lo) return kNoKey;  // never reads past the row part
        const uint4 v = __ldcs(reinterpret_cast<const uint4*>(K + p));
        uint64_t k = p >= lo ? (uint64_t(v.y) << 32) | v.x : kNoKey;
        if (p + 1 <= hi) k = kmin(k, (uint64_t(v.w) << 32) | v.z);
        return k;
    }
};

// Side [lo, hi] of element indices inside one k-block (act: this lane has the
// side) against the block's sub-block keys: the minimum over the covered
// sub-blocks whose key lies inside, and the edge rows left to scan.  The
// "inside" tests are on original positions [plo, phi] (for A_Q exact because
// the origins are non-decreasing: a key at the bound is also the key of an
// index inside, SPEC.md:231 / DESIGN 3.2).  ks = log2(k / 32).
template <bool DIRECT>
__device__ __forceinline__ uint64_t side_flat(const uint64_t* __restrict__ sub, bool act, uint32_t lo,
                                              uint32_t hi, uint32_t plo, uint32_t phi, uint32_t ks,
                                              RowTask& rl, RowTask& rr) {
    const uint32_t sl = lo >> 5, sr = hi >> 5, sb = (sl >> ks) << ks;
    const ulonglong2* sub2 = reinterpret_cast<const ulonglong2*>(sub + sb);
    // interior sub-blocks (sl, sr) as a bit mask over the block's <= 16 offsets:
    // one bit test per key (compile-time bit) instead of two range compares
    const uint32_t dl = sl - sb, dr = sr - sb;
    const uint32_t im = act ? (((1u << dr) - 1u) & ~((2u << dl) - 1u)) : 0u;
    ulonglong2 x[8];
#pragma unroll
    for (uint32_t c = 0; c < 8; ++c)
        x[c] = (im >> (2 * c)) & 3u ? __ldg(sub2 + c) : make_ulonglong2(kNoKey, kNoKey);
    const uint64_t kl = act ? __ldg(sub + sl) : kNoKey, kr = act ? __ldg(sub + sr) : kNoKey;
    uint64_t cand = kNoKey;
#pragma unroll
    for (uint32_t c = 0; c < 8; ++c) {
        if (im & (1u << (2 * c))) cand = kmin(cand, x[c].x);
        if (im & (2u << (2 * c))) cand = kmin(cand, x[c].y);
    }
    rl.need = rr.need = false;
    if (act) {
        if (key_pos(kl) >= plo && key_pos(kl) <= phi) cand = kmin(cand, kl);
        else rl = RowTask{lo, sl == sr ? hi : (sl << 5) + 31, key_hi(kl), DIRECT ? lo : plo, true};
        if (sr != sl) {
            if (key_pos(kr) <= phi) cand = kmin(cand, kr);
            else rr = RowTask{sr << 5, hi, key_hi(kr), DIRECT ? (sr << 5) : plo, true};
        }
    }
    return cand;
}

// One warp answers queries [g * 32, g * 32 + 32) (lane = query).  E: row loader
// of the scanned array (A, or A_Q), QP: query resolution (direct, or the
// contracted coordinates of BbST_CON).
// `pre`: the lane's query already resolved by the caller (before its PDL wait).
template <class E, class QP>
__device__ __forceinline__ void ml_flat_group(const E& elem, const QP& qp, uint32_t kshift,
                                              const uint64_t* __restrict__ ST, uint64_t stride,
                                              const uint64_t* __restrict__ sub, uint64_t q,
                                              uint64_t* __restrict__ answers, uint64_t g,
                                              uint4* s_rows, const Resolved* pre = nullptr) {
    const uint32_t lane = lane_id();
    const bool upper = lane >= 16;
    const uint32_t j = lane & 15u;
    const uint64_t i = g * 32 + lane;
    const uint32_t kmask = (1u << kshift) - 1u;

    // ---- the Sparse Table part (lane-private), as ml_one / answer_one
    uint32_t il = 0, ir = 0, pl = 0, pr = 0;
    bool s0 = false, s1 = false, inblk = false;  // sides: [il, min(ir, end of il's block)], [start of ir's block, ir]
    uint64_t best = kNoKey;
    bool write = false;
    if (i < q) {
        // queries, answers and the rows are streamed (evict-first): the Sparse
        // Table and the sub-block keys stay in L2 (measured: -7% on c3)
        const Resolved rq = pre ? *pre : qp.resolve(i);
        if (rq.done) {
            __stcs(reinterpret_cast<unsigned long long*>(answers + i), (unsigned long long)rq.direct);
        } else {
            write = true;
            il = uint32_t(rq.il);
            ir = uint32_t(rq.ir);
            pl = uint32_t(rq.pl);
            pr = uint32_t(rq.pr);
            const uint32_t bl = il >> kshift, br = ir >> kshift;
            const uint64_t Lk = __ldg(ST + bl);
            if (bl == br) {
                inblk = true;
                if (key_pos(Lk) >= pl && key_pos(Lk) <= pr) best = Lk;
                else s0 = true;
            } else {
                if (br - bl >= 2) {  // inner_span_min
                    const uint32_t e = 31 - __clz(br - bl - 1);
                    const uint64_t* row = ST + uint64_t(e) * stride;
                    best = kmin(__ldg(row + bl + 1), __ldg(row + br - (1u << e)));
                }
                const uint64_t Rk = __ldg(ST + br);
                if (best == kNoKey || key_hi(Rk) < key_hi(best)) {
                    if (key_pos(Rk) <= pr) best = kmin(best, Rk);
                    else s1 = true;
                }
                if (best == kNoKey || key_hi(Lk) <= key_hi(best)) {
                    if (key_pos(Lk) >= pl) best = kmin(best, Lk);
                    else s0 = true;
                }
            }
        }
    }

    // ---- sides (lane-private, one fixed-shape pass per warp)
    RowTask ra, rb;
    if (__any_sync(kFull, s0 || s1)) {
        RowTask r0l, r0r, r1l, r1r;
        const uint64_t c0 = side_flat<E::kDirect>(sub, s0, il, min(ir, il | kmask), pl,
                                                  inblk ? pr : 0xFFFFFFFFu, kshift - 5, r0l, r0r);
        const uint64_t c1 = side_flat<E::kDirect>(sub, s1, ir & ~kmask, ir, 0u, pr, kshift - 5, r1l, r1r);
        best = kmin(best, kmin(c0, c1));
        // side 1 starts on a sub-block boundary: one row at most (its left row when
        // it ends in its first sub-block, else its right row); side 0 has a right
        // row only inside one block, where there is no side 1: <= 2 rows per lane
        ra = r0l;
        rb = r0r.need ? r0r : r1l.need ? r1l : r1r;
    } else {
        ra.need = rb.need = false;
    }

    // ---- rows: pooled per warp, half-warp scans
    ra.need = ra.need && ((uint64_t(ra.v) << 32 | ra.a) < best);
    rb.need = rb.need && ((uint64_t(rb.v) << 32 | rb.a) < best);
    const unsigned ma = __ballot_sync(kFull, ra.need), mb = __ballot_sync(kFull, rb.need);
    if (ma | mb) {
        // entry: lo, (hi - lo) | owner << 8, (the bound needs no re-check: best only falls)
        const unsigned below = (1u << lane) - 1u;
        if (ra.need) s_rows[__popc(ma & below)] = make_uint4(ra.lo, (ra.hi - ra.lo) | (lane << 8), 0, 0);
        if (rb.need)
            s_rows[__popc(ma) + __popc(mb & below)] = make_uint4(rb.lo, (rb.hi - rb.lo) | (lane << 8), 0, 0);
        __syncwarp();
        const uint32_t nrows = __popc(ma) + __popc(mb);
        for (uint32_t e0 = 0; e0 < nrows; e0 += 2 * kMlBatch) {
            uint64_t key[kMlBatch];
            uint32_t own[kMlBatch];
#pragma unroll
            for (int u = 0; u < kMlBatch; ++u) {
                const uint32_t e = e0 + 2 * u + (upper ? 1u : 0u);
                const uint4 t = e < nrows ? s_rows[e] : make_uint4(0, 0, 0, 0);
                own[u] = t.y >> 8;
                key[u] = e < nrows ? elem.pair((uint64_t(t.x) & ~31ull) + 2 * j, t.x, t.x + (t.y & 31u))
                                   : kNoKey;
            }
#pragma unroll
            for (int u = 0; u < kMlBatch; ++u) {
                if (e0 + 2 * u >= nrows) break;  // warp-uniform
                const uint64_t cand = half_min_key(key[u], upper);
                const uint64_t c0 = shfl_u64(cand, 0), c1 = shfl_u64(cand, 16);
                const uint32_t o0 = __shfl_sync(kFull, own[u], 0), o1 = __shfl_sync(kFull, own[u], 16);
                if (lane == o0) best = kmin(best, c0);
                if (e0 + 2 * u + 1 < nrows && lane == o1) best = kmin(best, c1);
            }
        }
    }
    if (write) __stcs(reinterpret_cast<unsigned long long*>(answers + i), (unsigned long long)key_pos(best));
    __syncwarp();  // the row pool is reused by the warp's next group
}

template <class E, class QP, int NT>
__global__ void __launch_bounds__(NT, (NT == 128 ? BRMQ_FLAT_WARPS / 4 : 32)) k_query_flat(const E elem, const QP qp, uint32_t kshift,
                                                   const uint64_t* __restrict__ ST, uint64_t stride,
                                                   const uint64_t* __restrict__ sub, uint64_t q,
                                                   uint64_t* __restrict__ answers,
                                                   const CtlPublish pub) {
    constexpr int kRowCap = 64;  // <= 2 rows per lane
    __shared__ uint4 s_rows[NT / 32][kRowCap];
    const uint32_t warp = threadIdx.x >> 5;
    const uint64_t g = uint64_t(blockIdx.x) * (NT / 32) + warp;
    if constexpr (std::is_same<QP, QueryContractedWI>::value && NT == 32) {
        // BbST_CON (bitmap pipeline) small batches (one wave of 1-warp CTAs), a PDL secondary of the Sparse Table build:
        // the query and its contracted coordinates (the contraction's word info,
        // complete before the table build began) are read before the wait, while
        // the table's upper rows are still being written
        const uint64_t i = g * 32 + lane_id();
        Resolved rq{};
        if (i < q) rq = qp.resolve(i);
        brmq::pdl_wait();
        publish_early(pub);
        if (g < (q + 31) / 32) ml_flat_group(elem, qp, kshift, ST, stride, sub, q, answers, g, s_rows[warp], &rq);
    } else {
        brmq::pdl_wait();
        // BbST_CON only.  Compiled out of the BbST (QueryDirect) instances: there it
        // cost 8-16 bytes of spills per thread (c3 [32, 512] query 0.419 -> 0.413 ms).
        // (As a non-inlined call here: fewer spills, but the c3-con query 0.475 -> 0.491.)
        if constexpr (!std::is_same<QP, QueryDirect>::value) publish_early(pub);
        if (g < (q + 31) / 32) ml_flat_group(elem, qp, kshift, ST, stride, sub, q, answers, g, s_rows[warp]);
    }
}

// 128-thread CTAs for large batches: a CTA holds its slot until its slowest
// warp is done (measured vs 32 / 64 / 256: best over c3, c4 and c5)
constexpr int kFlatThreads = 128;

template <class E, class QP>
void launch_flat(const E& e, const QP& qp, uint32_t k, const uint64_t* ST, uint64_t stride,
                 const uint64_t* sub, uint64_t q, uint64_t* answers, cudaStream_t s,
                 const CtlPublish& pub) {
    // a batch whose warps all fit one wave of 1-warp CTAs (148 SMs x 32 CTAs) runs
    // with single-warp CTAs: no warp waits for a slower sibling (c2: -2.5 us)
    if (q <= uint64_t(148) * 32 * 32) {
        brmq::launch_k(k_query_flat<E, QP, 32>, dim3(unsigned((q + 31) / 32)), dim3(32), 0, s, e, qp, floor_log2_u64(k), ST,
                                                                       stride, sub, q, answers, pub);
        return;
    }
    const unsigned g = unsigned((q + kFlatThreads - 1) / kFlatThreads);
    brmq::launch_k(k_query_flat<E, QP, kFlatThreads>, dim3(g), dim3(kFlatThreads), 0, s, e, qp, floor_log2_u64(k), ST, stride,
                                                                  sub, q, answers, pub);
}

}  // namespace

int launch_query_ml(const int32_t* A, uint64_t n, uint32_t k, const uint64_t* ST, uint64_t b,
                    const uint64_t* sub, const uint64_t* Q, uint64_t q, uint64_t* answers,
                    uint32_t* err, cudaStream_t stream, const CtlPublish& pub) {
    if (q == 0) return 0;
    const unsigned grid = unsigned((q + kThreads - 1) / kThreads);
    if (k >= 64 && k <= 512 && (k & (k - 1)) == 0) {  // <= 16 sub-blocks per block
        if ((reinterpret_cast<uintptr_t>(A) & 7u) == 0)
            launch_flat(RowI32<true>{A, n}, QueryDirect{Q, n, err}, k, ST, b, sub, q, answers, stream, pub);
        else
            launch_flat(RowI32<false>{A, n}, QueryDirect{Q, n, err}, k, ST, b, sub, q, answers, stream, pub);
        return 1;
    }
    if ((reinterpret_cast<uintptr_t>(A) & 15u) == 0)
        brmq::launch_k(k_query_ml<true>, dim3(grid), dim3(kThreads), 0, stream, A, n, k, ST, b, sub, Q, q, answers, err, pub);
    else
        brmq::launch_k(k_query_ml<false>, dim3(grid), dim3(kThreads), 0, stream, A, n, k, ST, b, sub, Q, q, answers, err, pub);
    return 1;
}

// BbST_CON with a sub-block level over A_Q (power-of-two k in [64, 512]): the
// same flat answering as the multi-level BbST, over packed keys, from the
// contracted coordinates.  wi != nullptr: bitmap pipeline (coordinates from the
// per-word ranks), else cleft / cright_raw (radix pipeline).
int launch_query_con_flat(const uint64_t* AQ, uint32_t k, const uint64_t* ST, uint64_t b_max,
                          const uint64_t* sub, const uint64_t* Q, const uint2* word_info,
                          const uint32_t* cleft, const uint32_t* cright_raw, uint64_t n, uint64_t q,
                          uint64_t* answers, cudaStream_t stream, const CtlPublish& pub) {
    if (q == 0) return 0;
    if (word_info)
        launch_flat(RowKey{AQ}, QueryContractedWI{Q, word_info, n}, k, ST, b_max, sub, q, answers,
                    stream, pub);
    else
        launch_flat(RowKey{AQ}, QueryContracted{Q, cleft, cright_raw}, k, ST, b_max, sub, q, answers,
                    stream, pub);
    return 1;
}

}  // namespace brmq
