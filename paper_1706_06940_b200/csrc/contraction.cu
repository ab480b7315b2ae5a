// contraction.cu -- BbST_CON stage 2 on the device: contract A into A_Q.
//
// Replaces build_contracted / scan_areas (contraction.cpp:81-151): for the
// sorted, deduplicated endpoint positions b_0 < ... < b_{m-1}, area t is
// A[b_t .. b_{t+1}] INCLUSIVE of both ends (contraction.hpp:25-27) and A_Q[t]
// is its leftmost minimum.  Here A_Q[t] is one packed key (value, position),
// i.e. aq_values and aq_origin in a single 8-byte word.  Area t is closed with
// the boundary element A[b_{t+1}] that also opens area t+1, so every element
// of A is read exactly once (the reference reads the shared element once too,
// contraction.cpp:97-105).
//
// B200 design: ONE persistent, cooperatively launched kernel (all CTAs are
// co-resident, so its cross-CTA waits cannot deadlock).  The 4096-position
// tiles of A are partitioned into G fixed ranges of R tiles
// (contract_partition); CTA g works on range g clipped to the span
// [b_0, b_{m-1}], and splits it again into one contiguous piece per WARP.
// Every warp is an independent stream -- no block barrier in the loop:
//   - a warp tile is 1024 positions = 32 rows of 32; its data arrive with 8
//     coalesced 16-byte non-allocating loads per lane, issued one tile ahead
//     into registers, and are stored transposed into the warp's 4 KB of
//     shared memory so that lane r owns row r (chunk c of row r at
//     c ^ (r & 7): bank-conflict free on both sides).  Measured on this part
//     (tools/stream_bench.cu), register-destined loads stream at 5.6-5.9 TB/s
//     where TMA / bulk / cp.async rings into shared memory reach 4.7-5.1;
//   - lane r owns row r (32 positions = one bitmap word, prefetched with the
//     data) and reads it with 8 16-byte shared loads;
//   - a warp tile without boundaries costs a value-only row minimum, one
//     redux.min and a one-load leftmost search; rows holding boundaries are
//     closed cooperatively by the warp (sparse) or each by its lane (dense);
//   - the open segment and the running rank are carried in registers.
// Rank bases: per range, the boundary counts k_piece_count popcounted from the
// bitmap (bitmap pipeline) or the exclusive prefix k_unique wrote (sorted
// endpoints); per warp, the piece counts of k_piece_count or, with the prefix,
// a popcount of the warp's own piece while its first loads are in flight.
// Stitch: every warp publishes (tail of its piece, has-boundary); the area
// closed by a warp's first boundary folds the tails of the pieces before it
// back to the nearest piece holding a boundary -- in the CTA through shared
// memory, across CTAs through epoch-tagged descriptors (warp windows of 32).
// The kernel clears the bitmap words it consumed (the bitmap is never
// memset) and, for the bitmap pipeline, emits (rank prefix, bits) of every
// non-empty word for the query remap.
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "scan.cuh"

namespace brmq {
namespace {

constexpr int NW = int(kContractWarps);  // warps per CTA, one stream each (2 CTAs per SM at 128 registers)
static_assert(NW == int(kContractWarps), "piece layout shared with the endpoint stage");
constexpr int NT = NW * 32;
constexpr int kRow = 32;            // positions per lane = one 128-byte row
constexpr int kWTile = 32 * kRow;   // 1024 positions = 4 KB per warp tile
constexpr int kTile = 4 * kWTile;   // 4096: the partition unit
static_assert(kTile == (1 << kContractTileLog2), "partition tile size");
#ifndef BRMQ_CHUNKED_DENSE
#define BRMQ_CHUNKED_DENSE 1  // dense rows skip boundary-free chunk columns (instance with the sparse path)
#endif
#ifndef BRMQ_KDENSE
#define BRMQ_KDENSE 2
#endif
#ifndef BRMQ_CONTRACT_MINB
#define BRMQ_CONTRACT_MINB 2  // 2 CTAs per SM: <= 128 registers (129 would halve the residency)
#endif
constexpr int kDense = BRMQ_KDENSE;  // flagged rows per warp tile above which rows close per lane
#ifdef BRMQ_CONTRACT_STAMPS
// A/B diagnostics: per warp (start, loop end, stitch end) %globaltimer stamps of the
// last contraction launch (tools/contract_tail.py)
__device__ unsigned long long g_cstamp[kMaxContractRanges * 8][3];
__device__ unsigned long long g_cstamp2[kMaxContractRanges * 8][3];  // (entry, rank bases known, wait released)
__device__ __forceinline__ unsigned long long cgt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}
#endif
constexpr int kDenseEndpoints = 8;  // endpoints per warp tile from which only dense rows are compiled in

// Rows of the current warp tile in the warp's swizzled shared rows (16-byte
// chunk c of row r at byte r*128 + ((c ^ (r & 7)) << 4)), read with explicit
// shared loads.
struct Rows {
    uint32_t stage;    // shared address of the warp's rows
    uint32_t tile_lo;  // (positions fit 32 bits; those past n are masked)
    __device__ __forceinline__ int4 chunk(uint32_t r, int c) const {
        return lds128(stage + r * 128u + ((uint32_t(c) ^ (r & 7u)) << 4));
    }
    __device__ __forceinline__ int32_t elem(uint32_t r, int j) const {
        return lds32(stage + elem_offset(r, j));
    }
    __device__ __forceinline__ uint32_t pos(uint32_t r, int j) const {
        return tile_lo + r * uint32_t(kRow) + uint32_t(j);
    }
    static __device__ __forceinline__ uint32_t elem_offset(uint32_t r, int j) {
        return r * 128u + (((uint32_t(j) >> 2) ^ (r & 7u)) << 4) + ((j & 3) << 2);
    }
};

// A_Q slot of area `idx` (closed by the boundary of rank idx + 1).  BbST_CON:
// slot idx.  ST-RMQ_CON's marked contraction (SPEC.md "baseline"): entry 2t+1
// is the marked position b_t itself and entry 2t the unmarked run between
// b_{t-1} and b_t, so area idx (the run before b_{idx+1}) goes to 2 idx + 2.
template <bool MARKED>
__device__ __forceinline__ uint64_t aq_slot(uint64_t idx) {
    return MARKED ? 2 * idx + 2 : idx;
}

// Where a closed area goes.  FUSE (BbST_CON with a small A_Q): besides the
// store, its key is folded into the 32-key run minima (`sub`) and the k-block
// minima (row 0 of the block Sparse Table) with fire-and-forget reductions, so
// no block-argmin pass over A_Q follows (measured at c2: +4 us in the
// contraction for -7.5 us of block-argmin launch; a last-CTA build of the
// table's upper rows inside the contraction cost +8 us, rejected).
struct AqOut {
    uint64_t* aq;
    uint64_t* sub;
    uint64_t* blk;
    uint32_t kshift;
};
__device__ __forceinline__ void red_min_u64(uint64_t* p, uint64_t v) {
    asm volatile("red.relaxed.gpu.global.min.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
template <bool MARKED, bool FUSE>
__device__ __forceinline__ void put_area(const AqOut& o, uint64_t idx, uint64_t key) {
    o.aq[aq_slot<MARKED>(idx)] = key;
    if constexpr (FUSE && !MARKED) {
        red_min_u64(o.sub + (idx >> 5), key);
        red_min_u64(o.blk + (idx >> o.kshift), key);
    }
}

__device__ __forceinline__ int32_t comp(const int4& x, int e) {
    return e == 0 ? x.x : e == 1 ? x.y : e == 2 ? x.z : x.w;
}

// Leftmost minimum of row r over [lo, hi] (lo <= hi) as a packed key.  int32
// compares with a 5-bit local index (strict '<' over ascending positions keeps
// the leftmost); the 64-bit key is formed once.
template <bool FULL, class RW>
__device__ __forceinline__ uint64_t row_min(const RW& rw, uint32_t r, int lo, int hi) {
    if (FULL || (lo == 0 && hi == kRow - 1)) {
        // min per 16-byte chunk (3-way mins), leftmost winning chunk by strict '<',
        // then the leftmost element of that chunk equal to the minimum
        int4 x = rw.chunk(r, 0);
        int32_t bv = __vimin3_s32(x.x, x.y, min(x.z, x.w));
        int bc = 0;
#pragma unroll
        for (int c = 1; c < 8; ++c) {
            x = rw.chunk(r, c);
            const int32_t m = __vimin3_s32(x.x, x.y, min(x.z, x.w));
            if (m < bv) { bv = m; bc = c; }
        }
        x = rw.chunk(r, bc);
        const int e = x.x == bv ? 0 : x.y == bv ? 1 : x.z == bv ? 2 : 3;
        return pack_key(bv, uint32_t(rw.pos(r, 4 * bc + e)));
    }
    int32_t bv = 0x7FFFFFFF;
    int bi = -1;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        if (4 * c + 3 < lo || 4 * c > hi) continue;
        const int4 x = rw.chunk(r, c);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int j = 4 * c + e;
            const int32_t v = comp(x, e);
            if (j >= lo && j <= hi && (v < bv || bi < 0)) { bv = v; bi = j; }
        }
    }
    return pack_key(bv, uint32_t(rw.pos(r, bi)));
}

// Dense rows, one pass: the areas between consecutive boundaries of row r in
// [lo, hi] are stored (the first boundary has global rank `rank`, so the second
// closes area `rank`, ...); hp = min over [lo, first boundary] (the part of the
// area the row's first boundary closes, completed after the warp scan), run =
// min over [last boundary, hi] (the open segment the row hands on).
template <bool MARKED, bool FUSE, class RW>
__device__ __forceinline__ void row_pass(const RW& rw, uint32_t r, uint32_t fl, int lo, int hi,
                                         uint64_t rank, const AqOut& aq, uint64_t& hp,
                                         uint64_t& run) {
    int32_t rv = 0x7FFFFFFF;
    int ri = -1;
    bool seen = false;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        if (4 * c + 3 < lo || 4 * c > hi) continue;
        const int4 x = rw.chunk(r, c);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int j = 4 * c + e;
            if (j < lo || j > hi) continue;
            const int32_t v = comp(x, e);
            if ((fl >> j) & 1u) {
                uint64_t k = pack_key(v, uint32_t(rw.pos(r, j)));  // inclusive right end
                if (ri >= 0) k = kmin(k, pack_key(rv, uint32_t(rw.pos(r, ri))));
                if (seen) {
                    put_area<MARKED, FUSE>(aq, rank, k);
                    ++rank;
                } else {
                    hp = k;
                    seen = true;
                }
                rv = v;  // the boundary element opens the next area
                ri = j;
            } else if (v < rv || ri < 0) {
                rv = v;
                ri = j;
            }
        }
    }
    run = ri >= 0 ? pack_key(rv, uint32_t(rw.pos(r, ri))) : kNoKey;
}

// row_pass for an interior row (all 32 positions in the span), run by EVERY lane
// of a dense tile: a row without boundaries comes out with its minimum in
// `run`, so the unflagged lanes do their row minimum in the same instruction
// stream instead of a separate, serialised row_min pass; element 0 is peeled
// (the run is never empty after it).
template <bool MARKED, bool FUSE, class RW>
__device__ __forceinline__ void row_pass_all(const RW& rw, uint32_t r, uint32_t fl, uint64_t rank,
                                             const AqOut& aq, uint64_t& hp,
                                             uint64_t& run) {
    const uint32_t p0 = uint32_t(rw.pos(r, 0));
    int4 x = rw.chunk(r, 0);
    int32_t rv = x.x;
    uint32_t ri = 0;
    bool seen = fl & 1u;
    if (seen) hp = pack_key(rv, p0);
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        if (c) x = rw.chunk(r, c);
#pragma unroll
        for (int e = (c == 0 ? 1 : 0); e < 4; ++e) {
            const int j = 4 * c + e;
            const int32_t v = comp(x, e);
            if ((fl >> j) & 1u) {
                const uint64_t k = v < rv ? pack_key(v, p0 + j) : pack_key(rv, p0 + ri);
                if (seen) {
                    put_area<MARKED, FUSE>(aq, rank, k);
                    ++rank;
                } else {
                    hp = k;
                    seen = true;
                }
                rv = v;  // the boundary element opens the next area
                ri = j;
            } else if (v < rv) {
                rv = v;
                ri = j;
            }
        }
    }
    run = pack_key(rv, p0 + ri);
}

// row_pass_all without branches per element: the closing key of a boundary at
// j is m = leftmost-min(run state, (v_j, j)) -- the update a non-boundary
// element makes anyway -- so every element costs min / compare / select, and a
// boundary additionally captures m into the lane's shared-memory slots
// (predicated store, no branch) and restarts the run at (v_j, j).  The captures
// are emitted afterwards: capture 0 is the row's head part, capture i >= 1 closes
// area rank + i - 1.  Needs popc(fl) <= kCap (the caller checks; row_pass_all
// otherwise).  c5-con: the branchy per-element walk was ~15 instructions per
// element (BSSY/BRA/BSYNC around every compare), this one 8.
constexpr int kCap = 16;  // capture slots per lane
constexpr size_t kCapSmem = size_t(NW) * kCap * 32 * 8;  // dynamic shared memory of k_contract
// CHUNKED (the instance with the sparse path, few boundaries per dense tile): a
// 16-byte chunk in which no lane of the warp has a boundary is folded with one
// 3-way minimum and a leftmost-index select (~10 instructions instead of ~36);
// the per-element walk runs only for chunk columns where some lane has one
// (warp-uniform test, no divergence).
template <bool MARKED, bool FUSE, class RW, bool CHUNKED = false>
__device__ __forceinline__ void row_pass_cap(const RW& rw, uint32_t r, uint32_t fl, uint64_t rank,
                                             const AqOut& aq, uint64_t& hp, uint64_t& run,
                                             uint32_t cap /* shared address of slot 0 of this lane */) {
    const uint32_t p0 = uint32_t(rw.pos(r, 0));
    int32_t rv = 0x7FFFFFFF;
    uint32_t ri = 0;
    uint32_t at = cap;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int4 x = rw.chunk(r, c);
        if (CHUNKED && !__any_sync(kFull, ((fl >> (4 * c)) & 0xFu) != 0u)) {
            const int32_t m = __vimin3_s32(x.x, x.y, min(x.z, x.w));
            const uint32_t e = x.x == m ? 0u : x.y == m ? 1u : x.z == m ? 2u : 3u;
            if (m < rv) {  // strict: the earlier position keeps ties
                rv = m;
                ri = uint32_t(4 * c) + e;
            }
            continue;
        }
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const uint32_t j = uint32_t(4 * c + e);
            const int32_t v = comp(x, e);
            const bool lt = v < rv;  // strict: the earlier position keeps ties
            const int32_t mv = lt ? v : rv;
            const uint32_t mi = lt ? j : ri;
            const bool isb = (fl >> j) & 1u;
            if (isb) {  // predicated (no divergent branch): capture, advance, restart
                asm volatile("st.shared.v2.u32 [%0], {%1, %2};" ::"r"(at), "r"(uint32_t(mv)), "r"(mi) : "memory");
                at += 32u * 8u;
            }
            rv = isb ? v : mv;
            ri = isb ? j : mi;
        }
    }
    run = pack_key(rv, p0 + ri);
    const uint32_t nb = __popc(fl);
    for (uint32_t i = 0; i < nb; ++i) {
        uint32_t cv, ci;
        asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(cv), "=r"(ci) : "r"(cap + i * 32u * 8u) : "memory");
        const uint64_t k = pack_key(int32_t(cv), p0 + ci);
        if (i == 0) hp = k;
        else put_area<MARKED, FUSE>(aq, rank + i - 1, k);
    }
}

// Warp `warp`'s piece of CTA `cta`'s range: warp tiles [wa, wa + cnt) of range
// cta (R tiles), clipped to the span [b0, blast]; cnt = 0 when empty.  Shared by
// the contraction and the piece-count kernel, so both cut identically.
struct Piece {
    uint64_t wa, cnt;
};
__device__ __forceinline__ Piece piece_of(uint64_t cta, uint32_t warp, uint64_t R, uint32_t b0,
                                          uint32_t blast) {
    const uint64_t tfirst = b0 / kTile, tlast = blast / kTile, ra = cta * R;
    const uint64_t ta = ra > tfirst ? ra : tfirst;
    const uint64_t tb = ra + R - 1 < tlast ? ra + R - 1 : tlast;
    if (ta > tb) return Piece{0, 0};
    const uint64_t w0 = ta * 4 > b0 / kWTile ? ta * 4 : b0 / kWTile;
    const uint64_t w1 = tb * 4 + 3 < blast / kWTile ? tb * 4 + 3 : blast / kWTile;
    const uint64_t per = (w1 - w0 + NW) / NW;
    const uint64_t wa = w0 + warp * per;
    const uint64_t wb = wa + per - 1 < w1 ? wa + per - 1 : w1;
    return Piece{wa, wa <= wb ? wb - wa + 1 : 0};
}

// Boundaries per piece (pcnt[g * NW + w]) and per range (rcnt[g]), popcounted
// from the finished bitmap (L2-resident): one CTA per range, one warp per piece.
__global__ void __launch_bounds__(NT) k_piece_count(const uint32_t* __restrict__ bitmap,
                                                    const uint32_t* __restrict__ span, uint64_t R,
                                                    uint32_t* __restrict__ pcnt,
                                                    uint32_t* __restrict__ rcnt) {
    brmq::pdl_wait();
    brmq::pdl_trigger();  // small grid: dependents may be scheduled now
    __shared__ uint32_t s_c[NW];
    const uint32_t b0 = ~span[0], blast = span[1];
    const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
    uint32_t k = 0;
    if (b0 <= blast) {
        const Piece pc = piece_of(blockIdx.x, warp, R, b0, blast);
        const uint4* w4 = reinterpret_cast<const uint4*>(bitmap + pc.wa * 32);
        const uint64_t nv = pc.cnt * 8;
        // kPcU independent loads in flight per lane: a c2 piece (41.5 warp tiles =
        // 332 vectors) in one round trip instead of two
        constexpr int kPcU = 16;
        for (uint64_t j0 = lane; j0 < nv; j0 += 32 * kPcU) {
            uint4 w[kPcU];
#pragma unroll
            for (int u = 0; u < kPcU; ++u)
                w[u] = j0 + 32 * u < nv ? __ldg(w4 + j0 + 32 * u) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < kPcU; ++u) k += __popc(w[u].x) + __popc(w[u].y) + __popc(w[u].z) + __popc(w[u].w);
        }
    }
    k = __reduce_add_sync(kFull, k);
    if (lane == 0) {
        pcnt[uint64_t(blockIdx.x) * NW + warp] = k;
        s_c[warp] = k;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) t += s_c[w];
        rcnt[blockIdx.x] = t;
    }
}

struct ContractArgs {
    const int32_t* A;
    uint64_t n;
    uint32_t* bitmap;
    const uint32_t* span;
    uint64_t* aq;
    uint64_t* nb_out;
    uint64_t* aq_len;
    uint2* word_info;
    const uint32_t* rcnt;  // [G] boundaries per range, or (prefix) [G+1] exclusive prefix
    uint64_t range_tiles;  // R
    uint32_t prefix;
    uint64_t* st_part;   // [G * NW] epoch-tagged descriptors, one per piece
    uint64_t* key_tail;  // [G * NW]
    const uint32_t* pcnt;  // nullable: [G * NW] boundaries per piece (k_piece_count)
    const uint32_t* epoch_dev;  // device epoch counter (bumped once per solve)
    uint32_t epoch_off;
    // FUSE instances: 32-key run minima and row 0 of the k-block Sparse Table
    // over A_Q (filled by reductions), its row stride, log2(k), and b_dev =
    // ceil(|A_Q| / k)
    uint64_t* fuse_sub;
    uint64_t* fuse_st;
    uint64_t fuse_stride;
    uint32_t fuse_kshift;
    uint64_t* b_dev;
    // nullable: += the positions of A this kernel consumed (ContractionStats,
    // contraction.hpp:47-49), one reduction per warp
    uint64_t* reads;
};

// MARKED: ST-RMQ_CON's marked contraction -- marked positions read as +inf
// inside the areas (they get their own entries) and areas go to aq_slot.
// SPARSE = false: every warp tile holding a boundary takes the dense one-pass
// rows (the instance for high boundary densities: without the sparse path
// compiled in, c5-con's contraction runs 5% faster).
template <bool VEC, bool MARKED, bool SPARSE, bool FUSE>
__device__ __forceinline__ void contract_body(const ContractArgs& c) {
    const AqOut out{c.aq, c.fuse_sub, c.fuse_st, c.fuse_kshift};
    __shared__ __align__(128) int4 s_rows[NW][kWTile / 4];  // per warp: 32 rows x 128 B, swizzled
    extern __shared__ __align__(16) uint2 s_cap[];  // [NW][kCap][32] boundary captures (dense rows)
    __shared__ uint32_t s_cnt[NW];
    __shared__ unsigned long long s_base;
    __shared__ uint32_t s_red[NW];

#ifdef BRMQ_CONTRACT_STAMPS
    if ((threadIdx.x & 31u) == 0) g_cstamp2[uint64_t(blockIdx.x) * NW + (threadIdx.x >> 5)][0] = cgt();
#endif
    const uint32_t b0 = ~c.span[0], blast = c.span[1];
    if (b0 > blast) return;
    const uint32_t epoch = *c.epoch_dev + c.epoch_off;
    const uint64_t tfirst = b0 / kTile, tlast = blast / kTile;
    // fixed partition of ALL tiles of A into ranges of R tiles (contract_partition);
    // a CTA works on its range clipped to the span [b0, blast]
    const uint64_t cta = blockIdx.x, R = c.range_tiles;
    const uint64_t ra = cta * R;
    const uint64_t ta = ra > tfirst ? ra : tfirst;
    const uint64_t tb = ra + R - 1 < tlast ? ra + R - 1 : tlast;
    if (ta > tb) return;  // nothing of the span: never waited on by a CTA that has work
    const uint64_t cfirst = tfirst / R;  // the CTA holding b0
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;

    // this warp's piece: warp tiles [wa, wa + cnt) of the range, clipped to the span
    const Piece pc = piece_of(cta, warp, R, b0, blast);
    const uint64_t wa = pc.wa, cnt = pc.cnt;

    // Warp tile i (1024 positions): 8 coalesced 16-byte loads per lane into
    // registers one tile ahead, stored transposed into the warp's rows so that
    // lane r reads row r (128 B; chunk c at c ^ (r & 7): conflict-free both ways).
    int4 y[8];
    uint32_t fy = 0;  // bitmap word of the lane's row, one tile ahead
    // per-tile index arithmetic in 32 bits (warp tiles < 2^22): the loop's 64-bit
    // tile / interior / tail tests were ~8% of the kernel's instructions at c2
    const uint32_t wa32 = uint32_t(wa), cnt32 = uint32_t(cnt);
    const uint32_t full_tiles = uint32_t(c.n / kWTile);  // warp tiles entirely inside A
    const int4* A4base = reinterpret_cast<const int4*>(c.A) + lane;
    const uint32_t* Bbase = c.bitmap + lane;
    auto fetch = [&](uint32_t i) {
        const uint32_t t = wa32 + i;
        if (VEC && t < full_tiles) {
            const int4* A4 = A4base + size_t(t) * (kWTile / 4);
#pragma unroll
            for (int u = 0; u < 8; ++u) y[u] = ld_stream_v4(A4 + u * 32);

        } else {
            const uint64_t tile_lo = uint64_t(t) * kWTile;  // array tail / unaligned A: scalar loads, positions >= n read as 0 (masked later)
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint64_t p = tile_lo + 128u * u + 4u * lane;
                y[u].x = p + 0 < c.n ? __ldg(c.A + p + 0) : 0;
                y[u].y = p + 1 < c.n ? __ldg(c.A + p + 1) : 0;
                y[u].z = p + 2 < c.n ? __ldg(c.A + p + 2) : 0;
                y[u].w = p + 3 < c.n ? __ldg(c.A + p + 3) : 0;
            }
        }
        fy = Bbase[size_t(t) * 32];
    };
    auto stage = [&]() {
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t row = 4u * u + (lane >> 3), ch = lane & 7u;
            s_rows[warp][row * 8u + (ch ^ (row & 7u))] = y[u];
        }
        __syncwarp();
        if (MARKED && fy) {  // marked positions of the lane's row read as +inf
            const uint32_t base = smem_u32(s_rows[warp]);
            for (uint32_t m = fy; m; m &= m - 1) {
                const uint32_t off = Rows::elem_offset(lane, __ffs(m) - 1);
                asm volatile("st.shared.u32 [%0], %1;" ::"r"(base + off), "r"(0x7FFFFFFF) : "memory");
            }
        }
        if (MARKED) __syncwarp();
    };
    if (cnt32) fetch(0);
    // A PDL secondary of the piece count (BbST_CON) waits here: the span, the epoch
    // and the bitmap come from the endpoint kernel before it (complete when this
    // grid was scheduled), so the first tile of A is already in flight; the
    // per-piece / per-range counts below are the predecessor's (a no-op otherwise)
    brmq::pdl_wait();
    // dependents may be scheduled now -- after the wait, so that everything before
    // this grid is complete when they start (DESIGN 3.5: "two launches back")
    brmq::pdl_trigger();
#ifdef BRMQ_CONTRACT_STAMPS
    if (lane == 0) g_cstamp2[cta * NW + warp][2] = cgt();
#endif

    // ---- rank bases: the CTA's from the endpoint stage's per-range counts, the
    // warp's from a popcount of its piece of the bitmap (loads overlap the ring)
    {
        const uint4* w4 = reinterpret_cast<const uint4*>(c.bitmap + wa * 32);
        const uint64_t nvec = c.pcnt ? 0 : cnt * 8;  // counted already by k_piece_count
        uint32_t k = c.pcnt ? __ldg(c.pcnt + cta * NW + warp) : 0u;
        for (uint64_t j0 = lane; j0 < nvec; j0 += 32 * 8) {
            uint4 w[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                w[u] = j0 + u * 32 < nvec ? __ldg(w4 + j0 + u * 32) : make_uint4(0, 0, 0, 0);
#pragma unroll
            for (int u = 0; u < 8; ++u) k += __popc(w[u].x) + __popc(w[u].y) + __popc(w[u].z) + __popc(w[u].w);
        }
        if (!c.pcnt) k = __reduce_add_sync(kFull, k);
        uint32_t pre = 0;  // boundaries of earlier ranges (sum form)
        if (!c.prefix)
            for (uint64_t j = tid; j < cta; j += NT) pre += __ldg(c.rcnt + j);
        pre = __reduce_add_sync(kFull, pre);
        if (lane == 0) {
            s_cnt[warp] = k;
            s_red[warp] = pre;
        }
        __syncthreads();
        if (tid == 0) {
            uint64_t base = 0;
            if (c.prefix) {
                base = __ldg(c.rcnt + cta);
            } else {
#pragma unroll
                for (int w = 0; w < NW; ++w) base += s_red[w];
            }
            s_base = base;
            if (tb == tlast) {  // the CTA holding the span's last tile publishes the sizes
                uint64_t nb = base;
#pragma unroll
                for (int w = 0; w < NW; ++w) nb += s_cnt[w];
                *c.nb_out = nb;
                *c.aq_len = MARKED ? 2 * nb + 1 : nb - 1;
                if (FUSE) *c.b_dev = (nb - 1 + (1u << c.fuse_kshift) - 1) >> c.fuse_kshift;
            }
        }
        __syncthreads();
    }
#ifdef BRMQ_CONTRACT_STAMPS
    if (lane == 0) g_cstamp2[cta * NW + warp][1] = cgt();
#endif
    uint64_t rank_run = s_base;  // global rank of the warp's next boundary
    for (uint32_t w = 0; w < warp; ++w) rank_run += s_cnt[w];
    const uint64_t rank_first = rank_run;

    SegMin carry{kNoKey, 0};  // open segment after the warp tiles done so far (warp-uniform)
    uint64_t head = kNoKey;   // lane-local until published
    bool head_set = false;
    auto tile = [&](auto gen_tag, uint32_t i, uint32_t fl) {
        constexpr bool GEN = decltype(gen_tag)::value;
        const uint32_t t = wa32 + i;
        int jlo = 0, jhi = kRow - 1;
        bool any = true;
        if (GEN) {  // a tile crossing the span's ends (64-bit: positions past n may pass 2^32)
            const uint64_t p0 = uint64_t(t) * kWTile + uint64_t(lane) * kRow;
            any = p0 <= blast && p0 + kRow - 1 >= b0;
            jlo = p0 >= b0 ? 0 : int(b0 - p0);
            jhi = p0 + kRow - 1 <= blast ? kRow - 1 : int(int64_t(blast) - int64_t(p0));
        }
        const Rows rs{smem_u32(s_rows[warp]), t * uint32_t(kWTile)};
        const unsigned fm = __ballot_sync(kFull, fl != 0);

        if (fm == 0) {  // no boundary in the warp tile: one leftmost minimum
            uint64_t key;
            if (!GEN) {
                // value-only row minima, warp minimum, then the leftmost row holding it
                // is searched with one element per lane
                int32_t v = 0x7FFFFFFF;
#pragma unroll
                for (int cc = 0; cc < 8; ++cc) {
                    const int4 x = rs.chunk(lane, cc);
                    v = __vimin3_s32(v, x.x, x.y);
                    v = __vimin3_s32(v, x.z, x.w);
                }
                const int32_t wv = __reduce_min_sync(kFull, v);
                const int L = __ffs(__ballot_sync(kFull, v == wv)) - 1;
                const int e = __ffs(__ballot_sync(kFull, rs.elem(uint32_t(L), int(lane)) == wv)) - 1;
                key = pack_key(wv, uint32_t(rs.pos(uint32_t(L), e)));
            } else {
                uint64_t run = kNoKey;
                if (any) run = row_min<false>(rs, lane, jlo, jhi);
                key = warp_min_key(run);
            }
            carry.k = kmin(carry.k, key);
            return;
        }
        const bool dense = !SPARSE || __popc(fm) > kDense;

        // pass 1: open-segment key at the right end of the lane's row; a dense
        // tile's flagged rows are handled in one pass below instead
        uint64_t run = kNoKey;
        if (any && fl == 0 && (GEN || !dense))  // (dense interior tiles: row_pass_all below)
            run = !GEN ? row_min<true>(rs, lane, 0, kRow - 1) : row_min<false>(rs, lane, jlo, jhi);
        if (!dense) {  // sparse flagged rows: one element per lane
            for (unsigned m = fm; m; m &= m - 1) {
                const int s = __ffs(m) - 1;
                const uint32_t ft = __shfl_sync(kFull, fl, s);
                const int jh = __shfl_sync(kFull, jhi, s);
                const int lo = 31 - __clz(ft);
                const int32_t v = rs.elem(uint32_t(s), int(lane));
                const uint64_t key = pack_key(v, uint32_t(rs.pos(uint32_t(s), int(lane))));
                const uint64_t mk = warp_min_key(int(lane) >= lo && int(lane) <= jh ? key : kNoKey);
                if (lane == uint32_t(s)) run = mk;
            }
        }

        // pass 2: close the areas whose right boundary lies in a row
        const uint32_t cntb = __popc(fl);
        uint64_t my_rank = 0;  // global rank of the row's first boundary (flagged rows)
        SegMin wt;             // warp-tile total
        uint32_t wc;
        if (dense) {
            // ranks first (a count scan), then one pass per flagged row: its inner
            // areas are stored at once, its head / tail parts join the warp scan
            uint32_t cinc = cntb;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const uint32_t cy = __shfl_up_sync(kFull, cinc, o);
                if (lane >= uint32_t(o)) cinc += cy;
            }
            wc = __shfl_sync(kFull, cinc, 31);
            const uint64_t rank = rank_run + (cinc - cntb);
            uint64_t hp = kNoKey;
            if (!GEN) {
                if (!__any_sync(kFull, __popc(fl) > kCap))
                    row_pass_cap<MARKED, FUSE, Rows, SPARSE && BRMQ_CHUNKED_DENSE>(rs, lane, fl, rank, out, hp, run,
                                         smem_u32(s_cap) + (warp * kCap * 32u + lane) * 8u);
                else
                    row_pass_all<MARKED, FUSE>(rs, lane, fl, rank, out, hp, run);
            }
            else if (any && fl) row_pass<MARKED, FUSE>(rs, lane, fl, jlo, jhi, rank, out, hp, run);
            SegMin inc{run, cntb != 0};
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                SegMin y;
                y.k = __shfl_up_sync(kFull, inc.k, o);
                y.f = __shfl_up_sync(kFull, inc.f, o);
                if (lane >= uint32_t(o)) inc = seg_combine(y, inc);
            }
            wt.k = __shfl_sync(kFull, inc.k, 31);
            wt.f = __shfl_sync(kFull, inc.f, 31);
            SegMin we;
            we.k = __shfl_up_sync(kFull, inc.k, 1);
            we.f = __shfl_up_sync(kFull, inc.f, 1);
            if (lane == 0) we = SegMin{kNoKey, 0};
            if (fl) {
                const SegMin in = seg_combine(carry, we);  // open segment entering the row
                my_rank = rank;
                const uint64_t first = kmin(in.k, hp);   // the area the row's first boundary closes
                if (in.f) {
                    put_area<MARKED, FUSE>(out, rank - 1, first);
                } else {  // first boundary of the piece: its area opened in an earlier piece
                    head = first;
                    head_set = true;
                }
            }
        } else {
            const int L = 31 - __clz(fm);
            wt = SegMin{warp_min_key(int(lane) >= L ? run : kNoKey), 1};
            // rows holding one boundary each (the common sparse case): ranks are
            // popcounts of the flagged rows before, no reductions
            const bool multi = __any_sync(kFull, (fl & (fl - 1)) != 0);
            wc = multi ? __reduce_add_sync(kFull, cntb) : uint32_t(__popc(fm));
            for (unsigned m = fm; m; m &= m - 1) {
                const int s = __ffs(m) - 1;
                const uint32_t ft = __shfl_sync(kFull, fl, s);
                const int jl = __shfl_sync(kFull, jlo, s);
                // open segment entering row s: rows after the previous flagged row
                const unsigned below = fm & ((1u << s) - 1u);
                const int pf = below ? 31 - __clz(below) : -1;
                const int sl = pf < 0 ? 0 : pf;
                const uint64_t rank =
                    rank_run + (multi ? __reduce_add_sync(kFull, int(lane) < s ? cntb : 0u) : uint32_t(__popc(below)));
                if (lane == uint32_t(s)) my_rank = rank;
                if ((ft & (ft - 1)) == 0) {
                    // one boundary at column lo: its area = the open segment entering
                    // row s + the row's head part [jl, lo], in one reduction
                    const int lo = 31 - __clz(ft);
                    uint64_t x = int(lane) >= sl && int(lane) < s ? run : kNoKey;
                    if (int(lane) >= jl && int(lane) <= lo)
                        x = kmin(x, pack_key(rs.elem(uint32_t(s), int(lane)),
                                             uint32_t(rs.pos(uint32_t(s), int(lane)))));
                    uint64_t val = warp_min_key(x);
                    if (pf < 0) val = kmin(val, carry.k);
                    if (lane == uint32_t(s)) {
                        if (pf < 0 && !carry.f) {
                            head = val;
                            head_set = true;
                        } else {
                            put_area<MARKED, FUSE>(out, rank - 1, val);
                        }
                    }
                    continue;
                }
                const uint64_t seg = warp_min_key(int(lane) >= sl && int(lane) < s ? run : kNoKey);
                const SegMin in = pf >= 0 ? SegMin{seg, 1} : seg_combine(carry, SegMin{seg, 0});
                const int jh = __shfl_sync(kFull, jhi, s);
                const int32_t v = rs.elem(uint32_t(s), int(lane));
                const bool inr = int(lane) >= jl && int(lane) <= jh;
                const uint64_t key = inr ? pack_key(v, uint32_t(rs.pos(uint32_t(s), int(lane)))) : kNoKey;
                const bool isf = (ft >> lane) & 1u;
                SegMin Sg{key, isf};
                if (lane == 0 && !isf) Sg.k = kmin(Sg.k, in.k);  // the open segment joins the first part
#pragma unroll
                for (int o = 1; o < 32; o <<= 1) {
                    SegMin y;
                    y.k = __shfl_up_sync(kFull, Sg.k, o);
                    y.f = __shfl_up_sync(kFull, Sg.f, o);
                    if (lane >= uint32_t(o)) Sg = seg_combine(y, Sg);
                }
                uint64_t prev = __shfl_up_sync(kFull, Sg.k, 1);
                if (lane == 0) prev = in.k;
                if (isf) {
                    const uint32_t before = __popc(ft & ((1u << lane) - 1u));
                    const uint64_t rk = rank + before;
                    const uint64_t val = kmin(prev, key);  // inclusive right end
                    if (!in.f && before == 0) {
                        head = val;
                        head_set = true;
                    } else if (rk > 0) {
                        put_area<MARKED, FUSE>(out, rk - 1, val);
                    }
                }
            }
        }
        if (fl) {  // consumed bitmap word: (rank prefix, bits) for the remap, then clear
            const size_t w = size_t(t) * 32 + lane;
            if (c.word_info) c.word_info[w] = make_uint2(uint32_t(my_rank), fl);
            c.bitmap[w] = 0;
        }
        carry = seg_combine(carry, wt);
        rank_run += wc;
    };

    if (c.reads && cnt && lane == 0) {  // the warp's tiles, clipped to the span
        const uint64_t lo = wa * kWTile > b0 ? wa * kWTile : b0;
        const uint64_t hi = (wa + cnt) * kWTile - 1 < blast ? (wa + cnt) * kWTile - 1 : blast;
        if (hi >= lo) atomicAdd(reinterpret_cast<unsigned long long*>(c.reads), (unsigned long long)(hi - lo + 1));
    }
#ifdef BRMQ_CONTRACT_STAMPS
    const uint64_t gw_dbg = uint64_t(blockIdx.x) * NW + warp;
    if (lane == 0) g_cstamp[gw_dbg][0] = cgt();
#endif
    // tiles [i_in0, i_in1) of the piece lie entirely inside the span
    const uint32_t t_in0 = uint32_t((uint64_t(b0) + kWTile - 1) / kWTile), t_in1 = uint32_t((uint64_t(blast) + 1) / kWTile);
    const uint32_t i_in0 = t_in0 > wa32 ? t_in0 - wa32 : 0u;
    const uint32_t i_in1 = t_in1 > wa32 ? t_in1 - wa32 : 0u;
    if (cnt32) stage();
    for (uint32_t i = 0; i < cnt32; ++i) {
        const uint32_t fl = fy;
        if (i + 1 < cnt32) fetch(i + 1);  // in flight while tile i is reduced
        if (i >= i_in0 && i < i_in1) tile(std::false_type{}, i, fl);
        else tile(std::true_type{}, i, fl);
        __syncwarp();
        if (i + 1 < cnt32) stage();
    }

#ifdef BRMQ_CONTRACT_STAMPS
    if (lane == 0) g_cstamp[gw_dbg][1] = cgt();
#endif
    // ---- stitch: every warp publishes its piece's descriptor (the open segment at
    // its end, has-boundary) at once -- no block barrier, so a warp never waits
    // for the slowest warp of its CTA (c2: 7 us apart on average) -- and the area
    // closed by its first boundary folds the tails of the pieces before it back to
    // the nearest one holding a boundary (usually the previous warp's).
    const unsigned hl = __ballot_sync(kFull, head_set);
    if (hl) head = __shfl_sync(kFull, head, __ffs(hl) - 1);
    const int64_t gw = int64_t(cta) * NW + warp;
    if (lane == 0) {
        c.key_tail[gw] = carry.k;
        st_release_u64(c.st_part + gw, status_pack(epoch, kStInclusive, carry.f != 0, 0));
    }
#ifdef BRMQ_CONTRACT_STAMPS
    if (lane == 0 && (!carry.f || rank_first == 0)) g_cstamp[gw_dbg][2] = cgt();
#endif
    if (!carry.f || rank_first == 0) return;  // no boundary, or the global first one
    uint64_t acc = kNoKey;
    const int64_t wfirst = int64_t(cfirst) * NW;  // pieces before b0's CTA hold nothing
    for (int64_t p = gw - 1; p >= wfirst; p -= 32) {
        const int64_t j = p - int64_t(lane);
        const bool live = j >= wfirst;
        uint64_t sw = 0;
        bool ready = !live, has = false;
        while (true) {  // wait only for the descriptors up to the nearest boundary
            if (!ready) {
                sw = ld_relaxed_u64(c.st_part + j);
                ready = status_state(sw, epoch) != kStInvalid;
                has = ready && status_flag(sw);
            }
            const unsigned stop = __ballot_sync(kFull, has || !live);
            const int g = stop ? __ffs(stop) - 1 : 31;
            const unsigned need = g >= 31 ? kFull : ((2u << g) - 1u);
            if ((__ballot_sync(kFull, ready) & need) == need) break;
            // backoff: a spinning warp takes issue slots from the streaming warps
            __nanosleep(64);
        }
        __threadfence();  // acquire: the tails were stored before their descriptors
        const unsigned stop = __ballot_sync(kFull, has || !live);
        const int g = stop ? __ffs(stop) - 1 : 32;
        const uint64_t k = (live && int(lane) <= g) ? ld_relaxed_u64(c.key_tail + j) : kNoKey;
        acc = kmin(acc, warp_min_key(k));
        if (g < 32) break;
    }
    if (lane == 0) put_area<MARKED, FUSE>(out, rank_first - 1, kmin(acc, head));
#ifdef BRMQ_CONTRACT_STAMPS
    if (lane == 0) g_cstamp[gw_dbg][2] = cgt();
#endif
}

template <bool VEC, bool MARKED, bool SPARSE = true, bool FUSE = false>
__global__ void __launch_bounds__(NT, BRMQ_CONTRACT_MINB) k_contract(const __grid_constant__ ContractArgs c) {
    contract_body<VEC, MARKED, SPARSE, FUSE>(c);  // (its griddepcontrol.wait follows the first loads)
}

int contract_grid() {
    // per device: the shared-memory attribute belongs to the device's context
    // (the grid is the same on identical parts, kept per device anyway)
    static int grids[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    int& grid = grids[dev & 63];
    if (grid == 0) {
        int sms = 0, per_v = 0, per_s = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const void* fns[] = {reinterpret_cast<const void*>(k_contract<true, false>),
                             reinterpret_cast<const void*>(k_contract<true, false, false>),
                             reinterpret_cast<const void*>(k_contract<true, false, true, true>),
                             reinterpret_cast<const void*>(k_contract<true, false, false, true>),
                             reinterpret_cast<const void*>(k_contract<true, true>),
                             reinterpret_cast<const void*>(k_contract<true, true, false>),
                             reinterpret_cast<const void*>(k_contract<false, false>),
                             reinterpret_cast<const void*>(k_contract<false, true>)};
        for (const void* f : fns)  // the capture slots take the block past 48 KB of shared memory
            cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kCapSmem));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_v, k_contract<true, false>, NT, kCapSmem);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_s, k_contract<false, true>, NT, kCapSmem);
        int per = per_v < per_s ? per_v : per_s;
        if (per < 1) per = 1;
        grid = sms * per;
        if (grid > int(kMaxContractRanges)) grid = int(kMaxContractRanges);
    }
    return grid;
}

}  // namespace

#ifdef BRMQ_CONTRACT_STAMPS
extern "C" int brmq_debug_contract_stamps(unsigned long long* out, int n) {
    const int rc = int(cudaMemcpyFromSymbol(out, g_cstamp, size_t(n) * 3 * 8));
    static unsigned long long zero[kMaxContractRanges * 8][3];
    cudaMemcpyToSymbol(g_cstamp, zero, sizeof(zero));
    return rc;
}
extern "C" int brmq_debug_contract_stamps2(unsigned long long* out, int n) {
    return int(cudaMemcpyFromSymbol(out, g_cstamp2, size_t(n) * 3 * 8));
}
#endif

size_t contract_tiles(uint64_t n) { return (n + kTile - 1) / kTile; }
size_t contract_bitmap_words(uint64_t n) { return contract_tiles(n) * (kTile / 32) + 4; }
size_t contract_status_words() { return size_t(2) * kMaxContractRanges * NW; }  // st_part, key_tail (per piece)

int launch_piece_count(const uint32_t* bitmap, const uint32_t* span, uint64_t n, uint32_t* pcnt,
                       uint32_t* rcnt, cudaStream_t s) {
    uint32_t G = 0, R = 0;
    contract_partition(n, &G, &R);
    brmq::launch_k(k_piece_count, dim3(G), dim3(NT), 0, s, bitmap, span, R, pcnt, rcnt);
    return 1;
}

void contract_partition(uint64_t n, uint32_t* G, uint32_t* R) {
    const uint64_t tiles = contract_tiles(n);
    uint64_t g = uint64_t(contract_grid());
    if (g > tiles) g = tiles;
    if (g == 0) g = 1;
    const uint64_t r = (tiles + g - 1) / g;
    *R = uint32_t(r);
    *G = uint32_t(tiles ? (tiles + r - 1) / r : 1);
}

int launch_contract(const int32_t* A, uint64_t n, uint32_t* bitmap, const uint32_t* span,
                    const uint32_t* rcnt, bool prefix, uint64_t* aq, uint64_t* nb_out,
                    uint64_t* aq_len,
                    uint2* word_info, uint64_t* status, const uint32_t* epoch_dev,
                    uint32_t epoch_off, cudaStream_t s, bool marked, const uint32_t* pcnt,
                    uint64_t endpoints, const ContractFuse* fuse, bool* fused, uint64_t* array_reads) {
    if (fused) *fused = false;
    if (n == 0) return 0;
    uint32_t G = 0, R = 0;
    contract_partition(n, &G, &R);
    const bool vec = (reinterpret_cast<uintptr_t>(A) & 15u) == 0;
    // the fused block minima + table tail (small A_Q: the caller filled sub and
    // the table's row 0 with kNoKey)
    const bool fz = fuse && vec && !marked;
    ContractArgs args{A, n, bitmap, span, aq, nb_out, aq_len, word_info, rcnt, R,
                      prefix ? 1u : 0u, status, status + size_t(kMaxContractRanges) * NW, pcnt, epoch_dev,
                      epoch_off, fz ? fuse->sub : nullptr, fz ? fuse->st : nullptr,
                      fz ? fuse->b_max : 0, fz ? fuse->kshift : 0u, fz ? fuse->b_dev : nullptr,
                      array_reads};
    void* params[] = {&args};
    // >= 8 endpoints per 1024 positions on average: nearly every flagged warp tile
    // has more than kDense flagged rows, so the dense-only instance runs
    const bool dense = endpoints >= uint64_t(kDenseEndpoints) * (n / kWTile + 1);
    const void* fn = vec ? (marked ? (dense ? reinterpret_cast<const void*>(k_contract<true, true, false>)
                                            : reinterpret_cast<const void*>(k_contract<true, true>))
                                   : fz ? (dense ? reinterpret_cast<const void*>(k_contract<true, false, false, true>)
                                                 : reinterpret_cast<const void*>(k_contract<true, false, true, true>))
                                   : (dense ? reinterpret_cast<const void*>(k_contract<true, false, false>)
                                            : reinterpret_cast<const void*>(k_contract<true, false>)))
                         : (marked ? reinterpret_cast<const void*>(k_contract<false, true>)
                                   : reinterpret_cast<const void*>(k_contract<false, false>));
    if (fused) *fused = fz;
    // cooperative (co-residency checked); inside a solve also a PDL secondary: its
    // CTAs are placed as the predecessor's retire and wait in pdl_wait, and the
    // predecessor never waits on them, so co-residency is reached before any
    // cross-CTA wait begins
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(NT);
    cfg.dynamicSmemBytes = kCapSmem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    PdlState& st = pdl_state();
    if (st.on && !st.first) {
        at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[1].val.programmaticStreamSerializationAllowed = 1;
        cfg.numAttrs = 2;
    }
    st.first = false;
    cudaLaunchKernelExC(&cfg, fn, params);
    return 1;  // launch errors surface through the caller's cudaGetLastError
}

}  // namespace brmq
