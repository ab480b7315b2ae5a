// scan.cuh -- block-wide scans and the single-pass (decoupled look-back)
// tile-status protocol shared by the radix sort, the endpoint dedup/rank and
// the contraction kernels.
//
// Tile status words are 64-bit and self-describing, so a single relaxed
// 64-bit store publishes state and value atomically:
//     [63:40] epoch (24 bits)  [39:38] state  [37] flag  [36:0] value
// The epoch is a per-launch tag chosen by the host, so status arrays never
// need clearing between launches (stale words carry another epoch and read
// as "not ready").  Tiles are taken in launch order through an atomic ticket,
// so every predecessor of a tile is resident or finished when it looks back:
// a tile always publishes its aggregate BEFORE it waits, hence no deadlock.
#pragma once

#include "common.cuh"

namespace brmq {

constexpr uint64_t kStInvalid = 0, kStAggregate = 1, kStInclusive = 2;
constexpr uint64_t kValueMask = (1ull << 37) - 1;

__device__ __forceinline__ uint64_t status_pack(uint32_t epoch, uint64_t state, bool flag,
                                                uint64_t value) {
    return (uint64_t(epoch & 0xFFFFFFu) << 40) | (state << 38) | (uint64_t(flag) << 37) |
           (value & kValueMask);
}
__device__ __forceinline__ uint64_t status_state(uint64_t s, uint32_t epoch) {
    return (uint32_t(s >> 40) == (epoch & 0xFFFFFFu)) ? ((s >> 38) & 3ull) : kStInvalid;
}
__device__ __forceinline__ bool status_flag(uint64_t s) { return (s >> 37) & 1ull; }
__device__ __forceinline__ uint64_t status_value(uint64_t s) { return s & kValueMask; }

// Wait until tile p's status (epoch-tagged) is published; returns the word.
__device__ __forceinline__ uint64_t status_wait(const uint64_t* status, uint64_t p,
                                                uint32_t epoch) {
    uint64_t s;
    while (true) {
        s = ld_relaxed_u64(status + p);
        if (status_state(s, epoch) != kStInvalid) break;
        __nanosleep(32);
    }
    return s;
}

// Exclusive prefix sum over the tiles before `tile` (count look-back).
__device__ __forceinline__ uint64_t lookback_sum(const uint64_t* status, uint64_t tile,
                                                 uint32_t epoch) {
    uint64_t excl = 0;
    uint64_t p = tile;
    while (p > 0) {
        --p;
        const uint64_t s = status_wait(status, p, epoch);
        excl += status_value(s);
        if (status_state(s, epoch) == kStInclusive) break;
    }
    return excl;
}

__device__ __forceinline__ uint64_t warp_sum_u64(uint64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(kFull, v, o);
    return v;
}

// Warp-wide decoupled look-back (call with all 32 lanes of one warp).
// Reads the descriptors of 32 predecessors per round (lane i <- tile p - i),
// waits only until every lane up to the nearest inclusive ("P") one is
// published, and folds them: `excl` = sum of the values up to that tile;
// with KEYS, `carry` = min of the keys of the open segment entering `tile`
// (aggregate keys until the nearest tile holding a segment head, whose
// aggregate is its tail, or the nearest P tile, whose inclusive key is the
// open-segment min at its end).  Tiles before `tfirst` do not exist.
template <bool KEYS>
__device__ __forceinline__ void warp_lookback(const uint64_t* status, const uint64_t* key_agg,
                                              const uint64_t* key_inc, uint64_t tile,
                                              uint64_t tfirst, uint32_t epoch, uint64_t& excl,
                                              uint64_t& carry) {
    const unsigned lane = lane_id();
    excl = 0;
    carry = kNoKey;
    bool key_done = false;
    int64_t p = int64_t(tile) - 1;
    while (true) {
        const int64_t ti = p - int64_t(lane);
        const bool exists = ti >= int64_t(tfirst);
        uint64_t s = 0, st = kStInclusive;
        while (true) {
            if (exists) {
                s = ld_acquire_u64(status + ti);
                st = status_state(s, epoch);
            }
            const unsigned inv = __ballot_sync(kFull, st == kStInvalid);
            const unsigned pm = __ballot_sync(kFull, st == kStInclusive);
            const int lowp = pm ? __ffs(pm) - 1 : 31;
            const unsigned upto = lowp >= 31 ? kFull : ((2u << lowp) - 1u);
            if ((inv & upto) == 0) break;
            __nanosleep(20);
        }
        const unsigned pm = __ballot_sync(kFull, st == kStInclusive);
        const int g = pm ? __ffs(pm) - 1 : 32;  // nearest inclusive lane (32: none)
        excl += warp_sum_u64((int(lane) <= g && exists) ? status_value(s) : 0);
        if (KEYS && !key_done) {
            const unsigned fm = __ballot_sync(kFull, st == kStAggregate && status_flag(s));
            const int f = fm ? __ffs(fm) - 1 : 32;
            const int stop = f < g ? f : g;
            uint64_t kk = kNoKey;
            if (int(lane) <= stop && exists)
                kk = ld_relaxed_u64((st == kStInclusive ? key_inc : key_agg) + ti);
            carry = kmin(carry, warp_min_key(kk));
            key_done = stop < 32;
        }
        if (g < 32) break;
        p -= 32;
    }
}

// Block-wide exclusive sum (blockDim.x == NT, NT % 32 == 0).  `total` gets the
// block total.  Uses NT/32 + 1 words of shared scratch.
template <int NT>
__device__ __forceinline__ uint32_t block_excl_sum(uint32_t x, uint32_t* sh, uint32_t& total) {
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    uint32_t inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(kFull, inc, o);
        if (lane >= unsigned(o)) inc += y;
    }
    if (lane == 31) sh[warp] = inc;
    __syncthreads();
    if (warp == 0) {
        uint32_t w = lane < NT / 32 ? sh[lane] : 0;
        uint32_t wi = w;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(kFull, wi, o);
            if (lane >= unsigned(o)) wi += y;
        }
        if (lane < NT / 32) sh[lane] = wi - w;  // exclusive warp offsets
        if (lane == NT / 32 - 1) sh[NT / 32] = wi;
    }
    __syncthreads();
    total = sh[NT / 32];
    const uint32_t r = sh[warp] + inc - x;
    __syncthreads();
    return r;
}

// Segmented-min scan element: `f` = a segment head (boundary) lies inside,
// `k` = min key of the open segment at the element's right end.
struct SegMin {
    uint64_t k;
    uint32_t f;
};
// Associative: a then b (b to the right of a).
__device__ __forceinline__ SegMin seg_combine(SegMin a, SegMin b) {
    return SegMin{b.f ? b.k : kmin(a.k, b.k), a.f | b.f};
}

// Block-wide exclusive segmented-min scan combined with an exclusive sum.
template <int NT>
__device__ __forceinline__ void block_excl_segmin_sum(SegMin x, uint32_t c, SegMin& x_excl,
                                                      uint32_t& c_excl, SegMin& x_total,
                                                      uint32_t& c_total, uint64_t* shk,
                                                      uint32_t* shf, uint32_t* shc) {
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    SegMin inc = x;
    uint32_t cinc = c;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        SegMin y;
        y.k = __shfl_up_sync(kFull, inc.k, o);
        y.f = __shfl_up_sync(kFull, inc.f, o);
        const uint32_t cy = __shfl_up_sync(kFull, cinc, o);
        if (lane >= unsigned(o)) {
            inc = seg_combine(y, inc);
            cinc += cy;
        }
    }
    if (lane == 31) {
        shk[warp] = inc.k;
        shf[warp] = inc.f;
        shc[warp] = cinc;
    }
    __syncthreads();
    if (warp == 0) {
        SegMin w{kNoKey, 0};
        uint32_t wc = 0;
        if (lane < NT / 32) {
            w.k = shk[lane];
            w.f = shf[lane];
            wc = shc[lane];
        }
        SegMin wi = w;
        uint32_t wci = wc;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            SegMin y;
            y.k = __shfl_up_sync(kFull, wi.k, o);
            y.f = __shfl_up_sync(kFull, wi.f, o);
            const uint32_t cy = __shfl_up_sync(kFull, wci, o);
            if (lane >= unsigned(o)) {
                wi = seg_combine(y, wi);
                wci += cy;
            }
        }
        // exclusive warp prefix = inclusive of previous lane
        SegMin pe;
        pe.k = __shfl_up_sync(kFull, wi.k, 1);
        pe.f = __shfl_up_sync(kFull, wi.f, 1);
        uint32_t pc = __shfl_up_sync(kFull, wci, 1);
        if (lane == 0) {
            pe = SegMin{kNoKey, 0};
            pc = 0;
        }
        if (lane < NT / 32) {
            shk[lane] = pe.k;
            shf[lane] = pe.f;
            shc[lane] = pc;
        }
        if (lane == NT / 32 - 1) {
            shk[NT / 32] = wi.k;
            shf[NT / 32] = wi.f;
            shc[NT / 32] = wci;
        }
    }
    __syncthreads();
    // exclusive within warp: inclusive of the previous lane
    SegMin we;
    we.k = __shfl_up_sync(kFull, inc.k, 1);
    we.f = __shfl_up_sync(kFull, inc.f, 1);
    uint32_t wce = __shfl_up_sync(kFull, cinc, 1);
    if (lane == 0) {
        we = SegMin{kNoKey, 0};
        wce = 0;
    }
    const SegMin wp{shk[warp], shf[warp]};
    x_excl = seg_combine(wp, we);
    c_excl = shc[warp] + wce;
    x_total = SegMin{shk[NT / 32], shf[NT / 32]};
    c_total = shc[NT / 32];
    __syncthreads();
}

}  // namespace brmq
