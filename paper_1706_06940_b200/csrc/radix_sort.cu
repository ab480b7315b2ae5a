// radix_sort.cu -- on-device LSD radix sort of (pos, origin) endpoint pairs.
//
// Replaces radix_sort_by_pos (contraction.cpp:27-63): LSD over the bits of the
// 32-bit position, one up-front histogram for every digit (:35-41), a stable
// scatter per pass (:58).  Stability makes the output order identical to the
// reference's for equal positions (collect order).  The reference walks 8-bit
// digits and skips constant bytes; here the digits are as wide as 10 bits so
// that positions of up to 30 bits (n <= 2^30) take three passes, not four:
//   passes P = ceil(bits / 10), widths bits / P (+1 for the first bits % P),
//   e.g. 27 bits (n = 1e8) -> 9 + 9 + 9, 30 bits (n = 2^30) -> 10 + 10 + 10.
//
// B200 design (single-pass "onesweep" scheme):
//   k_rs_hist : one read of the keys (16-byte loads, 4 in flight per thread)
//               builds the histograms of all passes.
//   k_rs_pass : per pass ONE kernel.  A CTA takes a tile (atomic ticket =>
//               tiles start in order) of NT x ITEMS keys, item-major and
//               lane-minor per warp (coalesced loads), and ranks them stably
//               inside the warp: the peers of a key are found with one ballot
//               per digit bit (a "multisplit"; __match_any_sync took 47% of
//               the round-1 kernel's stall samples, and measured 0.65 vs 0.53 ms
//               at c3-con here), the running per-digit count lives in a 16-bit
//               warp-private counter whose per-warp totals give the tile's digit
//               counts (no histogram atomics).  Per digit: warp offsets, the
//               tile's count published as a 32-bit descriptor (zeroed by one
//               memset per sort, no epochs), a late decoupled look-back over
//               windows of 16 predecessors (while a wave's tiles all look back
//               at once an inclusive prefix propagates 16 tiles per round, not
//               one), and the tile is staged in shared memory sorted by digit,
//               then written out in runs (consecutive threads -> consecutive
//               addresses of a bucket).  No separate scan kernel, no global
//               barrier.
//   Yardstick (tools/cub_sort_bench.cu): cub::DeviceRadixSort::SortKeys on the
//   same 2e7 keys 0.53 ms (27 and 30 bits); this sort 0.53 ms (27 bits, 9-bit
//   digits) and 0.62 ms (30 bits, 10-bit digits).  It serves the stage API's
//   (pos, origin) pairs, ST-RMQ_CON and keys wider than 30 bits.
//
// The BbST_CON radix pipeline's sort + dedup is a two-level MSD radix sort
// instead (launch_radix_partition_mark): the collect kernel counts the top D
// bits, k_msd_partition scatters the keys by them (shared-atomic ranks, one
// global reservation per tile and digit -- no look-back, no stability needed),
// and k_bucket_mark finishes each bucket with a counting digit over the low L
// bits in shared memory, which also dedups and marks the boundary bitmap the
// contraction reads.  c3-con (2e7 endpoints, 27 bits): sort + dedup 0.57 ->
// 0.10 ms (+ ~12 us of histogram in the collect); c5-con (30 bits) 0.74 -> 0.15 ms.
#include <cstdint>

#include "common.cuh"
#include "kernels.h"
#include "scan.cuh"

namespace brmq {
namespace {

constexpr int kMaxBits = 10;
constexpr int kMaxRadix = 1 << kMaxBits;
constexpr int kMaxPasses = 4;
constexpr uint64_t kSmallM = 1u << 18;
// (NT, ITEMS): 512 x 16 = 8192-key tiles for large batches, 256 x 8 = 2048 for
// small ones (more tiles in flight; shorter per-tile latency)
#ifndef BRMQ_RS_NT
#define BRMQ_RS_NT 512
#endif
#ifndef BRMQ_RS_ITEMS
#define BRMQ_RS_ITEMS 16
#endif
constexpr int kNtLarge = BRMQ_RS_NT, kItemsLarge = BRMQ_RS_ITEMS;
constexpr int kNtSmall = 256, kItemsSmall = 8;
inline uint64_t tile_for(uint64_t m) {
    return m <= kSmallM ? uint64_t(kNtSmall) * kItemsSmall : uint64_t(kNtLarge) * kItemsLarge;
}

// Digit widths of pass p for `bits` key bits.
struct Plan {
    int passes;
    int width[kMaxPasses];
    int shift[kMaxPasses];
};
inline Plan plan_for(int bits) {
    Plan pl{};
    if (bits <= 0) return pl;
    pl.passes = (bits + kMaxBits - 1) / kMaxBits;
    if (pl.passes > kMaxPasses) pl.passes = kMaxPasses;
    const int base = bits / pl.passes, extra = bits % pl.passes;
    int sh = 0;
    for (int p = 0; p < pl.passes; ++p) {
        pl.width[p] = base + (p < extra ? 1 : 0);
        pl.shift[p] = sh;
        sh += pl.width[p];
    }
    return pl;
}

struct HistArgs {
    int passes;
    int width[kMaxPasses];
    int shift[kMaxPasses];
};

__global__ void __launch_bounds__(256) k_rs_hist(const uint32_t* __restrict__ keys, uint64_t m,
                                                 const __grid_constant__ HistArgs a,
                                                 unsigned long long* __restrict__ ghist) {
    brmq::pdl_wait();
    __shared__ uint32_t h[kMaxPasses][kMaxRadix];
    for (int i = threadIdx.x; i < kMaxPasses * kMaxRadix; i += 256) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint64_t stride = uint64_t(gridDim.x) * 256;
    auto add = [&](uint32_t k) {
        for (int p = 0; p < a.passes; ++p)
            atomicAdd(&h[p][(k >> a.shift[p]) & ((1u << a.width[p]) - 1u)], 1u);
    };
    // 16-byte loads, 4 in flight per thread (a 1-key-per-thread grid-stride loop was
    // latency-bound: 76 us for 2e7 keys)
    const uint64_t m4 = (reinterpret_cast<uintptr_t>(keys) & 15u) == 0 ? m / 4 : 0;
    const uint4* k4 = reinterpret_cast<const uint4*>(keys);
    constexpr int U = 4;
    for (uint64_t i0 = uint64_t(blockIdx.x) * 256 + threadIdx.x; i0 < m4; i0 += U * stride) {
        uint4 x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = i0 + u * stride < m4 ? __ldcs(k4 + i0 + u * stride) : make_uint4(0, 0, 0, 0);
#pragma unroll
        for (int u = 0; u < U; ++u)
            if (i0 + u * stride < m4) {
                add(x[u].x);
                add(x[u].y);
                add(x[u].z);
                add(x[u].w);
            }
    }
    for (uint64_t i = 4 * m4 + uint64_t(blockIdx.x) * 256 + threadIdx.x; i < m; i += stride) add(__ldg(keys + i));
    __syncthreads();
    for (int p = 0; p < a.passes; ++p)
        for (int d = threadIdx.x; d < (1 << a.width[p]); d += 256) {
            const uint32_t c = h[p][d];
            if (c) atomicAdd(ghist + p * kMaxRadix + d, (unsigned long long)c);
        }
}

// Dynamic shared memory of k_rs_pass<NT, ITEMS>.
template <int NT, int ITEMS>
struct PassSmem {
    static constexpr int NW = NT / 32;
    static constexpr int TILE = NT * ITEMS;
    static_assert(NW * kMaxRadix >= TILE, "the destination map reuses the warp counters");
    // per warp: running count, then the warp's offset in the digit; afterwards
    // reused as dest[] (the sorted slot of every tile item, in input order)
    uint16_t whist[NW][kMaxRadix];
    uint32_t thist[kMaxRadix];  // tile histogram (unordered smem atomics, published early)
    uint32_t texcl[kMaxRadix];  // tile-local start of each digit
    uint32_t gbase[kMaxRadix];  // global start of each digit's run of this tile
    uint32_t scan[NW + 1];
    uint32_t tile;
    uint32_t skey[TILE], sval[TILE];  // the tile, sorted by digit (stable)
};

// Look-back descriptors: one word per (tile, digit), zeroed by the sort's memset
// (no epochs): [top 2 bits] state 0 not ready / 1 aggregate / 2 inclusive,
// [rest] the count.  32-bit words while m < 2^30 (half the traffic of 64-bit
// epoch-tagged words; a tile's 1024 descriptors are the look-back's bytes).
template <class W>
struct Desc {
    static constexpr int kShift = int(sizeof(W) * 8) - 2;
    static constexpr W kMask = (W(1) << kShift) - 1;
    static __device__ __forceinline__ W pack(uint32_t state, uint64_t v) { return (W(state) << kShift) | W(v); }
    static __device__ __forceinline__ uint32_t state(W w) { return uint32_t(w >> kShift); }
    static __device__ __forceinline__ uint64_t value(W w) { return uint64_t(w & kMask); }
};
__device__ __forceinline__ uint32_t ld_vol(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ uint64_t ld_vol(const uint64_t* p) { return ld_relaxed_u64(p); }
__device__ __forceinline__ void st_vol(uint32_t* p, uint32_t v) {
    asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void st_vol(uint64_t* p, uint64_t v) { st_relaxed_u64(p, v); }

// WB: the digit width at compile time (8, 9, 10: the ballot loop unrolls), or 0
// for a run-time width.
template <int NT, int ITEMS, int WB, class W>
__global__ void __launch_bounds__(NT, (NT == 512 ? 2 : (NT == 256 && ITEMS > 8 ? 3 : 4))) k_rs_pass(
    const uint32_t* __restrict__ kin, const uint32_t* __restrict__ vin, uint32_t* __restrict__ kout,
    uint32_t* __restrict__ vout, uint64_t m, int shift, int width_rt,
    const unsigned long long* __restrict__ ghist, W* __restrict__ status,
    uint32_t* __restrict__ ticket) {
    brmq::pdl_wait();
    using S = PassSmem<NT, ITEMS>;
    using D = Desc<W>;
    constexpr int NW = S::NW, TILE = S::TILE;
    constexpr int DPT = kMaxRadix / NT;  // digits per thread (2 or 4), consecutive
    extern __shared__ __align__(16) unsigned char smem_raw[];
    S& sm = *reinterpret_cast<S*>(smem_raw);
    const int width = WB > 0 ? WB : width_rt;
    const uint32_t radix = 1u << width, dmask = radix - 1u;
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;

    if (threadIdx.x == 0) sm.tile = atomicAdd(ticket, 1u);
    for (int i = threadIdx.x; i < NW * kMaxRadix / 2; i += NT)
        reinterpret_cast<uint32_t*>(&sm.whist[0][0])[i] = 0u;
    for (int i = threadIdx.x; i < kMaxRadix; i += NT) sm.thist[i] = 0u;
    __syncthreads();
    const uint64_t tile = sm.tile;
    const uint64_t tbase = tile * TILE;
    const uint64_t base = tbase + uint64_t(warp) * (32 * ITEMS);

    // values are not held across the ranking: they are copied into their sorted
    // slots afterwards by a coalesced pass (dest[] map), which keeps the kernel at
    // 64 registers without spills
    uint32_t key[ITEMS];
    uint32_t rank2[(ITEMS + 1) / 2];  // two 16-bit in-warp ranks (later: sorted slots) per register
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const uint64_t idx = base + uint64_t(i) * 32 + lane;
        key[i] = idx < m ? __ldcs(kin + idx) : 0u;
    }

    // 1) stable warp ranking, item-major / lane-minor == input order.  The peers
    //    of a key (same digit) come from one ballot per digit bit.
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const bool ok = base + uint64_t(i) * 32 + lane < m;
        const uint32_t d = (key[i] >> shift) & dmask;
        unsigned peers = __ballot_sync(kFull, ok);
#pragma unroll
        for (int b = 0; b < (WB > 0 ? WB : kMaxBits); ++b) {
            if (WB == 0 && b >= width) break;
            const bool bit = (d >> b) & 1u;
            const unsigned bb = __ballot_sync(kFull, bit);
            peers &= bit ? bb : ~bb;
        }
        const uint32_t prev = ok ? sm.whist[warp][d] : 0u;
        __syncwarp();
        const uint32_t rk = prev + __popc(peers & lt);
        rank2[i / 2] = (i & 1) ? (rank2[i / 2] | (rk << 16)) : rk;
        if (ok && lane == unsigned(__ffs(peers) - 1)) sm.whist[warp][d] = uint16_t(prev + __popc(peers));
        __syncwarp();
    }
    __syncthreads();

    // 2) per digit (thread t owns digits t*DPT ...): the warps' offsets inside the
    //    tile's run of the digit and the tile count, published at once (the
    //    counts come from the warp counters: no histogram atomics)
    uint32_t tsum = 0;
    W* st = status + tile * kMaxRadix;
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
        const uint32_t d = threadIdx.x * DPT + j;
        uint32_t sum = 0;
        if (d < radix) {
#pragma unroll
            for (int w = 0; w < NW; ++w) {
                const uint32_t c = sm.whist[w][d];
                sm.whist[w][d] = uint16_t(sum);
                sum += c;
            }
            st_vol(st + d, D::pack(tile == 0 ? 2u : 1u, sum));
            sm.thist[d] = sum;
        }
        tsum += sum;
    }

    // 3) tile-local digit starts and the global histogram's exclusive prefix
    //    (gbase[d] gets the tile's look-back count added once it is known)
    {
        uint32_t ttot_unused, gtot;
        uint32_t run = block_excl_sum<NT>(tsum, sm.scan, ttot_unused);
        uint32_t gsum = 0;
#pragma unroll
        for (int j = 0; j < DPT; ++j) {
            const uint32_t d = threadIdx.x * DPT + j;
            gsum += d < radix ? uint32_t(ghist[d]) : 0u;
        }
        uint32_t grun = block_excl_sum<NT>(gsum, sm.scan, gtot);
#pragma unroll
        for (int j = 0; j < DPT; ++j) {
            const uint32_t d = threadIdx.x * DPT + j;
            if (d < radix) {
                sm.texcl[d] = run;
                sm.gbase[d] = grun;
                run += sm.thist[d];
                grun += uint32_t(ghist[d]);
            }
        }
    }
    __syncthreads();

    // 5) sorted slots: keys staged at once, the slot of every item recorded in
    //    input order (dest[] over the warp counters), then the values copied
    //    with coalesced reads
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const uint32_t d = (key[i] >> shift) & dmask;
        const uint32_t lp = sm.texcl[d] + sm.whist[warp][d] + ((rank2[i / 2] >> (16 * (i & 1))) & 0xFFFFu);
        rank2[i / 2] = (i & 1) ? ((rank2[i / 2] & 0xFFFFu) | (lp << 16)) : ((rank2[i / 2] & 0xFFFF0000u) | lp);
    }
    __syncthreads();  // every warp is done with whist: it becomes dest[]
    uint16_t* dest = &sm.whist[0][0];
    const bool with_vals = vin != nullptr;  // keys only: the endpoint positions alone
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const uint32_t o = warp * (32 * ITEMS) + i * 32 + lane;
        if (tbase + o < m) {
            const uint32_t lp = (rank2[i / 2] >> (16 * (i & 1))) & 0xFFFFu;
            sm.skey[lp] = key[i];
            if (with_vals) dest[o] = uint16_t(lp);
        }
    }
    // 6) look-back per digit, late (this tile's ranking and staging gave the
    //    predecessors time to turn inclusive)
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
        const uint32_t d = threadIdx.x * DPT + j;
        if (d < radix && tile > 0) {
            // a window of LB predecessors per round (independent loads in flight):
            // while the tiles of a wave all look back at once, an inclusive
            // prefix propagates LB tiles per round instead of one
            constexpr int LB = 16;
            uint64_t ex = 0;
            bool done = false;
            for (int64_t p0 = int64_t(tile) - 1; !done; p0 -= LB) {
                W w[LB];
#pragma unroll
                for (int u = 0; u < LB; ++u)
                    w[u] = p0 - u >= 0 ? ld_vol(status + uint64_t(p0 - u) * kMaxRadix + d) : W(0);
#pragma unroll
                for (int u = 0; u < LB; ++u) {
                    if (done) break;
                    if (p0 - u < 0) {
                        done = true;
                        break;
                    }
                    while (D::state(w[u]) == 0u) {
                        __nanosleep(32);
                        w[u] = ld_vol(status + uint64_t(p0 - u) * kMaxRadix + d);
                    }
                    ex += D::value(w[u]);
                    if (D::state(w[u]) == 2u) done = true;
                }
            }
            st_vol(st + d, D::pack(2u, ex + sm.thist[d]));
            sm.gbase[d] += uint32_t(ex);
        }
    }
    __syncthreads();
    if (with_vals) {
        constexpr int U = 4;
        for (uint32_t o0 = threadIdx.x; o0 < uint32_t(TILE); o0 += U * NT) {
            uint32_t v[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t o = o0 + u * NT;
                v[u] = (o < uint32_t(TILE) && tbase + o < m) ? __ldcs(vin + tbase + o) : 0u;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const uint32_t o = o0 + u * NT;
                if (o < uint32_t(TILE) && tbase + o < m) sm.sval[dest[o]] = v[u];
            }
        }
    }
    __syncthreads();
    const uint32_t ttot = uint32_t(m - tbase < uint64_t(TILE) ? m - tbase : uint64_t(TILE));
    for (uint32_t s = threadIdx.x; s < ttot; s += NT) {
        const uint32_t k = sm.skey[s];
        const uint32_t d = (k >> shift) & dmask;
        const uint32_t out = sm.gbase[d] + (s - sm.texcl[d]);
        kout[out] = k;
        if (with_vals) vout[out] = sm.sval[s];
    }
}

template <int NT, int ITEMS, int WB, class W>
void launch_pass(uint64_t tiles, const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                 uint64_t m, int shift, int width, const unsigned long long* gh, W* status,
                 uint32_t* ticket, cudaStream_t s) {
    const size_t sm = sizeof(PassSmem<NT, ITEMS>);
    static bool attr[64] = {};  // the attribute belongs to the function in each device's context
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr[dev & 63]) {
        cudaFuncSetAttribute(k_rs_pass<NT, ITEMS, WB, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
        attr[dev & 63] = true;
    }
    brmq::launch_k(k_rs_pass<NT, ITEMS, WB, W>, dim3(unsigned(tiles)), dim3(NT), sm, s, kin, vin, kout, vout,
                   m, shift, width, gh, status, ticket);
}

template <int NT, int ITEMS, class W>
void launch_pass_w(uint64_t tiles, const uint32_t* kin, const uint32_t* vin, uint32_t* kout, uint32_t* vout,
                   uint64_t m, int shift, int width, const unsigned long long* gh, W* status,
                   uint32_t* ticket, cudaStream_t s) {
    switch (width) {
        case 10: return launch_pass<NT, ITEMS, 10, W>(tiles, kin, vin, kout, vout, m, shift, width, gh, status, ticket, s);
        case 9: return launch_pass<NT, ITEMS, 9, W>(tiles, kin, vin, kout, vout, m, shift, width, gh, status, ticket, s);
        case 8: return launch_pass<NT, ITEMS, 8, W>(tiles, kin, vin, kout, vout, m, shift, width, gh, status, ticket, s);
        default: return launch_pass<NT, ITEMS, 0, W>(tiles, kin, vin, kout, vout, m, shift, width, gh, status, ticket, s);
    }
}

// MSD partition pass: tile of NT x ITEMS keys; the rank of a key inside its
// digit comes from a shared atomic on the tile's digit counter (the bucket
// order is all the next level needs, so no stable ranking), the tile's run of
// each digit is reserved with one global atomic on the digit's counter past the
// digit's start (the exclusive prefix of the collect-time histogram) -- no
// look-back chain -- and the tile is staged sorted by digit and written in runs.
#ifndef BRMQ_PART_NT
#define BRMQ_PART_NT 512
#endif
#ifndef BRMQ_PART_ITEMS
#define BRMQ_PART_ITEMS 16
#endif
#ifndef BRMQ_PART_MINB
#define BRMQ_PART_MINB 1
#endif
constexpr int kNtPart = BRMQ_PART_NT, kItemsPart = BRMQ_PART_ITEMS;
template <int NT, int ITEMS>
__global__ void __launch_bounds__(NT, (NT == kNtPart ? BRMQ_PART_MINB : 1)) k_msd_partition(const uint32_t* __restrict__ kin,
                                                      uint32_t* __restrict__ kout, uint64_t m, int shift,
                                                      uint32_t dmask,
                                                      const unsigned long long* __restrict__ ghist,
                                                      uint32_t* __restrict__ gcnt,
                                                      uint32_t* __restrict__ bstart) {
    brmq::pdl_wait();
    constexpr int NW = NT / 32, TILE = NT * ITEMS, DPT = kMaxRadix / NT;
    static_assert(TILE <= 65536, "16-bit ranks");
    __shared__ uint32_t th[kMaxRadix], texcl[kMaxRadix], base[kMaxRadix];
    __shared__ uint32_t scan[NW + 1];
    __shared__ uint32_t skey[TILE];
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    for (int i = threadIdx.x; i < kMaxRadix; i += NT) th[i] = 0u;
    __syncthreads();
    const uint64_t tbase = uint64_t(blockIdx.x) * TILE;
    const uint64_t wbase = tbase + uint64_t(warp) * (32 * ITEMS);
    uint32_t key[ITEMS];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const uint64_t idx = wbase + uint64_t(i) * 32 + lane;
        key[i] = idx < m ? __ldcs(kin + idx) : 0u;
    }
    uint32_t rk2[(ITEMS + 1) / 2];
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        const bool ok = wbase + uint64_t(i) * 32 + lane < m;
        const uint32_t r = ok ? atomicAdd(&th[(key[i] >> shift) & dmask], 1u) : 0u;
        rk2[i / 2] = (i & 1) ? (rk2[i / 2] | (r << 16)) : r;
    }
    __syncthreads();
    // reservations first: their latency overlaps the two block scans
    uint32_t tsum = 0, gsum = 0, c[DPT], got[DPT], gh[DPT];
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
        const uint32_t d = threadIdx.x * DPT + j;
        c[j] = th[d];
        got[j] = c[j] ? atomicAdd(gcnt + d, c[j]) : 0u;
        gh[j] = d <= dmask ? uint32_t(ghist[d]) : 0u;
        tsum += c[j];
        gsum += gh[j];
    }
    uint32_t tot;
    uint32_t run = block_excl_sum<NT>(tsum, scan, tot);
    uint32_t grun = block_excl_sum<NT>(gsum, scan, tot);
#pragma unroll
    for (int j = 0; j < DPT; ++j) {
        const uint32_t d = threadIdx.x * DPT + j;
        texcl[d] = run;
        if (c[j]) base[d] = grun + got[j];
        if (blockIdx.x == 0) bstart[d] = grun;  // the buckets' starts, for k_bucket_mark
        run += c[j];
        grun += gh[j];
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
        if (wbase + uint64_t(i) * 32 + lane < m) {
            const uint32_t d = (key[i] >> shift) & dmask;
            skey[texcl[d] + ((rk2[i / 2] >> (16 * (i & 1))) & 0xFFFFu)] = key[i];
        }
    }
    __syncthreads();
    const uint32_t ttot = uint32_t(m - tbase < uint64_t(TILE) ? m - tbase : uint64_t(TILE));
    for (uint32_t s = threadIdx.x; s < ttot; s += NT) {
        const uint32_t k = skey[s];
        const uint32_t d = (k >> shift) & dmask;
        kout[base[d] + (s - texcl[d])] = k;
    }
}

// MSD partition + per-bucket marking (launch_radix_partition_mark): bucket b of
// the top-digit partition holds exactly the keys in [b << L, (b + 1) << L); its
// CTA sorts and dedups them by one counting digit of L bits -- a presence bitmap
// of 2^L bits in shared memory, set by shared atomics -- and writes the bucket's
// nonzero bitmap words (the global bitmap is all-zero on entry: the contraction
// clears every word it consumes); err bit 2 for positions >= n.
#ifndef BRMQ_MARK_U
#define BRMQ_MARK_U 8
#endif
template <int NT>
__global__ void __launch_bounds__(NT) k_bucket_mark(
    const uint32_t* __restrict__ keys, uint64_t n, int L, const unsigned long long* __restrict__ ghist,
    const uint32_t* __restrict__ bstart, uint32_t* __restrict__ bitmap, uint64_t bitmap_words,
    uint32_t* __restrict__ err) {
    brmq::pdl_wait();
    constexpr int kMarkThreads = NT;
    extern __shared__ __align__(16) uint32_t bm[];
    const uint32_t b = blockIdx.x;
    const uint64_t cnt = ghist[b];
    if (cnt == 0) return;  // nothing to mark: the bucket's words stay zero
    const uint32_t nw = 1u << (L - 5);  // bitmap words of the bucket (L >= 7)
    for (uint32_t w = threadIdx.x * 4; w < nw; w += kMarkThreads * 4)
        *reinterpret_cast<uint4*>(bm + w) = make_uint4(0, 0, 0, 0);
    __syncthreads();
    const uint64_t start = bstart[b], lo = uint64_t(b) << L;
    uint32_t bad = 0;
    constexpr int U = BRMQ_MARK_U;
    for (uint64_t i0 = threadIdx.x; i0 < cnt; i0 += U * kMarkThreads) {
        uint32_t x[U];
#pragma unroll
        for (int u = 0; u < U; ++u) x[u] = i0 + u * kMarkThreads < cnt ? __ldcs(keys + start + i0 + u * kMarkThreads) : 0xFFFFFFFFu;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (i0 + u * kMarkThreads >= cnt) break;
            if (x[u] >= n) {
                bad = 2u;
                continue;
            }
            const uint32_t r = uint32_t(x[u] - lo);
            atomicOr(bm + (r >> 5), 1u << (r & 31));
        }
    }
    if (bad) atomicOr(err, bad);
    __syncthreads();
    const uint64_t w0 = lo >> 5;
    for (uint32_t w = threadIdx.x * 4; w < nw; w += kMarkThreads * 4) {
        const uint4 v = *reinterpret_cast<const uint4*>(bm + w);
        if ((v.x | v.y | v.z | v.w) == 0u) continue;
        if (w0 + w + 4 <= bitmap_words) {
            *reinterpret_cast<uint4*>(bitmap + w0 + w) = v;
        } else {
            const uint32_t e[4] = {v.x, v.y, v.z, v.w};
            for (int j = 0; j < 4; ++j)
                if (w0 + w + j < bitmap_words && e[j]) bitmap[w0 + w + j] = e[j];
        }
    }
}

}  // namespace

bool radix_partition_shape(int bits, uint64_t m, uint64_t bitmap_words, int* D, int* L) {
    // small batches keep the LSD passes (c1, m = 2e3: 0.022 vs 0.028 ms)
    if (bits < 8 || bits > 30 || m < (1u << 14) || m >= (uint64_t(1) << 32) || (bitmap_words & 3u)) return false;
    *D = bits - 7 < kMaxBits ? bits - 7 : kMaxBits;
    *L = bits - *D;
    return *L <= 20;
}

unsigned long long* radix_partition_hist(void* tmp) { return static_cast<unsigned long long*>(tmp); }

// The partitioned keys land in alt_keys; the top-digit histogram is in tmp[0..),
// the reservation counters (zeroed with it) at tmp + 8 KB, the buckets' starts
// at tmp + 12 KB.
int launch_radix_partition_mark(const uint32_t* keys, uint32_t* alt_keys, uint64_t m, int bits, uint64_t n,
                                void* tmp, uint32_t* bitmap, uint64_t bitmap_words, uint32_t* err,
                                cudaStream_t stream) {
    int D = 0, L = 0;
    if (!radix_partition_shape(bits, m, bitmap_words, &D, &L)) return -1;
    const auto* ghist = static_cast<const unsigned long long*>(tmp);
    auto* gcnt = reinterpret_cast<uint32_t*>(static_cast<char*>(tmp) + kMaxRadix * 8);
    auto* bstart = gcnt + kMaxRadix;
    if (m <= kSmallM) {
        constexpr int T = kNtSmall * kItemsSmall;
        brmq::launch_k(k_msd_partition<kNtSmall, kItemsSmall>, dim3(unsigned((m + T - 1) / T)), dim3(kNtSmall), 0,
                       stream, keys, alt_keys, m, L, (1u << D) - 1u, ghist, gcnt, bstart);
    } else {
        constexpr int T = kNtPart * kItemsPart;
        brmq::launch_k(k_msd_partition<kNtPart, kItemsPart>, dim3(unsigned((m + T - 1) / T)), dim3(kNtPart), 0,
                       stream, keys, alt_keys, m, L, (1u << D) - 1u, ghist, gcnt, bstart);
    }
    // 1024 threads for the largest buckets (L >= 18: 32 KB+ of bitmap, 1 CTA per
    // SM at L = 20), 512 below (c3-con: 0.120 -> 0.108 ms partition + marks)
    const size_t smem = size_t(1u << (L - 5)) * 4;
    static bool attr[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr[dev & 63]) {
        cudaFuncSetAttribute(k_bucket_mark<1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
        cudaFuncSetAttribute(k_bucket_mark<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 128 * 1024);
        attr[dev & 63] = true;
    }
    if (L >= 18)
        brmq::launch_k(k_bucket_mark<1024>, dim3(1u << D), dim3(1024), smem, stream, alt_keys, n, L, ghist, bstart,
                       bitmap, bitmap_words, err);
    else
        brmq::launch_k(k_bucket_mark<512>, dim3(1u << D), dim3(512), smem, stream, alt_keys, n, L, ghist, bstart,
                       bitmap, bitmap_words, err);
    return 2;
}

// [ghist: 4 x 1024 u64][tickets: 4 u32 padded to 256 B], zeroed by every sort
size_t radix_sort_temp_bytes(uint64_t, int) { return size_t(kMaxPasses * kMaxRadix * 8) + 256; }

// 64-bit words of look-back descriptors (32-bit descriptors while m < 2^30,
// packed two per word)
size_t radix_sort_status_words(uint64_t m, int bits) {
    const Plan pl = plan_for(bits);
    const uint64_t tile = tile_for(m);
    const size_t d = size_t(pl.passes) * ((m + tile - 1) / tile) * kMaxRadix;
    return m < (uint64_t(1) << 30) ? (d + 1) / 2 : d;
}

int radix_sort_passes(int bits) { return plan_for(bits).passes; }

int launch_radix_sort(uint32_t* keys, uint32_t* vals, uint32_t* alt_keys, uint32_t* alt_vals,
                      uint64_t m, int bits, void* tmp, uint64_t* status, cudaStream_t stream,
                      bool* result_in_alt, const uint32_t* /*epoch_dev*/, uint32_t /*epoch_off*/) {
    *result_in_alt = false;
    if (m <= 1 || bits <= 0) return 0;
    const Plan pl = plan_for(bits);
    const uint64_t tile = tile_for(m);
    const uint64_t tiles = (m + tile - 1) / tile;
    auto* ghist = static_cast<unsigned long long*>(tmp);
    auto* tickets = reinterpret_cast<uint32_t*>(static_cast<char*>(tmp) + kMaxPasses * kMaxRadix * 8);
    cudaMemsetAsync(tmp, 0, radix_sort_temp_bytes(m, bits), stream);
    pdl_break();  // a memset node precedes the histogram: plain launch
    int launches = 0;
    {
        HistArgs ha{};
        ha.passes = pl.passes;
        for (int p = 0; p < pl.passes; ++p) {
            ha.width[p] = pl.width[p];
            ha.shift[p] = pl.shift[p];
        }
        uint64_t blocks = (m + 256 * 16 - 1) / (256 * 16);
        if (blocks > 148 * 4) blocks = 148 * 4;
        brmq::launch_k(k_rs_hist, dim3(unsigned(blocks)), dim3(256), 0, stream, keys, m, ha, ghist);
        ++launches;
    }
    // the descriptors start zeroed (state "not ready"): one memset per sort
    const bool narrow = m < (uint64_t(1) << 30);
    cudaMemsetAsync(status, 0, radix_sort_status_words(m, bits) * 8, stream);
    pdl_break();
    const uint32_t* kin = keys;
    const uint32_t* vin = vals;
    uint32_t* kout = alt_keys;
    uint32_t* vout = alt_vals;
    for (int p = 0; p < pl.passes; ++p) {
        const uint64_t off = uint64_t(p) * tiles * kMaxRadix;
        uint32_t* st32 = reinterpret_cast<uint32_t*>(status) + off;
        uint64_t* st64 = status + off;
        const unsigned long long* gh = ghist + p * kMaxRadix;
        if (m <= kSmallM) {
            if (narrow) launch_pass_w<kNtSmall, kItemsSmall>(tiles, kin, vin, kout, vout, m, pl.shift[p], pl.width[p], gh, st32, tickets + p, stream);
            else launch_pass_w<kNtSmall, kItemsSmall>(tiles, kin, vin, kout, vout, m, pl.shift[p], pl.width[p], gh, st64, tickets + p, stream);
        } else {
            if (narrow) launch_pass_w<kNtLarge, kItemsLarge>(tiles, kin, vin, kout, vout, m, pl.shift[p], pl.width[p], gh, st32, tickets + p, stream);
            else launch_pass_w<kNtLarge, kItemsLarge>(tiles, kin, vin, kout, vout, m, pl.shift[p], pl.width[p], gh, st64, tickets + p, stream);
        }
        ++launches;
        const uint32_t* tk = kin;
        const uint32_t* tv = vin;
        kin = kout;
        vin = vout;
        kout = const_cast<uint32_t*>(tk);
        vout = const_cast<uint32_t*>(tv);
    }
    *result_in_alt = (pl.passes & 1) != 0;
    return launches;
}

}  // namespace brmq
