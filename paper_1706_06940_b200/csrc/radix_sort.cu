// radix_sort.cu -- on-device LSD radix sort of (pos, origin) endpoint pairs.
//
// Replaces radix_sort_by_pos (contraction.cpp:27-63): LSD by 8-bit digits of
// the 32-bit position, one up-front histogram for every digit (:35-41),
// stable scatter per pass (:58).  Stability makes the output order identical
// to the reference's for equal positions (collect order).
//
// B200 design (single-pass "onesweep" scheme):
//   k_rs_hist : one read of the keys builds the histograms of all passes.
//   k_rs_pass : per pass ONE kernel.  A CTA takes a 4096-key tile (atomic
//               ticket => tiles start in order), ranks keys stably inside the
//               warp with __match_any_sync, turns per-warp digit counts into
//               tile offsets, publishes its 256 digit counts, looks back over
//               the predecessors' epoch-tagged counts (decoupled look-back,
//               one thread per digit) and scatters.  No separate scan kernel,
//               no global barrier, no status clearing between launches.
// Only ceil(bits/8) passes run, with bits = bit_width(n-1) chosen by the
// caller (positions < n), e.g. 27 bits -> 4 passes, the last one 3 bits wide.
#include "common.cuh"
#include "kernels.h"
#include "scan.cuh"

namespace brmq {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kItemsLarge = 16;  // 4096-key tiles for large batches
constexpr int kItemsSmall = 8;   // 2048-key tiles: shorter per-tile latency for small batches (measured vs 1024, 4096)
constexpr uint64_t kSmallM = 1u << 18;
inline int items_for(uint64_t m) { return m <= kSmallM ? kItemsSmall : kItemsLarge; }
constexpr int kRadix = 256;
constexpr int kMaxPasses = 4;

__global__ void __launch_bounds__(kThreads) k_rs_hist(const uint32_t* __restrict__ keys, uint64_t m,
                                                      int passes,
                                                      unsigned long long* __restrict__ ghist) {
    __shared__ uint32_t h[kMaxPasses][kRadix];
    for (int i = threadIdx.x; i < kMaxPasses * kRadix; i += kThreads) (&h[0][0])[i] = 0;
    __syncthreads();
    const uint64_t stride = uint64_t(gridDim.x) * kThreads;
    for (uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i < m; i += stride) {
        const uint32_t k = __ldg(keys + i);
        for (int p = 0; p < passes; ++p) atomicAdd(&h[p][(k >> (8 * p)) & 0xFF], 1u);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < passes * kRadix; i += kThreads) {
        const uint32_t c = (&h[0][0])[i];
        if (c) atomicAdd(ghist + i, (unsigned long long)c);
    }
}

template <int kItems>
__global__ void __launch_bounds__(kThreads) k_rs_pass(const uint32_t* __restrict__ kin,
                                                      const uint32_t* __restrict__ vin,
                                                      uint32_t* __restrict__ kout,
                                                      uint32_t* __restrict__ vout, uint64_t m,
                                                      int shift,
                                                      const unsigned long long* __restrict__ ghist,
                                                      uint64_t* __restrict__ status,
                                                      uint32_t* __restrict__ ticket,
                                                      const uint32_t* __restrict__ epoch_dev,
                                                      uint32_t epoch_off) {
    const uint32_t epoch = *epoch_dev + epoch_off;
    constexpr int kTile = kThreads * kItems;
    __shared__ uint32_t s_tile;
    __shared__ uint32_t whist[kWarps][kRadix];
    __shared__ uint32_t thist[kRadix];
    __shared__ uint32_t texcl[kRadix];
    __shared__ unsigned long long s_base[kRadix];
    __shared__ uint32_t s_scan[kWarps + 1];
    __shared__ uint32_t skey[kTile], sval[kTile];  // the tile, locally sorted by digit
    const unsigned lane = lane_id(), warp = threadIdx.x >> 5;
    const uint32_t d = threadIdx.x;  // the digit this thread publishes / looks back for

    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    for (int i = threadIdx.x; i < kWarps * kRadix; i += kThreads) (&whist[0][0])[i] = 0;
    thist[d] = 0;
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t base = tile * kTile + uint64_t(warp) * (32 * kItems);

    uint32_t key[kItems], val[kItems], dig[kItems], rank[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const uint64_t idx = base + uint64_t(i) * 32 + lane;
        const bool ok = idx < m;
        key[i] = ok ? __ldg(kin + idx) : 0u;
        val[i] = ok ? __ldg(vin + idx) : 0u;
        dig[i] = ok ? ((key[i] >> shift) & 0xFFu) : 0x100u;  // 0x100 = no key
    }
    // 1) tile digit histogram, published at once so successors never wait on
    //    this tile's ranking work (decoupled look-back)
#pragma unroll
    for (int i = 0; i < kItems; ++i)
        if (dig[i] < 0x100u) atomicAdd(&thist[dig[i]], 1u);
    __syncthreads();
    const uint32_t tcount = thist[d];
    uint64_t* st = status + tile * kRadix;
    st_relaxed_u64(st + d, status_pack(epoch, tile == 0 ? kStInclusive : kStAggregate, false, tcount));

    // 2) stable warp-level ranking: item-major, lane-minor == input order
    const unsigned lt = (1u << lane) - 1u;
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        const unsigned peers = __match_any_sync(kFull, dig[i]);
        const uint32_t before = __popc(peers & lt);
        uint32_t prev = 0;
        if (dig[i] < 0x100u) prev = whist[warp][dig[i]];
        __syncwarp();
        rank[i] = prev + before;
        if (dig[i] < 0x100u && lane == unsigned(__ffs(peers) - 1))
            whist[warp][dig[i]] = prev + __popc(peers);
        __syncwarp();
    }
    __syncthreads();

    // 3) per digit: warp offsets, global digit base, look-back over tiles
    uint32_t sum = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
        const uint32_t c = whist[w][d];
        whist[w][d] = sum;
        sum += c;
    }
    uint32_t gtot, ttot;
    const uint32_t gex = block_excl_sum<kThreads>(uint32_t(ghist[d]), s_scan, gtot);
    texcl[d] = block_excl_sum<kThreads>(tcount, s_scan, ttot);
    // look-back for digit d, 8 predecessors per round (independent loads in flight)
    uint64_t excl = 0;
    if (tile > 0) {
        int64_t p = int64_t(tile) - 1;
        bool done = false;
        while (!done) {
            uint64_t w[8];
#pragma unroll
            for (int u = 0; u < 8; ++u)
                w[u] = p - u >= 0 ? ld_relaxed_u64(status + uint64_t(p - u) * kRadix + d) : 0;
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                if (done) break;
                if (p - u < 0) { done = true; break; }
                while (status_state(w[u], epoch) == kStInvalid)
                    w[u] = ld_relaxed_u64(status + uint64_t(p - u) * kRadix + d);
                excl += status_value(w[u]);
                if (status_state(w[u], epoch) == kStInclusive) done = true;
            }
            p -= 8;
        }
        st_relaxed_u64(st + d, status_pack(epoch, kStInclusive, false, excl + tcount));
    }
    s_base[d] = (unsigned long long)gex + excl;
    __syncthreads();

    // 4) stage the tile in shared memory sorted by digit (stable), then write
    //    out so that consecutive threads hit consecutive addresses of a bucket
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
        if (dig[i] < 0x100u) {
            const uint32_t lp = texcl[dig[i]] + whist[warp][dig[i]] + rank[i];
            skey[lp] = key[i];
            sval[lp] = val[i];
        }
    }
    __syncthreads();
    for (uint32_t s = threadIdx.x; s < ttot; s += kThreads) {
        const uint32_t k = skey[s];
        const uint32_t dd = (k >> shift) & 0xFFu;
        const uint64_t out = s_base[dd] + (s - texcl[dd]);
        kout[out] = k;
        vout[out] = sval[s];
    }
}

}  // namespace

// [ghist: 4*256 u64][tickets: 4 u32 padded to 256 B], zeroed by every sort
size_t radix_sort_temp_bytes(uint64_t, int) { return size_t(kMaxPasses * kRadix * 8) + 256; }

size_t radix_sort_status_words(uint64_t m, int bits) {
    const int passes = bits <= 0 ? 0 : (bits + 7) / 8;
    const uint64_t tile = uint64_t(kThreads) * items_for(m);
    return size_t(passes) * ((m + tile - 1) / tile) * kRadix;
}

int radix_sort_passes(int bits) { return bits <= 0 ? 0 : (bits + 7) / 8; }

int launch_radix_sort(uint32_t* keys, uint32_t* vals, uint32_t* alt_keys, uint32_t* alt_vals,
                      uint64_t m, int bits, void* tmp, uint64_t* status, cudaStream_t stream,
                      bool* result_in_alt, const uint32_t* epoch_dev, uint32_t epoch_off) {
    *result_in_alt = false;
    if (m <= 1 || bits <= 0) return 0;
    const int passes = (bits + 7) / 8;
    const int items = items_for(m);
    const uint64_t tiles = (m + uint64_t(kThreads) * items - 1) / (uint64_t(kThreads) * items);
    auto* ghist = static_cast<unsigned long long*>(tmp);
    auto* tickets = reinterpret_cast<uint32_t*>(static_cast<char*>(tmp) + kMaxPasses * kRadix * 8);
    cudaMemsetAsync(tmp, 0, radix_sort_temp_bytes(m, bits), stream);
    int launches = 0;
    {
        uint64_t blocks = (m + kThreads * 8 - 1) / (kThreads * 8);
        if (blocks > 148 * 8) blocks = 148 * 8;
        k_rs_hist<<<unsigned(blocks), kThreads, 0, stream>>>(keys, m, passes, ghist);
        ++launches;
    }
    const uint32_t* kin = keys;
    const uint32_t* vin = vals;
    uint32_t* kout = alt_keys;
    uint32_t* vout = alt_vals;
    for (int p = 0; p < passes; ++p) {
        auto kern = items == kItemsSmall ? k_rs_pass<kItemsSmall> : k_rs_pass<kItemsLarge>;
        kern<<<unsigned(tiles), kThreads, 0, stream>>>(kin, vin, kout, vout, m, 8 * p,
                                                            ghist + p * kRadix,
                                                            status + uint64_t(p) * tiles * kRadix,
                                                            tickets + p, epoch_dev, epoch_off + uint32_t(p));
        ++launches;
        const uint32_t* tk = kin;
        const uint32_t* tv = vin;
        kin = kout;
        vin = vout;
        kout = const_cast<uint32_t*>(tk);
        vout = const_cast<uint32_t*>(tv);
    }
    *result_in_alt = (passes & 1) != 0;
    return launches;
}

}  // namespace brmq
