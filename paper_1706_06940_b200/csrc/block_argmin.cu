// block_argmin.cu -- level 0 of the block Sparse Table (K1).
//
// SPEC.md:199-203 / :213 / :253: level-0 entry j is the leftmost-minimum
// position of block B_j = [j*k, min((j+1)*k, m)); the trailing partial block
// is clipped (no +inf padding).  PAPER.md:304-309 (BbST stage 1).
//
// B200 design: this is one streaming pass over A (4n bytes, HBM-bound).
// One warp owns one block: each lane issues 128-bit non-allocating loads
// (ld.global.nc.L1::no_allocate.v4), 4 vectors per lane in flight per round,
// keeps its leftmost minimum in registers, and the warp combines lanes with
// two redux.sync (value, then leftmost position) -- no shared memory, no
// block barrier.  Output is one packed key per block (8 B).
#include "common.cuh"
#include "kernels.h"

namespace brmq {
namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = 4;  // 16-byte vectors per lane in flight
constexpr int kKeysU = 8;   // A_Q keys pass: a k = 512 block (256 vectors) in one round trip

// k % 128 == 0, A 16-byte aligned: full blocks [0, nfull) with vector loads;
// the trailing partial block (blk == nfull < nblk) with lane-strided scalars.
__global__ void __launch_bounds__(kThreads) k_block_argmin_i32_vec(const int32_t* __restrict__ A,
                                                                   uint64_t n, uint64_t nfull,
                                                                   uint64_t nblk, uint32_t k,
                                                                   uint64_t* __restrict__ keys) {
    brmq::pdl_wait();
    const uint64_t blk = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    if (blk >= nblk) return;
    const unsigned lane = lane_id();
    if (blk >= nfull) {  // clipped trailing block
        const uint64_t lo = blk * k;
        uint64_t best = kNoKey;
        for (uint64_t i = lo + lane; i < n; i += 32) best = kmin(best, pack_key(__ldg(A + i), uint32_t(i)));
        best = warp_min_key(best);
        if (lane == 0) keys[blk] = best;
        return;
    }
    const uint32_t base_pos = uint32_t(blk * k);
    const int4* v4 = reinterpret_cast<const int4*>(A + uint64_t(base_pos));
    const uint32_t nvec = k >> 2;  // multiple of 32
    int32_t bv = 0x7FFFFFFF;
    uint32_t bp = 0xFFFFFFFFu;
    for (uint32_t v0 = 0; v0 < nvec; v0 += 32 * kUnroll) {
        int4 x[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            if (v0 + 32 * u < nvec) x[u] = ld_stream_v4(v4 + v0 + 32 * u + lane);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (v0 + 32 * u >= nvec) break;
            const uint32_t p = base_pos + 4 * (v0 + 32 * u + lane);
            // ascending positions + strict '<' => lane-local leftmost minimum;
            // the (bp == ~0) test seeds the first element even if it is INT32_MAX.
            if (x[u].x < bv || bp == 0xFFFFFFFFu) { bv = x[u].x; bp = p; }
            if (x[u].y < bv) { bv = x[u].y; bp = p + 1; }
            if (x[u].z < bv) { bv = x[u].z; bp = p + 2; }
            if (x[u].w < bv) { bv = x[u].w; bp = p + 3; }
        }
    }
    const uint64_t key = warp_min_key(pack_key(bv, bp));
    if (lane == 0) keys[blk] = key;
}

// Any k / alignment: warp per block, lane-strided coalesced scalar loads.
__global__ void __launch_bounds__(kThreads) k_block_argmin_i32_gen(const int32_t* __restrict__ A,
                                                                   uint64_t n, uint32_t k,
                                                                   uint64_t first, uint64_t nblk,
                                                                   uint64_t* __restrict__ keys) {
    brmq::pdl_wait();
    const uint64_t blk = first + ((uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5);
    if (blk >= nblk) return;
    const unsigned lane = lane_id();
    const uint64_t lo = blk * k;
    const uint64_t hi = lo + k < n ? lo + k : n;
    uint64_t best = kNoKey;
    for (uint64_t i = lo + lane; i < hi; i += 32) best = kmin(best, pack_key(__ldg(A + i), uint32_t(i)));
    best = warp_min_key(best);
    if (lane == 0) keys[blk] = best;
}

// Packed-key input (A_Q).  Device-side length: blocks past ceil(len/k) exit.
__global__ void __launch_bounds__(kThreads) k_block_argmin_keys(const uint64_t* __restrict__ K,
                                                                uint64_t len_max,
                                                                const uint64_t* __restrict__ len_dev,
                                                                uint32_t k,
                                                                uint64_t* __restrict__ keys,
                                                                uint64_t* __restrict__ b_dev) {
    brmq::pdl_wait();
    brmq::pdl_trigger();  // small grid: dependents may be scheduled now
    const uint64_t len = len_dev ? *len_dev : len_max;
    const uint64_t blk = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    if (b_dev && blockIdx.x == 0 && threadIdx.x == 0) *b_dev = (len + k - 1) / k;
    const uint64_t lo = blk * k;
    if (lo >= len) return;
    const unsigned lane = lane_id();
    const uint64_t hi = lo + k < len ? lo + k : len;
    uint64_t best = kNoKey;
    if ((k & 63u) == 0 && hi - lo == k && (reinterpret_cast<uintptr_t>(K) & 15u) == 0) {
        const uint4* v4 = reinterpret_cast<const uint4*>(K + lo);
        const uint32_t nvec = k >> 1;  // multiple of 32
        for (uint32_t v0 = 0; v0 < nvec; v0 += 32 * kUnroll) {
            uint4 x[kUnroll];
#pragma unroll
            for (int u = 0; u < kUnroll; ++u)
                if (v0 + 32 * u < nvec) x[u] = ld_stream_u4(v4 + v0 + 32 * u + lane);
#pragma unroll
            for (int u = 0; u < kUnroll; ++u) {
                if (v0 + 32 * u >= nvec) break;
                best = kmin(best, (uint64_t(x[u].y) << 32) | x[u].x);
                best = kmin(best, (uint64_t(x[u].w) << 32) | x[u].z);
            }
        }
    } else {
        for (uint64_t i = lo + lane; i < hi; i += 32) best = kmin(best, __ldg(K + i));
    }
    best = warp_min_key(best);
    if (lane == 0) keys[blk] = best;
}

// Small blocks (k < 32, the lower levels of a multi-level chain): one thread per
// block, its k cells read in order (a warp covers 32k contiguous cells, so every
// sector is fetched once through L1); ascending positions + strict '<' = leftmost.
__global__ void __launch_bounds__(kThreads) k_block_argmin_i32_small(const int32_t* __restrict__ A,
                                                                     uint64_t n, uint32_t k,
                                                                     uint64_t nblk,
                                                                     uint64_t* __restrict__ keys) {
    brmq::pdl_wait();
    const uint64_t blk = uint64_t(blockIdx.x) * kThreads + threadIdx.x;
    if (blk >= nblk) return;
    const uint64_t lo = blk * k, hi = lo + k < n ? lo + k : n;
    int32_t bv = __ldg(A + lo);
    uint64_t bp = lo;
    for (uint64_t i = lo + 1; i < hi; ++i) {
        const int32_t v = __ldg(A + i);
        if (v < bv) { bv = v; bp = i; }
    }
    keys[blk] = pack_key(bv, uint32_t(bp));
}

__global__ void __launch_bounds__(kThreads) k_block_argmin_keys_small(const uint64_t* __restrict__ K,
                                                                      uint64_t len, uint32_t k,
                                                                      uint64_t nblk,
                                                                      uint64_t* __restrict__ keys) {
    brmq::pdl_wait();
    const uint64_t blk = uint64_t(blockIdx.x) * kThreads + threadIdx.x;
    if (blk >= nblk) return;
    const uint64_t lo = blk * k, hi = lo + k < len ? lo + k : len;
    uint64_t best = kNoKey;
    for (uint64_t i = lo; i < hi; ++i) best = kmin(best, __ldg(K + i));
    keys[blk] = best;
}

// k = 4V, V in {1, 2, 4, 8, 16, 32} (k = 4 .. 128), A 16-byte aligned: one
// 128-bit vector per lane, V lanes per block, 4 rounds of 32 vectors per warp in
// flight; the lane-local leftmost minimum of its 4 cells is combined over the
// V-lane group with shuffles (lower lanes hold lower positions: kmin is leftmost).
template <int V>
__global__ void __launch_bounds__(kThreads) k_block_argmin_i32_grp(const int32_t* __restrict__ A,
                                                                   uint64_t nfull,
                                                                   uint64_t* __restrict__ keys) {
    brmq::pdl_wait();
    constexpr int kR = 4;
    const uint64_t warp = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    const unsigned lane = lane_id();
    const int4* A4 = reinterpret_cast<const int4*>(A);
    const uint64_t nvec = nfull * V;
    int4 x[kR];
#pragma unroll
    for (int u = 0; u < kR; ++u) {
        const uint64_t v = (warp * kR + u) * 32 + lane;
        if (v < nvec) x[u] = ld_stream_v4(A4 + v);
    }
#pragma unroll
    for (int u = 0; u < kR; ++u) {
        const uint64_t v = (warp * kR + u) * 32 + lane;
        if ((warp * kR + u) * 32 >= nvec) break;  // warp-uniform
        uint64_t key = kNoKey;
        if (v < nvec) {
            const uint32_t p = uint32_t(v * 4);
            int32_t bv = x[u].x;
            uint32_t bp = p;
            if (x[u].y < bv) { bv = x[u].y; bp = p + 1; }
            if (x[u].z < bv) { bv = x[u].z; bp = p + 2; }
            if (x[u].w < bv) { bv = x[u].w; bp = p + 3; }
            key = pack_key(bv, bp);
        }
        key = group_min_key<V>(key);
        if (v < nvec && lane % V == 0) keys[v / V] = key;
    }
}

inline unsigned grid_for_warps(uint64_t warps) {
    return unsigned((warps + kWarps - 1) / kWarps);
}

}  // namespace

// k = 1 (the element Sparse Table of the harness's "sparse" algorithm): keys only
__global__ void k_pack_keys(const int32_t* __restrict__ A, uint64_t n, uint64_t* __restrict__ keys) {
    brmq::pdl_wait();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < n) keys[i] = pack_key(__ldg(A + i), uint32_t(i));
}

int launch_block_argmin_i32(const int32_t* A, uint64_t n, uint32_t k, uint64_t* keys,
                            cudaStream_t stream) {
    const uint64_t nblk = (n + k - 1) / k;
    if (nblk == 0) return 0;
    if (k == 1) {
        brmq::launch_k(k_pack_keys, dim3(unsigned((n + 255) / 256)), dim3(256), 0, stream, A, n, keys);
        return 1;
    }
    const bool al = (reinterpret_cast<uintptr_t>(A) & 15u) == 0;
    if (al && k <= 128 && (k & (k - 1)) == 0 && k >= 4 && n / k > 0) {
        const uint64_t nfull = n / k;
        const unsigned grid = unsigned((nfull * (k / 4) + 32 * 4 * kWarps - 1) / (32 * 4 * kWarps));
        switch (k) {
            case 4: brmq::launch_k(k_block_argmin_i32_grp<1>, dim3(grid), dim3(kThreads), 0, stream, A, nfull, keys); break;
            case 8: brmq::launch_k(k_block_argmin_i32_grp<2>, dim3(grid), dim3(kThreads), 0, stream, A, nfull, keys); break;
            case 16: brmq::launch_k(k_block_argmin_i32_grp<4>, dim3(grid), dim3(kThreads), 0, stream, A, nfull, keys); break;
            case 32: brmq::launch_k(k_block_argmin_i32_grp<8>, dim3(grid), dim3(kThreads), 0, stream, A, nfull, keys); break;
            case 64: brmq::launch_k(k_block_argmin_i32_grp<16>, dim3(grid), dim3(kThreads), 0, stream, A, nfull, keys); break;
            default: brmq::launch_k(k_block_argmin_i32_grp<32>, dim3(grid), dim3(kThreads), 0, stream, A, nfull, keys); break;
        }
        if (nblk > nfull)  // the clipped trailing block
            brmq::launch_k(k_block_argmin_i32_gen, dim3(1), dim3(kThreads), 0, stream, A, n, k, nfull, nblk, keys);
        return nblk > nfull ? 2 : 1;
    }
    if (k < 32) {
        brmq::launch_k(k_block_argmin_i32_small, dim3(unsigned((nblk + kThreads - 1) / kThreads)), dim3(kThreads), 0, stream, A, n, k, nblk,
                                                                                                  keys);
    } else if ((k & 127u) == 0 && (reinterpret_cast<uintptr_t>(A) & 15u) == 0) {
        brmq::launch_k(k_block_argmin_i32_vec, dim3(grid_for_warps(nblk)), dim3(kThreads), 0, stream, A, n, n / k, nblk, k, keys);
    } else {
        brmq::launch_k(k_block_argmin_i32_gen, dim3(grid_for_warps(nblk)), dim3(kThreads), 0, stream, A, n, k, 0, nblk, keys);
    }
    return 1;
}

int launch_block_argmin_keys(const uint64_t* K, uint64_t len_max, const uint64_t* len_dev,
                             uint32_t k, uint64_t* keys, uint64_t* b_dev, cudaStream_t stream) {
    uint64_t nblk = (len_max + k - 1) / k;
    if (k < 32 && !len_dev && !b_dev) {  // host-known length (multi-level chains)
        if (nblk == 0) return 0;
        brmq::launch_k(k_block_argmin_keys_small, dim3(unsigned((nblk + kThreads - 1) / kThreads)), dim3(kThreads), 0, stream, 
            K, len_max, k, nblk, keys);
        return 1;
    }
    if (nblk == 0) nblk = 1;  // still publish *b_dev
    brmq::launch_k(k_block_argmin_keys, dim3(grid_for_warps(nblk)), dim3(kThreads), 0, stream, K, len_max, len_dev, k, keys,
                                                                       b_dev);
    return 1;
}

}  // namespace brmq

// ---------------------------------------------------------------------------
// Two-level block minima for multi-level BbST
// with k1 = 32: besides the k-block keys (level 0 of the Sparse Table) the same
// single pass over A stores the leftmost-min key of every 32-element sub-block
// (one 128-byte row), 8 B per 128 B read (+6% traffic).  Vector path: lane l of
// round u holds 16-byte vector 32u + l of the block, so the 8 lanes of a quarter
// warp cover one sub-block and reduce it with two masked redux.sync.
namespace brmq {
namespace {

__global__ void __launch_bounds__(kThreads) k_block_argmin_ml_vec(const int32_t* __restrict__ A,
                                                                  uint64_t n, uint64_t nfull,
                                                                  uint64_t nblk, uint32_t k,
                                                                  uint64_t* __restrict__ keys,
                                                                  uint64_t* __restrict__ sub) {
    brmq::pdl_wait();
    const uint64_t blk = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    if (blk >= nblk) return;
    const unsigned lane = lane_id();
    const uint64_t lo = blk * k;
    if (blk >= nfull) {  // clipped trailing block: sub-block by sub-block, scalar
        uint64_t best = kNoKey;
        for (uint64_t sb = lo; sb < n; sb += 32) {
            const uint64_t i = sb + lane;
            uint64_t kk = i < n ? pack_key(__ldg(A + i), uint32_t(i)) : kNoKey;
            kk = warp_min_key(kk);
            if (lane == 0) sub[sb >> 5] = kk;
            best = kmin(best, kk);
        }
        if (lane == 0) keys[blk] = best;
        return;
    }
    const int4* v4 = reinterpret_cast<const int4*>(A + lo);
    const uint32_t nvec = k >> 2;  // multiple of 32
    uint64_t best = kNoKey;
    for (uint32_t v0 = 0; v0 < nvec; v0 += 32 * kUnroll) {
        int4 x[kUnroll];
#pragma unroll
        for (int u = 0; u < kUnroll; ++u)
            if (v0 + 32 * u < nvec) x[u] = ld_stream_v4(v4 + v0 + 32 * u + lane);
#pragma unroll
        for (int u = 0; u < kUnroll; ++u) {
            if (v0 + 32 * u >= nvec) break;
            const uint32_t p = uint32_t(lo) + 4 * (v0 + 32 * u + lane);
            int32_t bv = x[u].x;
            uint32_t bp = p;
            if (x[u].y < bv) { bv = x[u].y; bp = p + 1; }
            if (x[u].z < bv) { bv = x[u].z; bp = p + 2; }
            if (x[u].w < bv) { bv = x[u].w; bp = p + 3; }
            const uint64_t sk = group_min_key<8>(pack_key(bv, bp));  // the quarter warp's sub-block
            if ((lane & 7u) == 0) sub[(lo >> 5) + ((v0 + 32 * u + lane) >> 3)] = sk;
            best = kmin(best, sk);
        }
    }
    best = warp_min_key(best);
    if (lane == 0) keys[blk] = best;
}

// any k (multiple of 32) / alignment: sub-block by sub-block with coalesced scalars
__global__ void __launch_bounds__(kThreads) k_block_argmin_ml_gen(const int32_t* __restrict__ A,
                                                                  uint64_t n, uint64_t nblk,
                                                                  uint32_t k,
                                                                  uint64_t* __restrict__ keys,
                                                                  uint64_t* __restrict__ sub) {
    brmq::pdl_wait();
    const uint64_t blk = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) >> 5;
    if (blk >= nblk) return;
    const unsigned lane = lane_id();
    const uint64_t lo = blk * k, hi = lo + k < n ? lo + k : n;
    uint64_t best = kNoKey;
    for (uint64_t sb = lo; sb < hi; sb += 32) {
        const uint64_t i = sb + lane;
        uint64_t kk = i < hi ? pack_key(__ldg(A + i), uint32_t(i)) : kNoKey;
        kk = warp_min_key(kk);
        if (lane == 0) sub[sb >> 5] = kk;
        best = kmin(best, kk);
    }
    if (lane == 0) keys[blk] = best;
}

// Two-level minima over packed keys (A_Q of BbST_CON, device-side length): the
// k-block keys and the 32-key sub-block keys in one pass.  k a multiple of 64,
// A_Q 16-byte aligned and padded to an even count: lane l of round u holds keys
// 2(32u + l) and 2(32u + l) + 1 of the block, so a half warp covers one
// sub-block.
__global__ void __launch_bounds__(kThreads) k_block_argmin_keys_ml(
    const uint64_t* __restrict__ K, const uint64_t* __restrict__ len_dev, uint64_t len_max,
    uint32_t k, uint64_t* __restrict__ keys, uint64_t* __restrict__ sub,
    uint64_t* __restrict__ b_dev) {
    brmq::pdl_wait();
    brmq::pdl_trigger();  // small grid: dependents may be scheduled now
    const uint64_t blk = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t lo = blk * k;
    const unsigned lane = lane_id();
    const uint4* v4 = reinterpret_cast<const uint4*>(K + lo);
    const uint32_t nvec = k >> 1;  // multiple of 32
    // the first round's loads go out before the true length (written by the
    // contraction) is read: within the allocation (len_max, padded to an even
    // count) they are harmless, and the length masks them below -- one dependent
    // round trip fewer per block
    uint4 x[kKeysU];
#pragma unroll
    for (int u = 0; u < kKeysU; ++u) {
        const uint64_t e = lo + 2 * uint64_t(32 * u + lane);
        x[u] = 32u * u < nvec && e < len_max ? ld_stream_u4(v4 + 32 * u + lane) : make_uint4(~0u, ~0u, ~0u, ~0u);
    }
    const uint64_t len = len_dev ? *len_dev : len_max;
    if (b_dev && blockIdx.x == 0 && threadIdx.x == 0) *b_dev = (len + k - 1) / k;
    if (lo >= len) return;
    uint64_t best = kNoKey;
    for (uint32_t v0 = 0; v0 < nvec; v0 += 32 * kKeysU) {
        if (v0) {
#pragma unroll
            for (int u = 0; u < kKeysU; ++u) {
                const uint64_t e = lo + 2 * uint64_t(v0 + 32 * u + lane);
                x[u] = v0 + 32 * u < nvec && e < len ? ld_stream_u4(v4 + v0 + 32 * u + lane)
                                                     : make_uint4(~0u, ~0u, ~0u, ~0u);
            }
        }
#pragma unroll
        for (int u = 0; u < kKeysU; ++u) {
            if (v0 + 32 * u >= nvec) break;
            const uint64_t e = lo + 2 * uint64_t(v0 + 32 * u + lane);
            uint64_t kk = e < len ? (uint64_t(x[u].y) << 32) | x[u].x : kNoKey;
            if (e + 1 < len) kk = kmin(kk, (uint64_t(x[u].w) << 32) | x[u].z);
            kk = group_min_key<16>(kk);  // the half warp's sub-block
            if ((lane & 15u) == 0 && e < len) sub[e >> 5] = kk;
            best = kmin(best, kk);
        }
    }
    best = warp_min_key(best);
    if (lane == 0) keys[blk] = best;
}

}  // namespace

int launch_block_argmin_ml(const int32_t* A, uint64_t n, uint32_t k, uint64_t* keys,
                           uint64_t* sub, cudaStream_t stream) {
    const uint64_t nblk = (n + k - 1) / k;
    if (nblk == 0) return 0;
    if ((k & 127u) == 0 && (reinterpret_cast<uintptr_t>(A) & 15u) == 0)
        brmq::launch_k(k_block_argmin_ml_vec, dim3(grid_for_warps(nblk)), dim3(kThreads), 0, stream, A, n, n / k, nblk, k, keys,
                                                                            sub);
    else
        brmq::launch_k(k_block_argmin_ml_gen, dim3(grid_for_warps(nblk)), dim3(kThreads), 0, stream, A, n, nblk, k, keys, sub);
    return 1;
}

int launch_block_argmin_keys_ml(const uint64_t* K, uint64_t len_max, const uint64_t* len_dev,
                                uint32_t k, uint64_t* keys, uint64_t* sub, uint64_t* b_dev,
                                cudaStream_t stream) {
    uint64_t nblk = (len_max + k - 1) / k;
    if (k < 32 && !len_dev && !b_dev) {  // host-known length (multi-level chains)
        if (nblk == 0) return 0;
        brmq::launch_k(k_block_argmin_keys_small, dim3(unsigned((nblk + kThreads - 1) / kThreads)), dim3(kThreads), 0, stream, 
            K, len_max, k, nblk, keys);
        return 1;
    }
    if (nblk == 0) nblk = 1;  // still publish *b_dev
    // few blocks (A_Q of a small batch): one warp per CTA spreads them over all SMs
    const unsigned nt = nblk <= uint64_t(148) * 32 ? 32u : unsigned(kThreads);
    brmq::launch_k(k_block_argmin_keys_ml, dim3(unsigned((nblk * 32 + nt - 1) / nt)), dim3(nt), 0, stream, K, len_dev, len_max,
                                                                                 k, keys, sub, b_dev);
    return 1;
}

}  // namespace brmq
