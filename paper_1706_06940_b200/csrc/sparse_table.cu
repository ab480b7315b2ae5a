// sparse_table.cu -- levels 1..L-1 of the block Sparse Table (K2).
//
// Recurrence (element_sparse_table.cpp:20-31): cell (e, j) =
// min(cell(e-1, j), cell(e-1, j + 2^(e-1))), valid where j + 2^e <= b.  On
// packed keys the unsigned min is the leftmost-on-ties arg-smaller.
//
// B200 design: instead of one launch per level (18-22 launches, each a full
// L2 round trip), several levels are produced per launch from shared memory.
// Columns that interact at levels base+1..base+D from level `base` are those
// congruent modulo s = 2^base, so a CTA owns R residues x T consecutive
// "t" positions (column = r + s*t) plus a halo of 2^D - 1 t-positions,
// doubles D times in shared memory (ping-pong buffers, one barrier per level)
// and writes each finished level straight to its row.  base = 0 uses R = 1
// (plain contiguous columns, D <= 10); higher bases use R = 8 residues so
// every global access is a 64-byte contiguous run.  b = 2M (n = 2^30,
// k = 512, 22 levels) needs 3 launches instead of 21.
#include "common.cuh"
#include "kernels.h"

namespace brmq {
namespace {

constexpr int kThreads = 256;

template <int R>
__global__ void __launch_bounds__(kThreads) k_st_tile(uint64_t* __restrict__ ST, uint64_t b_max,
                                                      const uint64_t* __restrict__ b_dev,
                                                      uint32_t base, uint32_t D, uint32_t T,
                                                      uint64_t groups) {
    extern __shared__ uint64_t smem[];
    const uint64_t b = b_dev ? *b_dev : b_max;
    const uint64_t s = 1ull << base;
    const uint32_t H = (1u << D) - 1;
    const uint32_t W = T + H;
    const uint64_t g = blockIdx.x % groups;         // residue group
    const uint64_t tt = blockIdx.x / groups;        // t tile
    const uint64_t r0 = g * R;
    const uint64_t t0 = tt * T;
    if (b < s || r0 + s * t0 + s > b) return;       // no valid level-`base` cell in this tile
    uint64_t* buf0 = smem;
    uint64_t* buf1 = smem + size_t(W) * R;
    const uint64_t* row_in = ST + uint64_t(base) * b_max;
    const uint64_t last_valid = b - s;              // level-base cell c valid iff c <= b - 2^base
    for (uint32_t idx = threadIdx.x; idx < W * R; idx += kThreads) {
        const uint32_t rl = idx % R, tl = idx / R;
        const uint64_t c = r0 + rl + s * (t0 + tl);
        buf0[idx] = c <= last_valid ? row_in[c] : kNoKey;
    }
    __syncthreads();
    uint64_t* cur = buf0;
    uint64_t* nxt = buf1;
    for (uint32_t d = 1; d <= D; ++d) {
        const uint32_t half = 1u << (d - 1);
        const uint32_t live = W - half;             // t positions with both operands in window
        const uint32_t lvl = base + d;
        const uint64_t span = 1ull << lvl;
        uint64_t* row_out = ST + uint64_t(lvl) * b_max;
        for (uint32_t idx = threadIdx.x; idx < live * R; idx += kThreads) {
            const uint64_t v = kmin(cur[idx], cur[idx + half * R]);
            nxt[idx] = v;
            const uint32_t rl = idx % R, tl = idx / R;
            if (tl < T) {
                const uint64_t c = r0 + rl + s * (t0 + tl);
                if (c + span <= b) row_out[c] = v;
            }
        }
        __syncthreads();
        uint64_t* t = cur;
        cur = nxt;
        nxt = t;
    }
}

}  // namespace

int launch_sparse_table(uint64_t* ST, uint64_t b, const uint64_t* b_dev, cudaStream_t stream) {
    if (b < 2) return 0;
    const uint32_t L = floor_log2_u64(b) + 1;
    int launches = 0;
    uint32_t base = 0;
    while (base < L - 1) {
        if (base == 0) {
            const uint32_t D = (L - 1) < 10 ? (L - 1) : 10;
            const uint32_t T = b >= 65536 ? 256 : 1024;  // >= 2-5 CTAs per SM on big tables
            const uint64_t tiles = (b + T - 1) / T;
            const size_t sm = size_t(2) * (T + (1u << D) - 1) * sizeof(uint64_t);
            cudaFuncSetAttribute(k_st_tile<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
            k_st_tile<1><<<unsigned(tiles), kThreads, sm, stream>>>(ST, b, b_dev, 0, D, T, 1);
            base = D;
        } else {
            const uint32_t D = (L - 1 - base) < 7 ? (L - 1 - base) : 7;
            const uint32_t T = 32;
            const uint64_t s = 1ull << base;
            const uint64_t groups = s / 8;  // base >= 10 here; 8 residues = 64-byte runs
            const uint64_t tcount = (b + s - 1) / s;
            const uint64_t tiles = (tcount + T - 1) / T;
            const size_t sm = size_t(2) * (T + (1u << D) - 1) * 8 * sizeof(uint64_t);
            cudaFuncSetAttribute(k_st_tile<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
            k_st_tile<8><<<unsigned(groups * tiles), kThreads, sm, stream>>>(ST, b, b_dev, base, D, T,
                                                                             groups);
            base += D;
        }
        ++launches;
    }
    return launches;
}

}  // namespace brmq
