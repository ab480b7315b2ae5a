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
// (plain contiguous columns, D <= 10, T = 2048); higher bases use R = 16
// residues (128-byte runs, D <= 7, T = 128), and the last launch of a large
// table, which has at most 32 t-positions, trades them for 32 or 64 residues.  The loops are split so that the
// store predicate is a single 32-bit compare against a per-level limit.
// b = 2M (n = 2^30, k = 512, 22 levels) needs 3 launches instead of 21.
#include "common.cuh"
#include "kernels.h"

namespace brmq {
namespace {

template <int R, int T, int NT>
__global__ void __launch_bounds__(NT) k_st_tile(uint64_t* __restrict__ ST, uint64_t b_max,
                                                const uint64_t* __restrict__ b_dev, uint32_t base,
                                                uint32_t D, uint32_t groups) {
    brmq::pdl_wait();
    brmq::pdl_trigger();  // small grid: dependents may be scheduled now
    extern __shared__ uint64_t smem[];
    const uint64_t s = 1ull << base;
    const uint32_t W = T + (1u << D) - 1;
    const uint32_t g = blockIdx.x % groups;  // residue group
    const uint32_t tt = blockIdx.x / groups;  // t tile
    const uint64_t r0 = uint64_t(g) * R;
    const uint64_t t0 = uint64_t(tt) * T;
    uint64_t* cur = smem;
    uint64_t* nxt = smem + size_t(W) * R;
    const uint64_t* row_in = ST + uint64_t(base) * b_max;
    // The window's first kPV cells per thread are loaded before the true block
    // count (written by the block-keys kernel) is read: within the table's
    // allocation (b_max) they are harmless and the count masks them -- one
    // dependent round trip fewer
    constexpr int kPV = 4;
    uint64_t pv[kPV];
#pragma unroll
    for (int u = 0; u < kPV; ++u) {
        const uint32_t i = threadIdx.x + uint32_t(u) * NT;
        const uint64_t c = r0 + i % R + ((t0 + i / R) << base);
        pv[u] = i < W * R && c + s <= b_max ? row_in[c] : kNoKey;
    }
    const uint64_t b = b_dev ? *b_dev : b_max;
    if (b < s || r0 + s * t0 + s > b) return;  // no valid level-`base` cell in this tile
    // level-`base` cell (r, t) is valid iff r + s*t <= b - s  <=>  t <= (b - s - r) >> base
#pragma unroll
    for (int u = 0; u < kPV; ++u) {
        const uint32_t i = threadIdx.x + uint32_t(u) * NT;
        const uint64_t c = r0 + i % R + ((t0 + i / R) << base);
        if (i < W * R) cur[i] = c + s <= b ? pv[u] : kNoKey;
    }
    for (uint32_t i = threadIdx.x + kPV * NT; i < W * R; i += NT) {
        const uint32_t rl = i % R, tl = i / R;
        const uint64_t c = r0 + rl + ((t0 + tl) << base);
        cur[i] = c + s <= b ? row_in[c] : kNoKey;
    }
    __syncthreads();
    for (uint32_t d = 1; d <= D; ++d) {
        const uint32_t half = 1u << (d - 1);
        const uint32_t live = (W - half) * R;  // items with both operands in the window
        const uint32_t lvl = base + d;
        const uint64_t span = 1ull << lvl;
        uint64_t* row_out = ST + uint64_t(lvl) * b_max + r0 + (t0 << base);
        // stored cells: tl < T and column + span <= b
        const int64_t room = int64_t(b) - int64_t(span) - int64_t(r0) - int64_t(t0 << base);
        const uint32_t stored = T * R;
        for (uint32_t i = threadIdx.x; i < stored; i += NT) {
            const uint64_t v = kmin(cur[i], cur[i + half * R]);
            nxt[i] = v;
            const uint32_t rl = i % R, tl = i / R;
            const int64_t off = int64_t(rl) + (int64_t(tl) << base);
            if (off <= room) row_out[off] = v;
        }
        for (uint32_t i = stored + threadIdx.x; i < live; i += NT)
            nxt[i] = kmin(cur[i], cur[i + half * R]);
        __syncthreads();
        uint64_t* t = cur;
        cur = nxt;
        nxt = t;
    }
}

template <int R, int T, int NT>
int launch_tile(uint64_t* ST, uint64_t b, const uint64_t* b_dev, uint32_t base, uint32_t D,
                cudaStream_t stream) {
    const uint64_t s = 1ull << base;
    const uint64_t groups = s >= uint64_t(R) ? s / R : 1;
    const uint64_t tcount = (b + s - 1) / s;
    const uint64_t tiles = (tcount + T - 1) / T;
    const size_t sm = size_t(2) * (T + (1u << D) - 1) * R * sizeof(uint64_t);
    cudaFuncSetAttribute(k_st_tile<R, T, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(sm));
    brmq::launch_k(k_st_tile<R, T, NT>, dim3(unsigned(groups * tiles)), dim3(NT), sm, stream, ST, b, b_dev, base, D,
                                                                      uint32_t(groups));
    return 1;
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
            // small tables: narrow tiles so that several CTAs share the work
            launches += b >= (1u << 16) ? launch_tile<1, 2048, 512>(ST, b, b_dev, 0, D, stream)
                                        : launch_tile<1, 256, 256>(ST, b, b_dev, 0, D, stream);
            base = D;
        } else {
            const uint32_t D = (L - 1 - base) < 7 ? (L - 1 - base) : 7;
            // base >= 10.  The last launch of a table has few t-positions
            // (tcount = b >> base, 2^D of them at most): trade t for residues so
            // its CTAs are not mostly empty windows
            const uint64_t tcount = (b + (1ull << base) - 1) >> base;
            if (tcount <= 16)
                launches += launch_tile<64, 16, 256>(ST, b, b_dev, base, D, stream);
            else if (tcount <= 32)
                launches += launch_tile<32, 32, 256>(ST, b, b_dev, base, D, stream);
            else  // (measured: T = 128 x 512 threads beats 64 x 256 and 256 x 512)
                launches += launch_tile<16, 128, 512>(ST, b, b_dev, base, D, stream);
            base += D;
        }
    }
    return launches;
}

}  // namespace brmq
