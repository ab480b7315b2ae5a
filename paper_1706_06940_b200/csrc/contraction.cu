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
// co-resident, so its cross-CTA waits cannot deadlock).  The 4096-element tiles
// of the span [b_0, b_{m-1}] are split into G contiguous ranges, one per CTA:
//   A. count:  popcount of the CTA's words of the boundary bitmap, published at
//              once; the CTA's rank base is the sum of ALL predecessors' counts
//              (independent reads, no look-back chain).
//   B. stream: the CTA's tiles in order through a 4-deep ring of TMA tensor
//              loads -- 16 KB of A as 128 rows x 128 B with the 128-byte
//              swizzle plus the tile's 512 bitmap bytes, one mbarrier per
//              stage.  Thread t owns row t (32 positions = one bitmap word) and
//              reads it with 8 bank-conflict-free 16-byte shared loads.  One
//              block barrier per tile: a segmented-min + count scan whose warp
//              totals are double-buffered; the stage consumed by the previous
//              tile is refilled right after that barrier.  The open segment is
//              carried from tile to tile in registers, so every area inside
//              the range is stored directly.  Rows holding boundaries are closed
//              cooperatively by their warp (one element per lane, a 5-step
//              segmented warp scan) when they are sparse, or each by its own
//              thread when they are dense.
//   C. stitch: the CTA publishes (head partial, tail partial, has-boundary);
//              the area closed by its first boundary is finished by folding
//              the predecessors' tails back to the nearest CTA holding a
//              boundary (warp windows of 32 CTAs).
// The kernel clears the bitmap words it consumed (the bitmap is never
// memset) and, for the bitmap pipeline, emits (rank prefix, bits) of every
// non-empty word for the query remap.
#include <cstdlib>
#include <cstring>
#include <type_traits>

#include "common.cuh"
#include "kernels.h"
#include "scan.cuh"
#include "tma_host.h"

namespace brmq {
namespace {

constexpr int NT = 128;             // consumer threads per CTA (one row each)
constexpr int NW = NT / 32;         // consumer warps per CTA
constexpr int NTP = NT + 32;        // + one producer warp issuing the TMA ring
constexpr int kRow = 32;            // positions per thread = one 128-byte row
constexpr int kTile = NT * kRow;    // 4096 positions = 16 KB per tile
static_assert(kTile == (1 << kContractTileLog2), "partition tile size");
constexpr int kMaxStages = 4;       // TMA ring depth (runtime: ContractArgs::stages)
constexpr int kDense = 4;           // flagged rows per warp above which rows close per thread

struct __align__(1024) Stage {
    int4 a[kTile / 4];  // NT swizzled rows: 16-byte chunk c of row r at chunk c ^ (r & 7)
};

// Rows of the current tile.  In SMEM mode they come from the swizzled TMA stage
// (16-byte chunk c of row r at byte r*128 + ((c ^ (r & 7)) << 4)) with explicit
// shared loads; otherwise (array tail past the tensor map, unaligned A) from
// global memory, bounded by n.
template <bool SMEM>
struct Rows {
    uint32_t stage;  // shared address of the stage
    const int32_t* g;
    uint64_t tile_lo, n;
    __device__ __forceinline__ int4 chunk(uint32_t r, int c) const {
        if (SMEM) return lds128(stage + r * 128u + ((uint32_t(c) ^ (r & 7u)) << 4));
        const uint64_t q = tile_lo + uint64_t(r) * kRow + 4 * c;
        int4 y;
        y.x = q + 0 < n ? __ldg(g + q + 0) : 0;
        y.y = q + 1 < n ? __ldg(g + q + 1) : 0;
        y.z = q + 2 < n ? __ldg(g + q + 2) : 0;
        y.w = q + 3 < n ? __ldg(g + q + 3) : 0;
        return y;
    }
    __device__ __forceinline__ int32_t elem(uint32_t r, int j) const {
        if (SMEM)
            return lds32(stage + r * 128u + (((uint32_t(j) >> 2) ^ (r & 7u)) << 4) + ((j & 3) << 2));
        const uint64_t q = tile_lo + uint64_t(r) * kRow + j;
        return q < n ? __ldg(g + q) : 0;
    }
    __device__ __forceinline__ uint64_t pos(uint32_t r, int j) const {
        return tile_lo + uint64_t(r) * kRow + j;
    }
};

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

// Per-thread closing of the areas whose right boundary (bit of fl) lies in
// [lo, hi] of row r; `cur` = open-segment key entering lo, `rank` =
// boundaries before.  Used when boundaries are dense.
template <class RW>
__device__ __forceinline__ void row_close_areas(const RW& rw, uint32_t r, uint32_t fl, int lo,
                                                int hi, uint64_t cur, uint64_t rank,
                                                uint64_t* __restrict__ aq) {
    int32_t rv = 0x7FFFFFFF;
    int ri = -1;
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
                uint64_t k = cur;
                if (ri >= 0) k = kmin(k, pack_key(rv, uint32_t(rw.pos(r, ri))));
                k = kmin(k, pack_key(v, uint32_t(rw.pos(r, j))));  // inclusive right end
                if (rank > 0) aq[rank - 1] = k;
                ++rank;
                cur = kNoKey;
                rv = v;  // the boundary element opens the next area
                ri = j;
            } else if (v < rv || ri < 0) {
                rv = v;
                ri = j;
            }
        }
    }
}

struct ContractArgs {
    const int32_t* A;
    uint64_t n;
    uint64_t rows;  // rows (of 32) covered by the tensor map; 0 = no TMA
    uint32_t* bitmap;
    const uint32_t* span;
    uint64_t* aq;
    uint64_t* nb_out;
    uint64_t* aq_len;
    uint2* word_info;
    const uint32_t* rcnt;  // [G] boundaries per range, or (prefix) [G+1] exclusive prefix
    uint64_t range_tiles;  // R
    uint32_t prefix;
    uint64_t* st_part;   // [G] epoch-tagged partial descriptors (phase C)
    uint64_t* key_tail;  // [G]
    const uint32_t* epoch_dev;  // device epoch counter (bumped once per solve)
    uint32_t epoch_off;
    uint32_t stages;  // TMA ring depth, 2..kMaxStages
    uint32_t debug;   // profiling knob: 1 = stream only (no compute)
};

template <bool TMA>
__global__ void __launch_bounds__(NTP) k_contract(const __grid_constant__ CUtensorMap tmap,
                                                 const ContractArgs c) {
    extern __shared__ unsigned char smem_raw[];
    const uint32_t raw = smem_u32(smem_raw);
    const uint32_t sbase = (raw + 1023u) & ~1023u;  // 1024-byte aligned: 128-byte swizzle atoms
    unsigned char* base_ptr = smem_raw + (sbase - raw);
    Stage* stg = reinterpret_cast<Stage*>(base_ptr);
    const uint32_t kStages = c.stages;
    uint32_t* sbits = reinterpret_cast<uint32_t*>(base_ptr + (TMA ? kStages * sizeof(Stage) : 0));
    uint64_t* bars = reinterpret_cast<uint64_t*>(sbits + (TMA ? kStages * NT : 0));  // full[S]
    uint64_t* empties = bars + kMaxStages;                                             // empty[S]
    __shared__ uint64_t s_tk[2][NW];  // double-buffered warp totals of the tile scan
    __shared__ uint32_t s_tf[2][NW], s_tc[2][NW];
    __shared__ uint32_t s_red[NW];
    __shared__ unsigned long long s_base;
    __shared__ uint64_t s_head;  // partial of the area closed by the range's first boundary
    __shared__ unsigned long long s_first_rank;

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
    const uint64_t my_count = tb - ta + 1;
    const uint32_t tid = threadIdx.x, lane = tid & 31u, warp = tid >> 5;

    auto issue = [&](uint64_t i) {  // thread 0: tile ta+i -> stage i % kStages
        const uint64_t t = ta + i;
        const uint32_t st = uint32_t(i % kStages);
        fence_proxy_async();
        mbar_arrive_expect_tx(&bars[st], uint32_t(sizeof(Stage)) + NT * 4u);
        tma_load_2d(stg[st].a, &tmap, 0, int(t * NT), &bars[st]);
        bulk_g2s(sbits + st * NT, c.bitmap + t * NT, NT * 4u, &bars[st]);
    };
    const bool producer = warp == NW;
    if (TMA && tid == 0) {
        for (uint32_t st = 0; st < kStages; ++st) {
            mbar_init(&bars[st], 1);       // TMA bytes land
            mbar_init(&empties[st], NW);   // every consumer warp is done with the stage
        }
        fence_mbar_init();
    }
    if (tid == 0) s_head = kNoKey;
    __syncthreads();
    if (TMA && producer && lane == 0)  // prologue: the first kStages tiles, before phase A
        for (uint64_t i = 0; i < my_count && i < uint64_t(kStages); ++i) issue(i);

    // ---- A: rank base = boundaries in all earlier ranges.  The endpoint stage
    // counted them per range while marking the bitmap (rcnt), so this is one
    // read of at most G counts from L2 -- no dependence on other CTAs' progress.
    if (c.prefix) {
        if (tid == 0) {
            s_base = __ldg(c.rcnt + cta);
            if (tb == tlast) {  // the CTA holding the span's last tile publishes the sizes
                const uint64_t nb = __ldg(c.rcnt + cta + 1);
                *c.nb_out = nb;
                *c.aq_len = nb - 1;
            }
        }
        __syncthreads();
    } else {
        uint32_t sum = 0;
        for (uint64_t j = tid; !producer && j < cta; j += NT) sum += __ldg(c.rcnt + j);
        sum = __reduce_add_sync(kFull, sum);
        if (lane == 0 && !producer) s_red[warp] = sum;
        __syncthreads();
        if (tid == 0) {
            uint64_t base = 0;
#pragma unroll
            for (int w = 0; w < NW; ++w) base += s_red[w];
            s_base = base;
            if (tb == tlast) {
                const uint64_t nb = base + __ldg(c.rcnt + cta);
                *c.nb_out = nb;
                *c.aq_len = nb - 1;
            }
        }
        __syncthreads();
    }

    // ---- B: stream the range
    if (producer) {  // refill each stage as soon as all consumer warps released it
        if (TMA && lane == 0)
            for (uint64_t i = kStages; i < my_count; ++i) {
                const uint32_t st = uint32_t(i % kStages);
                mbar_wait(&empties[st], uint32_t(i / kStages - 1) & 1u);
                issue(i);
            }
        return;
    }
    SegMin carry{kNoKey, 0};  // open segment after the tiles done so far (block-uniform)
    uint64_t rank_run = s_base;
    const uint64_t tensor_end = c.rows * 32;  // positions >= this are read from global

    // One tile.  GEN: the tile holds b0 or blast (partial rows) or lies past
    // the tensor map; otherwise every row is full and comes from shared memory.
    uint32_t st = 0, phase = 0;  // ring position of tile i: i % kStages, (i / kStages) & 1
    auto tile = [&](auto gen_tag, uint64_t i) {
        constexpr bool GEN = decltype(gen_tag)::value;
        const int par = int(i & 1);
        const uint64_t t = ta + i;
        const uint64_t tile_lo = t * kTile;
        const bool smem_rows = TMA && tile_lo + kTile <= tensor_end;
        uint32_t fl;
        if (TMA) {
            mbar_wait(&bars[st], phase);
            fl = sbits[st * NT + tid];
        } else {
            fl = c.bitmap[t * NT + tid];
        }
        const uint64_t p0 = tile_lo + uint64_t(tid) * kRow;
        int jlo = 0, jhi = kRow - 1;
        bool any = true;
        if (GEN) {
            any = p0 <= blast && p0 + kRow - 1 >= b0;
            jlo = p0 >= b0 ? 0 : int(b0 - p0);
            jhi = p0 + kRow - 1 <= blast ? kRow - 1 : int(int64_t(blast) - int64_t(p0));
        }
        const Rows<true> rs{sbase + uint32_t(st) * uint32_t(sizeof(Stage)), c.A, tile_lo, c.n};
        const Rows<false> rg{0, c.A, tile_lo, c.n};
        if (c.debug >= 1) {  // profiling: the memory pipeline alone
            __syncwarp();
            if (TMA && lane == 0) mbar_arrive(&empties[st]);
            if (++st == kStages) { st = 0; phase ^= 1u; }
            return;
        }
        const unsigned fm = __ballot_sync(kFull, fl != 0);
        const bool dense = __popc(fm) > kDense;

        // pass 1: open-segment key at the right end of the thread's row
        uint64_t run = kNoKey;
        if (any && (fl == 0 || dense)) {
            const int lo = fl ? 31 - __clz(fl) : jlo;
            if (!GEN || smem_rows)
                run = (!GEN && fl == 0) ? row_min<true>(rs, tid, 0, kRow - 1) : row_min<false>(rs, tid, lo, jhi);
            else
                run = row_min<false>(rg, tid, lo, jhi);
        }
        if (fm == 0) {  // nothing of this stage is read again: release it before the barrier
            __syncwarp();
            if (TMA && lane == 0) mbar_arrive(&empties[st]);
        }
        uint64_t hd = kNoKey;  // single-boundary row: min over [jlo, boundary], carry excluded
        if (fm && !dense) {  // sparse flagged rows: one element per lane
            for (unsigned m = fm; m; m &= m - 1) {
                const int s = __ffs(m) - 1;
                const uint32_t ft = __shfl_sync(kFull, fl, s);
                const int jl = __shfl_sync(kFull, jlo, s);
                const int jh = __shfl_sync(kFull, jhi, s);
                const uint32_t r = warp * 32 + s;
                const int lo = 31 - __clz(ft);
                const int32_t v = (!GEN || smem_rows) ? rs.elem(r, int(lane)) : rg.elem(r, int(lane));
                const uint64_t key = pack_key(v, uint32_t(rs.pos(r, int(lane))));
                const uint64_t mk = warp_min_key(int(lane) >= lo && int(lane) <= jh ? key : kNoKey);
                if ((ft & (ft - 1)) == 0) {  // one boundary: its head part now, no scan later
                    const uint64_t mh = warp_min_key(int(lane) >= jl && int(lane) <= lo ? key : kNoKey);
                    if (lane == uint32_t(s)) hd = mh;
                }
                if (lane == uint32_t(s)) run = mk;
            }
        }

        // warp totals (scan only when dense), one block barrier, fold earlier warps
        const uint32_t cnt = __popc(fl);
        SegMin inc{run, cnt != 0};
        uint32_t cinc = cnt;
        SegMin wt;
        uint32_t wc;
        if (dense) {
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                SegMin y;
                y.k = __shfl_up_sync(kFull, inc.k, o);
                y.f = __shfl_up_sync(kFull, inc.f, o);
                const uint32_t cy = __shfl_up_sync(kFull, cinc, o);
                if (lane >= uint32_t(o)) {
                    inc = seg_combine(y, inc);
                    cinc += cy;
                }
            }
            wt.k = __shfl_sync(kFull, inc.k, 31);
            wt.f = __shfl_sync(kFull, inc.f, 31);
            wc = __shfl_sync(kFull, cinc, 31);
        } else if (fm == 0) {
            wt = SegMin{warp_min_key(run), 0};
            wc = 0;
        } else {
            const int L = 31 - __clz(fm);
            wt = SegMin{warp_min_key(int(lane) >= L ? run : kNoKey), 1};
            wc = __reduce_add_sync(kFull, cnt);
        }
        if (lane == 0) {
            s_tk[par][warp] = wt.k;
            s_tf[par][warp] = wt.f;
            s_tc[par][warp] = wc;
        }
        bar_sync_named(1, NT);  // the only consumer barrier of the tile
        SegMin wp{kNoKey, 0}, xt{kNoKey, 0};
        uint32_t cp = 0, ct = 0;
#pragma unroll
        for (int w = 0; w < NW; ++w) {
            const SegMin tw{s_tk[par][w], s_tf[par][w]};
            if (w < int(warp)) {
                wp = seg_combine(wp, tw);
                cp += s_tc[par][w];
            }
            xt = seg_combine(xt, tw);
            ct += s_tc[par][w];
        }

        // pass 2: close the areas whose right boundary lies in a row
        uint64_t my_rank = 0;  // boundaries before this thread's row (flagged rows only)
        if (fm) {
            const SegMin cw = seg_combine(carry, wp);  // open segment entering the warp
            if (dense) {
                SegMin we;
                we.k = __shfl_up_sync(kFull, inc.k, 1);
                we.f = __shfl_up_sync(kFull, inc.f, 1);
                uint32_t wce = __shfl_up_sync(kFull, cinc, 1);
                if (lane == 0) { we = SegMin{kNoKey, 0}; wce = 0; }
                if (fl) {
                    const SegMin in = seg_combine(cw, we);
                    const uint64_t rank = rank_run + cp + wce;
                    my_rank = rank;
                    auto close = [&](const auto& rw) {
                        if (in.f) {
                            row_close_areas(rw, tid, fl, jlo, jhi, in.k, rank, c.aq);
                        } else {  // first boundary of the range: its area opened in an earlier CTA
                            const int f = __ffs(fl) - 1;
                            s_head = kmin(in.k, row_min<false>(rw, tid, jlo, f));
                            s_first_rank = rank;
                            row_close_areas(rw, tid, fl & (fl - 1), f, jhi, kNoKey, rank + 1, c.aq);
                        }
                    };
                    if (!GEN || smem_rows) close(rs); else close(rg);
                }
            } else {
                for (unsigned m = fm; m; m &= m - 1) {
                    const int s = __ffs(m) - 1;
                    const uint32_t ft = __shfl_sync(kFull, fl, s);
                    // open segment entering row s: rows after the previous flagged row
                    const unsigned below = fm & ((1u << s) - 1u);
                    const int pf = below ? 31 - __clz(below) : -1;
                    const uint64_t seg = warp_min_key((int(lane) >= (pf < 0 ? 0 : pf) && int(lane) < s) ? run : kNoKey);
                    const SegMin in = pf >= 0 ? SegMin{seg, 1} : seg_combine(cw, SegMin{seg, 0});
                    const uint64_t rank = rank_run + cp + __reduce_add_sync(kFull, int(lane) < s ? cnt : 0u);
                    if (lane == uint32_t(s)) my_rank = rank;
                    if ((ft & (ft - 1)) == 0) {  // one boundary: area = carry + head part
                        if (lane == uint32_t(s)) {
                            const uint64_t val = kmin(in.k, hd);
                            if (!in.f) {
                                s_head = val;
                                s_first_rank = rank;
                            } else if (rank > 0) {
                                c.aq[rank - 1] = val;
                            }
                        }
                        continue;
                    }
                    const int jl = __shfl_sync(kFull, jlo, s);
                    const int jh = __shfl_sync(kFull, jhi, s);
                    const uint32_t r = warp * 32 + s;
                    const int32_t v = (!GEN || smem_rows) ? rs.elem(r, int(lane)) : rg.elem(r, int(lane));
                    const bool inr = int(lane) >= jl && int(lane) <= jh;
                    const uint64_t key = inr ? pack_key(v, uint32_t(rs.pos(r, int(lane)))) : kNoKey;
                    const bool isf = (ft >> lane) & 1u;
                    SegMin S{key, isf};
                    if (lane == 0 && !isf) S.k = kmin(S.k, in.k);  // the carry joins the first segment
#pragma unroll
                    for (int o = 1; o < 32; o <<= 1) {
                        SegMin y;
                        y.k = __shfl_up_sync(kFull, S.k, o);
                        y.f = __shfl_up_sync(kFull, S.f, o);
                        if (lane >= uint32_t(o)) S = seg_combine(y, S);
                    }
                    uint64_t prev = __shfl_up_sync(kFull, S.k, 1);
                    if (lane == 0) prev = in.k;
                    if (isf) {
                        const uint32_t before = __popc(ft & ((1u << lane) - 1u));
                        const uint64_t rk = rank + before;
                        const uint64_t val = kmin(prev, key);  // inclusive right end
                        if (!in.f && before == 0) {
                            s_head = val;
                            s_first_rank = rk;
                        } else if (rk > 0) {
                            c.aq[rk - 1] = val;
                        }
                    }
                }
            }
            if (fl) {  // consumed bitmap word: (rank prefix, bits) for the remap, then clear
                const uint64_t w = t * NT + tid;
                if (c.word_info) c.word_info[w] = make_uint2(uint32_t(my_rank), fl);
                c.bitmap[w] = 0;
            }
        }
        carry = seg_combine(carry, xt);
        rank_run += ct;
        if (fm) {
            __syncwarp();
            if (TMA && lane == 0) mbar_arrive(&empties[st]);  // this warp is done with the stage
        }
        if (++st == kStages) { st = 0; phase ^= 1u; }
    };

    for (uint64_t i = 0; i < my_count; ++i) {
        const uint64_t t = ta + i;
        const uint64_t tile_lo = t * kTile;
        const bool interior = tile_lo >= b0 && tile_lo + kTile - 1 <= blast &&
                              (!TMA || tile_lo + kTile <= tensor_end);
        if (interior) tile(std::false_type{}, i);
        else tile(std::true_type{}, i);
    }
    bar_sync_named(1, NT);  // s_head / s_first_rank visible (consumers only)

    // ---- C: stitch the area that crosses into this range from the left
    if (warp == 0) {
        if (lane == 0) {
            c.key_tail[cta] = carry.k;
            st_release_u64(c.st_part + cta, status_pack(epoch, kStInclusive, carry.f != 0, 0));
        }
        if (carry.f && ta != tfirst) {
            const uint64_t head = s_head;
            uint64_t acc = kNoKey;
            int64_t p = int64_t(cta) - 1;
            bool done = false;
            while (!done) {
                const int64_t j = p - int64_t(lane);
                uint64_t sw = 0, k = kNoKey;
                bool has = false;
                const bool live = j >= int64_t(cfirst);  // CTAs before b0's hold nothing
                if (live) {
                    while (status_state(sw = ld_relaxed_u64(c.st_part + j), epoch) == kStInvalid) {
                    }
                    has = status_flag(sw);
                }
                __threadfence();  // acquire: the tails were stored before their descriptors
                if (live) k = ld_relaxed_u64(c.key_tail + j);
                const unsigned hm = __ballot_sync(kFull, has || !live);
                const int g = hm ? __ffs(hm) - 1 : 32;
                acc = kmin(acc, warp_min_key(int(lane) <= g ? k : kNoKey));
                done = g < 32;
                p -= 32;
            }
            if (lane == 0) c.aq[s_first_rank - 1] = kmin(acc, head);
        }
    }
}

struct ContractLaunch {
    int grid = 0;  // co-resident CTAs of both kernel variants (cooperative launch)
    size_t smem_tma = 0;
    uint32_t stages = 0, debug = 0;
};

ContractLaunch& contract_cfg() {
    static ContractLaunch cfg;
    if (cfg.grid == 0) {
        int dev = 0, sms = 0, per_tma = 0, per_ldg = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        const char* e = getenv("BRMQ_CONTRACT_STAGES");  // tuning knob, default 2
        cfg.stages = e ? uint32_t(atoi(e)) : 2u;
        const char* d = getenv("BRMQ_CONTRACT_DEBUG");
        cfg.debug = d ? uint32_t(atoi(d)) : 0u;
        if (cfg.stages < 2) cfg.stages = 2;
        if (cfg.stages > kMaxStages) cfg.stages = kMaxStages;
        cfg.smem_tma = 1024 + cfg.stages * (sizeof(Stage) + NT * 4) + 2 * kMaxStages * 8;
        cudaFuncSetAttribute(k_contract<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(cfg.smem_tma));
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_tma, k_contract<true>, NTP, cfg.smem_tma);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_ldg, k_contract<false>, NTP,
                                                      1024 + 2 * kMaxStages * 8);
        int per = per_tma < per_ldg ? per_tma : per_ldg;
        if (per < 1) per = 1;
        cfg.grid = sms * per;
        if (cfg.grid > int(kMaxContractRanges)) cfg.grid = int(kMaxContractRanges);
    }
    return cfg;
}

}  // namespace

size_t contract_tiles(uint64_t n) { return (n + kTile - 1) / kTile; }
size_t contract_bitmap_words(uint64_t n) { return contract_tiles(n) * NT + 4; }
size_t contract_status_words() { return size_t(2) * kMaxContractRanges; }  // st_part, key_tail

void contract_partition(uint64_t n, uint32_t* G, uint32_t* R) {
    const uint64_t tiles = contract_tiles(n);
    uint64_t g = uint64_t(contract_cfg().grid);
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
                    uint32_t epoch_off, cudaStream_t s) {
    if (n == 0) return 0;
    const ContractLaunch& cfg = contract_cfg();
    CUtensorMap tmap;
    std::memset(&tmap, 0, sizeof(tmap));
    const uint64_t rows = n / 32;
    // TMA needs a 16-byte aligned base; arrays without a full row use the plain path
    const bool tma = (reinterpret_cast<uintptr_t>(A) & 15u) == 0 && rows > 0 &&
                     make_tmap_rows128(&tmap, A, rows, NT);
    uint32_t G = 0, R = 0;
    contract_partition(n, &G, &R);
    ContractArgs args{A, n, tma ? rows : 0, bitmap, span, aq, nb_out, aq_len, word_info,
                      rcnt, R, prefix ? 1u : 0u, status, status + kMaxContractRanges, epoch_dev, epoch_off,
                      cfg.stages, cfg.debug};
    void* params[] = {&tmap, &args};
    cudaLaunchCooperativeKernel(tma ? reinterpret_cast<const void*>(k_contract<true>)
                                    : reinterpret_cast<const void*>(k_contract<false>),
                                dim3(G), dim3(NTP), params,
                                tma ? cfg.smem_tma : 1024 + 2 * kMaxStages * 8, s);
    return 1;  // launch errors surface through the caller's cudaGetLastError
}

}  // namespace brmq
