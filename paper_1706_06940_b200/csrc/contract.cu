// contract.cu -- BbST_CON stage 1 on the device: endpoints, dedup/rank and the
// boundary bitmap consumed by the contraction kernel (contraction.cu), plus
// the bitmap remap and the stage-API helper kernels.
//
// Reference stages replaced:
//   collect_endpoints          contraction.cpp:13-23
//   dedup -> boundary          contraction.cpp:118-127
//   scan_areas / build_contracted   contraction.cpp:81-151 (inclusive areas)
//   remap_queries_from_sorted  contraction.cpp:174-199
//
// B200 design.  The boundary set is handed to the contraction kernel as a
// bitmap over A (bit p set <=> p is a query endpoint), so a tile of A finds its
// area boundaries with one coalesced read of its bitmap words instead of a
// search in the sorted boundary list (see contraction.cu for the scan of A).
//
// Two ways to produce the bitmap + query ranks (BRMQ_SORT_* in brmq.h):
//   radix  : k_collect -> device radix sort (radix_sort.cu) -> k_unique
//            (dedup, ranks = cleft / cright, marks the bitmap)
//   bitmap : k_collect marks the bitmap directly (a counting sort by
//            position with one presence bit per key); ranks come afterwards
//            from per-word prefix counts the contraction kernel emits.
#include "common.cuh"
#include "kernels.h"
#include "scan.cuh"

namespace brmq {
namespace {

constexpr int kThreads = 256;
constexpr int kItems = 8;   // 2048-endpoint dedup tiles (measured vs 1024 and 4096)
constexpr int kTile = kThreads * kItems;
constexpr int kCollectU = 4;  // queries per thread in flight in k_collect

// ------------------------------------------------------------------ collect
// span[0] = max(~pos) (= ~min pos), span[1] = max(pos); control block starts zeroed.
// Grid-stride with a capped grid so the span needs only 2 atomics per CTA.
// With a bitmap, marks every endpoint with a fire-and-forget reduction (the
// boundaries per contraction piece are popcounted afterwards: k_piece_count).
__global__ void __launch_bounds__(kThreads) k_collect(const ulonglong2* __restrict__ Q, uint64_t q,
                                                      uint64_t n, uint32_t* __restrict__ keys,
                                                      uint32_t* __restrict__ vals,
                                                      uint32_t* __restrict__ bitmap,
                                                      uint32_t* __restrict__ span,
                                                      uint32_t* __restrict__ err,
                                                      uint32_t* __restrict__ epoch_bump,
                                                      uint32_t epoch_by, uint32_t mark_lo,
                                                      uint32_t mark_hi, uint64_t* __restrict__ fill0,
                                                      uint64_t fill0_n, uint64_t* __restrict__ fill1,
                                                      uint64_t fill1_n,
                                                      unsigned long long* __restrict__ hist,
                                                      uint32_t hshift, uint32_t hmask) {
    brmq::pdl_wait();
    brmq::pdl_trigger();  // small grid: dependents may be scheduled now
    {
        const uint64_t t = uint64_t(blockIdx.x) * kThreads + threadIdx.x, nt = uint64_t(gridDim.x) * kThreads;
        for (uint64_t i = t; i < fill0_n; i += nt) fill0[i] = kNoKey;
        for (uint64_t i = t; i < fill1_n; i += nt) fill1[i] = kNoKey;
    }
    // the solve's epoch reservation rides on this first kernel (no extra launch)
    if (epoch_bump && blockIdx.x == 0 && threadIdx.x == 0) *epoch_bump += epoch_by;
    __shared__ uint32_t s_lo, s_hi;
    __shared__ uint32_t s_hist[1024];  // hist: the radix partition's top-digit counts
    if (threadIdx.x == 0) { s_lo = 0xFFFFFFFFu; s_hi = 0; }
    if (hist)
        for (uint32_t d = threadIdx.x; d <= hmask; d += kThreads) s_hist[d] = 0;
    __syncthreads();
    uint32_t lo_acc = 0xFFFFFFFFu, hi_acc = 0;
    const uint64_t stride = uint64_t(gridDim.x) * kThreads;
    // kCollectU queries per thread in flight (ncu, c5-con: 75% of the stall
    // samples waited on the single streamed query load of the plain loop)
    constexpr int U = kCollectU;
    for (uint64_t i0 = uint64_t(blockIdx.x) * kThreads + threadIdx.x; i0 < q; i0 += U * stride) {
      ulonglong2 xs[U];
#pragma unroll
      for (int u = 0; u < U; ++u)
          xs[u] = i0 + u * stride < q ? __ldcs(Q + i0 + u * stride) : make_ulonglong2(0, 0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t i = i0 + u * stride;
        if (i >= q) break;
        const ulonglong2 x = xs[u];
        uint64_t l = x.x, r = x.y;
        if (l > r) { const uint64_t t = l; l = r; r = t; }  // types.hpp:18-20
        if (r >= n) {                                        // naive.hpp:14-15 (range)
            atomicOr(err, 2u);
            r = n - 1;
            if (l > r) l = r;
        }
        const uint32_t lo = uint32_t(l), hi = uint32_t(r);
        if (keys) reinterpret_cast<uint2*>(keys)[i] = make_uint2(lo, hi);
        if (vals)
            reinterpret_cast<uint2*>(vals)[i] =
                make_uint2(uint32_t(i << 1), uint32_t((i << 1) | 1u));  // contraction.hpp:16-18
        if (hist) {
            atomicAdd(&s_hist[(lo >> hshift) & hmask], 1u);
            atomicAdd(&s_hist[(hi >> hshift) & hmask], 1u);
        }
        if (bitmap) {  // only the endpoints in this pass's slice [mark_lo, mark_hi]
            if (lo - mark_lo <= mark_hi - mark_lo) atomicOr(bitmap + (lo >> 5), 1u << (lo & 31));
            if (hi - mark_lo <= mark_hi - mark_lo) atomicOr(bitmap + (hi >> 5), 1u << (hi & 31));
        }
        lo_acc = lo < lo_acc ? lo : lo_acc;
        hi_acc = hi > hi_acc ? hi : hi_acc;
      }
    }
    if (span) {
        const uint32_t wlo = __reduce_min_sync(kFull, lo_acc);
        const uint32_t whi = __reduce_max_sync(kFull, hi_acc);
        if (lane_id() == 0 && wlo != 0xFFFFFFFFu) {
            atomicMin(&s_lo, wlo);
            atomicMax(&s_hi, whi);
        }
        __syncthreads();
        if (threadIdx.x == 0 && s_lo != 0xFFFFFFFFu) {
            atomicMax(span + 0, ~s_lo);
            atomicMax(span + 1, s_hi);
        }
    }
    if (hist) {
        __syncthreads();
        for (uint32_t d = threadIdx.x; d <= hmask; d += kThreads)
            if (const uint32_t c = s_hist[d]) atomicAdd(hist + d, (unsigned long long)c);
    }
}

// ------------------------------------------------------------------- unique
// Sorted endpoints -> ranks.  rank(j) = (#distinct positions among 0..j) - 1.
// With a bitmap, also rfirst[g] (g = 0..G) = rank of the first boundary at or
// after the start of contraction range g (= |boundary| past the last one): the
// head of every range change writes the entries it crosses, so the
// contraction gets its rank bases without counting.
__global__ void __launch_bounds__(kThreads) k_unique(
    const uint32_t* __restrict__ pos, const uint32_t* __restrict__ org, uint64_t m, uint64_t n,
    uint32_t* __restrict__ boundary, uint32_t* __restrict__ cleft, uint32_t* __restrict__ cright_raw,
    uint32_t* __restrict__ bitmap, uint32_t* __restrict__ rfirst, uint32_t R, uint32_t G,
    uint32_t* __restrict__ span, uint64_t* __restrict__ nb_out,
    uint32_t* __restrict__ err, uint64_t* __restrict__ status, uint32_t* __restrict__ ticket,
    const uint32_t* __restrict__ epoch_dev, uint32_t epoch_off) {
    brmq::pdl_wait();
    const uint32_t epoch = *epoch_dev + epoch_off;
    __shared__ uint32_t s_tile;
    __shared__ uint32_t s_scan[kThreads / 32 + 1];
    __shared__ unsigned long long s_excl;
    if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    const uint64_t base = tile * kTile + uint64_t(threadIdx.x) * kItems;

    uint32_t p[kItems];
    if (base + kItems <= m) {
        const uint4* v = reinterpret_cast<const uint4*>(pos + base);
#pragma unroll
        for (int j = 0; j < kItems / 4; ++j) {
            const uint4 x = __ldcs(v + j);  // streamed: keeps cleft / cright in L2
            p[4 * j] = x.x; p[4 * j + 1] = x.y; p[4 * j + 2] = x.z; p[4 * j + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < kItems; ++j) p[j] = base + j < m ? __ldg(pos + base + j) : 0u;
    }
    uint32_t prev = base > 0 && base - 1 < m ? __ldg(pos + base - 1) : 0u;
    // the origins are loaded now: in flight during the look-back below
    uint4 o4[kItems / 4];
    if (base + kItems <= m && cleft) {
        const uint4* v = reinterpret_cast<const uint4*>(org + base);
#pragma unroll
        for (int j = 0; j < kItems / 4; ++j) o4[j] = __ldcs(v + j);
    }
    uint32_t heads = 0, cnt = 0;
    bool unsorted = false;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const uint64_t idx = base + j;
        if (idx < m) {
            const bool h = idx == 0 || p[j] != prev;
            unsorted |= idx > 0 && p[j] < prev;            // contraction.cpp:123
            heads |= uint32_t(h) << j;
            cnt += h;
            prev = p[j];
        }
    }
    if (unsorted) atomicOr(err, 4u);
    uint32_t total;
    const uint32_t excl = block_excl_sum<kThreads>(cnt, s_scan, total);
    if (threadIdx.x < 32) {
        if (tile == 0) {
            if (threadIdx.x == 0) {
                st_release_u64(status, status_pack(epoch, kStInclusive, false, total));
                s_excl = 0;
            }
        } else {
            if (threadIdx.x == 0)
                st_release_u64(status + tile, status_pack(epoch, kStAggregate, false, total));
            uint64_t e, unused;
            warp_lookback<false>(status, nullptr, nullptr, tile, 0, epoch, e, unused);
            if (threadIdx.x == 0) {
                st_release_u64(status + tile, status_pack(epoch, kStInclusive, false, e + total));
                s_excl = e;
            }
        }
    }
    __syncthreads();
    uint64_t r = s_excl + excl;  // rank of the next head; item rank = r - 1 after its head
    const uint32_t* o = reinterpret_cast<const uint32_t*>(o4);
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        const uint64_t idx = base + j;
        if (idx >= m) break;
        if ((heads >> j) & 1u) {
            ++r;
            if (p[j] >= n) {
                atomicOr(err, 2u);  // position past the array: range error
            } else if (bitmap) {
                atomicOr(bitmap + (p[j] >> 5), 1u << (p[j] & 31));
                const uint32_t g = (p[j] >> kContractTileLog2) / R;
                uint32_t g0 = 0;  // first range not yet covered by an earlier head
                if (idx > 0) {
                    const uint32_t pp = j > 0 ? p[j - 1] : __ldg(pos + idx - 1);
                    g0 = (pp >> kContractTileLog2) / R + 1;
                }
                for (uint32_t x = g0; x <= g; ++x) rfirst[x] = uint32_t(r - 1);
            }
            if (boundary) boundary[r - 1] = p[j];
        }
        if (cleft) {
            const uint32_t og = base + kItems <= m ? o[j] : __ldg(org + idx);
            const uint32_t qi = og >> 1;
            ((og & 1u) ? cright_raw : cleft)[qi] = uint32_t(r - 1);
        }
        if (idx == 0 && span) span[0] = ~p[j];
        if (idx == m - 1) {
            *nb_out = r;
            if (span) span[1] = p[j];
            if (bitmap && p[j] < n)
                for (uint32_t x = (p[j] >> kContractTileLog2) / R + 1; x <= G; ++x) rfirst[x] = uint32_t(r);
        }
    }
}

// ------------------------------------------------------------- mark sorted
// Sorted endpoint positions -> the boundary bitmap (the dedup of
// contraction.cpp:118-127: a position present any number of times is one bit).
// Each thread walks 8 consecutive sorted positions and ORs the bits of a word
// locally; a word strictly inside the thread's run is owned by it (plain
// store: the bitmap is all-zero between solves), the first and last words may be
// shared with the neighbours (atomicOr).  Checks the order (contraction.cpp:123)
// and the range, and publishes the span.  The boundary ranks then come from the
// bitmap (k_piece_count) and the query kernel's per-word ranks, as in the
// bitmap pipeline: no look-back, no rank scatter.
__global__ void __launch_bounds__(kThreads) k_mark_sorted(const uint32_t* __restrict__ pos, uint64_t m,
                                                          uint64_t n, uint32_t* __restrict__ bitmap,
                                                          uint32_t* __restrict__ span,
                                                          uint32_t* __restrict__ err) {
    brmq::pdl_wait();
    const uint64_t base = (uint64_t(blockIdx.x) * kThreads + threadIdx.x) * kItems;
    if (base >= m) return;
    uint32_t p[kItems];
    if (base + kItems <= m) {
        const uint4* v = reinterpret_cast<const uint4*>(pos + base);
#pragma unroll
        for (int j = 0; j < kItems / 4; ++j) {
            const uint4 x = __ldcs(v + j);
            p[4 * j] = x.x; p[4 * j + 1] = x.y; p[4 * j + 2] = x.z; p[4 * j + 3] = x.w;
        }
    } else {
#pragma unroll
        for (int j = 0; j < kItems; ++j) p[j] = base + j < m ? __ldg(pos + base + j) : 0u;
    }
    uint32_t prev = base > 0 ? __ldg(pos + base - 1) : 0u;
    uint32_t bad = 0, word = 0xFFFFFFFFu, bits = 0;
    bool first = true;
#pragma unroll
    for (int j = 0; j < kItems; ++j) {
        if (base + j >= m) break;
        const uint32_t x = p[j];
        if (base + j > 0 && x < prev) bad |= 4u;  // contraction.cpp:123
        prev = x;
        if (x >= n) {
            bad |= 2u;
            continue;
        }
        if ((x >> 5) != word) {
            if (bits) {
                if (first) atomicOr(bitmap + word, bits);
                else bitmap[word] = bits;
                first = false;
            }
            word = x >> 5;
            bits = 0;
        }
        bits |= 1u << (x & 31);
    }
    if (bits) atomicOr(bitmap + word, bits);
    if (bad) atomicOr(err, bad);
    if (base == 0) span[0] = ~p[0];
    if (base + kItems >= m) span[1] = p[(m - 1 - base) < kItems ? (m - 1 - base) : 0];
}

// ------------------------------------------------------------ bitmap remap
__global__ void __launch_bounds__(kThreads) k_remap_bitmap(const ulonglong2* __restrict__ Q,
                                                           uint64_t q, uint64_t n,
                                                           const uint2* __restrict__ word_info,
                                                           uint32_t* __restrict__ cleft,
                                                           uint32_t* __restrict__ cright_raw) {
    brmq::pdl_wait();
    const uint64_t i = uint64_t(blockIdx.x) * kThreads + threadIdx.x;
    if (i >= q) return;
    const ulonglong2 x = __ldg(Q + i);
    uint64_t l = x.x, r = x.y;
    if (l > r) { const uint64_t t = l; l = r; r = t; }
    if (r >= n) { r = n - 1; if (l > r) l = r; }
    const uint2 wl = __ldg(word_info + (l >> 5)), wr = __ldg(word_info + (r >> 5));
    cleft[i] = wl.x + __popc(wl.y & ((1u << (l & 31)) - 1u));
    cright_raw[i] = wr.x + __popc(wr.y & ((1u << (r & 31)) - 1u));
}

// --------------------------------------------------- stage-API helper kernels
__global__ void k_split_eps(const uint2* __restrict__ eps, uint64_t m, uint32_t* __restrict__ keys,
                            uint32_t* __restrict__ vals) {
    brmq::pdl_wait();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < m) {
        const uint2 e = eps[i];
        keys[i] = e.x;
        vals[i] = e.y;
    }
}
__global__ void k_join_eps(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ vals,
                           uint64_t m, uint2* __restrict__ eps) {
    brmq::pdl_wait();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < m) eps[i] = make_uint2(keys[i], vals[i]);
}
__global__ void k_split_aq(const uint64_t* __restrict__ aq, const uint64_t* __restrict__ len,
                           uint64_t len_max, int32_t* __restrict__ values,
                           uint64_t* __restrict__ origin) {
    brmq::pdl_wait();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < len_max && i < *len) {
        values[i] = key_value(aq[i]);
        origin[i] = key_pos(aq[i]);
    }
}
__global__ void k_u32_to_u64(const uint32_t* __restrict__ a, const uint64_t* __restrict__ len,
                             uint64_t len_max, uint64_t* __restrict__ out) {
    brmq::pdl_wait();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < len_max && i < *len) out[i] = a[i];
}
// remap_queries_from_sorted semantics by binary search in the boundary list
// (contraction.cpp:153-199): missing endpoint -> err |= 8 (logic_error).
__global__ void k_remap_search(const uint32_t* __restrict__ pos, const uint32_t* __restrict__ org,
                               uint64_t m, const uint64_t* __restrict__ boundary, uint64_t nb,
                               uint64_t q, uint32_t* __restrict__ cl, uint32_t* __restrict__ cr,
                               uint32_t* __restrict__ err) {
    brmq::pdl_wait();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= m) return;
    const uint64_t p = pos[i];
    uint64_t lo = 0, hi = nb;
    while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (boundary[mid] < p) lo = mid + 1; else hi = mid;
    }
    const uint32_t og = org[i];
    if (lo >= nb || boundary[lo] != p || (og >> 1) >= q) {
        atomicOr(err, 8u);
        return;
    }
    ((og & 1u) ? cr : cl)[og >> 1] = uint32_t(lo);
}
__global__ void k_remap_finish(uint64_t q, const uint32_t* __restrict__ cl, uint32_t* __restrict__ cr,
                               uint8_t* __restrict__ dg) {
    brmq::pdl_wait();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= q) return;
    if (cr[i] == cl[i]) dg[i] = 1;  // contraction.cpp:191-197
    else { dg[i] = 0; cr[i] -= 1; }
}
// remap_queries (contraction.cpp:152-171): per query, lower_bound of each end in
// the boundary list; a degenerate query (left == right) keeps cleft = cright = 0;
// an end missing from the list -> err |= 8 (logic_error).  Queries are
// normalised left <= right first (the Query constructor, types.hpp:18-20).
__global__ void k_remap_queries(const ulonglong2* __restrict__ Q, uint64_t q,
                                const uint64_t* __restrict__ boundary, uint64_t nb,
                                uint32_t* __restrict__ cl, uint32_t* __restrict__ cr,
                                uint8_t* __restrict__ dg, uint32_t* __restrict__ err) {
    brmq::pdl_wait();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= q) return;
    const ulonglong2 x = __ldg(Q + i);
    const uint64_t l = x.x < x.y ? x.x : x.y, r = x.x < x.y ? x.y : x.x;
    if (l == r) {
        cl[i] = cr[i] = 0;
        dg[i] = 1;
        return;
    }
    uint64_t idx[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
        const uint64_t p = e ? r : l;
        uint64_t lo = 0, hi = nb;
        while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (__ldg(boundary + mid) < p) lo = mid + 1; else hi = mid;
        }
        if (lo >= nb || __ldg(boundary + lo) != p) {
            atomicOr(err, 8u);
            return;
        }
        idx[e] = lo;
    }
    cl[i] = uint32_t(idx[0]);
    cr[i] = uint32_t(idx[1] - 1);
    dg[i] = 0;
}
__global__ void k_keys_to_pos(uint64_t* __restrict__ t, uint64_t count) {
    brmq::pdl_wait();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < count) t[i] = t[i] == kNoKey ? ~0ull : uint64_t(key_pos(t[i]));
}

// ------------------------------------------------ ST-RMQ_CON (SPEC.md "baseline")
// Marked contraction E: E[2t+1] = A[b_t] (every marked
// position verbatim), E[2t] = the unmarked run between b_{t-1} and b_t, E[0] /
// E[2m] the runs before b_0 / after b_{m-1}.  The contraction kernel in MARKED
// mode wrote E[2t] as the leftmost minimum of [b_{t-1}, b_t] with both marks read
// as +inf; when that minimum landed on the mark b_{t-1} the run is empty (no
// entry: +inf) or all +inf (its first position).
__global__ void k_marked_fill(const int32_t* __restrict__ A, const uint32_t* __restrict__ bnd,
                              const uint64_t* __restrict__ m_dev, uint64_t* __restrict__ E) {
    brmq::pdl_wait();
    const uint64_t m = *m_dev;
    const uint64_t t = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (t >= m) return;
    const uint32_t b = bnd[t];
    E[2 * t + 1] = pack_key(__ldg(A + b), b);
    if (t == 0) {
        E[0] = kNoKey;
        E[2 * m] = kNoKey;
    } else {
        const uint32_t p = bnd[t - 1];
        const uint64_t x = E[2 * t];
        if (x == kNoKey || key_pos(x) == p) E[2 * t] = b - p >= 2 ? pack_key(0x7FFFFFFF, p + 1) : kNoKey;
    }
}

// E[0] = leftmost minimum of A[0, b_0), E[2m] = of A(b_{m-1}, n): grid-stride,
// warp reductions, one 64-bit atomicMin per warp and side.
__global__ void k_marked_edges(const int32_t* __restrict__ A, uint64_t n,
                               const uint32_t* __restrict__ span, const uint64_t* __restrict__ m_dev,
                               uint64_t* __restrict__ E) {
    brmq::pdl_wait();
    const uint32_t b0 = ~span[0], blast = span[1];
    if (b0 > blast) return;
    const uint64_t pre = b0, suf = n - 1 - blast;  // lengths
    const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
    uint64_t kp = kNoKey, ks = kNoKey;
    for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < pre + suf; i += stride) {
        const uint64_t p = i < pre ? i : blast + 1 + (i - pre);
        const uint64_t k = pack_key(__ldg(A + p), uint32_t(p));
        if (i < pre) kp = kmin(kp, k);
        else ks = kmin(ks, k);
    }
    kp = warp_min_key(kp);
    ks = warp_min_key(ks);
    if (lane_id() == 0) {
        if (kp != kNoKey) atomicMin(reinterpret_cast<unsigned long long*>(E), kp);
        if (ks != kNoKey) atomicMin(reinterpret_cast<unsigned long long*>(E + 2 * *m_dev), ks);
    }
}

// Query i: [2 cl + 1, 2 cr + 1] in E through the element Sparse Table (row e at
// ST + e * stride), the two-range trick of element_sparse_table.cpp:35-44.
__device__ __forceinline__ void st_one(const ulonglong2* __restrict__ Q,
                                       const uint32_t* __restrict__ cleft,
                                       const uint32_t* __restrict__ cright_raw, uint64_t i,
                                       const uint64_t* __restrict__ ST, uint64_t stride,
                                       uint64_t* __restrict__ answers) {
    const ulonglong2 x = __ldg(Q + i);
    const uint64_t l = x.x < x.y ? x.x : x.y;
    const uint64_t il = 2 * uint64_t(__ldg(cleft + i)) + 1, ir = 2 * uint64_t(__ldg(cright_raw + i)) + 1;
    if (il == ir) {  // l == r
        answers[i] = l;
        return;
    }
    const uint32_t e = floor_log2_u64(ir - il + 1);
    const uint64_t* row = ST + uint64_t(e) * stride;
    answers[i] = key_pos(kmin(__ldg(row + il), __ldg(row + ir + 1 - (1ull << e))));
}
__global__ void k_query_st(const ulonglong2* __restrict__ Q, const uint32_t* __restrict__ cleft,
                           const uint32_t* __restrict__ cright_raw, uint64_t q,
                           const uint64_t* __restrict__ ST, uint64_t stride,
                           uint64_t* __restrict__ answers, const CtlPublish pub) {
    brmq::pdl_wait();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i < q) st_one(Q, cleft, cright_raw, i, ST, stride, answers);
}

inline unsigned g256(uint64_t x) { return unsigned((x + 255) / 256); }

}  // namespace

// ------------------------------------------------------------------ launchers
uint32_t collect_mark_slices(uint64_t n, uint64_t q) {
    const uint64_t bm_bytes = 2 * q >= n / 256 ? n / 8 : 0;
    constexpr uint64_t kSliceBytes = uint64_t(32) << 20;
    return uint32_t((bm_bytes + kSliceBytes - 1) / kSliceBytes);
}

int launch_collect(const uint64_t* Q, uint64_t q, uint64_t n, uint32_t* keys, uint32_t* vals,
                   uint32_t* bitmap, uint32_t* span, uint32_t* err, cudaStream_t s,
                   uint32_t* epoch_bump, uint32_t epoch_by, uint64_t* fill0, uint64_t fill0_n,
                   uint64_t* fill1, uint64_t fill1_n, unsigned long long* hist, uint32_t hshift,
                   uint32_t hmask) {
    if (q == 0) return 0;
    if (hist && hmask >= 1024u) return -1;
    // small batches: one CTA per SM (fewer span atomics, c2 -1.3 us); large ones
    // need the wide grid for the loads in flight (c5 at 148 CTAs: 0.25 -> 0.70 ms)
    const unsigned cap = q <= (uint64_t(1) << 18) ? 148u : 148u * 16u;
    const unsigned grid = g256(q) < cap ? g256(q) : cap;
    // A bitmap larger than the L2 (2^30 positions: 128 MiB) hit by many endpoints
    // (at least one per 8 words) is marked in 32 MiB slices, one pass over the
    // queries each, so that the random-position reductions hit lines resident in
    // L2 instead of missing to HBM: c5's 2e7 endpoints 0.47 -> 0.26 ms (64 MiB
    // slices: 0.28, 16 MiB: 0.34); c4's 2e6 would pay more for the extra passes
    // (0.10 -> 0.15 ms)
    const uint32_t slices = bitmap ? collect_mark_slices(n, q) : 0u;
    if (slices <= 1) {
        brmq::launch_k(k_collect, dim3(grid), dim3(kThreads), 0, s, reinterpret_cast<const ulonglong2*>(Q), q, n, keys, vals,
                                               bitmap, span, err, epoch_bump, epoch_by, 0u, ~0u,
                                               fill0, fill0_n, fill1, fill1_n, hist, hshift, hmask);
        return 1;
    }
    const uint64_t per = (n + slices - 1) / slices;
    for (uint32_t t = 0; t < slices; ++t) {
        const uint64_t a = t * per, b = (t + 1) * per < n ? (t + 1) * per : n;
        brmq::launch_k(k_collect, dim3(grid), dim3(kThreads), 0, s, reinterpret_cast<const ulonglong2*>(Q), q, n, keys, vals,
                                               bitmap, span, err, t == 0 ? epoch_bump : nullptr,
                                               epoch_by, uint32_t(a), uint32_t(b - 1),
                                               t == 0 ? fill0 : nullptr, t == 0 ? fill0_n : 0,
                                               t == 0 ? fill1 : nullptr, t == 0 ? fill1_n : 0,
                                               t == 0 ? hist : nullptr, hshift, hmask);
    }
    return int(slices);
}

size_t unique_status_words(uint64_t m) { return (m + kTile - 1) / kTile; }

int launch_mark_sorted(const uint32_t* pos, uint64_t m, uint64_t n, uint32_t* bitmap, uint32_t* span,
                       uint32_t* err, cudaStream_t s) {
    if (m == 0) return 0;
    const uint64_t threads = (m + kItems - 1) / kItems;
    brmq::launch_k(k_mark_sorted, dim3(unsigned((threads + kThreads - 1) / kThreads)), dim3(kThreads), 0, s,
                   pos, m, n, bitmap, span, err);
    return 1;
}

int launch_unique(const uint32_t* pos, const uint32_t* org, uint64_t m, uint64_t n, uint32_t* boundary,
                  uint32_t* cleft, uint32_t* cright_raw, uint32_t* bitmap, uint32_t* rfirst,
                  uint32_t range_tiles, uint32_t* span, uint64_t* nb_out, uint32_t* err,
                  uint64_t* status, uint32_t* ticket, const uint32_t* epoch_dev,
                  uint32_t epoch_off, cudaStream_t s) {
    if (m == 0) return 0;
    uint32_t G = 0, R = 1;
    if (bitmap) contract_partition(n, &G, &R);
    if (bitmap && R != range_tiles) return -1;
    brmq::launch_k(k_unique, dim3(unsigned((m + kTile - 1) / kTile)), dim3(kThreads), 0, s, 
        pos, org, m, n, boundary, cleft, cright_raw, bitmap, rfirst, R, G, span, nb_out, err,
        status, ticket, epoch_dev, epoch_off);
    return 1;
}

int launch_remap_bitmap(const uint64_t* Q, uint64_t q, uint64_t n, const uint2* word_info,
                        uint32_t* cleft, uint32_t* cright_raw, cudaStream_t s) {
    if (q == 0) return 0;
    brmq::launch_k(k_remap_bitmap, dim3(g256(q)), dim3(kThreads), 0, s, reinterpret_cast<const ulonglong2*>(Q), q, n,
                                                word_info, cleft, cright_raw);
    return 1;
}

int launch_split_eps(const void* eps, uint64_t m, uint32_t* keys, uint32_t* vals, cudaStream_t s) {
    if (!m) return 0;
    brmq::launch_k(k_split_eps, dim3(g256(m)), dim3(256), 0, s, static_cast<const uint2*>(eps), m, keys, vals);
    return 1;
}
int launch_join_eps(const uint32_t* keys, const uint32_t* vals, uint64_t m, void* eps,
                    cudaStream_t s) {
    if (!m) return 0;
    brmq::launch_k(k_join_eps, dim3(g256(m)), dim3(256), 0, s, keys, vals, m, static_cast<uint2*>(eps));
    return 1;
}
int launch_split_aq(const uint64_t* aq, const uint64_t* len, uint64_t len_max, int32_t* values,
                    uint64_t* origin, cudaStream_t s) {
    if (!len_max) return 0;
    brmq::launch_k(k_split_aq, dim3(g256(len_max)), dim3(256), 0, s, aq, len, len_max, values, origin);
    return 1;
}
int launch_u32_to_u64(const uint32_t* a, const uint64_t* len, uint64_t len_max, uint64_t* out,
                      cudaStream_t s) {
    if (!len_max) return 0;
    brmq::launch_k(k_u32_to_u64, dim3(g256(len_max)), dim3(256), 0, s, a, len, len_max, out);
    return 1;
}
int launch_remap_search(const uint32_t* pos, const uint32_t* org, uint64_t m,
                        const uint64_t* boundary, uint64_t nb, uint64_t q, uint32_t* cl,
                        uint32_t* cr, uint8_t* dg, uint32_t* err, cudaStream_t s) {
    int l = 0;
    if (m) {
        brmq::launch_k(k_remap_search, dim3(g256(m)), dim3(256), 0, s, pos, org, m, boundary, nb, q, cl, cr, err);
        ++l;
    }
    if (q) {
        brmq::launch_k(k_remap_finish, dim3(g256(q)), dim3(256), 0, s, q, cl, cr, dg);
        ++l;
    }
    return l;
}
int launch_remap_queries(const uint64_t* Q, uint64_t q, const uint64_t* boundary, uint64_t nb,
                         uint32_t* cl, uint32_t* cr, uint8_t* dg, uint32_t* err, cudaStream_t s) {
    if (!q) return 0;
    brmq::launch_k(k_remap_queries, dim3(g256(q)), dim3(256), 0, s, reinterpret_cast<const ulonglong2*>(Q), q, boundary, nb,
                                             cl, cr, dg, err);
    return 1;
}
int launch_marked_fill(const int32_t* A, const uint32_t* boundary, const uint64_t* m_dev,
                       uint64_t m_max, uint64_t* E, cudaStream_t s) {
    if (!m_max) return 0;
    brmq::launch_k(k_marked_fill, dim3(g256(m_max)), dim3(256), 0, s, A, boundary, m_dev, E);
    return 1;
}

int launch_marked_edges(const int32_t* A, uint64_t n, const uint32_t* span, const uint64_t* m_dev,
                        uint64_t* E, cudaStream_t s) {
    if (!n) return 0;
    const uint64_t g = (n + 255) / 256;
    brmq::launch_k(k_marked_edges, dim3(unsigned(g < 148 * 8 ? g : 148 * 8)), dim3(256), 0, s, A, n, span, m_dev, E);
    return 1;
}

int launch_query_st(const uint64_t* Q, const uint32_t* cleft, const uint32_t* cright_raw,
                    uint64_t q, const uint64_t* ST, uint64_t stride, uint64_t* answers,
                    cudaStream_t s, const CtlPublish& pub) {
    if (!q) return 0;
    brmq::launch_k(k_query_st, dim3(g256(q)), dim3(256), 0, s, reinterpret_cast<const ulonglong2*>(Q), cleft, cright_raw,
                                        q, ST, stride, answers, pub);
    return 1;
}

int launch_keys_to_pos(uint64_t* t, uint64_t count, cudaStream_t s) {
    if (!count) return 0;
    brmq::launch_k(k_keys_to_pos, dim3(g256(count)), dim3(256), 0, s, t, count);
    return 1;
}

}  // namespace brmq
