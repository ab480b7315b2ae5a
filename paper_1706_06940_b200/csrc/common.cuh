// common.cuh -- shared device helpers for the batched-RMQ kernels (sm_100a).
//
// Every argmin in the engine carries a packed 64-bit key
//     key = (uint64(uint32(v) ^ 0x80000000) << 32) | pos32
// so that unsigned min(key) is exactly "smallest value, then leftmost
// position" for signed int32 values -- the reference's answer contract
// (naive.hpp:18 strict '<', element_sparse_table.cpp:29,43 leftmost on ties).
// Valid because positions fit 32 bits (n <= 2^32-1, contraction.hpp:13).
#pragma once

#include "kernels.h"  // CtlPublish

#include <cstdint>

#include <cuda_runtime.h>

namespace brmq {

constexpr uint64_t kNoKey = ~0ull;  // never a real key: pos 0xFFFFFFFF is not a valid position
constexpr unsigned kFull = 0xFFFFFFFFu;

__host__ __device__ __forceinline__ uint64_t pack_key(int32_t v, uint32_t pos) {
    return (uint64_t(uint32_t(v) ^ 0x80000000u) << 32) | pos;
}
__host__ __device__ __forceinline__ uint32_t key_hi(uint64_t k) { return uint32_t(k >> 32); }
__host__ __device__ __forceinline__ uint32_t key_pos(uint64_t k) { return uint32_t(k); }
__host__ __device__ __forceinline__ int32_t key_value(uint64_t k) {
    return int32_t(uint32_t(k >> 32) ^ 0x80000000u);
}
__host__ __device__ __forceinline__ uint64_t kmin(uint64_t a, uint64_t b) { return a < b ? a : b; }

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// PDL (kernels.h launch_k): the first statement of every kernel.  Waits until
// the predecessor grid has completed and flushed (a no-op for a plain launch).
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
// Lets this grid's dependents be scheduled before it exits.  Only in kernels
// with small grids: every CTA of a large grid paying it cost ~1-2 ns per CTA of
// serialised front-end work (measured: c5 BbST block argmin, 262K CTAs, +0.55 ms).
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// Warp-wide min of packed keys with two redux.sync (no 64-bit shuffles):
// min of the high words, then min of the low words among lanes holding it.
__device__ __forceinline__ uint64_t warp_min_key(uint64_t k) {
    const uint32_t hi = key_hi(k);
    const uint32_t whi = __reduce_min_sync(kFull, hi);
    const uint32_t wlo = __reduce_min_sync(kFull, hi == whi ? uint32_t(k) : 0xFFFFFFFFu);
    return (uint64_t(whi) << 32) | wlo;
}

// Min over lanes of a sub-group of `G` consecutive lanes (G power of two <= 32).
template <int G>
__device__ __forceinline__ uint64_t group_min_key(uint64_t k) {
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) k = kmin(k, __shfl_xor_sync(kFull, k, o));
    return k;
}

__host__ __device__ __forceinline__ uint32_t floor_log2_u64(uint64_t x) {
#ifdef __CUDA_ARCH__
    return 63u - uint32_t(__clzll(x));
#else
    return 63u - uint32_t(__builtin_clzll(x));
#endif
}

// Streaming 128-bit read-only load that does not allocate in L1 (A is read once).
__device__ __forceinline__ int4 ld_stream_v4(const int4* p) {
    int4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

__device__ __forceinline__ uint4 ld_stream_u4(const uint4* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Release / acquire flag accesses for single-pass (decoupled look-back) scans.
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
    asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
    uint32_t v;
    asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_acquire_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_relaxed_u64(uint64_t* p, uint64_t v) {
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ uint64_t ld_relaxed_u64(const uint64_t* p) {
    uint64_t v;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}

// ------------------------------------------------ shared-memory helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return uint32_t(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ int4 lds128(uint32_t addr) {
    int4 r;
    asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "r"(addr));
    return r;
}
__device__ __forceinline__ int32_t lds32(uint32_t addr) {
    int32_t r;
    asm volatile("ld.shared.s32 %0, [%1];" : "=r"(r) : "r"(addr));
    return r;
}

// Publication of the control header by the final kernel of a solve whose final
// kernel writes nothing into the header itself (BbST_CON): every earlier kernel
// has completed (stream order), so the first warp of CTA 0 copies the header to
// the host-mapped mirror at once and re-zeroes the accumulating fields for the
// next solve -- no tail launch (k_publish: ~3 us per solve at c2).
__device__ __forceinline__ void publish_early(const CtlPublish& p) {
    if (!p.host || blockIdx.x != 0 || threadIdx.x >= 32) return;
    for (uint32_t i = threadIdx.x; i < p.words; i += 32) p.host[i] = __ldcg(p.ctl + i);
    __syncwarp();
    for (uint32_t i = threadIdx.x; i < p.reset_words; i += 32) const_cast<uint32_t*>(p.ctl)[i] = 0u;
}
}  // namespace brmq
