// stream_bench.cu -- microbenchmark of read-streaming methods on B200 (tooling,
// not shipped).  Streams N int32 once and reduces them to a checksum, timing
// each method with CUDA events (L2 flushed between runs).
//   ldg   : non-persistent, warp per 512 elements, 4 x 16 B loads per lane
//   ldgp  : persistent grid-stride warps, 4 x 16 B per lane per step
//   bulk  : persistent CTAs, 1D cp.async.bulk ring of S x T-byte stages
//   tma2d : persistent CTAs, 2D tensor-map ring (128 B rows, 128B swizzle)
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I include -I tools
//        tools/stream_bench.cu -o /tmp/sb -lcuda
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "tma_dev.cuh"
#include "tma_host.h"

using namespace brmq;

__global__ void k_ldg(const int4* __restrict__ a, uint64_t nvec, unsigned* out) {
    const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    const uint64_t base = w * 128;
    if (base >= nvec) return;
    int m = 0x7FFFFFFF;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        const int4 x = ld_stream_v4(a + base + u * 32 + lane);
        m = __vimin3_s32(m, x.x, x.y);
        m = __vimin3_s32(m, x.z, x.w);
    }
    m = __reduce_min_sync(0xffffffffu, m);
    if (lane == 0 && m == 0x12345678) atomicAdd(out, 1u);
}

__global__ void k_ldgp(const int4* __restrict__ a, uint64_t nvec, unsigned* out) {
    const uint64_t nw = uint64_t(gridDim.x) * blockDim.x / 32;
    const unsigned lane = threadIdx.x & 31;
    int m = 0x7FFFFFFF;
    for (uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; w * 128 < nvec; w += nw) {
        int4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = ld_stream_v4(a + w * 128 + u * 32 + lane);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            m = __vimin3_s32(m, x[u].x, x[u].y);
            m = __vimin3_s32(m, x[u].z, x[u].w);
        }
    }
    m = __reduce_min_sync(0xffffffffu, m);
    if (lane == 0 && m == 0x12345678) atomicAdd(out, 1u);
}

// persistent, each warp streams its own contiguous piece (PF: prefetch next step)
template <bool PF>
__global__ void k_ldgc(const int4* __restrict__ a, uint64_t nvec, unsigned* out) {
    const uint64_t nw = uint64_t(gridDim.x) * blockDim.x / 32;
    const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31;
    const uint64_t steps = nvec / 128;
    const uint64_t per = (steps + nw - 1) / nw;
    const uint64_t s0 = w * per, s1 = s0 + per < steps ? s0 + per : steps;
    int m = 0x7FFFFFFF;
    if (!PF) {
        for (uint64_t s = s0; s < s1; ++s) {
            int4 x[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = ld_stream_v4(a + s * 128 + u * 32 + lane);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                m = __vimin3_s32(m, x[u].x, x[u].y);
                m = __vimin3_s32(m, x[u].z, x[u].w);
            }
        }
    } else {
        int4 x[4], y[4];
        if (s0 < s1)
#pragma unroll
            for (int u = 0; u < 4; ++u) x[u] = ld_stream_v4(a + s0 * 128 + u * 32 + lane);
        for (uint64_t s = s0; s < s1; ++s) {
            if (s + 1 < s1)
#pragma unroll
                for (int u = 0; u < 4; ++u) y[u] = ld_stream_v4(a + (s + 1) * 128 + u * 32 + lane);
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                m = __vimin3_s32(m, x[u].x, x[u].y);
                m = __vimin3_s32(m, x[u].z, x[u].w);
                x[u] = y[u];
            }
        }
    }
    m = __reduce_min_sync(0xffffffffu, m);
    if (lane == 0 && m == 0x12345678) atomicAdd(out, 1u);
}

// persistent per-warp contiguous pieces through a per-warp cp.async ring of S
// stages x 2 KB in shared memory (each lane copies and reads back its own 64 B)
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src) {
    asm volatile("cp.async.cg.shared.global.L2::128B [%0], [%1], 16;" ::"r"(dst), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int S>
__global__ void k_cpa(const int4* __restrict__ a, uint64_t nvec, unsigned* out) {
    extern __shared__ int4 ring[];  // [warps][S][128]
    const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint64_t nw = uint64_t(gridDim.x) * blockDim.x / 32;
    const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const uint64_t steps = nvec / 128;
    const uint64_t per = (steps + nw - 1) / nw;
    const uint64_t s0 = w * per, s1 = s0 + per < steps ? s0 + per : steps;
    const uint32_t base = smem_u32(ring + warp * S * 128);
    auto issue = [&](uint64_t s) {
        if (s < s1) {
            const uint32_t st = uint32_t((s - s0) % S);
#pragma unroll
            for (int u = 0; u < 4; ++u) cp_async16(base + (st * 128 + u * 32 + lane) * 16, a + s * 128 + u * 32 + lane);
        }
        cp_commit();
    };
    for (int i = 0; i < S - 1; ++i) issue(s0 + i);
    int m = 0x7FFFFFFF;
    for (uint64_t s = s0; s < s1; ++s) {
        issue(s + S - 1);
        cp_wait<S - 1>();
        const uint32_t st = uint32_t((s - s0) % S);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int4 x = lds128(base + (st * 128 + u * 32 + lane) * 16);
            m = __vimin3_s32(m, x.x, x.y);
            m = __vimin3_s32(m, x.z, x.w);
        }
    }
    m = __reduce_min_sync(0xffffffffu, m);
    if (lane == 0 && m == 0x12345678) atomicAdd(out, 1u);
}

// persistent per-warp pieces, LDG into registers (prefetch 1 step), then a
// transposed round trip through shared memory (STS, syncwarp, LDS of the lane's row)
__global__ void k_ldg_sts(const int4* __restrict__ a, uint64_t nvec, unsigned* out) {
    __shared__ int4 sx[8][128];
    const uint64_t nw = uint64_t(gridDim.x) * blockDim.x / 32;
    const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint64_t steps = nvec / 128;
    const uint64_t per = (steps + nw - 1) / nw;
    const uint64_t s0 = w * per, s1 = s0 + per < steps ? s0 + per : steps;
    int m = 0x7FFFFFFF;
    int4 y[4];
    if (s0 < s1)
#pragma unroll
        for (int u = 0; u < 4; ++u) y[u] = ld_stream_v4(a + s0 * 128 + u * 32 + lane);
    for (uint64_t s = s0; s < s1; ++s) {
        int4 x[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) x[u] = y[u];
        if (s + 1 < s1)
#pragma unroll
            for (int u = 0; u < 4; ++u) y[u] = ld_stream_v4(a + (s + 1) * 128 + u * 32 + lane);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const uint32_t row = 8u * u + (lane >> 2), c = lane & 3u;
            sx[warp][4 * row + (c ^ ((row >> 1) & 3u))] = x[u];
        }
        __syncwarp();
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const int4 v = sx[warp][4 * lane + (q ^ ((lane >> 1) & 3u))];
            m = __vimin3_s32(m, v.x, v.y);
            m = __vimin3_s32(m, v.z, v.w);
        }
        __syncwarp();
    }
    m = __reduce_min_sync(0xffffffffu, m);
    if (lane == 0 && m == 0x12345678) atomicAdd(out, 1u);
}

// non-persistent, one warp per 4 KB warp tile (8 x 16 B per lane in flight), the
// contraction's shared-memory transpose, lane r reads row r; residency set by
// the dynamic shared memory the launch asks for
__global__ void k_ldg8_sts(const int4* __restrict__ a, uint64_t nvec, unsigned* out) {
    __shared__ __align__(128) int4 sx[8][256];
    const uint64_t w = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (w * 256 >= nvec) return;
    int4 y[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) y[u] = ld_stream_v4(a + w * 256 + u * 32 + lane);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
        const uint32_t row = 4u * u + (lane >> 3), ch = lane & 7u;
        sx[warp][row * 8u + (ch ^ (row & 7u))] = y[u];
    }
    __syncwarp();
    int m = 0x7FFFFFFF;
#pragma unroll
    for (int c = 0; c < 8; ++c) {
        const int4 v = sx[warp][lane * 8u + (c ^ (lane & 7u))];
        m = __vimin3_s32(m, v.x, v.y);
        m = __vimin3_s32(m, v.z, v.w);
    }
    m = __reduce_min_sync(0xffffffffu, m);
    if (lane == 0 && m == 0x12345678) atomicAdd(out, 1u);
}

// persistent 4 KB warp tiles with the contraction's transpose and one tile of
// prefetch; the tiles a warp takes: CH = 0 one contiguous piece per warp (the
// contraction today), else chunks of CH consecutive tiles dealt round-robin over
// the warps (the grid sweeps A front to back, the tail is balanced to one chunk)
template <int CH>
__global__ void k_ldg8p_sts(const int4* __restrict__ a, uint64_t nvec, unsigned* out) {
    __shared__ __align__(128) int4 sx[8][256];
    const uint32_t nw = gridDim.x * blockDim.x / 32;
    const uint32_t w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const unsigned lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t tiles = uint32_t(nvec / 256);
    auto tile_at = [&](uint32_t i) -> uint32_t {  // i-th tile of this warp, or ~0u
        if (CH == 0) {
            const uint32_t per = (tiles + nw - 1) / nw, t = w * per + i;
            return i < per && t < tiles ? t : ~0u;
        }
        constexpr uint32_t C = CH ? CH : 1;
        const uint32_t t = ((i / C) * nw + w) * C + i % C;
        return t < tiles ? t : ~0u;
    };
    int m = 0x7FFFFFFF;
    int4 y[8];
    uint32_t t = tile_at(0);
    if (t != ~0u)
#pragma unroll
        for (int u = 0; u < 8; ++u) y[u] = ld_stream_v4(a + uint64_t(t) * 256 + u * 32 + lane);
    for (uint32_t i = 0; t != ~0u; ++i) {
        int4 x[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) x[u] = y[u];
        t = tile_at(i + 1);
        if (t != ~0u)
#pragma unroll
            for (int u = 0; u < 8; ++u) y[u] = ld_stream_v4(a + uint64_t(t) * 256 + u * 32 + lane);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint32_t row = 4u * u + (lane >> 3), ch = lane & 7u;
            sx[warp][row * 8u + (ch ^ (row & 7u))] = x[u];
        }
        __syncwarp();
#pragma unroll
        for (int c = 0; c < 8; ++c) {
            const int4 v = sx[warp][lane * 8u + (c ^ (lane & 7u))];
            m = __vimin3_s32(m, v.x, v.y);
            m = __vimin3_s32(m, v.z, v.w);
        }
        __syncwarp();
    }
    m = __reduce_min_sync(0xffffffffu, m);
    if (lane == 0 && m == 0x12345678) atomicAdd(out, 1u);
}

// persistent: CTA c streams contiguous range of tiles; S stages of T bytes.
template <bool TMA2D>
__global__ void k_ring(const __grid_constant__ CUtensorMap tmap, const int32_t* __restrict__ a,
                       uint64_t ntiles, uint32_t T, uint32_t S, unsigned* out) {
    extern __shared__ unsigned char raw[];
    const uint32_t r0 = smem_u32(raw);
    const uint32_t sb = (r0 + 1023u) & ~1023u;
    unsigned char* base = raw + (sb - r0);
    uint64_t* full = reinterpret_cast<uint64_t*>(base + S * T);
    const uint64_t per = (ntiles + gridDim.x - 1) / gridDim.x;
    const uint64_t t0 = blockIdx.x * per;
    const uint64_t t1 = t0 + per < ntiles ? t0 + per : ntiles;
    if (t0 >= t1) return;
    const uint64_t cnt = t1 - t0;
    const unsigned tid = threadIdx.x, nt = blockDim.x;
    auto issue = [&](uint64_t i) {
        const uint32_t st = uint32_t(i % S);
        fence_proxy_async();
        mbar_arrive_expect_tx(&full[st], T);
        if (TMA2D)
            tma_load_2d(base + st * T, &tmap, 0, int((t0 + i) * (T / 128)), &full[st]);
        else
            bulk_g2s(base + st * T, a + (t0 + i) * (T / 4), T, &full[st]);
    };
    if (tid == 0) {
        for (uint32_t s = 0; s < S; ++s) mbar_init(&full[s], 1);
        fence_mbar_init();
        for (uint64_t i = 0; i < cnt && i < S; ++i) issue(i);
    }
    __syncthreads();
    int m = 0x7FFFFFFF;
    for (uint64_t i = 0; i < cnt; ++i) {
        const uint32_t st = uint32_t(i % S);
        mbar_wait(&full[st], uint32_t(i / S) & 1u);
        const uint32_t sa = sb + st * T;
        for (uint32_t o = tid * 16; o < T; o += nt * 16) {
            const int4 x = lds128(sa + o);
            m = __vimin3_s32(m, x.x, x.y);
            m = __vimin3_s32(m, x.z, x.w);
        }
        __syncthreads();
        if (tid == 0 && i + S < cnt) issue(i + S);
    }
    m = __reduce_min_sync(0xffffffffu, m);
    if ((tid & 31) == 0 && m == 0x12345678) atomicAdd(out, 1u);
}

int main(int argc, char** argv) {
    const uint64_t n = argc > 1 ? strtoull(argv[1], nullptr, 10) : 100000000ull;
    const uint64_t nbytes = n * 4;
    int32_t* a;
    cudaMalloc(&a, nbytes + (1 << 20));
    cudaMemset(a, 1, nbytes);
    unsigned* out;
    cudaMalloc(&out, 4);
    char* flush;
    const size_t fb = size_t(512) << 20;
    cudaMalloc(&flush, fb);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto timeit = [&](const char* name, auto&& launch) {
        std::vector<float> v;
        for (int it = 0; it < 8; ++it) {
            cudaMemsetAsync(flush, it, fb);  // evict A from L2 ...
            k_ldg<<<unsigned(fb / 16 / 128 * 32 / 256), 256>>>(reinterpret_cast<int4*>(flush), fb / 16, out);
            // ... and drain the memset's dirty lines before the window (bench.py's L2Flush)
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            if (it >= 2) v.push_back(ms);
        }
        float s = 0;
        for (float x : v) s += x;
        s /= v.size();
        const cudaError_t err = cudaGetLastError();
        printf("%-28s %8.2f us  %7.0f GB/s  %s\n", name, s * 1e3, nbytes / (s * 1e-3) / 1e9,
               err == cudaSuccess ? "" : cudaGetErrorString(err));
    };
    const uint64_t nvec = n / 4;
    for (int tpb : {128, 256, 512})
        timeit((std::string("ldg tpb=") + std::to_string(tpb)).c_str(), [&] {
            k_ldg<<<unsigned((nvec / 128 * 32 + tpb - 1) / tpb), tpb>>>(reinterpret_cast<int4*>(a), nvec, out);
        });
    for (int per : {4, 8, 16})
        timeit((std::string("ldgp warps/sm=") + std::to_string(per * 8)).c_str(), [&] {
            k_ldgp<<<sms * per, 256>>>(reinterpret_cast<int4*>(a), nvec, out);
        });
    for (int per : {4, 8})
        for (int pf = 0; pf < 2; ++pf)
            timeit((std::string("ldgc pf=") + std::to_string(pf) + " warps/sm=" + std::to_string(per * 8)).c_str(), [&] {
                if (pf) k_ldgc<true><<<sms * per, 256>>>(reinterpret_cast<int4*>(a), nvec, out);
                else k_ldgc<false><<<sms * per, 256>>>(reinterpret_cast<int4*>(a), nvec, out);
            });
    for (int per : {3, 4, 6})
        timeit((std::string("ldg+sts warps/sm=") + std::to_string(per * 8)).c_str(), [&] {
            k_ldg_sts<<<sms * per, 256>>>(reinterpret_cast<int4*>(a), nvec, out);
        });
    for (int per : {2, 3, 4, 8}) {
        const int smem = (200 * 1024) / per - 32 * 1024 - 1024;  // static 32 KB + dynamic
        cudaFuncSetAttribute(k_ldg8_sts, cudaFuncAttributeMaxDynamicSharedMemorySize, smem > 0 ? smem : 0);
        timeit((std::string("ldg8+sts np cta/sm=") + std::to_string(per)).c_str(), [&] {
            k_ldg8_sts<<<unsigned((nvec / 256 * 32 + 255) / 256), 256, smem > 0 ? smem : 0>>>(
                reinterpret_cast<int4*>(a), nvec, out);
        });
    }
    auto p8 = [&](auto kern, const char* nm) {
        for (int per : {2, 3})
            timeit((std::string(nm) + " cta/sm=" + std::to_string(per)).c_str(),
                   [&] { kern<<<sms * per, 256>>>(reinterpret_cast<int4*>(a), nvec, out); });
    };
    p8(k_ldg8p_sts<0>, "p8 contiguous");
    p8(k_ldg8p_sts<1>, "p8 chunk=1");
    p8(k_ldg8p_sts<2>, "p8 chunk=2");
    p8(k_ldg8p_sts<4>, "p8 chunk=4");
    p8(k_ldg8p_sts<8>, "p8 chunk=8");
    if (argc > 3) return 0;
    auto cpa = [&](auto kern, int S, int cpsm) {
        const size_t smem = size_t(8) * S * 2048;
        cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
        char name[64];
        snprintf(name, sizeof name, "cp.async S=%d cta/sm=%d", S, cpsm);
        timeit(name, [&] { kern<<<sms * cpsm, 256, smem>>>(reinterpret_cast<int4*>(a), nvec, out); });
    };
    cpa(k_cpa<2>, 2, 4); cpa(k_cpa<3>, 3, 3); cpa(k_cpa<4>, 4, 3); cpa(k_cpa<4>, 4, 2); cpa(k_cpa<6>, 6, 2); cpa(k_cpa<8>, 8, 1);
    if (argc > 2) return 0;
    CUtensorMap tm;
    for (uint32_t T : {4096u, 8192u, 16384u, 32768u}) {
        for (uint32_t S : {2u, 3u, 4u, 6u}) {
            const size_t smem = 1024 + size_t(S) * T + 64;
            if (smem > 200 * 1024) continue;
            for (int tma2d = 0; tma2d < 2; ++tma2d) {
                if (tma2d && !make_tmap_rows128(&tm, a, n / 32, T / 128)) continue;
                auto kern = tma2d ? k_ring<true> : k_ring<false>;
                cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));
                int per = 0;
                cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, kern, 128, smem);
                const uint64_t ntiles = nbytes / T;
                char name[64];
                snprintf(name, sizeof name, "%s T=%u S=%u cta/sm=%d", tma2d ? "tma2d" : "bulk", T, S, per);
                timeit(name, [&] { kern<<<sms * per, 128, smem>>>(tm, a, ntiles, T, S, out); });
            }
        }
    }
    return 0;
}
