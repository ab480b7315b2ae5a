// staging.cpp -- pinned-ring staging of pageable host buffers (staging.h).
#include "staging.h"

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>

namespace brmq {

Stager::~Stager() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_.store(true);
    }
    cv_.notify_all();
    for (auto& t : pool_) t.join();
    for (unsigned b = 0; b < kSlots; ++b) {
        if (ev_[b]) cudaEventDestroy(ev_[b]);
        if (buf_[b]) cudaFreeHost(buf_[b]);
    }
}

bool Stager::is_pinned(const void* p) {
    cudaPointerAttributes a{};
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();  // unregistered pointers may report an error on older drivers
        return false;
    }
    return a.type == cudaMemoryTypeHost || a.type == cudaMemoryTypeManaged;
}

cudaError_t Stager::init() {
    if (ready_) return cudaSuccess;
    if (const char* g = getenv("BRMQ_STAGE_CHUNK_KB")) chunk_ = size_t(atol(g)) << 10;
    if (const char* g = getenv("BRMQ_STAGE_DEBUG")) debug_ = atoi(g) != 0;
    for (unsigned b = 0; b < kSlots; ++b) {
        if (cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&buf_[b]), chunk_, cudaHostAllocDefault))
            return e;
        if (cudaError_t e = cudaEventCreateWithFlags(&ev_[b], cudaEventDisableTiming)) return e;
    }
    // memcpy threads: a few are enough to outrun PCIe (measured ~8-12 GB/s each)
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    parts_ = std::min(8u, hw);
    if (const char* g = getenv("BRMQ_STAGE_THREADS")) parts_ = std::max(1, atoi(g));
    for (unsigned i = 1; i < parts_; ++i) pool_.emplace_back(&Stager::worker, this, i);
    ready_ = true;
    return cudaSuccess;
}

// Workers spin on the job generation while copies keep coming (a staged H2D
// hands out one job per chunk; a futex wake per job costs tens of microseconds),
// and sleep on the condition variable after kSpinMs without one.
namespace {
constexpr double kSpinMs = 2.0;
inline void cpu_relax() {
#if defined(__x86_64__) || defined(__i386__)
    __builtin_ia32_pause();
#endif
}
}  // namespace

void Stager::worker(unsigned id) {
    uint64_t seen = 0;
    for (;;) {
        uint64_t g;
        auto t0 = std::chrono::steady_clock::now();
        for (unsigned spins = 0; (g = gen_.load()) == seen;) {
            if (stop_.load()) return;
            cpu_relax();
            if ((++spins & 1023u) == 0 &&
                std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count() > kSpinMs) {
                std::unique_lock<std::mutex> lk(mu_);
                ++sleepers_;
                cv_.wait(lk, [&] { return stop_.load() || gen_.load() != seen; });
                --sleepers_;
                t0 = std::chrono::steady_clock::now();
            }
        }
        seen = g;
        char* d = jdst_;
        const char* s = jsrc_;
        const size_t n = jbytes_, per = (n + parts_ - 1) / parts_;
        const size_t a = std::min(n, size_t(id) * per), b = std::min(n, a + per);
        if (b > a) std::memcpy(d + a, s + a, b - a);
        pending_.fetch_sub(1);
    }
}

void Stager::par_copy(void* dst, const void* src, size_t bytes) {
    if (parts_ <= 1 || bytes < (size_t(1) << 20)) {
        std::memcpy(dst, src, bytes);
        return;
    }
    jdst_ = static_cast<char*>(dst);  // published by the generation bump below
    jsrc_ = static_cast<const char*>(src);
    jbytes_ = bytes;
    pending_.store(parts_ - 1);
    gen_.fetch_add(1);
    if (sleepers_.load() > 0) {
        std::lock_guard<std::mutex> lk(mu_);
        cv_.notify_all();
    }
    const size_t per = (bytes + parts_ - 1) / parts_;
    std::memcpy(dst, src, std::min(bytes, per));  // part 0 on the calling thread
    while (pending_.load() != 0) cpu_relax();
}

cudaError_t Stager::h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return cudaSuccess;
    static const bool off_ = getenv("BRMQ_STAGE") && atoi(getenv("BRMQ_STAGE")) == 0;
    if (bytes < (size_t(1) << 20) || off_ || is_pinned(src))
        return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
    if (cudaError_t e = init()) return e;
    using clk = std::chrono::steady_clock;
    double t_wait = 0, t_copy = 0;
    const auto t0 = clk::now();
    // chunk sizes grow from kHead to chunk_: the first DMA starts after a short copy
    size_t len = std::min(kHead, chunk_);
    for (size_t off = 0; off < bytes; off += len, len = std::min(2 * len, chunk_)) {
        len = std::min(len, bytes - off);
        const unsigned b = slot_;
        slot_ = (slot_ + 1) % kSlots;
        const auto a = clk::now();
        if (cudaError_t e = cudaEventSynchronize(ev_[b])) return e;  // its previous DMA is done
        const auto m = clk::now();
        par_copy(buf_[b], static_cast<const char*>(src) + off, len);
        t_wait += std::chrono::duration<double, std::milli>(m - a).count();
        t_copy += std::chrono::duration<double, std::milli>(clk::now() - m).count();
        if (cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + off, buf_[b], len,
                                            cudaMemcpyHostToDevice, s))
            return e;
        if (cudaError_t e = cudaEventRecord(ev_[b], s)) return e;
    }
    if (debug_)
        std::fprintf(stderr, "stage h2d %zu B: %.3f ms total, %.3f ms copy (%.1f GB/s), %.3f ms waiting\n", bytes,
                     std::chrono::duration<double, std::milli>(clk::now() - t0).count(), t_copy,
                     bytes / t_copy * 1e-6, t_wait);
    return cudaSuccess;
}

cudaError_t Stager::d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return cudaSuccess;
    static const bool off_ = getenv("BRMQ_STAGE") && atoi(getenv("BRMQ_STAGE")) == 0;
    if (bytes < (size_t(1) << 20) || off_ || is_pinned(dst))
        return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
    if (cudaError_t e = init()) return e;
    const size_t chunks = (bytes + chunk_ - 1) / chunk_;
    // every slot's earlier use is complete: the copy-outs below are synchronous
    for (unsigned b = 0; b < kSlots; ++b)
        if (cudaError_t e = cudaEventSynchronize(ev_[b])) return e;
    auto issue = [&](size_t i) -> cudaError_t {
        const unsigned b = unsigned(i % kSlots);
        const size_t off = i * chunk_, len = std::min(chunk_, bytes - off);
        if (cudaError_t e = cudaMemcpyAsync(buf_[b], static_cast<const char*>(src) + off, len,
                                            cudaMemcpyDeviceToHost, s))
            return e;
        return cudaEventRecord(ev_[b], s);
    };
    // up to kSlots - 1 DMAs ahead of the chunk being copied out
    for (size_t i = 0; i + 1 < kSlots && i < chunks; ++i)
        if (cudaError_t e = issue(i)) return e;
    for (size_t i = 0; i < chunks; ++i) {
        if (i + kSlots - 1 < chunks)  // that slot's previous copy-out finished before this point
            if (cudaError_t e = issue(i + kSlots - 1)) return e;
        const unsigned b = unsigned(i % kSlots);
        if (cudaError_t e = cudaEventSynchronize(ev_[b])) return e;
        const size_t off = i * chunk_, len = std::min(chunk_, bytes - off);
        par_copy(static_cast<char*>(dst) + off, buf_[b], len);
    }
    return cudaSuccess;
}

}  // namespace brmq
