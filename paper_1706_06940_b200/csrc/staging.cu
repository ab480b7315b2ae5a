// staging.cpp -- pinned-ring staging of pageable host buffers (staging.h).
#include "staging.h"

#include <algorithm>
#include <cstring>

namespace brmq {

Stager::~Stager() {
    {
        std::lock_guard<std::mutex> lk(mu_);
        stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : pool_) t.join();
    for (int b = 0; b < 2; ++b) {
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
    for (int b = 0; b < 2; ++b) {
        if (cudaError_t e = cudaHostAlloc(reinterpret_cast<void**>(&buf_[b]), kChunk, cudaHostAllocDefault))
            return e;
        if (cudaError_t e = cudaEventCreateWithFlags(&ev_[b], cudaEventDisableTiming)) return e;
    }
    // memcpy threads: a few are enough to outrun PCIe (measured ~8-12 GB/s each)
    unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    parts_ = std::min(8u, hw);
    for (unsigned i = 1; i < parts_; ++i) pool_.emplace_back(&Stager::worker, this, i);
    ready_ = true;
    return cudaSuccess;
}

void Stager::worker(unsigned id) {
    uint64_t seen = 0;
    for (;;) {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
        if (stop_) return;
        seen = gen_;
        char* d = jdst_;
        const char* s = jsrc_;
        const size_t n = jbytes_, per = (n + parts_ - 1) / parts_;
        lk.unlock();
        const size_t a = std::min(n, size_t(id) * per), b = std::min(n, a + per);
        if (b > a) std::memcpy(d + a, s + a, b - a);
        lk.lock();
        if (--pending_ == 0) done_cv_.notify_one();
    }
}

void Stager::par_copy(void* dst, const void* src, size_t bytes) {
    if (parts_ <= 1 || bytes < (size_t(1) << 20)) {
        std::memcpy(dst, src, bytes);
        return;
    }
    {
        std::lock_guard<std::mutex> lk(mu_);
        jdst_ = static_cast<char*>(dst);
        jsrc_ = static_cast<const char*>(src);
        jbytes_ = bytes;
        pending_ = parts_ - 1;
        ++gen_;
    }
    cv_.notify_all();
    const size_t per = (bytes + parts_ - 1) / parts_;
    std::memcpy(dst, src, std::min(bytes, per));  // part 0 on the calling thread
    std::unique_lock<std::mutex> lk(mu_);
    done_cv_.wait(lk, [&] { return pending_ == 0; });
}

cudaError_t Stager::h2d(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return cudaSuccess;
    if (bytes < (size_t(1) << 20) || is_pinned(src))
        return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, s);
    if (cudaError_t e = init()) return e;
    for (size_t off = 0, i = 0; off < bytes; off += kChunk, ++i) {
        const int b = int(i & 1);
        const size_t len = std::min(kChunk, bytes - off);
        if (cudaError_t e = cudaEventSynchronize(ev_[b])) return e;  // its previous DMA is done
        par_copy(buf_[b], static_cast<const char*>(src) + off, len);
        if (cudaError_t e = cudaMemcpyAsync(static_cast<char*>(dst) + off, buf_[b], len,
                                            cudaMemcpyHostToDevice, s))
            return e;
        if (cudaError_t e = cudaEventRecord(ev_[b], s)) return e;
    }
    return cudaSuccess;
}

cudaError_t Stager::d2h(void* dst, const void* src, size_t bytes, cudaStream_t s) {
    if (bytes == 0) return cudaSuccess;
    if (bytes < (size_t(1) << 20) || is_pinned(dst))
        return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, s);
    if (cudaError_t e = init()) return e;
    const size_t chunks = (bytes + kChunk - 1) / kChunk;
    auto issue = [&](size_t i) -> cudaError_t {
        const int b = int(i & 1);
        const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
        if (cudaError_t e = cudaMemcpyAsync(buf_[b], static_cast<const char*>(src) + off, len,
                                            cudaMemcpyDeviceToHost, s))
            return e;
        return cudaEventRecord(ev_[b], s);
    };
    if (cudaError_t e = issue(0)) return e;
    for (size_t i = 0; i < chunks; ++i) {
        if (i + 1 < chunks) {  // the next chunk's DMA overlaps this chunk's CPU copy
            // its slot's previous copy-out finished (sequentially) before this point
            if (cudaError_t e = issue(i + 1)) return e;
        }
        const int b = int(i & 1);
        if (cudaError_t e = cudaEventSynchronize(ev_[b])) return e;
        const size_t off = i * kChunk, len = std::min(kChunk, bytes - off);
        par_copy(static_cast<char*>(dst) + off, buf_[b], len);
    }
    return cudaSuccess;
}

}  // namespace brmq
