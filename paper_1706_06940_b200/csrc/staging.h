// staging.h -- host <-> device copies for host-pointer solves (api.cu).
//
// The reference API takes its inputs as std::span / std::vector (pageable
// memory, contraction.hpp:61-64, types.hpp:26).  cudaMemcpyAsync from pageable
// memory goes through the driver's own small bounce buffer; this stager moves
// pageable data through a ring of pinned chunks instead (3 slots; chunk sizes
// grow from 1 MiB to 16 MiB, so the first DMA starts early): the CPU copy of
// chunk i+1, spread over a persistent pool of spinning host threads, overlaps
// the DMA of chunk i.  Pinned (page-locked / registered) buffers are copied
// directly.  Copies are issued on the context's stream; a staged H2D returns
// once its last chunk is enqueued, a staged D2H once the data is in the
// destination.  Measured (c2, 400 MB, 16-core host, tools/stage_ab.py): a
// pageable solve 7.9 ms vs 7.4 ms from pinned buffers and 35 ms through the
// driver's own pageable path; 2 MiB chunks 12.3 ms, 8 MiB 8.0-8.4 ms (per-chunk
// DMA / API cost).
#pragma once

#include <atomic>
#include <condition_variable>
#include <cstddef>
#include <cstdint>
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

namespace brmq {

class Stager {
public:
    Stager() = default;
    ~Stager();
    Stager(const Stager&) = delete;
    Stager& operator=(const Stager&) = delete;

    // dst (device) <- src (host) / dst (host) <- src (device), on stream s
    cudaError_t h2d(void* dst, const void* src, size_t bytes, cudaStream_t s);
    cudaError_t d2h(void* dst, const void* src, size_t bytes, cudaStream_t s);
    static bool is_pinned(const void* p);


private:
    cudaError_t init();
    void par_copy(void* dst, const void* src, size_t bytes);
    void worker(unsigned id);

    static constexpr unsigned kSlots = 3;
    static constexpr size_t kHead = size_t(1) << 20;  // first chunk of a staged H2D
    bool ready_ = false;
    bool debug_ = false;
    size_t chunk_ = size_t(16) << 20;  // per ring slot
    char* buf_[kSlots] = {};
    cudaEvent_t ev_[kSlots] = {};
    unsigned slot_ = 0;  // next ring slot of a staged H2D
    // copy pool: job = (dst, src, bytes) split into equal parts, published by a
    // bump of gen_; workers spin between jobs (staging.cu)
    std::vector<std::thread> pool_;
    std::mutex mu_;
    std::condition_variable cv_;
    std::atomic<uint64_t> gen_{0};
    std::atomic<unsigned> pending_{0};
    std::atomic<unsigned> sleepers_{0};
    std::atomic<bool> stop_{false};
    char* jdst_ = nullptr;
    const char* jsrc_ = nullptr;
    size_t jbytes_ = 0;
    unsigned parts_ = 1;
};

}  // namespace brmq
