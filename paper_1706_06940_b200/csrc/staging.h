// staging.h -- host <-> device copies for host-pointer solves (api.cu).
//
// The reference API takes its inputs as std::span / std::vector (pageable
// memory, contraction.hpp:61-64, types.hpp:26).  cudaMemcpyAsync from pageable
// memory goes through the driver's own small bounce buffer; this stager moves
// pageable data through a double-buffered ring of pinned chunks instead, the
// CPU copy of chunk i+1 (spread over a persistent pool of host threads)
// overlapping the DMA of chunk i.  Pinned (page-locked / registered) buffers
// are copied directly.  Copies are issued on the context's stream; a staged
// H2D returns once its last chunk is enqueued, a staged D2H once the data is
// in the destination.
#pragma once

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

    static constexpr size_t kChunk = size_t(16) << 20;  // per ring slot

private:
    cudaError_t init();
    void par_copy(void* dst, const void* src, size_t bytes);
    void worker(unsigned id);

    bool ready_ = false;
    char* buf_[2] = {nullptr, nullptr};
    cudaEvent_t ev_[2] = {nullptr, nullptr};
    // copy pool: job = (dst, src, bytes) split into equal parts
    std::vector<std::thread> pool_;
    std::mutex mu_;
    std::condition_variable cv_, done_cv_;
    uint64_t gen_ = 0;
    unsigned pending_ = 0;
    bool stop_ = false;
    char* jdst_ = nullptr;
    const char* jsrc_ = nullptr;
    size_t jbytes_ = 0;
    unsigned parts_ = 1;
};

}  // namespace brmq
