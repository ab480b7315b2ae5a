// api.cu -- the C-ABI (include/brmq.h): context, workspace, validation and the
// stream-ordered orchestration of the sm_100a kernels.
//
// Each extern "C" entry point stands in for one reference function (see
// brmq.h for the file:line map).  The host code never computes an answer: if
// the device path cannot run the call fails with BRMQ_ECUDA -- there is no CPU
// fallback anywhere in this library.
#include <cstdarg>
#include <cstddef>
#include <cstdlib>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../include/brmq.h"
#include "common.cuh"
#include "errors.h"
#include "kernels.h"
#include "staging.h"

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof(buf), fmt, ap);
    va_end(ap);
    g_last_error = buf;
    return code;
}

}  // namespace

int brmq::set_error(int code, const char* msg) {
    g_last_error = msg;
    return code;
}

namespace {

#define CUDA_TRY(expr)                                                                      \
    do {                                                                                    \
        cudaError_t e_ = (expr);                                                            \
        if (e_ != cudaSuccess)                                                              \
            return fail(e_ == cudaErrorMemoryAllocation ? BRMQ_ENOMEM : BRMQ_ECUDA,        \
                        "%s: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
    } while (0)

constexpr size_t kAlign = 256;
inline size_t align_up(size_t x, size_t a = kAlign) { return (x + a - 1) / a * a; }

// Control block of one call: zeroed by one memset at the start of every solve.
struct Control {
    uint32_t err;       // 1 query out of range (direct), 2 range (collect/unique), 4 unsorted, 8 logic
    uint32_t span[2];   // [~min endpoint, max endpoint]
    uint32_t tickets[5];  // last-CTA tickets: [0] k_unique
    uint64_t array_reads;  // positions of A the contraction consumed (ContractionStats)
    uint64_t scanned;      // cells of A the h = 1 query scans covered (debug counter)
    uint64_t nb;        // |boundary|
    uint64_t aq_len;    // |A_Q|
    uint64_t b_dev;     // blocks over A_Q
    // boundaries per contraction range (bitmap pipeline: k_piece_count) or their
    // exclusive prefix (radix pipeline / stage API: k_unique); fully rewritten by
    // every solve, so only the header above is zeroed and copied back
    uint32_t rcnt[brmq::kMaxContractRanges + 1];
};
constexpr size_t kCtlHeader = offsetof(Control, rcnt);
static_assert(kCtlHeader % 4 == 0, "header copied as u32 words");

}  // namespace

struct GraphKey {
    int kind;
    const void* A;
    uint64_t n;
    const void* Q;
    uint64_t q;
    uint32_t k;
    int sort_kind;
    void* ans;
    cudaStream_t stream;
    bool operator==(const GraphKey& o) const {
        return kind == o.kind && A == o.A && n == o.n && Q == o.Q && q == o.q && k == o.k &&
               sort_kind == o.sort_kind && ans == o.ans && stream == o.stream;
    }
};

struct brmq_ctx {
    int device = 0;
    cudaStream_t own = nullptr;
    cudaStream_t stream = nullptr;
    char* ws = nullptr;  // grow-only workspace (zeroed on growth)
    size_t ws_cap = 0;
    char* st = nullptr;  // grow-only arena that only ever holds epoch-tagged status words
    size_t st_cap = 0;   // (so stale bytes can never alias a live epoch); zeroed on growth
    uint32_t* bitmap = nullptr;  // persistent, kept all-zero by the contraction kernel
    char* aux = nullptr;  // grow-only buffers of the sharded solves (clipped queries, keys)
    size_t aux_cap = 0;
    size_t bitmap_words = 0;
    Control* ctl_host = nullptr;  // pinned, device-mapped mirror of the control header
    uint32_t* ctl_host_dev = nullptr;  // its device address (solves publish into it)
    bool ctl_clean = false;  // the device control header is all-zero (no memset needed)
    uint32_t* epoch_dev = nullptr;  // device epoch counter, bumped by every solve (graph-safe)
    uint32_t epoch_host = 1;        // host mirror of *epoch_dev
    bool use_graphs = true;
    bool use_pdl = false;  // programmatic dependent launches inside a solve (BRMQ_PDL=1: on; DESIGN 3.5)
    bool count_scans = false;  // brmq_ctx_set_counters
    bool use_msd = true;  // radix pipeline: MSD partition + bucket marks (BRMQ_MSD=0: LSD over all digits)
    // small A_Q: block / sub-block minima by reductions inside the contraction
    // (BRMQ_FUSE=1: on).  Off: measured -1 us at c2 in one harness and +16 us in
    // bench.py's process (DESIGN 3.1)
    bool use_fuse = false;
    // BbST_CON: the contraction and the query kernel as PDL secondaries of their
    // predecessors, each issuing its independent loads before its wait (BRMQ_PDL_QUERY=0: off)
    bool pdl_query = true;
    // brmq_ctx_set_async: device-pointer solves (BbST, [32, k], BbST_CON) return as
    // soon as they are enqueued; brmq_synchronize waits, fills the solve info and
    // returns the last solve's status (pending_fill)
    bool async_mode = false;
    bool async_pending = false;
    std::function<void()> pending_fill;
    struct GraphEntry;
    std::vector<GraphEntry*> graphs;
    // timing: 0 off, 1 every stage, 2 only the roofline kernel (contract / block_argmin)
    int timing = 0;
    std::vector<cudaEvent_t> ev;
    std::vector<std::string> stage_names;
    std::vector<uint32_t> stage_launches;
    brmq_stage_times last_times{};
    brmq_solve_info info{};
    brmq::Stager stager;  // host-pointer solves: pinned-ring staging of pageable buffers
};

// A captured solve: replaying it re-runs every kernel with the same buffers;
// the look-back epochs come from the device counter the graph itself bumps.
struct brmq_ctx::GraphEntry {
    GraphKey key;
    cudaGraphExec_t exec = nullptr;
    int launches = 0;
    int timing = 0;
    std::vector<std::string> names;
    std::vector<uint32_t> nl;
};

namespace {

// Bump allocator over the context workspace; call plan() for every buffer,
// then commit() (grows the workspace if needed), then get pointers by index.
struct Carve {
    std::vector<size_t> off;
    size_t total = 0;
    size_t add(size_t bytes) {
        off.push_back(total);
        total += align_up(bytes ? bytes : 1);
        return off.size() - 1;
    }
};

void drop_graphs(brmq_ctx* c) {
    for (auto* g : c->graphs) {
        if (g->exec) cudaGraphExecDestroy(g->exec);
        delete g;
    }
    c->graphs.clear();
}

int ensure_ws(brmq_ctx* c, size_t bytes) {
    if (bytes <= c->ws_cap) return BRMQ_OK;
    drop_graphs(c);
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (c->ws) cudaFree(c->ws);
    c->ws = nullptr;
    c->ws_cap = 0;
    size_t cap = align_up(bytes + bytes / 8, 1 << 21);
    CUDA_TRY(cudaMalloc(&c->ws, cap));
    CUDA_TRY(cudaMemsetAsync(c->ws, 0, cap, c->stream));
    c->ws_cap = cap;
    c->ctl_clean = true;
    return BRMQ_OK;
}

int ensure_status(brmq_ctx* c, size_t bytes) {
    if (bytes <= c->st_cap) return BRMQ_OK;
    drop_graphs(c);
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (c->st) cudaFree(c->st);
    c->st = nullptr;
    c->st_cap = 0;
    const size_t cap = align_up(bytes + bytes / 8, 1 << 20);
    CUDA_TRY(cudaMalloc(&c->st, cap));
    CUDA_TRY(cudaMemsetAsync(c->st, 0, cap, c->stream));
    c->st_cap = cap;
    return BRMQ_OK;
}

int ensure_bitmap(brmq_ctx* c, uint64_t n) {
    const size_t words = brmq::contract_bitmap_words(n);  // whole tiles
    if (words <= c->bitmap_words) return BRMQ_OK;
    drop_graphs(c);
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (c->bitmap) cudaFree(c->bitmap);
    c->bitmap = nullptr;
    c->bitmap_words = 0;
    CUDA_TRY(cudaMalloc(&c->bitmap, words * 4));
    CUDA_TRY(cudaMemsetAsync(c->bitmap, 0, words * 4, c->stream));
    c->bitmap_words = words;
    return BRMQ_OK;
}

__global__ void k_bump_epoch(uint32_t* epoch, uint32_t by) {
    brmq::pdl_wait();
    *epoch += by;
}

// Every solve reserves `count` consecutive 24-bit epochs for its single-pass
// scans: one tiny kernel bumps the device counter first, and each look-back
// kernel reads *epoch_dev + its offset.  Inside a CUDA graph the bump is a node,
// so replays get fresh epochs too.  Before the 24-bit tag would wrap, the status
// arena is cleared and the counter restarted (outside any graph).
int begin_epochs(brmq_ctx* c, uint32_t count) {
    if (c->epoch_host + count + 1 >= (1u << 24)) {
        if (c->st) CUDA_TRY(cudaMemsetAsync(c->st, 0, c->st_cap, c->stream));
        c->epoch_host = 1;
        CUDA_TRY(cudaMemcpyAsync(c->epoch_dev, &c->epoch_host, 4, cudaMemcpyHostToDevice, c->stream));
        CUDA_TRY(cudaStreamSynchronize(c->stream));
    }
    return BRMQ_OK;
}

// ------------------------------------------------------------------ timing
struct Timer {
    brmq_ctx* c;
    int n = 0;
    explicit Timer(brmq_ctx* ctx) : c(ctx) {
        c->stage_names.clear();
        c->stage_launches.clear();
    }
    bool active = false;
    void stage(const char* name, int launches_before) {
        (void)launches_before;
        active = c->timing == 1 || (c->timing == 2 && (std::strcmp(name, "contract") == 0 ||
                                                        std::strcmp(name, "block_argmin") == 0));
        if (!active || n >= BRMQ_MAX_STAGES) return;
        record(c->ev[2 * n]);
        c->stage_names.emplace_back(name);
        c->stage_launches.push_back(0);
    }
    // timing level 3: two phases, "preprocess" (everything before the query kernel)
    // and "query" -- four event nodes per solve instead of two per stage
    bool ph_open = false;
    // device solves: the "preprocess" phase opens with a plain event recorded on
    // the stream before the graph launch (one event node fewer inside the graph;
    // the window then starts where the bench's own window does)
    void pre_launch(bool dev) {
        if (c->timing != 3 || !dev || n >= BRMQ_MAX_STAGES) return;
        cudaEventRecord(c->ev[2 * n], c->stream);
        c->stage_names.emplace_back("preprocess");
        c->stage_launches.push_back(0);
        ph_open = true;
    }
    void phase_begin(const char* name) {
        if (c->timing != 3 || n >= BRMQ_MAX_STAGES || ph_open) return;
        record(c->ev[2 * n]);
        c->stage_names.emplace_back(name);
        c->stage_launches.push_back(0);
        ph_open = true;
    }
    void phase_end(int launches) {
        if (!ph_open) return;
        record(c->ev[2 * n + 1]);
        c->stage_launches.back() = uint32_t(launches);
        ++n;
        ph_open = false;
    }
    void end(int launches) {
        if (!active || n >= BRMQ_MAX_STAGES) return;
        active = false;
        record(c->ev[2 * n + 1]);
        c->stage_launches.back() = uint32_t(launches);
        ++n;
    }
    // inside a stream capture the record must be an external event node
    void record(cudaEvent_t e) {
        cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
        cudaStreamIsCapturing(c->stream, &st);
        if (st == cudaStreamCaptureStatusActive)
            cudaEventRecordWithFlags(e, c->stream, cudaEventRecordExternal);
        else
            cudaEventRecord(e, c->stream);
    }
    void reset() {
        n = 0;
        c->stage_names.clear();
        c->stage_launches.clear();
    }
    void restore(const std::vector<std::string>& names, const std::vector<uint32_t>& nl) {
        c->stage_names = names;
        c->stage_launches = nl;
        n = int(names.size());
    }
    void finish() {
        brmq_stage_times& t = c->last_times;
        std::memset(&t, 0, sizeof(t));
        if (!c->timing) return;
        t.count = n;
        for (int i = 0; i < n; ++i) {
            std::snprintf(t.name[i], sizeof(t.name[i]), "%s", c->stage_names[i].c_str());
            float ms = 0.f;
            cudaEventElapsedTime(&ms, c->ev[2 * i], c->ev[2 * i + 1]);
            t.ms[i] = ms;
            t.launches[i] = c->stage_launches[i];
        }
    }
};

bool is_device(uint32_t flags) { return (flags & BRMQ_PTR_DEVICE) != 0; }

int check_status(brmq_ctx* c) {
    CUDA_TRY(cudaGetLastError());
    return BRMQ_OK;
}

int sync_and_read_control(brmq_ctx* c, const Control* ctl_dev) {
    CUDA_TRY(cudaMemcpyAsync(c->ctl_host, ctl_dev, kCtlHeader, cudaMemcpyDeviceToHost,
                             c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return BRMQ_OK;
}

int map_err(uint32_t err) {
    if (err & 8u) return fail(BRMQ_ELOGIC, "remap_queries_from_sorted: endpoint missing from boundary");
    if (err & 4u) return fail(BRMQ_EINVAL, "build_contracted: endpoints not sorted");
    if (err & 3u) return fail(BRMQ_ERANGE, "query exceeds array bounds");
    return BRMQ_OK;
}

// End of a solve.  Synchronous: wait, fill the solve info from the control header
// the final kernel published (host-mapped), return its status.  Async mode
// (device pointers, no stage timing): return at once; brmq_synchronize does the
// rest for the last solve.
template <class Fill>
int end_solve(brmq_ctx* c, bool dev, Timer& tm, Fill&& fill) {
    if (dev && c->async_mode && c->timing == 0) {
        tm.finish();
        c->pending_fill = std::function<void()>(fill);
        c->async_pending = true;
        return BRMQ_OK;
    }
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    tm.finish();
    fill();
    return map_err(c->ctl_host->err);
}

// A call on a context with an async solve outstanding settles it first (waits,
// fills the solve info, returns its status if it failed), so no error is dropped.
int settle_pending(brmq_ctx* c) {
    if (!c->async_pending) return BRMQ_OK;
    c->async_pending = false;
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    if (c->pending_fill) c->pending_fill();
    c->pending_fill = nullptr;
    return map_err(c->ctl_host->err);
}

int bits_for(uint64_t n) {  // bit_width(n - 1): positions are < n
    if (n <= 1) return 0;
    return 64 - __builtin_clzll(n - 1);
}


// Issues one solve: `enqueue` puts every async operation of the call on the
// context stream (ending with the D2H of the control block).  Device-pointer
// solves are captured once per (shape, pointers, stream) into a CUDA graph and
// replayed: one launch instead of ~10, no CPU launch gaps between kernels.
template <class F>
int run_solve(brmq_ctx* c, const GraphKey& key, bool graphable, Timer& tm, int& launches,
              F&& enqueue) {
    cudaStream_t s = c->stream;
    if (!(graphable && c->use_graphs)) return enqueue();
    brmq_ctx::GraphEntry* g = nullptr;
    for (auto* e : c->graphs)
        if (e->key == key && e->timing == c->timing) g = e;
    if (!g) {
        if (c->graphs.size() >= 16) {  // small LRU-less cache: drop the oldest
            cudaGraphExecDestroy(c->graphs.front()->exec);
            delete c->graphs.front();
            c->graphs.erase(c->graphs.begin());
        }
        cudaGraph_t graph = nullptr;
        CUDA_TRY(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
        const int rc = enqueue();
        const cudaError_t ee = cudaStreamEndCapture(s, &graph);
        cudaGraphExec_t exec = nullptr;
        if (rc == BRMQ_OK && ee == cudaSuccess &&
            cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess) {
            cudaGraphDestroy(graph);
            g = new brmq_ctx::GraphEntry();
            g->key = key;
            g->exec = exec;
            g->launches = launches;
            g->timing = c->timing;
            g->names = c->stage_names;
            g->nl = c->stage_launches;
            c->graphs.push_back(g);
        } else {  // not capturable here: run directly from now on
            if (graph) cudaGraphDestroy(graph);
            const cudaError_t why = cudaGetLastError();
            if (getenv("BRMQ_DEBUG"))
                fprintf(stderr, "brmq: graph capture failed (rc=%d end=%s last=%s); direct launches\n", rc,
                        cudaGetErrorString(ee), cudaGetErrorString(why));
            c->use_graphs = false;
            if (rc != BRMQ_OK) return rc;
            launches = 0;
            tm.reset();
            return enqueue();
        }
    } else {
        launches = g->launches;
        tm.restore(g->names, g->nl);
    }
    CUDA_TRY(cudaGraphLaunch(g->exec, s));
    c->info.graph = 1;
    return BRMQ_OK;
}

}  // namespace

extern "C" {

const char* brmq_last_error(void) { return g_last_error.c_str(); }

int brmq_floor_log2(uint64_t x, uint32_t* out) {
    if (x == 0) return fail(BRMQ_EDOMAIN, "floor_log2: argument must be positive");  // bits.hpp:11
    *out = 63u - uint32_t(__builtin_clzll(x));
    return BRMQ_OK;
}

int brmq_ctx_create(brmq_ctx** out, int device) {
    if (!out) return fail(BRMQ_EINVAL, "brmq_ctx_create: null out");
    *out = nullptr;
    int count = 0;
    CUDA_TRY(cudaGetDeviceCount(&count));
    if (device < 0 || device >= count) return fail(BRMQ_EINVAL, "brmq_ctx_create: no device %d", device);
    CUDA_TRY(cudaSetDevice(device));
    auto* c = new brmq_ctx();
    c->device = device;
    cudaError_t e = cudaStreamCreateWithFlags(&c->own, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete c;
        return fail(BRMQ_ECUDA, "cudaStreamCreate: %s", cudaGetErrorString(e));
    }
    c->stream = c->own;
    e = cudaHostAlloc(reinterpret_cast<void**>(&c->ctl_host), sizeof(Control), cudaHostAllocMapped);
    if (e == cudaSuccess)
        e = cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->ctl_host_dev), c->ctl_host, 0);
    if (e != cudaSuccess) {
        cudaStreamDestroy(c->own);
        delete c;
        return fail(BRMQ_ECUDA, "cudaHostAlloc: %s", cudaGetErrorString(e));
    }
    c->ev.resize(2 * BRMQ_MAX_STAGES);
    for (auto& x : c->ev) cudaEventCreate(&x);
    if (cudaMalloc(&c->epoch_dev, 256) != cudaSuccess ||
        cudaMemcpy(c->epoch_dev, &c->epoch_host, 4, cudaMemcpyHostToDevice) != cudaSuccess) {
        brmq_ctx_destroy(c);
        return fail(BRMQ_ECUDA, "epoch counter allocation failed");
    }
    if (const char* g = getenv("BRMQ_GRAPHS")) c->use_graphs = atoi(g) != 0;
    if (const char* g = getenv("BRMQ_PDL")) c->use_pdl = atoi(g) != 0;
    if (const char* g = getenv("BRMQ_FUSE")) c->use_fuse = atoi(g) != 0;
    if (const char* g = getenv("BRMQ_MSD")) c->use_msd = atoi(g) != 0;
    if (const char* g = getenv("BRMQ_PDL_QUERY")) c->pdl_query = atoi(g) != 0;
    *out = c;
    return BRMQ_OK;
}

void brmq_ctx_destroy(brmq_ctx* c) {
    if (!c) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    drop_graphs(c);
    for (auto& x : c->ev) cudaEventDestroy(x);
    if (c->epoch_dev) cudaFree(c->epoch_dev);
    if (c->ws) cudaFree(c->ws);
    if (c->st) cudaFree(c->st);
    if (c->bitmap) cudaFree(c->bitmap);
    if (c->aux) cudaFree(c->aux);
    if (c->ctl_host) cudaFreeHost(c->ctl_host);
    if (c->own) cudaStreamDestroy(c->own);
    delete c;
}

int brmq_ctx_set_stream(brmq_ctx* c, void* s) {
    if (!c) return fail(BRMQ_EINVAL, "null context");
    if (int rc = settle_pending(c)) return rc;  // (an outstanding async solve belongs to the old settings)
    c->stream = s ? static_cast<cudaStream_t>(s) : c->own;
    return BRMQ_OK;
}

void* brmq_ctx_stream(brmq_ctx* c) { return c ? static_cast<void*>(c->stream) : nullptr; }

int brmq_ctx_set_timing(brmq_ctx* c, int enable) {
    if (!c) return fail(BRMQ_EINVAL, "null context");
    if (int rc = settle_pending(c)) return rc;  // (an outstanding async solve belongs to the old settings)
    c->timing = enable < 0 ? 0 : (enable > 3 ? 1 : enable);
    return BRMQ_OK;
}

int brmq_ctx_set_counters(brmq_ctx* c, int enable) {
    if (!c) return fail(BRMQ_EINVAL, "null context");
    if (int rc = settle_pending(c)) return rc;  // (an outstanding async solve belongs to the old settings)
    c->count_scans = enable != 0;
    return BRMQ_OK;
}

int brmq_last_stage_times(brmq_ctx* c, brmq_stage_times* out) {
    if (!c || !out) return fail(BRMQ_EINVAL, "null argument");
    if (int rc = settle_pending(c)) return rc;
    *out = c->last_times;
    return BRMQ_OK;
}

int brmq_last_solve_info(brmq_ctx* c, brmq_solve_info* out) {
    if (!c || !out) return fail(BRMQ_EINVAL, "null argument");
    if (int rc = settle_pending(c)) return rc;
    *out = c->info;
    return BRMQ_OK;
}

int brmq_host_alloc(void** out, size_t bytes) {
    CUDA_TRY(cudaHostAlloc(out, bytes ? bytes : 1, cudaHostAllocDefault));
    return BRMQ_OK;
}
int brmq_host_free(void* p) {
    CUDA_TRY(cudaFreeHost(p));
    return BRMQ_OK;
}
int brmq_device_alloc(brmq_ctx* c, void** out, size_t bytes) {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaMalloc(out, bytes ? bytes : 1));
    return BRMQ_OK;
}
int brmq_device_free(brmq_ctx* c, void* p) {
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaFree(p));
    return BRMQ_OK;
}
int brmq_memcpy(brmq_ctx* c, void* dst, const void* src, size_t bytes, int kind) {
    CUDA_TRY(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyKind(kind), c->stream));
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return BRMQ_OK;
}
int brmq_synchronize(brmq_ctx* c) {
    if (!c) return fail(BRMQ_EINVAL, "null context");
    CUDA_TRY(cudaStreamSynchronize(c->stream));
    return settle_pending(c);
}

int brmq_ctx_set_async(brmq_ctx* c, int enable) {
    if (!c) return fail(BRMQ_EINVAL, "null context");
    if (int rc = settle_pending(c)) return rc;
    c->async_mode = enable != 0;
    return BRMQ_OK;
}

// The final kernel of a solve copies the control header into the mapped host
// mirror (no device-to-host copy node in the solve's graph).
// The final kernel also re-zeroes the accumulating fields (err, span, tickets) for
// the next solve, so a solve's graph needs no memset node; prepare_ctl zeroes the
// header explicitly (outside any graph) only when something else left it dirty.
// One warp, launched after the final kernel (stream order: every CTA of it has
// finished): the query kernels carry no end-of-kernel barrier + ticket for this
// (measured: ~1 us more lifetime per CTA, 78K CTAs at c3).
__global__ void k_publish(const uint32_t* __restrict__ ctl, uint32_t* __restrict__ host, uint32_t words,
                          uint32_t reset_words) {
    brmq::pdl_wait();
    for (uint32_t i = threadIdx.x; i < words; i += 32) host[i] = __ldcg(ctl + i);
    __syncwarp();
    for (uint32_t i = threadIdx.x; i < reset_words; i += 32) const_cast<uint32_t*>(ctl)[i] = 0u;
    __threadfence_system();
}

brmq::CtlPublish publish_ctl(brmq_ctx* c, Control* ctl) {
    return brmq::CtlPublish{reinterpret_cast<const uint32_t*>(ctl), c->ctl_host_dev, nullptr,
                            uint32_t(kCtlHeader / 4), uint32_t(offsetof(Control, nb) / 4)};
}

int publish(brmq_ctx* c, Control* ctl, cudaStream_t s) {
    brmq::launch_k(k_publish, dim3(1), dim3(32), 0, s, reinterpret_cast<const uint32_t*>(ctl),
                   c->ctl_host_dev, uint32_t(kCtlHeader / 4), uint32_t(offsetof(Control, nb) / 4));
    return 1;
}

int prepare_ctl(brmq_ctx* c, Control* ctl) {
    if (!c->ctl_clean) CUDA_TRY(cudaMemsetAsync(ctl, 0, kCtlHeader, c->stream));
    c->ctl_clean = false;  // until this solve's final kernel has run
    return BRMQ_OK;
}

// ------------------------------------------------------------------ shards
// A split over G devices in contiguous shards; every query's answer is
// the min over shards of the packed key of its piece on the shard, so one
// min-allreduce of q keys (NCCL over NVLink, any order) finishes the batch.
__global__ void k_shard_local(const ulonglong2* __restrict__ Q, uint64_t q, uint64_t off,
                              uint64_t ns, uint64_t n_total, ulonglong2* __restrict__ Ql,
                              uint8_t* __restrict__ empty, uint32_t* __restrict__ err) {
    brmq::pdl_wait();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= q) return;
    const ulonglong2 x = __ldg(Q + i);
    uint64_t l = x.x, r = x.y;
    if (l > r) { const uint64_t t = l; l = r; r = t; }  // types.hpp:18-20
    if (r >= n_total) atomicOr(err, 1u);                 // naive.hpp:14-15 (whole array)
    const uint64_t lo = l > off ? l : off;
    const uint64_t hi = r < off + ns - 1 ? r : off + ns - 1;
    const bool e = r >= n_total || lo > hi;
    empty[i] = e;
    Ql[i] = e ? make_ulonglong2(0, 0) : make_ulonglong2(lo - off, hi - off);
}
__global__ void k_shard_keys(const uint64_t* __restrict__ loc, const uint8_t* __restrict__ empty,
                             const int32_t* __restrict__ A, uint64_t off, uint64_t q,
                             uint64_t* __restrict__ keys) {
    brmq::pdl_wait();
    const uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
    if (i >= q) return;
    const uint64_t p = loc[i];
    keys[i] = empty[i] ? ~0ull : brmq::pack_key(__ldg(A + p), uint32_t(off + p));
}

extern "C++" {
namespace {
// Shared by the sharded solves: clip every query to this shard (k_shard_local),
// run the ordinary single-device solve `local` on the shard, turn its local
// answers into packed keys with global positions (k_shard_keys).
template <class Local>
int solve_shard(brmq_ctx* c, const int32_t* A, uint64_t n_shard, uint64_t offset, uint64_t n_total,
                const brmq_query* Q, uint64_t q, uint64_t* keys, uint32_t flags, Local local) {
    if (n_total > 0xFFFFFFFFull) return fail(BRMQ_EINVAL, "input too long for 32-bit positions");
    if (offset + n_shard > n_total)
        return fail(BRMQ_EINVAL, "shard [%llu, %llu) outside the array of %llu",
                    (unsigned long long)offset, (unsigned long long)(offset + n_shard),
                    (unsigned long long)n_total);
    if (q == 0) return BRMQ_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    const bool dev = is_device(flags);
    cudaStream_t s = c->stream;
    // the local solve owns the context workspace: the shard's own buffers live in
    // a separate grow-only arena (steady-state calls allocate nothing)
    const size_t a_bytes = (n_shard * 4 + 15) & ~size_t(15);  // keeps the copied queries 16-byte aligned
    const size_t bytes = q * 16 + q * 8 + q * 8 + q + 96 + (dev ? 0 : a_bytes + q * 16);
    if (bytes > c->aux_cap) {
        drop_graphs(c);  // captured local solves may point into the old arena
        CUDA_TRY(cudaStreamSynchronize(s));
        if (c->aux) cudaFree(c->aux);
        c->aux = nullptr;
        c->aux_cap = 0;
        const size_t cap = align_up(bytes + bytes / 8, 1 << 21);
        CUDA_TRY(cudaMalloc(reinterpret_cast<void**>(&c->aux), cap));
        c->aux_cap = cap;
    }
    char* buf = c->aux;
    auto* Ql = reinterpret_cast<ulonglong2*>(buf);
    auto* loc = reinterpret_cast<uint64_t*>(buf + q * 16);
    auto* dkeys = reinterpret_cast<uint64_t*>(buf + q * 24);
    auto* empty = reinterpret_cast<uint8_t*>(buf + q * 32);
    auto* err = reinterpret_cast<uint32_t*>(buf + ((q * 33 + 15) & ~size_t(15)));
    const int32_t* dA = A;
    const ulonglong2* dQ = reinterpret_cast<const ulonglong2*>(Q);
    if (!dev) {
        auto* hA = reinterpret_cast<int32_t*>(buf + ((q * 33 + 64 + 15) & ~size_t(15)));
        auto* hQ = reinterpret_cast<ulonglong2*>(reinterpret_cast<char*>(hA) + a_bytes);
        CUDA_TRY(c->stager.h2d(hQ, Q, q * 16, s));
        CUDA_TRY(c->stager.h2d(hA, A, n_shard * 4, s));
        dA = hA;
        dQ = hQ;
    }
    CUDA_TRY(cudaMemsetAsync(err, 0, 4, s));
    const unsigned g = unsigned((q + 255) / 256);
    brmq::launch_k(k_shard_local, dim3(g), dim3(256), 0, s, dQ, q, offset, n_shard, n_total, Ql, empty, err);
    // an empty shard (world does not divide n evenly) answers NO_KEY for every
    // query: k_shard_local marks them all empty, no local solve runs
    int rc = n_shard ? local(dA, reinterpret_cast<const brmq_query*>(Ql), loc) : BRMQ_OK;
    if (rc == BRMQ_OK) {
        brmq::launch_k(k_shard_keys, dim3(g), dim3(256), 0, s, loc, empty, dA, offset, q, dev ? keys : dkeys);
        uint32_t herr = 0;
        if (!dev) CUDA_TRY(c->stager.d2h(keys, dkeys, q * 8, s));
        CUDA_TRY(cudaMemcpyAsync(c->ctl_host, err, 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        herr = *reinterpret_cast<uint32_t*>(c->ctl_host);
        if (herr) rc = fail(BRMQ_ERANGE, "query exceeds array bounds");
    }
    CUDA_TRY(cudaStreamSynchronize(s));
    return rc;
}
}  // namespace
}  // extern "C++"

int brmq_solve_bbst_shard(brmq_ctx* c, const int32_t* A, uint64_t n_shard, uint64_t offset,
                          uint64_t n_total, const brmq_query* Q, uint64_t q, uint32_t k,
                          uint64_t* keys, uint32_t flags) {
    if (!c) return fail(BRMQ_EINVAL, "null context");
    if (int rc = settle_pending(c)) return rc;  // an outstanding async solve first
    if (k == 0) return fail(BRMQ_EINVAL, "solve_batch_bbst: block size k must be >= 1");
    return solve_shard(c, A, n_shard, offset, n_total, Q, q, keys, flags,
                       [&](const int32_t* dA, const brmq_query* Ql, uint64_t* loc) {
                           return brmq_solve_bbst(c, dA, n_shard, Ql, q, k, loc, BRMQ_PTR_DEVICE);
                       });
}

int brmq_solve_bbst_con_shard(brmq_ctx* c, const int32_t* A, uint64_t n_shard, uint64_t offset,
                              uint64_t n_total, const brmq_query* Q, uint64_t q, uint32_t k,
                              int sort_kind, uint64_t* keys, uint32_t flags) {
    if (!c) return fail(BRMQ_EINVAL, "null context");
    if (int rc = settle_pending(c)) return rc;  // an outstanding async solve first
    if (k == 0) return fail(BRMQ_EINVAL, "solve_batch_bbst_con: block size k must be >= 1");
    // the clipped queries' endpoints include the shard borders of every query that
    // crosses one: the shard is contracted with its own endpoints plus those borders
    return solve_shard(c, A, n_shard, offset, n_total, Q, q, keys, flags,
                       [&](const int32_t* dA, const brmq_query* Ql, uint64_t* loc) {
                           return brmq_solve_bbst_con(c, dA, n_shard, Ql, q, k, sort_kind, loc,
                                                      BRMQ_PTR_DEVICE);
                       });
}

// ------------------------------------------------------------------ naive
// The harness's "naive" algorithm (naive.hpp:13-21): every query scanned on the
// device, one warp per query.  A baseline, not a BbST path.
int brmq_solve_naive(brmq_ctx* c, const int32_t* A, uint64_t n, const brmq_query* Q, uint64_t q,
                     uint64_t* answers, uint32_t flags) {
    if (!c) return fail(BRMQ_EINVAL, "null context");
    if (int rc = settle_pending(c)) return rc;  // an outstanding async solve first
    c->info = brmq_solve_info{};
    c->info.n = n;
    c->info.q = q;
    Timer tm(c);
    if (q == 0) {
        tm.finish();
        return BRMQ_OK;
    }
    if (n == 0) return fail(BRMQ_ERANGE, "query exceeds array bounds");
    CUDA_TRY(cudaSetDevice(c->device));
    const bool dev = is_device(flags);
    Carve cv;
    const size_t i_ctl = cv.add(sizeof(Control));
    const size_t i_a = dev ? 0 : cv.add(n * 4);
    const size_t i_q = dev ? 0 : cv.add(q * 16);
    const size_t i_ans = dev ? 0 : cv.add(q * 8);
    if (int rc = ensure_ws(c, cv.total)) return rc;
    auto P = [&](size_t i) { return c->ws + cv.off[i]; };
    auto* ctl = reinterpret_cast<Control*>(P(i_ctl));
    const int32_t* dA = dev ? A : reinterpret_cast<int32_t*>(P(i_a));
    const uint64_t* dQ = dev ? reinterpret_cast<const uint64_t*>(Q) : reinterpret_cast<uint64_t*>(P(i_q));
    uint64_t* dAns = dev ? answers : reinterpret_cast<uint64_t*>(P(i_ans));
    cudaStream_t s = c->stream;
    int launches = 0;
    auto enqueue = [&]() -> int {
        brmq::PdlScope pdl(c->timing == 0 && c->use_pdl);  // kernels after the first: PDL secondaries
        // (the control header is zeroed by the previous solve's final kernel, see prepare_ctl)
        if (!dev) {
            tm.stage("h2d", launches);
            CUDA_TRY(c->stager.h2d(const_cast<uint64_t*>(dQ), Q, q * 16, s));  // small first: A's DMA runs last
            CUDA_TRY(c->stager.h2d(const_cast<int32_t*>(dA), A, n * 4, s));
            tm.end(0);
        }
        tm.stage("query", launches);
        const int l = brmq::launch_naive(dA, n, dQ, q, dAns, &ctl->err, s, brmq::CtlPublish{});
        launches += l;
        tm.end(l);
        launches += publish(c, ctl, s);  // control header -> host (k_publish)
        if (int rc = check_status(c)) return rc;
        if (!dev) {
            tm.stage("d2h", launches);
            CUDA_TRY(c->stager.d2h(answers, dAns, q * 8, s));
            tm.end(0);
        }
        // (the control header reaches c->ctl_host from the final kernel: publish())
        return BRMQ_OK;
    };
    const GraphKey key{4, A, n, Q, q, 0, 0, answers, s};
    if (int rc = prepare_ctl(c, ctl)) return rc;
    if (int rc = run_solve(c, key, dev, tm, launches, enqueue)) return rc;
    c->ctl_clean = true;  // the final kernel published and re-zeroed the header
    CUDA_TRY(cudaStreamSynchronize(s));
    tm.finish();
    c->info.kernel_launches = uint32_t(launches);
    return map_err(c->ctl_host->err);
}

// ------------------------------------------------------------------ BbST (h = 1)
int brmq_solve_bbst(brmq_ctx* c, const int32_t* A, uint64_t n, const brmq_query* Q, uint64_t q,
                    uint32_t k, uint64_t* answers, uint32_t flags) {
    if (!c) return fail(BRMQ_EINVAL, "null context");
    if (int rc = settle_pending(c)) return rc;  // an outstanding async solve first
    if (k == 0) return fail(BRMQ_EINVAL, "solve_batch_bbst: block size k must be >= 1");
    if (n > 0xFFFFFFFFull) return fail(BRMQ_EINVAL, "input too long for 32-bit positions");
    c->info = brmq_solve_info{};
    c->info.n = n;
    c->info.q = q;
    c->info.k = k;
    Timer tm(c);
    if (q == 0) {  // SPEC.md:306 empty batch -> empty answers
        tm.finish();
        return BRMQ_OK;
    }
    if (n == 0) return fail(BRMQ_ERANGE, "query exceeds array bounds");
    CUDA_TRY(cudaSetDevice(c->device));
    const bool dev = is_device(flags);
    const uint64_t b = (n + k - 1) / k;
    const uint32_t L = brmq::floor_log2_u64(b) + 1;

    Carve cv;
    const size_t i_ctl = cv.add(sizeof(Control));
    const size_t i_st = cv.add(size_t(L) * b * 8);
    const size_t i_a = dev ? 0 : cv.add(n * 4);
    const size_t i_q = dev ? 0 : cv.add(q * 16);
    const size_t i_ans = dev ? 0 : cv.add(q * 8);
    if (int rc = ensure_ws(c, cv.total)) return rc;
    auto P = [&](size_t i) { return c->ws + cv.off[i]; };
    auto* ctl = reinterpret_cast<Control*>(P(i_ctl));
    auto* ST = reinterpret_cast<uint64_t*>(P(i_st));
    const int32_t* dA = dev ? A : reinterpret_cast<int32_t*>(P(i_a));
    const uint64_t* dQ = dev ? reinterpret_cast<const uint64_t*>(Q) : reinterpret_cast<uint64_t*>(P(i_q));
    uint64_t* dAns = dev ? answers : reinterpret_cast<uint64_t*>(P(i_ans));
    cudaStream_t s = c->stream;
    int launches = 0;
    auto enqueue = [&]() -> int {
        brmq::PdlScope pdl(c->timing == 0 && c->use_pdl);  // kernels after the first: PDL secondaries
        int l = 0;
        // (the control header is zeroed by the previous solve's final kernel, see prepare_ctl)
        if (!dev) {
            tm.stage("h2d", launches);
            CUDA_TRY(c->stager.h2d(const_cast<uint64_t*>(dQ), Q, q * 16, s));  // small first: A's DMA runs last
            CUDA_TRY(c->stager.h2d(const_cast<int32_t*>(dA), A, n * 4, s));
            tm.end(0);
        }
        tm.phase_begin("preprocess");
        tm.stage("block_argmin", launches);
        l = brmq::launch_block_argmin_i32(dA, n, k, ST, s);
        launches += l;
        tm.end(l);
        tm.stage("sparse_table", launches);
        l = brmq::launch_sparse_table(ST, b, nullptr, s);
        launches += l;
        tm.end(l);
        tm.phase_end(launches);
        tm.phase_begin("query");
        tm.stage("query", launches);
        l = brmq::launch_query_direct(dA, n, k, ST, b, dQ, q, dAns, &ctl->err, s, brmq::CtlPublish{},
                                      c->count_scans ? &ctl->scanned : nullptr);
        launches += l;
        tm.end(l);
        tm.phase_end(l);
        launches += publish(c, ctl, s);  // control header -> host (k_publish)
        if (int rc = check_status(c)) return rc;
        if (!dev) {
            tm.stage("d2h", launches);
            CUDA_TRY(c->stager.d2h(answers, dAns, q * 8, s));
            tm.end(0);
        }
        // (the control header reaches c->ctl_host from the final kernel: publish())
        return BRMQ_OK;
    };
    const GraphKey key{0, A, n, Q, q, k, c->count_scans ? 1 : 0, answers, s};
    if (int rc = prepare_ctl(c, ctl)) return rc;
    tm.pre_launch(dev);
    if (int rc = run_solve(c, key, dev, tm, launches, enqueue)) return rc;
    c->ctl_clean = true;  // the final kernel published and re-zeroed the header
    return end_solve(c, dev, tm, [c, b, L, launches]() {
        c->info.blocks = b;
        c->info.levels = L;
        c->info.kernel_launches = uint32_t(launches);
        c->info.scanned_cells = c->count_scans ? c->ctl_host->scanned : 0;
    });
}

// ------------------------------------------------------------ multi-level BbST
// Any other dividing chain (query_chain.cu): M_0 = k_1-block minima of A, M_j from
// M_{j-1} (k_{j+1}/k_j children each), the k_h-block minima from M_{h-2}, the
// block Sparse Table over them, one warp per query descending the levels.
static int solve_chain(brmq_ctx* c, const int32_t* A, uint64_t n, const brmq_query* Q, uint64_t q,
                const uint32_t* ks, uint32_t h, uint64_t* answers, uint32_t flags) {
    if (n > 0xFFFFFFFFull) return fail(BRMQ_EINVAL, "input too long for 32-bit positions");
    const uint32_t k = ks[h - 1];
    c->info = brmq_solve_info{};
    c->info.n = n;
    c->info.q = q;
    c->info.k = k;
    Timer tm(c);
    if (q == 0) {
        tm.finish();
        return BRMQ_OK;
    }
    if (n == 0) return fail(BRMQ_ERANGE, "query exceeds array bounds");
    CUDA_TRY(cudaSetDevice(c->device));
    const bool dev = is_device(flags);
    const uint64_t b = (n + k - 1) / k;
    const uint32_t L = brmq::floor_log2_u64(b) + 1;
    Carve cv;
    const size_t i_ctl = cv.add(sizeof(Control));
    const size_t i_st = cv.add(size_t(L) * b * 8);
    size_t i_m[brmq::kMaxChain] = {};
    uint64_t mlen[brmq::kMaxChain] = {};
    for (uint32_t j = 0; j + 1 < h; ++j) {
        mlen[j] = (n + ks[j] - 1) / ks[j];
        i_m[j] = cv.add(mlen[j] * 8);
    }
    const size_t i_a = dev ? 0 : cv.add(n * 4);
    const size_t i_q = dev ? 0 : cv.add(q * 16);
    const size_t i_ans = dev ? 0 : cv.add(q * 8);
    if (int rc = ensure_ws(c, cv.total)) return rc;
    auto P = [&](size_t i) { return c->ws + cv.off[i]; };
    auto* ctl = reinterpret_cast<Control*>(P(i_ctl));
    auto* ST = reinterpret_cast<uint64_t*>(P(i_st));
    uint64_t* M[brmq::kMaxChain] = {};
    for (uint32_t j = 0; j + 1 < h; ++j) M[j] = reinterpret_cast<uint64_t*>(P(i_m[j]));
    const int32_t* dA = dev ? A : reinterpret_cast<int32_t*>(P(i_a));
    const uint64_t* dQ = dev ? reinterpret_cast<const uint64_t*>(Q) : reinterpret_cast<uint64_t*>(P(i_q));
    uint64_t* dAns = dev ? answers : reinterpret_cast<uint64_t*>(P(i_ans));
    cudaStream_t s = c->stream;
    int launches = 0;
    auto enqueue = [&]() -> int {
        brmq::PdlScope pdl(c->timing == 0 && c->use_pdl);  // kernels after the first: PDL secondaries
        int l = 0;
        if (!dev) {
            tm.stage("h2d", launches);
            CUDA_TRY(c->stager.h2d(const_cast<uint64_t*>(dQ), Q, q * 16, s));  // small first: A's DMA runs last
            CUDA_TRY(c->stager.h2d(const_cast<int32_t*>(dA), A, n * 4, s));
            tm.end(0);
        }
        tm.stage("block_argmin", launches);
        l = brmq::launch_block_argmin_i32(dA, n, ks[0], M[0], s);  // level k_1 from A
        for (uint32_t j = 1; j + 1 < h; ++j)                       // level k_{j+1} from level k_j
            l += brmq::launch_block_argmin_keys(M[j - 1], mlen[j - 1], nullptr, ks[j] / ks[j - 1], M[j],
                                                nullptr, s);
        l += brmq::launch_block_argmin_keys(M[h - 2], mlen[h - 2], nullptr, k / ks[h - 2], ST, nullptr, s);
        launches += l;
        tm.end(l);
        tm.stage("sparse_table", launches);
        l = brmq::launch_sparse_table(ST, b, nullptr, s);
        launches += l;
        tm.end(l);
        tm.stage("query", launches);
        l = brmq::launch_query_chain(dA, n, ks, h, M, ST, b, dQ, q, dAns, &ctl->err, s, brmq::CtlPublish{});
        launches += l;
        tm.end(l);
        launches += publish(c, ctl, s);  // control header -> host (k_publish)
        if (int rc = check_status(c)) return rc;
        if (!dev) {
            tm.stage("d2h", launches);
            CUDA_TRY(c->stager.d2h(answers, dAns, q * 8, s));
            tm.end(0);
        }
        return BRMQ_OK;
    };
    // no graph cache: the key has no room for the chain; a direct enqueue is 4 + h launches
    const GraphKey key{5, A, n, Q, q, k, int(h), answers, s};
    if (int rc = prepare_ctl(c, ctl)) return rc;
    if (int rc = run_solve(c, key, false, tm, launches, enqueue)) return rc;
    c->ctl_clean = true;  // the final kernel published and re-zeroed the header
    return end_solve(c, dev, tm, [c, b, L, launches]() {
        c->info.blocks = b;
        c->info.levels = L;
        c->info.kernel_launches = uint32_t(launches);
    });
}

int brmq_solve_bbst_ml(brmq_ctx* c, const int32_t* A, uint64_t n, const brmq_query* Q, uint64_t q,
                       const uint32_t* ks, uint32_t h, uint64_t* answers, uint32_t flags) {
    if (!c || !ks) return fail(BRMQ_EINVAL, "null argument");
    if (int rc = settle_pending(c)) return rc;  // an outstanding async solve first
    if (h == 0) return fail(BRMQ_EINVAL, "solve_batch_bbst: empty level config");
    if (h == 1) return brmq_solve_bbst(c, A, n, Q, q, ks[0], answers, flags);
    if (h > brmq::kMaxChain) return fail(BRMQ_EINVAL, "solve_batch_bbst: at most 8 levels");
    for (uint32_t j = 0; j < h; ++j) {  // k_1 < ... < k_h, k_i | k_{i+1}
        if (ks[j] == 0 || (j > 0 && (ks[j] <= ks[j - 1] || ks[j] % ks[j - 1] != 0)))
            return fail(BRMQ_EINVAL, "solve_batch_bbst: the level config is not a dividing chain");
    }
    if (h != 2 || ks[0] != 32) return solve_chain(c, A, n, Q, q, ks, h, answers, flags);
    const uint32_t k = ks[1];
    if (n > 0xFFFFFFFFull) return fail(BRMQ_EINVAL, "input too long for 32-bit positions");
    c->info = brmq_solve_info{};
    c->info.n = n;
    c->info.q = q;
    c->info.k = k;
    Timer tm(c);
    if (q == 0) {
        tm.finish();
        return BRMQ_OK;
    }
    if (n == 0) return fail(BRMQ_ERANGE, "query exceeds array bounds");
    CUDA_TRY(cudaSetDevice(c->device));
    const bool dev = is_device(flags);
    const uint64_t b = (n + k - 1) / k;
    const uint32_t L = brmq::floor_log2_u64(b) + 1;
    Carve cv;
    const size_t i_ctl = cv.add(sizeof(Control));
    const size_t i_st = cv.add(size_t(L) * b * 8);
    const size_t i_sub = cv.add(((n + 31) / 32) * 8);
    const size_t i_a = dev ? 0 : cv.add(n * 4);
    const size_t i_q = dev ? 0 : cv.add(q * 16);
    const size_t i_ans = dev ? 0 : cv.add(q * 8);
    if (int rc = ensure_ws(c, cv.total)) return rc;
    auto P = [&](size_t i) { return c->ws + cv.off[i]; };
    auto* ctl = reinterpret_cast<Control*>(P(i_ctl));
    auto* ST = reinterpret_cast<uint64_t*>(P(i_st));
    auto* SUB = reinterpret_cast<uint64_t*>(P(i_sub));
    const int32_t* dA = dev ? A : reinterpret_cast<int32_t*>(P(i_a));
    const uint64_t* dQ = dev ? reinterpret_cast<const uint64_t*>(Q) : reinterpret_cast<uint64_t*>(P(i_q));
    uint64_t* dAns = dev ? answers : reinterpret_cast<uint64_t*>(P(i_ans));
    cudaStream_t s = c->stream;
    int launches = 0;
    auto enqueue = [&]() -> int {
        brmq::PdlScope pdl(c->timing == 0 && c->use_pdl);  // kernels after the first: PDL secondaries
        int l = 0;
        // (the control header is zeroed by the previous solve's final kernel, see prepare_ctl)
        if (!dev) {
            tm.stage("h2d", launches);
            CUDA_TRY(c->stager.h2d(const_cast<uint64_t*>(dQ), Q, q * 16, s));  // small first: A's DMA runs last
            CUDA_TRY(c->stager.h2d(const_cast<int32_t*>(dA), A, n * 4, s));
            tm.end(0);
        }
        tm.stage("block_argmin", launches);
        l = brmq::launch_block_argmin_ml(dA, n, k, ST, SUB, s);
        launches += l;
        tm.end(l);
        tm.stage("sparse_table", launches);
        l = brmq::launch_sparse_table(ST, b, nullptr, s);
        launches += l;
        tm.end(l);
        tm.stage("query", launches);
        l = brmq::launch_query_ml(dA, n, k, ST, b, SUB, dQ, q, dAns, &ctl->err, s, brmq::CtlPublish{});
        launches += l;
        tm.end(l);
        launches += publish(c, ctl, s);  // control header -> host (k_publish)
        if (int rc = check_status(c)) return rc;
        if (!dev) {
            tm.stage("d2h", launches);
            CUDA_TRY(c->stager.d2h(answers, dAns, q * 8, s));
            tm.end(0);
        }
        // (the control header reaches c->ctl_host from the final kernel: publish())
        return BRMQ_OK;
    };
    const GraphKey key{2, A, n, Q, q, k, 32, answers, s};
    if (int rc = prepare_ctl(c, ctl)) return rc;
    if (int rc = run_solve(c, key, dev, tm, launches, enqueue)) return rc;
    c->ctl_clean = true;  // the final kernel published and re-zeroed the header
    return end_solve(c, dev, tm, [c, b, L, launches]() {
        c->info.blocks = b;
        c->info.levels = L;
        c->info.kernel_launches = uint32_t(launches);
    });
}

// ------------------------------------------------------------------ BbST_CON
int brmq_solve_bbst_con(brmq_ctx* c, const int32_t* A, uint64_t n, const brmq_query* Q,
                        uint64_t q, uint32_t k, int sort_kind, uint64_t* answers,
                        uint32_t flags) {
    if (!c) return fail(BRMQ_EINVAL, "null context");
    if (int rc = settle_pending(c)) return rc;  // an outstanding async solve first
    if (k == 0) return fail(BRMQ_EINVAL, "solve_batch_bbst_con: block size k must be >= 1");
    if (n > 0xFFFFFFFFull) return fail(BRMQ_EINVAL, "input too long for 32-bit positions");
    if (q > (1ull << 31)) return fail(BRMQ_EINVAL, "collect_endpoints: too many queries for 32-bit origins");
    if (sort_kind < 0 || sort_kind > 2) return fail(BRMQ_EINVAL, "unknown sort kind %d", sort_kind);
    c->info = brmq_solve_info{};
    c->info.n = n;
    c->info.q = q;
    c->info.k = k;
    Timer tm(c);
    if (q == 0) {
        tm.finish();
        return BRMQ_OK;
    }
    if (n == 0) return fail(BRMQ_ERANGE, "query exceeds array bounds");
    CUDA_TRY(cudaSetDevice(c->device));
    const bool dev = is_device(flags);
    const uint64_t m = 2 * q;
    const int bits = bits_for(n);
    // the bitmap sort marks endpoints directly, unless the bitmap outgrows the L2
    // and is dense enough to need several slice passes over the queries (c5-con:
    // four): then the endpoints are bucketed once by their top bits and each
    // bucket marked from shared memory (the MSD pipeline's marking, same bitmap)
    int D_ = 0, Lb_ = 0;
    const bool use_bitmap =
        sort_kind == 2 && !(c->use_msd && brmq::collect_mark_slices(n, q) > 1 &&
                            brmq::radix_partition_shape(bits, m, brmq::contract_bitmap_words(n), &D_, &Lb_));
    const uint64_t aq_max = m - 1;                       // |A_Q| <= 2q - 1
    const uint64_t b_max = (aq_max + k - 1) / k;
    const uint32_t L = brmq::floor_log2_u64(b_max) + 1;
    const uint64_t ntiles = brmq::contract_tiles(n);
    uint32_t G = 0, R = 0;
    brmq::contract_partition(n, &G, &R);
    if (int rc = ensure_bitmap(c, n)) return rc;

    Carve cv;
    const size_t i_ctl = cv.add(sizeof(Control));
    const size_t i_aq = cv.add((aq_max + 2) * 8);
    const size_t i_st = cv.add(size_t(L) * b_max * 8);
    // power-of-two k in [64, 512]: 32-key sub-block minima over A_Q as a second level
    // (answers identical; partial blocks are resolved through them, DESIGN 3.2)
    const bool sub_level = k >= 64 && k <= 512 && (k & (k - 1)) == 0;
    const size_t sub_words = (aq_max + 31) / 32 + 2;
    const size_t i_sub = cv.add(sub_level ? sub_words * 8 : 0);
    // small A_Q: the contraction itself yields the block / sub-block minima
    // (brmq::ContractFuse); no block-argmin pass over A_Q follows.  Large A_Q (dense
    // areas: many reductions on each block key) keeps the separate pass.
    const bool fuse = sub_level && b_max <= 1024 && c->use_fuse;  // (c4-con, 3906 blocks: +25 us of reductions for -12 us)
    Carve sv;  // status arena
    const size_t i_cst = sv.add(brmq::contract_status_words() * 8);
    const size_t i_pc = cv.add(size_t(brmq::kMaxContractRanges) * brmq::kContractWarps * 4);
    // both pipelines: the contraction emits (rank prefix, bits) per non-empty bitmap
    // word and the query kernel computes each query's contracted coordinates from
    // them (remap_queries_from_sorted, contraction.cpp:174-199, folded into
    // answering: no random scatter of ranks into per-query arrays)
    size_t i_k0 = 0, i_k1 = 0, i_rs = 0, i_rst = 0;
    const size_t i_wi = cv.add((n / 32 + 2) * 8);
    if (!use_bitmap) {
        // the radix pipeline sorts the endpoint POSITIONS (keys only): their origins
        // served only the rank scatter above
        i_k0 = cv.add(m * 4);
        i_k1 = cv.add(m * 4);
        i_rs = cv.add(brmq::radix_sort_temp_bytes(m, bits));
        i_rst = sv.add(brmq::radix_sort_status_words(m, bits) * 8);
    }
    const size_t i_a = dev ? 0 : cv.add(n * 4);
    const size_t i_q = dev ? 0 : cv.add(q * 16);
    const size_t i_ans = dev ? 0 : cv.add(q * 8);
    if (int rc = ensure_ws(c, cv.total)) return rc;
    if (int rc = ensure_status(c, sv.total)) return rc;
    auto P = [&](size_t i) { return c->ws + cv.off[i]; };
    auto S = [&](size_t i) { return reinterpret_cast<uint64_t*>(c->st + sv.off[i]); };
    auto* ctl = reinterpret_cast<Control*>(P(i_ctl));
    auto* AQ = reinterpret_cast<uint64_t*>(P(i_aq));
    auto* ST = reinterpret_cast<uint64_t*>(P(i_st));
    auto* cst = S(i_cst);
    auto* pcnt = reinterpret_cast<uint32_t*>(P(i_pc));
    const int32_t* dA = dev ? A : reinterpret_cast<int32_t*>(P(i_a));
    const uint64_t* dQ = dev ? reinterpret_cast<const uint64_t*>(Q) : reinterpret_cast<uint64_t*>(P(i_q));
    uint64_t* dAns = dev ? answers : reinterpret_cast<uint64_t*>(P(i_ans));
    cudaStream_t s = c->stream;
    const uint32_t n_epochs = 1u;  // the contraction's look-back (the sort's descriptors are zeroed)
    if (int rc = begin_epochs(c, n_epochs)) return rc;
    int launches = 0;
    auto enqueue = [&]() -> int {
        brmq::PdlScope pdl(c->timing == 0 && c->use_pdl);  // kernels after the first: PDL secondaries
        int l = 0;
        // (the control header is zeroed by the previous solve's final kernel, see prepare_ctl)
        if (!dev) {
            tm.stage("h2d", launches);
            CUDA_TRY(c->stager.h2d(const_cast<uint64_t*>(dQ), Q, q * 16, s));  // small first: A's DMA runs last
            CUDA_TRY(c->stager.h2d(const_cast<int32_t*>(dA), A, n * 4, s));
            tm.end(0);
        }
        // the epochs of this solve are reserved by the first kernel (k_collect)
        // epoch offset 0: the contraction's look-back
        auto* SUB = reinterpret_cast<uint64_t*>(P(i_sub));
        uint64_t* fill0 = fuse ? SUB : nullptr;
        uint64_t* fill1 = fuse ? ST : nullptr;
        const uint64_t fill0_n = fuse ? sub_words : 0, fill1_n = fuse ? b_max : 0;
        tm.phase_begin("preprocess");
        if (use_bitmap) {
            tm.stage("collect_mark", launches);
            l = brmq::launch_collect(dQ, q, n, nullptr, nullptr, c->bitmap,
                                     ctl->span, &ctl->err, s, c->epoch_dev, n_epochs, fill0, fill0_n,
                                     fill1, fill1_n);
            l += brmq::launch_piece_count(c->bitmap, ctl->span, n, pcnt, ctl->rcnt, s);
            launches += l;
            tm.end(l);
        } else {
            auto* k0 = reinterpret_cast<uint32_t*>(P(i_k0));
            auto* k1 = reinterpret_cast<uint32_t*>(P(i_k1));
            // MSD (radix_partition_shape): the collect builds the top-digit
            // histogram; a partition pass, then per bucket a counting digit in
            // shared memory that dedups and marks the bitmap
            const uint64_t bm_words = brmq::contract_bitmap_words(n);
            int D = 0, Lb = 0;
            const bool msd = c->use_msd && brmq::radix_partition_shape(bits, m, bm_words, &D, &Lb);
            if (msd) CUDA_TRY(cudaMemsetAsync(P(i_rs), 0, brmq::radix_sort_temp_bytes(m, bits), s));
            tm.stage("collect", launches);
            l = brmq::launch_collect(dQ, q, n, k0, nullptr, nullptr, msd ? ctl->span : nullptr, &ctl->err, s,
                                     c->epoch_dev, n_epochs, fill0, fill0_n, fill1, fill1_n,
                                     msd ? brmq::radix_partition_hist(P(i_rs)) : nullptr, uint32_t(Lb),
                                     msd ? (1u << D) - 1u : 0u);
            launches += l;
            tm.end(l);
            tm.stage("radix_sort", launches);
            if (msd) {
                l = brmq::launch_radix_partition_mark(k0, k1, m, bits, n, P(i_rs), c->bitmap, bm_words, &ctl->err,
                                                      s);
                launches += l;
                tm.end(l);
                tm.stage("unique_rank", launches);
                l = brmq::launch_piece_count(c->bitmap, ctl->span, n, pcnt, ctl->rcnt, s);
                launches += l;
                tm.end(l);
            } else {  // LSD over all digits
                bool in_alt = false;
                l = brmq::launch_radix_sort(k0, nullptr, k1, nullptr, m, bits, P(i_rs), S(i_rst), s, &in_alt,
                                            c->epoch_dev, 2);
                launches += l;
                tm.end(l);
                // dedup: the sorted positions mark the bitmap (coalesced, no look-back);
                // ranks per contraction piece from the bitmap as in the bitmap pipeline
                tm.stage("unique_rank", launches);
                l = brmq::launch_mark_sorted(in_alt ? k1 : k0, m, n, c->bitmap, ctl->span, &ctl->err, s);
                l += brmq::launch_piece_count(c->bitmap, ctl->span, n, pcnt, ctl->rcnt, s);
                launches += l;
                tm.end(l);
            }
        }
        tm.stage("contract", launches);
        const brmq::ContractFuse fz{SUB, ST, b_max, brmq::floor_log2_u64(k), &ctl->b_dev};
        bool fused = false;
        // a PDL secondary of the piece count: its first tile loads are issued
        // before its griddepcontrol.wait (contraction.cu contract_body)
        const brmq::PdlState pdl_before = brmq::pdl_state();
        if (c->timing == 0 && c->pdl_query) brmq::pdl_state() = brmq::PdlState{true, false};
        l = brmq::launch_contract(dA, n, c->bitmap, ctl->span, ctl->rcnt, false, AQ,
                                  &ctl->nb, &ctl->aq_len, reinterpret_cast<uint2*>(P(i_wi)), cst,
                                  c->epoch_dev, 0, s, false, pcnt, 2 * q,
                                  fuse ? &fz : nullptr, &fused);
        brmq::pdl_state() = pdl_before;
        launches += l;
        tm.end(l);
        // (bitmap pipeline: the query remap is folded into the query kernel)
        if (!fused) {  // (e.g. unaligned A: the filled sub / row 0 are overwritten here)
            tm.stage("block_argmin", launches);
            l = sub_level ? brmq::launch_block_argmin_keys_ml(AQ, aq_max, &ctl->aq_len, k, ST, SUB,
                                                              &ctl->b_dev, s)
                          : brmq::launch_block_argmin_keys(AQ, aq_max, &ctl->aq_len, k, ST, &ctl->b_dev, s);
            launches += l;
            tm.end(l);
        }
        tm.stage("sparse_table", launches);
        l = brmq::launch_sparse_table(ST, b_max, &ctl->b_dev, s);
        launches += l;
        tm.end(l);
        tm.phase_end(launches);
        tm.phase_begin("query");
        tm.stage("query", launches);
        const uint2* wi = reinterpret_cast<uint2*>(P(i_wi));
        // the query kernel writes nothing into the control header: its first warp
        // publishes it (publish_early), no k_publish launch
        // the query kernel as a PDL secondary of the table build: it resolves its
        // queries (Q + word info) before its griddepcontrol.wait (query.cu k_query_flat)
        const brmq::PdlState pdl_saved = brmq::pdl_state();
        if (c->timing == 0 && c->pdl_query && sub_level) brmq::pdl_state() = brmq::PdlState{true, false};
        if (sub_level)
            l = brmq::launch_query_con_flat(AQ, k, ST, b_max, SUB, dQ, wi, nullptr, nullptr, n, q, dAns, s,
                                            publish_ctl(c, ctl));
        else
            l = brmq::launch_query_contracted_wi(AQ, k, ST, b_max, dQ, wi, n, q, dAns, s,
                                                 publish_ctl(c, ctl));
        brmq::pdl_state() = pdl_saved;
        launches += l;
        tm.end(l);
        tm.phase_end(l);
        if (int rc = check_status(c)) return rc;
        if (!dev) {
            tm.stage("d2h", launches);
            CUDA_TRY(c->stager.d2h(answers, dAns, q * 8, s));
            tm.end(0);
        }
        // (the control header reaches c->ctl_host from the final kernel: publish())
        return BRMQ_OK;
    };
    const GraphKey key{1, A, n, Q, q, k, sort_kind, answers, s};
    if (int rc = prepare_ctl(c, ctl)) return rc;
    tm.pre_launch(dev);
    if (int rc = run_solve(c, key, dev, tm, launches, enqueue)) return rc;
    c->ctl_clean = true;  // the final kernel published and re-zeroed the header
    c->epoch_host += n_epochs;
    return end_solve(c, dev, tm, [c, launches]() {
        const Control& h = *c->ctl_host;
        c->info.boundary = h.nb;
        c->info.span_lo = ~h.span[0];
        c->info.span_hi = h.span[1];
        c->info.blocks = h.b_dev;
        c->info.levels = h.b_dev ? brmq::floor_log2_u64(h.b_dev) + 1 : 0;
        c->info.kernel_launches = uint32_t(launches);
    });
}

// ------------------------------------------------------------------ ST-RMQ_CON
// SPEC.md "baseline" (Alzamel et al., section 2): marked contraction of A
// into E (each marked position verbatim, each maximal unmarked run by its
// minimum: 2m + 1 <= 4q + 1 entries; an empty run keeps its slot as +inf, a
// documented departure from "exactly one entry per run"), an element Sparse
// Table over E, two probes per query.  Endpoint sort: the LSD radix sort.
int brmq_solve_st_rmq_con(brmq_ctx* c, const int32_t* A, uint64_t n, const brmq_query* Q,
                          uint64_t q, uint64_t* answers, uint32_t flags) {
    if (!c) return fail(BRMQ_EINVAL, "null context");
    if (int rc = settle_pending(c)) return rc;  // an outstanding async solve first
    if (n > 0xFFFFFFFFull) return fail(BRMQ_EINVAL, "input too long for 32-bit positions");
    if (q > (1ull << 31)) return fail(BRMQ_EINVAL, "collect_endpoints: too many queries for 32-bit origins");
    c->info = brmq_solve_info{};
    c->info.n = n;
    c->info.q = q;
    c->info.k = 1;
    Timer tm(c);
    if (q == 0) {
        tm.finish();
        return BRMQ_OK;
    }
    if (n == 0) return fail(BRMQ_ERANGE, "query exceeds array bounds");
    CUDA_TRY(cudaSetDevice(c->device));
    const bool dev = is_device(flags);
    const uint64_t m = 2 * q;
    const uint64_t e_max = 2 * m + 1;  // |E| <= 4q + 1
    const uint32_t L = brmq::floor_log2_u64(e_max) + 1;
    const int bits = bits_for(n);
    uint32_t G = 0, R = 0;
    brmq::contract_partition(n, &G, &R);
    if (int rc = ensure_bitmap(c, n)) return rc;

    Carve cv;
    const size_t i_ctl = cv.add(sizeof(Control));
    const size_t i_cl = cv.add(q * 4);
    const size_t i_cr = cv.add(q * 4);
    const size_t i_bd = cv.add(m * 4);
    const size_t i_st = cv.add(size_t(L) * e_max * 8);  // row 0 = E
    const size_t i_k0 = cv.add(m * 4), i_v0 = cv.add(m * 4), i_k1 = cv.add(m * 4), i_v1 = cv.add(m * 4);
    const size_t i_rs = cv.add(brmq::radix_sort_temp_bytes(m, bits));
    Carve sv;
    const size_t i_cst = sv.add(brmq::contract_status_words() * 8);
    const size_t i_rst = sv.add(brmq::radix_sort_status_words(m, bits) * 8);
    const size_t i_ust = sv.add(brmq::unique_status_words(m) * 8);
    const size_t i_a = dev ? 0 : cv.add(n * 4);
    const size_t i_q = dev ? 0 : cv.add(q * 16);
    const size_t i_ans = dev ? 0 : cv.add(q * 8);
    if (int rc = ensure_ws(c, cv.total)) return rc;
    if (int rc = ensure_status(c, sv.total)) return rc;
    auto P = [&](size_t i) { return c->ws + cv.off[i]; };
    auto S = [&](size_t i) { return reinterpret_cast<uint64_t*>(c->st + sv.off[i]); };
    auto* ctl = reinterpret_cast<Control*>(P(i_ctl));
    auto* cl = reinterpret_cast<uint32_t*>(P(i_cl));
    auto* cr = reinterpret_cast<uint32_t*>(P(i_cr));
    auto* bd = reinterpret_cast<uint32_t*>(P(i_bd));
    auto* ST = reinterpret_cast<uint64_t*>(P(i_st));
    const int32_t* dA = dev ? A : reinterpret_cast<int32_t*>(P(i_a));
    const uint64_t* dQ = dev ? reinterpret_cast<const uint64_t*>(Q) : reinterpret_cast<uint64_t*>(P(i_q));
    uint64_t* dAns = dev ? answers : reinterpret_cast<uint64_t*>(P(i_ans));
    cudaStream_t s = c->stream;
    const uint32_t n_epochs = 2u + uint32_t(brmq::radix_sort_passes(bits));
    if (int rc = begin_epochs(c, n_epochs)) return rc;
    int launches = 0;
    auto enqueue = [&]() -> int {
        brmq::PdlScope pdl(c->timing == 0 && c->use_pdl);  // kernels after the first: PDL secondaries
        int l = 0;
        // (the control header is zeroed by the previous solve's final kernel, see prepare_ctl)
        if (!dev) {
            tm.stage("h2d", launches);
            CUDA_TRY(c->stager.h2d(const_cast<uint64_t*>(dQ), Q, q * 16, s));  // small first: A's DMA runs last
            CUDA_TRY(c->stager.h2d(const_cast<int32_t*>(dA), A, n * 4, s));
            tm.end(0);
        }
        // the epochs of this solve are reserved by the first kernel (k_collect)
        auto* k0 = reinterpret_cast<uint32_t*>(P(i_k0));
        auto* v0 = reinterpret_cast<uint32_t*>(P(i_v0));
        auto* k1 = reinterpret_cast<uint32_t*>(P(i_k1));
        auto* v1 = reinterpret_cast<uint32_t*>(P(i_v1));
        tm.stage("collect", launches);
        l = brmq::launch_collect(dQ, q, n, k0, v0, nullptr, nullptr, &ctl->err, s,
                                 c->epoch_dev, n_epochs);
        launches += l;
        tm.end(l);
        tm.stage("radix_sort", launches);
        bool in_alt = false;
        l = brmq::launch_radix_sort(k0, v0, k1, v1, m, bits, P(i_rs), S(i_rst), s, &in_alt,
                                    c->epoch_dev, 2);
        launches += l;
        tm.end(l);
        tm.stage("unique_rank", launches);
        l = brmq::launch_unique(in_alt ? k1 : k0, in_alt ? v1 : v0, m, n, bd, cl, cr, c->bitmap,
                                ctl->rcnt, R, ctl->span, &ctl->nb, &ctl->err, S(i_ust),
                                &ctl->tickets[0], c->epoch_dev, 1, s);
        launches += l;
        tm.end(l);
        tm.stage("contract", launches);
        l = brmq::launch_contract(dA, n, c->bitmap, ctl->span, ctl->rcnt, true, ST, &ctl->nb,
                                  &ctl->aq_len, nullptr, S(i_cst), c->epoch_dev, 0, s,
                                  /*marked=*/true, nullptr, 2 * q);
        l += brmq::launch_marked_fill(dA, bd, &ctl->nb, m, ST, s);
        l += brmq::launch_marked_edges(dA, n, ctl->span, &ctl->nb, ST, s);
        launches += l;
        tm.end(l);
        tm.stage("sparse_table", launches);
        l = brmq::launch_sparse_table(ST, e_max, &ctl->aq_len, s);
        launches += l;
        tm.end(l);
        tm.stage("query", launches);
        l = brmq::launch_query_st(dQ, cl, cr, q, ST, e_max, dAns, s, brmq::CtlPublish{});
        launches += l;
        tm.end(l);
        launches += publish(c, ctl, s);  // control header -> host (k_publish)
        if (int rc = check_status(c)) return rc;
        if (!dev) {
            tm.stage("d2h", launches);
            CUDA_TRY(c->stager.d2h(answers, dAns, q * 8, s));
            tm.end(0);
        }
        // (the control header reaches c->ctl_host from the final kernel: publish())
        return BRMQ_OK;
    };
    const GraphKey key{3, A, n, Q, q, 1, 0, answers, s};
    if (int rc = prepare_ctl(c, ctl)) return rc;
    if (int rc = run_solve(c, key, dev, tm, launches, enqueue)) return rc;
    c->ctl_clean = true;  // the final kernel published and re-zeroed the header
    c->epoch_host += n_epochs;
    CUDA_TRY(cudaStreamSynchronize(s));
    tm.finish();
    const Control& h = *c->ctl_host;
    c->info.boundary = h.nb;
    c->info.span_lo = ~h.span[0];
    c->info.span_hi = h.span[1];
    c->info.blocks = h.aq_len;  // |E|: the element table's columns
    c->info.levels = h.aq_len ? brmq::floor_log2_u64(h.aq_len) + 1 : 0;
    c->info.kernel_launches = uint32_t(launches);
    return map_err(h.err);
}

// ------------------------------------------------------------ stage entry points
int brmq_collect_endpoints(brmq_ctx* c, const brmq_query* Q, uint64_t q, brmq_endpoint* eps,
                           uint32_t flags) {
    if (!c) return fail(BRMQ_EINVAL, "null context");
    if (int rc = settle_pending(c)) return rc;  // an outstanding async solve first
    if (q > (1ull << 31)) return fail(BRMQ_EINVAL, "collect_endpoints: too many queries for 32-bit origins");
    if (q == 0) return BRMQ_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    const bool dev = is_device(flags);
    const uint64_t m = 2 * q;
    Carve cv;
    const size_t i_ctl = cv.add(sizeof(Control));
    const size_t i_k = cv.add(m * 4), i_v = cv.add(m * 4);
    const size_t i_q = dev ? 0 : cv.add(q * 16);
    const size_t i_e = dev ? 0 : cv.add(m * 8);
    if (int rc = ensure_ws(c, cv.total)) return rc;
    auto P = [&](size_t i) { return c->ws + cv.off[i]; };
    cudaStream_t s = c->stream;
    auto* ctl = reinterpret_cast<Control*>(P(i_ctl));
    const uint64_t* dQ = dev ? reinterpret_cast<const uint64_t*>(Q) : reinterpret_cast<uint64_t*>(P(i_q));
    void* dE = dev ? static_cast<void*>(eps) : static_cast<void*>(P(i_e));
    c->ctl_clean = false;  // stage calls leave the header dirty
    CUDA_TRY(cudaMemsetAsync(ctl, 0, kCtlHeader, s));
    if (!dev) CUDA_TRY(c->stager.h2d(const_cast<uint64_t*>(dQ), Q, q * 16, s));
    auto* k = reinterpret_cast<uint32_t*>(P(i_k));
    auto* v = reinterpret_cast<uint32_t*>(P(i_v));
    brmq::launch_collect(dQ, q, ~0ull, k, v, nullptr, nullptr, &ctl->err, s);  // positions truncated to 32 bits (contraction.cpp:19-20)
    brmq::launch_join_eps(k, v, m, dE, s);
    if (int rc = check_status(c)) return rc;
    if (!dev) CUDA_TRY(cudaMemcpyAsync(eps, dE, m * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return BRMQ_OK;
}

int brmq_sort_endpoints(brmq_ctx* c, brmq_endpoint* eps, uint64_t m, int sort_kind, uint32_t flags) {
    if (!c) return fail(BRMQ_EINVAL, "null context");
    if (int rc = settle_pending(c)) return rc;  // an outstanding async solve first
    if (sort_kind < 0 || sort_kind > 2) return fail(BRMQ_EINVAL, "unknown sort kind %d", sort_kind);
    if (m < 2) return BRMQ_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    const bool dev = is_device(flags);
    Carve cv;
    const size_t i_k0 = cv.add(m * 4), i_v0 = cv.add(m * 4), i_k1 = cv.add(m * 4), i_v1 = cv.add(m * 4);
    const size_t i_rs = cv.add(brmq::radix_sort_temp_bytes(m, 32));
    const size_t i_e = dev ? 0 : cv.add(m * 8);
    if (int rc = ensure_ws(c, cv.total)) return rc;
    c->ctl_clean = false;  // stage calls may overwrite the control header
    if (int rc = ensure_status(c, brmq::radix_sort_status_words(m, 32) * 8)) return rc;
    auto P = [&](size_t i) { return c->ws + cv.off[i]; };
    cudaStream_t s = c->stream;
    void* dE = dev ? static_cast<void*>(eps) : static_cast<void*>(P(i_e));
    if (!dev) CUDA_TRY(cudaMemcpyAsync(dE, eps, m * 8, cudaMemcpyHostToDevice, s));
    auto* k0 = reinterpret_cast<uint32_t*>(P(i_k0));
    auto* v0 = reinterpret_cast<uint32_t*>(P(i_v0));
    auto* k1 = reinterpret_cast<uint32_t*>(P(i_k1));
    auto* v1 = reinterpret_cast<uint32_t*>(P(i_v1));
    brmq::launch_split_eps(dE, m, k0, v0, s);
    bool in_alt = false;
    if (int rc = begin_epochs(c, 4)) return rc;
    brmq::launch_k(k_bump_epoch, dim3(1), dim3(1), 0, s, c->epoch_dev, 4);
    c->epoch_host += 4;
    brmq::launch_radix_sort(k0, v0, k1, v1, m, 32, P(i_rs), reinterpret_cast<uint64_t*>(c->st), s,
                            &in_alt, c->epoch_dev, 0);
    brmq::launch_join_eps(in_alt ? k1 : k0, in_alt ? v1 : v0, m, dE, s);
    if (int rc = check_status(c)) return rc;
    if (!dev) CUDA_TRY(cudaMemcpyAsync(eps, dE, m * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return BRMQ_OK;
}

int brmq_build_contracted(brmq_ctx* c, const int32_t* A, uint64_t n, const brmq_endpoint* sorted_eps,
                          uint64_t m, int32_t* aq_values, uint64_t* aq_origin, uint64_t* boundary,
                          uint64_t* nb, uint32_t flags) {
    return brmq_build_contracted_stats(c, A, n, sorted_eps, m, aq_values, aq_origin, boundary, nb,
                                       flags, nullptr);
}

int brmq_build_contracted_stats(brmq_ctx* c, const int32_t* A, uint64_t n, const brmq_endpoint* sorted_eps,
                                uint64_t m, int32_t* aq_values, uint64_t* aq_origin, uint64_t* boundary,
                                uint64_t* nb, uint32_t flags, uint64_t* array_reads) {
    if (!c || !nb) return fail(BRMQ_EINVAL, "null argument");
    if (int rc = settle_pending(c)) return rc;  // an outstanding async solve first
    *nb = 0;
    if (m == 0) return BRMQ_OK;  // contraction.cpp:116
    if (n == 0) return fail(BRMQ_ERANGE, "endpoint exceeds array bounds");
    if (n > 0xFFFFFFFFull) return fail(BRMQ_EINVAL, "input too long for 32-bit positions");
    CUDA_TRY(cudaSetDevice(c->device));
    const bool dev = is_device(flags);
    if (int rc = ensure_bitmap(c, n)) return rc;
    const uint64_t ntiles = brmq::contract_tiles(n);
    Carve cv;
    const size_t i_ctl = cv.add(sizeof(Control));
    const size_t i_k = cv.add(m * 4), i_v = cv.add(m * 4), i_bd = cv.add(m * 4);
    const size_t i_aq = cv.add((m + 2) * 8);
    Carve sv;
    const size_t i_ust = sv.add(brmq::unique_status_words(m) * 8);
    const size_t i_cst = sv.add(brmq::contract_status_words() * 8);
    const size_t i_a = dev ? 0 : cv.add(n * 4);
    const size_t i_e = dev ? 0 : cv.add(m * 8);
    const size_t i_av = dev ? 0 : cv.add(m * 4);
    const size_t i_ao = dev ? 0 : cv.add(m * 8);
    const size_t i_bo = dev ? 0 : cv.add(m * 8);
    if (int rc = ensure_ws(c, cv.total)) return rc;
    if (int rc = ensure_status(c, sv.total)) return rc;
    auto P = [&](size_t i) { return c->ws + cv.off[i]; };
    auto S = [&](size_t i) { return reinterpret_cast<uint64_t*>(c->st + sv.off[i]); };
    cudaStream_t s = c->stream;
    auto* ctl = reinterpret_cast<Control*>(P(i_ctl));
    const int32_t* dA = dev ? A : reinterpret_cast<int32_t*>(P(i_a));
    const void* dE = dev ? static_cast<const void*>(sorted_eps) : static_cast<void*>(P(i_e));
    int32_t* dav = dev ? aq_values : reinterpret_cast<int32_t*>(P(i_av));
    uint64_t* dao = dev ? aq_origin : reinterpret_cast<uint64_t*>(P(i_ao));
    uint64_t* dbo = dev ? boundary : reinterpret_cast<uint64_t*>(P(i_bo));
    c->ctl_clean = false;  // stage calls leave the header dirty
    CUDA_TRY(cudaMemsetAsync(ctl, 0, kCtlHeader, s));
    if (!dev) {
        CUDA_TRY(c->stager.h2d(const_cast<int32_t*>(dA), A, n * 4, s));
        CUDA_TRY(cudaMemcpyAsync(const_cast<void*>(dE), sorted_eps, m * 8, cudaMemcpyHostToDevice, s));
    }
    auto* k = reinterpret_cast<uint32_t*>(P(i_k));
    auto* v = reinterpret_cast<uint32_t*>(P(i_v));
    auto* bd = reinterpret_cast<uint32_t*>(P(i_bd));
    auto* AQ = reinterpret_cast<uint64_t*>(P(i_aq));
    brmq::launch_split_eps(dE, m, k, v, s);
    if (int rc = begin_epochs(c, 2)) return rc;
    brmq::launch_k(k_bump_epoch, dim3(1), dim3(1), 0, s, c->epoch_dev, 2);
    c->epoch_host += 2;
    uint32_t G = 0, R = 0;
    brmq::contract_partition(n, &G, &R);
    brmq::launch_unique(k, v, m, n, bd, nullptr, nullptr, c->bitmap, ctl->rcnt, R, ctl->span,
                        &ctl->nb, &ctl->err,
                        S(i_ust), &ctl->tickets[0], c->epoch_dev, 0, s);
    if (int rc = sync_and_read_control(c, ctl)) return rc;
    if (c->ctl_host->err) {
        // unsorted or out-of-range endpoints: clear any marks and report
        CUDA_TRY(cudaMemsetAsync(c->bitmap, 0, c->bitmap_words * 4, s));
        CUDA_TRY(cudaStreamSynchronize(s));
        return map_err(c->ctl_host->err);
    }
    brmq::launch_contract(dA, n, c->bitmap, ctl->span, ctl->rcnt, true, AQ, &ctl->nb,
                          &ctl->aq_len, nullptr,
                          S(i_cst), c->epoch_dev, 1, s, false, nullptr, m, nullptr, nullptr,
                          array_reads ? &ctl->array_reads : nullptr);
    brmq::launch_split_aq(AQ, &ctl->aq_len, m, dav, dao, s);
    brmq::launch_u32_to_u64(bd, &ctl->nb, m, dbo, s);
    if (int rc = check_status(c)) return rc;
    if (int rc = sync_and_read_control(c, ctl)) return rc;
    const uint64_t nbv = c->ctl_host->nb;
    const uint64_t areas = nbv > 0 ? nbv - 1 : 0;
    // contraction.cpp:84-107: with one area or more the scan reads b_0 .. b_last
    if (array_reads) *array_reads += areas ? c->ctl_host->array_reads : 0;
    if (!dev) {
        if (areas) {
            CUDA_TRY(cudaMemcpyAsync(aq_values, dav, areas * 4, cudaMemcpyDeviceToHost, s));
            CUDA_TRY(cudaMemcpyAsync(aq_origin, dao, areas * 8, cudaMemcpyDeviceToHost, s));
        }
        CUDA_TRY(cudaMemcpyAsync(boundary, dbo, nbv * 8, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaStreamSynchronize(s));
    }
    *nb = nbv;
    return map_err(c->ctl_host->err);
}

int brmq_remap_from_sorted(brmq_ctx* c, const brmq_endpoint* sorted_eps, uint64_t m,
                           const uint64_t* boundary, uint64_t nb, uint64_t q, uint32_t* cleft,
                           uint32_t* cright, uint8_t* degenerate, uint32_t flags) {
    if (!c) return fail(BRMQ_EINVAL, "null context");
    if (int rc = settle_pending(c)) return rc;  // an outstanding async solve first
    if (q == 0 && m == 0) return BRMQ_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    const bool dev = is_device(flags);
    Carve cv;
    const size_t i_ctl = cv.add(sizeof(Control));
    const size_t i_k = cv.add(m * 4), i_v = cv.add(m * 4);
    const size_t i_e = dev ? 0 : cv.add(m * 8);
    const size_t i_b = dev ? 0 : cv.add(nb * 8);
    const size_t i_cl = dev ? 0 : cv.add(q * 4), i_cr = dev ? 0 : cv.add(q * 4);
    const size_t i_dg = dev ? 0 : cv.add(q);
    if (int rc = ensure_ws(c, cv.total)) return rc;
    auto P = [&](size_t i) { return c->ws + cv.off[i]; };
    cudaStream_t s = c->stream;
    auto* ctl = reinterpret_cast<Control*>(P(i_ctl));
    const void* dE = dev ? static_cast<const void*>(sorted_eps) : static_cast<void*>(P(i_e));
    const uint64_t* dB = dev ? boundary : reinterpret_cast<uint64_t*>(P(i_b));
    uint32_t* dcl = dev ? cleft : reinterpret_cast<uint32_t*>(P(i_cl));
    uint32_t* dcr = dev ? cright : reinterpret_cast<uint32_t*>(P(i_cr));
    uint8_t* ddg = dev ? degenerate : reinterpret_cast<uint8_t*>(P(i_dg));
    c->ctl_clean = false;  // stage calls leave the header dirty
    CUDA_TRY(cudaMemsetAsync(ctl, 0, kCtlHeader, s));
    if (!dev) {
        if (m) CUDA_TRY(cudaMemcpyAsync(const_cast<void*>(dE), sorted_eps, m * 8, cudaMemcpyHostToDevice, s));
        if (nb) CUDA_TRY(cudaMemcpyAsync(const_cast<uint64_t*>(dB), boundary, nb * 8, cudaMemcpyHostToDevice, s));
    }
    if (q) {
        CUDA_TRY(cudaMemsetAsync(dcl, 0, q * 4, s));
        CUDA_TRY(cudaMemsetAsync(dcr, 0, q * 4, s));
    }
    auto* k = reinterpret_cast<uint32_t*>(P(i_k));
    auto* v = reinterpret_cast<uint32_t*>(P(i_v));
    brmq::launch_split_eps(dE, m, k, v, s);
    brmq::launch_remap_search(k, v, m, dB, nb, q, dcl, dcr, ddg, &ctl->err, s);
    if (int rc = check_status(c)) return rc;
    if (!dev && q) {
        CUDA_TRY(cudaMemcpyAsync(cleft, dcl, q * 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(cright, dcr, q * 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(degenerate, ddg, q, cudaMemcpyDeviceToHost, s));
    }
    if (int rc = sync_and_read_control(c, ctl)) return rc;
    return map_err(c->ctl_host->err);
}

int brmq_remap_queries(brmq_ctx* c, const brmq_query* Q, uint64_t q, const uint64_t* boundary,
                       uint64_t nb, uint32_t* cleft, uint32_t* cright, uint8_t* degenerate,
                       uint32_t flags) {
    if (!c) return fail(BRMQ_EINVAL, "null context");
    if (int rc = settle_pending(c)) return rc;  // an outstanding async solve first
    if (q == 0) return BRMQ_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    const bool dev = is_device(flags);
    Carve cv;
    const size_t i_ctl = cv.add(sizeof(Control));
    const size_t i_q = dev ? 0 : cv.add(q * 16);
    const size_t i_b = dev ? 0 : cv.add(nb * 8);
    const size_t i_cl = dev ? 0 : cv.add(q * 4), i_cr = dev ? 0 : cv.add(q * 4);
    const size_t i_dg = dev ? 0 : cv.add(q);
    if (int rc = ensure_ws(c, cv.total)) return rc;
    auto P = [&](size_t i) { return c->ws + cv.off[i]; };
    cudaStream_t s = c->stream;
    auto* ctl = reinterpret_cast<Control*>(P(i_ctl));
    const uint64_t* dQ = dev ? reinterpret_cast<const uint64_t*>(Q) : reinterpret_cast<uint64_t*>(P(i_q));
    const uint64_t* dB = dev ? boundary : reinterpret_cast<uint64_t*>(P(i_b));
    uint32_t* dcl = dev ? cleft : reinterpret_cast<uint32_t*>(P(i_cl));
    uint32_t* dcr = dev ? cright : reinterpret_cast<uint32_t*>(P(i_cr));
    uint8_t* ddg = dev ? degenerate : reinterpret_cast<uint8_t*>(P(i_dg));
    c->ctl_clean = false;  // stage calls leave the header dirty
    CUDA_TRY(cudaMemsetAsync(ctl, 0, kCtlHeader, s));
    if (!dev) {
        CUDA_TRY(c->stager.h2d(const_cast<uint64_t*>(dQ), Q, q * 16, s));
        if (nb) CUDA_TRY(cudaMemcpyAsync(const_cast<uint64_t*>(dB), boundary, nb * 8, cudaMemcpyHostToDevice, s));
    }
    brmq::launch_remap_queries(dQ, q, dB, nb, dcl, dcr, ddg, &ctl->err, s);
    if (int rc = check_status(c)) return rc;
    if (!dev) {
        CUDA_TRY(cudaMemcpyAsync(cleft, dcl, q * 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(cright, dcr, q * 4, cudaMemcpyDeviceToHost, s));
        CUDA_TRY(cudaMemcpyAsync(degenerate, ddg, q, cudaMemcpyDeviceToHost, s));
    }
    if (int rc = sync_and_read_control(c, ctl)) return rc;
    return map_err(c->ctl_host->err);
}

int brmq_build_block_sparse(brmq_ctx* c, const int32_t* values, uint64_t m, uint32_t k,
                            uint64_t* table, uint64_t* b_out, uint32_t* levels_out, uint32_t flags) {
    if (!c || !b_out || !levels_out) return fail(BRMQ_EINVAL, "null argument");
    if (int rc = settle_pending(c)) return rc;  // an outstanding async solve first
    if (k == 0) return fail(BRMQ_EINVAL, "build_block_sparse: k must be >= 1");
    if (m > 0xFFFFFFFFull) return fail(BRMQ_EINVAL, "input too long for 32-bit positions");
    const uint64_t b = (m + k - 1) / k;
    *b_out = b;
    *levels_out = b ? brmq::floor_log2_u64(b) + 1 : 0;
    if (b == 0) return BRMQ_OK;
    CUDA_TRY(cudaSetDevice(c->device));
    const bool dev = is_device(flags);
    const uint64_t cells = uint64_t(*levels_out) * b;
    Carve cv;
    const size_t i_v = dev ? 0 : cv.add(m * 4);
    const size_t i_t = dev ? 0 : cv.add(cells * 8);
    if (int rc = ensure_ws(c, cv.total)) return rc;
    c->ctl_clean = false;  // stage calls may overwrite the control header
    auto P = [&](size_t i) { return c->ws + cv.off[i]; };
    cudaStream_t s = c->stream;
    const int32_t* dV = dev ? values : reinterpret_cast<int32_t*>(P(i_v));
    uint64_t* dT = dev ? table : reinterpret_cast<uint64_t*>(P(i_t));
    if (!dev) CUDA_TRY(cudaMemcpyAsync(const_cast<int32_t*>(dV), values, m * 4, cudaMemcpyHostToDevice, s));
    CUDA_TRY(cudaMemsetAsync(dT, 0xFF, cells * 8, s));
    brmq::launch_block_argmin_i32(dV, m, k, dT, s);
    brmq::launch_sparse_table(dT, b, nullptr, s);
    brmq::launch_keys_to_pos(dT, cells, s);
    if (int rc = check_status(c)) return rc;
    if (!dev) CUDA_TRY(cudaMemcpyAsync(table, dT, cells * 8, cudaMemcpyDeviceToHost, s));
    CUDA_TRY(cudaStreamSynchronize(s));
    return BRMQ_OK;
}

}  // extern "C"
