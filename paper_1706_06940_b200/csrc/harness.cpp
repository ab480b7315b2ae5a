// harness.cpp -- host side of the bench-harness contract (include/brmq_harness.h,
// SPEC.md:379-456): RMQA / RMQQ / RMQR files, the Table 2 memory model, the
// value checksum and the answer verifier.  Plain C++, no CUDA.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "../../include/brmq_harness.h"
#include "errors.h"

namespace {

using brmq::set_error;

uint32_t floor_log2(uint64_t x) { return 63u - uint32_t(__builtin_clzll(x)); }

// ceil(m / k) blocks x (floor_log2(blocks) + 1) levels
uint64_t block_cells(uint64_t m, uint64_t k) {
    if (m == 0 || k == 0) return 0;
    const uint64_t b = (m + k - 1) / k;
    return b * (floor_log2(b) + 1);
}

// jagged element table: sum over levels e of (m - 2^e + 1) cells (element_sparse_table.cpp:16-31)
uint64_t jagged_cells(uint64_t m) {
    if (m == 0) return 0;
    const uint32_t L = floor_log2(m) + 1;
    uint64_t c = 0;
    for (uint32_t e = 0; e < L; ++e) c += m - (uint64_t(1) << e) + 1;
    return c;
}

// ---- files
struct File {
    FILE* f = nullptr;
    ~File() {
        if (f) fclose(f);
    }
};

int write_file(const char* path, const char magic[4], uint64_t count, const void* body,
               size_t elem) {
    if (!path) return set_error(BRMQ_EINVAL, "null path");
    if (count && !body) return set_error(BRMQ_EINVAL, "null buffer");
    File fh;
    fh.f = fopen(path, "wb");
    if (!fh.f) return set_error(BRMQ_EIO, (std::string("cannot open for writing: ") + path).c_str());
    unsigned char hdr[13];
    std::memcpy(hdr, magic, 4);
    hdr[4] = 1;
    for (int i = 0; i < 8; ++i) hdr[5 + i] = uint8_t(count >> (8 * i));  // little-endian u64
    if (fwrite(hdr, 1, sizeof hdr, fh.f) != sizeof hdr ||
        (count && fwrite(body, elem, count, fh.f) != count) || fflush(fh.f) != 0)
        return set_error(BRMQ_EIO, (std::string("write failed: ") + path).c_str());
    return BRMQ_OK;
}

int read_file(const char* path, const char magic[4], void* body, size_t elem, uint64_t cap,
              uint64_t* count) {
    if (!path || !count) return set_error(BRMQ_EINVAL, "null argument");
    File fh;
    fh.f = fopen(path, "rb");
    if (!fh.f) return set_error(BRMQ_EIO, (std::string("cannot open: ") + path).c_str());
    unsigned char hdr[13];
    if (fread(hdr, 1, sizeof hdr, fh.f) != sizeof hdr)
        return set_error(BRMQ_EINVAL, (std::string("truncated header: ") + path).c_str());
    if (std::memcmp(hdr, magic, 4) != 0)
        return set_error(BRMQ_EINVAL, (std::string("bad magic (want ") + std::string(magic, 4) +
                                       "): " + path).c_str());
    if (hdr[4] != 1) return set_error(BRMQ_EINVAL, (std::string("unsupported version: ") + path).c_str());
    uint64_t c = 0;
    for (int i = 0; i < 8; ++i) c |= uint64_t(hdr[5 + i]) << (8 * i);
    *count = c;
    if (!body) return BRMQ_OK;
    if (c > cap) return set_error(BRMQ_EINVAL, "buffer too small for the file's count");
    if (c && fread(body, elem, c, fh.f) != c)
        return set_error(BRMQ_EINVAL, (std::string("truncated body: ") + path).c_str());
    return BRMQ_OK;
}

static_assert(sizeof(brmq_query) == 16, "query layout");

template <class F>
void par_for(uint64_t total, unsigned threads, F&& f) {
    if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
    const uint64_t parts = std::max<uint64_t>(1, std::min<uint64_t>(threads, total / 1024 + 1));
    const uint64_t chunk = (total + parts - 1) / parts;
    std::vector<std::thread> pool;
    for (uint64_t w = 1; w < parts; ++w) {
        const uint64_t b = w * chunk, e = std::min(total, b + chunk);
        if (b < e) pool.emplace_back([&f, b, e, w] { f(b, e, w); });
    }
    f(0, std::min(total, chunk), 0);
    for (auto& t : pool) t.join();
}

}  // namespace

extern "C" {

int brmq_account_memory(int algo, uint64_t n, uint64_t q, const uint32_t* ks, uint32_t h,
                        uint64_t* extra_bytes, double* extra_pct) {
    if (!extra_bytes) return set_error(BRMQ_EINVAL, "null output");
    const bool needs_k = algo == BRMQ_ALGO_BBST || algo == BRMQ_ALGO_BBST_CON || algo == BRMQ_ALGO_BBST_ML;
    if (needs_k && (!ks || h == 0 || ks[0] == 0)) return set_error(BRMQ_EINVAL, "block size required");
    uint64_t b = 0;
    switch (algo) {
        case BRMQ_ALGO_NAIVE:
            b = 0;
            break;
        case BRMQ_ALGO_SPARSE:
            b = 4 * jagged_cells(n);
            break;
        case BRMQ_ALGO_ST_RMQ_CON: {
            const uint64_t M = 4 * q + 1;
            b = (n + 7) / 8 + 12 * M + 4 * jagged_cells(M);
            break;
        }
        case BRMQ_ALGO_BBST_CON:
            b = 20 * 2 * q + 8 * block_cells(2 * q, ks[h - 1]);
            break;
        case BRMQ_ALGO_BBST:
            b = 8 * block_cells(n, ks[h - 1]);
            break;
        case BRMQ_ALGO_BBST_ML:
            b = 8 * block_cells(n, ks[h - 1]);
            if (h >= 2) b += 8 * ((n + ks[0] - 1) / ks[0]);
            break;
        default:
            return set_error(BRMQ_EINVAL, "unknown algorithm id");
    }
    *extra_bytes = b;
    if (extra_pct) *extra_pct = n ? 100.0 * double(b) / (4.0 * double(n)) : 0.0;
    return BRMQ_OK;
}

int brmq_answers_checksum(const int32_t* A, uint64_t n, const uint64_t* answers, uint64_t q,
                          uint64_t* out) {
    if (!out || (q && !answers) || (n && !A)) return set_error(BRMQ_EINVAL, "null argument");
    uint64_t h = 0xcbf29ce484222325ull;  // FNV-1a offset basis
    for (uint64_t i = 0; i < q; ++i) {
        const uint32_t v = answers[i] < n ? uint32_t(A[answers[i]]) : 0xFFFFFFFFu;
        for (int b = 0; b < 4; ++b) {
            h ^= (v >> (8 * b)) & 0xFFu;
            h *= 0x100000001b3ull;  // FNV prime
        }
    }
    *out = h;
    return BRMQ_OK;
}

int brmq_write_array_file(const char* path, const int32_t* A, uint64_t n) {
    return write_file(path, "RMQA", n, A, sizeof(int32_t));
}
int brmq_read_array_file(const char* path, int32_t* A, uint64_t cap, uint64_t* n) {
    return read_file(path, "RMQA", A, sizeof(int32_t), cap, n);
}
int brmq_write_query_file(const char* path, const brmq_query* Q, uint64_t q) {
    return write_file(path, "RMQQ", q, Q, sizeof(brmq_query));
}
int brmq_read_query_file(const char* path, brmq_query* Q, uint64_t cap, uint64_t* q) {
    return read_file(path, "RMQQ", Q, sizeof(brmq_query), cap, q);
}
int brmq_write_answer_file(const char* path, const uint64_t* answers, uint64_t q) {
    return write_file(path, "RMQR", q, answers, sizeof(uint64_t));
}
int brmq_read_answer_file(const char* path, uint64_t* answers, uint64_t cap, uint64_t* q) {
    return read_file(path, "RMQR", answers, sizeof(uint64_t), cap, q);
}

int brmq_verify_answers(const int32_t* A, uint64_t n, const brmq_query* Q, uint64_t q,
                        const uint64_t* answers, unsigned threads, uint64_t* bad,
                        uint64_t* first_bad) {
    if (!bad || !first_bad || (q && (!Q || !answers)) || (n && !A))
        return set_error(BRMQ_EINVAL, "null argument");
    *bad = 0;
    *first_bad = q;
    if (q == 0) return BRMQ_OK;
    // block minima (values) and a sparse table over them
    constexpr uint64_t kB = 1024;
    const uint64_t nb = (n + kB - 1) / kB;
    std::vector<int32_t> bmin(nb ? nb : 1, INT32_MAX);
    par_for(nb, threads, [&](uint64_t b, uint64_t e, uint64_t) {
        for (uint64_t j = b; j < e; ++j) {
            int32_t m = INT32_MAX;
            for (uint64_t i = j * kB; i < std::min(n, j * kB + kB); ++i) m = std::min(m, A[i]);
            bmin[j] = m;
        }
    });
    const uint32_t L = nb ? floor_log2(nb) + 1 : 1;
    std::vector<std::vector<int32_t>> st(L);
    st[0] = bmin;
    for (uint32_t e = 1; e < L; ++e) {
        const uint64_t half = uint64_t(1) << (e - 1), cnt = nb - (uint64_t(1) << e) + 1;
        st[e].resize(cnt);
        for (uint64_t j = 0; j < cnt; ++j) st[e][j] = std::min(st[e - 1][j], st[e - 1][j + half]);
    }
    // minimum value of A[lo..hi] (lo <= hi < n)
    auto range_min = [&](uint64_t lo, uint64_t hi) {
        int32_t m = INT32_MAX;
        const uint64_t bl = lo / kB, br = hi / kB;
        if (bl == br) {
            for (uint64_t i = lo; i <= hi; ++i) m = std::min(m, A[i]);
            return m;
        }
        for (uint64_t i = lo; i < bl * kB + kB; ++i) m = std::min(m, A[i]);
        for (uint64_t i = br * kB; i <= hi; ++i) m = std::min(m, A[i]);
        if (br - bl >= 2) {
            const uint64_t s = br - bl - 1;
            const uint32_t e = floor_log2(s);
            m = std::min(m, std::min(st[e][bl + 1], st[e][br - (uint64_t(1) << e)]));
        }
        return m;
    };
    const unsigned T = threads ? threads : std::max(1u, std::thread::hardware_concurrency());
    std::vector<uint64_t> nbad(T + 1, 0), fbad(T + 1, q);
    par_for(q, threads, [&](uint64_t b, uint64_t e, uint64_t w) {
        for (uint64_t i = b; i < e; ++i) {
            uint64_t l = Q[i].left, r = Q[i].right;
            if (l > r) std::swap(l, r);  // types.hpp:18-20
            const uint64_t a = answers[i];
            bool ok = r < n && a >= l && a <= r;
            if (ok) {
                const int32_t v = A[a];
                // leftmost minimum: nothing smaller in [l, r], nothing <= v in [l, a)
                ok = range_min(l, r) == v && (a == l || range_min(l, a - 1) > v);
            }
            if (!ok) {
                ++nbad[w];
                fbad[w] = std::min(fbad[w], i);
            }
        }
    });
    for (unsigned w = 0; w <= T; ++w) {
        *bad += nbad[w];
        *first_bad = std::min(*first_bad, fbad[w]);
    }
    return BRMQ_OK;
}

}  // extern "C"
