// workload.cpp -- deterministic synthetic workloads (include/brmq_workload.h).
// Measurement infrastructure: host-only, counter-based (any thread can produce
// any element), so multi-threaded generation is bit-identical to serial.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "../../include/brmq_workload.h"

namespace {

inline uint64_t mix64(uint64_t z) {
    z ^= z >> 30;
    z *= 0xBF58476D1CE4E5B9ull;
    z ^= z >> 27;
    z *= 0x94D049BB133111EBull;
    z ^= z >> 31;
    return z;
}
inline uint64_t stream_base(uint64_t seed, uint64_t s) {
    return mix64(seed ^ (0xA0761D6478BD642Full * (s + 1)));
}
inline uint64_t draw(uint64_t base, uint64_t i) { return mix64(base + (i + 1) * 0x9E3779B97F4A7C15ull); }
inline uint64_t mulhi(uint64_t x, uint64_t m) {
    return uint64_t((unsigned __int128)x * m >> 64);
}

template <class F>
void par_for(uint64_t total, unsigned threads, F&& f) {
    if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
    if (total < (1u << 16)) threads = 1;
    const uint64_t parts = std::min<uint64_t>(threads, total ? total : 1);
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

uint64_t brmq_workload_mix64(uint64_t z) { return mix64(z); }

int brmq_workload_array(int kind, uint64_t n, uint64_t seed, int32_t* out, unsigned threads) {
    if (n == 0) return 0;
    if (!out) return 3;
    const uint64_t base = stream_base(seed, 0);
    switch (kind) {
        case BRMQ_ARRAY_UNIFORM31:
            par_for(n, threads, [&](uint64_t b, uint64_t e, uint64_t) {
                for (uint64_t i = b; i < e; ++i) out[i] = int32_t(draw(base, i) >> 33);
            });
            return 0;
        case BRMQ_ARRAY_TIES16:
            par_for(n, threads, [&](uint64_t b, uint64_t e, uint64_t) {
                for (uint64_t i = b; i < e; ++i) out[i] = int32_t(draw(base, i) >> 60);
            });
            return 0;
        case BRMQ_ARRAY_WALK: {
            // two-pass parallel prefix over +-1 steps, then subtract the minimum
            if (n > (1ull << 31)) return 3;  // keeps |walk| < 2^31
            if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
            std::vector<int64_t> sums(threads + 1, 0), mins(threads + 1, 0);
            const uint64_t parts = std::min<uint64_t>(threads, n);
            const uint64_t chunk = (n + parts - 1) / parts;
            auto step = [&](uint64_t i) -> int64_t { return i == 0 ? 0 : ((draw(base, i) & 1) ? 1 : -1); };
            std::vector<std::thread> pool;
            auto pass1 = [&](uint64_t w) {
                const uint64_t b = w * chunk, e = std::min(n, b + chunk);
                int64_t s = 0;
                for (uint64_t i = b; i < e; ++i) s += step(i);
                sums[w + 1] = s;
            };
            for (uint64_t w = 1; w < parts; ++w) pool.emplace_back(pass1, w);
            pass1(0);
            for (auto& t : pool) t.join();
            pool.clear();
            for (uint64_t w = 1; w <= parts; ++w) sums[w] += sums[w - 1];
            auto pass2 = [&](uint64_t w) {
                const uint64_t b = w * chunk, e = std::min(n, b + chunk);
                int64_t s = sums[w], mn = INT64_MAX;
                for (uint64_t i = b; i < e; ++i) {
                    s += step(i);
                    out[i] = int32_t(s);
                    mn = std::min(mn, s);
                }
                mins[w] = mn;
            };
            for (uint64_t w = 1; w < parts; ++w) pool.emplace_back(pass2, w);
            pass2(0);
            for (auto& t : pool) t.join();
            int64_t mn = INT64_MAX;
            for (uint64_t w = 0; w < parts; ++w) mn = std::min(mn, mins[w]);
            par_for(n, threads, [&](uint64_t b, uint64_t e, uint64_t) {
                for (uint64_t i = b; i < e; ++i) out[i] = int32_t(int64_t(out[i]) - mn);
            });
            return 0;
        }
        case BRMQ_ARRAY_PERMUTATION: {
            // [1..n], then floor(n/2) swaps of uniform index pairs
            if (n > 0x7FFFFFFFull) return 3;
            for (uint64_t i = 0; i < n; ++i) out[i] = int32_t(i + 1);
            for (uint64_t s = 0; s < n / 2; ++s) {
                const uint64_t a = mulhi(draw(base, 2 * s), n), b = mulhi(draw(base, 2 * s + 1), n);
                std::swap(out[a], out[b]);
            }
            return 0;
        }
        default:
            return 3;
    }
}

int brmq_workload_array_range(int kind, uint64_t n, uint64_t seed, uint64_t first, uint64_t count,
                              int32_t* out, unsigned threads) {
    // elements [first, first + count) of brmq_workload_array(kind, n, seed): the
    // counter-based draws make any slice independent of the rest (a sharded run
    // generates only its own shard)
    if (count == 0) return 0;
    if (!out || first + count > n) return 3;
    const uint64_t base = stream_base(seed, 0);
    switch (kind) {
        case BRMQ_ARRAY_UNIFORM31:
            par_for(count, threads, [&](uint64_t b, uint64_t e, uint64_t) {
                for (uint64_t i = b; i < e; ++i) out[i] = int32_t(draw(base, first + i) >> 33);
            });
            return 0;
        case BRMQ_ARRAY_TIES16:
            par_for(count, threads, [&](uint64_t b, uint64_t e, uint64_t) {
                for (uint64_t i = b; i < e; ++i) out[i] = int32_t(draw(base, first + i) >> 60);
            });
            return 0;
        default:
            return 3;  // the walk and the permutation are not slice-local
    }
}

int brmq_workload_queries(int kind, uint64_t n, uint64_t q, uint64_t seed, uint64_t* out,
                          unsigned threads) {
    if (q == 0) return 0;
    if (n == 0 || !out) return 3;
    const uint64_t base = stream_base(seed, 1);
    const double ln_n = std::log(double(n));
    switch (kind) {
        case BRMQ_QUERIES_UNIFORM:
            par_for(q, threads, [&](uint64_t b, uint64_t e, uint64_t) {
                for (uint64_t i = b; i < e; ++i) {
                    uint64_t l = mulhi(draw(base, 2 * i), n), r = mulhi(draw(base, 2 * i + 1), n);
                    if (l > r) std::swap(l, r);
                    out[2 * i] = l;
                    out[2 * i + 1] = r;
                }
            });
            return 0;
        case BRMQ_QUERIES_LOGUNIFORM:
            par_for(q, threads, [&](uint64_t b, uint64_t e, uint64_t) {
                for (uint64_t i = b; i < e; ++i) {
                    const double u = double(draw(base, 2 * i) >> 11) * 0x1.0p-53;
                    double lenf = std::floor(std::exp(u * ln_n));
                    uint64_t len = lenf < 1.0 ? 1 : (lenf >= double(n) ? n : uint64_t(lenf));
                    if (len < 1) len = 1;
                    if (len > n) len = n;
                    const uint64_t l = mulhi(draw(base, 2 * i + 1), n - len + 1);
                    out[2 * i] = l;
                    out[2 * i + 1] = l + len - 1;
                }
            });
            return 0;
        case BRMQ_QUERIES_MIXED:
            par_for(q, threads, [&](uint64_t b, uint64_t e, uint64_t) {
                for (uint64_t i = b; i < e; ++i) {
                    uint64_t len = (i & 1) == 0 ? 1 + mulhi(draw(base, 2 * i), 256)
                                                : 1 + mulhi(draw(base, 2 * i), n);
                    if (len > n) len = n;
                    const uint64_t l = mulhi(draw(base, 2 * i + 1), n - len + 1);
                    out[2 * i] = l;
                    out[2 * i + 1] = l + len - 1;
                }
            });
            return 0;
        default:
            return 3;
    }
}

}  // extern "C"
