// harness.cpp -- host side of the bench-harness contract (include/brmq_harness.h,
// SPEC.md:379-456): RMQA / RMQQ / RMQR files, the Table 2 memory model, the
// value checksum and the answer verifier.  Plain C++, no CUDA.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
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
            // the structures the chain solve allocates (api.cu solve_chain): the
            // Sparse Table over the k_h-blocks plus one 8-byte key per k_j-block of
            // every lower level j < h - 1
            b = 8 * block_cells(n, ks[h - 1]);
            for (uint32_t j = 0; j + 1 < h; ++j) b += 8 * ((n + ks[j] - 1) / ks[j]);
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

// ---- emit_plot
int brmq_emit_plot(const char* csv_path, const char* svg_path) {
    if (!csv_path || !svg_path) return set_error(BRMQ_EINVAL, "null path");
    FILE* f = fopen(csv_path, "rb");
    if (!f) return set_error(BRMQ_EIO, "emit_plot: cannot read the CSV");
    std::string text;
    char buf[4096];
    for (size_t r; (r = fread(buf, 1, sizeof(buf), f)) > 0;) text.append(buf, r);
    fclose(f);
    // columns of emit_csv: algo, n, q, k_chain, ..., t_total_ns (index 10)
    struct Pt { double q, t; };
    std::map<std::string, std::vector<Pt>> series;  // ordered: deterministic output
    uint64_t n0 = 0;
    bool first = true, header = true;
    size_t pos = 0;
    while (pos < text.size()) {
        size_t e = text.find('\n', pos);
        if (e == std::string::npos) e = text.size();
        std::string line = text.substr(pos, e - pos);
        pos = e + 1;
        if (!line.empty() && line.back() == '\r') line.pop_back();
        if (line.empty()) continue;
        if (header) {  // the header row
            header = false;
            if (line.compare(0, 5, "algo,") == 0) continue;
        }
        std::vector<std::string> col;
        for (size_t a = 0;;) {
            const size_t b = line.find(',', a);
            col.push_back(line.substr(a, b == std::string::npos ? std::string::npos : b - a));
            if (b == std::string::npos) break;
            a = b + 1;
        }
        if (col.size() < 11) return set_error(BRMQ_EINVAL, "emit_plot: malformed CSV row");
        const uint64_t n = strtoull(col[1].c_str(), nullptr, 10);
        if (first) n0 = n;
        else if (n != n0) return set_error(BRMQ_EINVAL, "emit_plot: records do not share n");
        first = false;
        const double q = strtod(col[2].c_str(), nullptr), t = strtod(col[10].c_str(), nullptr);
        if (q > 0 && t > 0) series[col[0] + (col[3].empty() ? "" : " k=" + col[3])].push_back({q, t});
    }
    if (series.empty()) {
        fprintf(stderr, "brmq: emit_plot: no records, nothing written\n");
        return BRMQ_OK;
    }
    double qlo = 1e300, qhi = 0, tlo = 1e300, thi = 0;
    for (auto& kv : series) {
        std::sort(kv.second.begin(), kv.second.end(), [](const Pt& a, const Pt& b) { return a.q < b.q; });
        for (const Pt& p : kv.second) {
            qlo = std::min(qlo, p.q); qhi = std::max(qhi, p.q);
            tlo = std::min(tlo, p.t); thi = std::max(thi, p.t);
        }
    }
    const double lq0 = std::floor(std::log10(qlo)), lq1 = std::max(lq0 + 1, std::ceil(std::log10(qhi)));
    const double lt0 = std::floor(std::log10(tlo)), lt1 = std::max(lt0 + 1, std::ceil(std::log10(thi)));
    const double W = 720, H = 480, L = 80, R = 220, T = 30, B = 60;
    auto X = [&](double q) { return L + (std::log10(q) - lq0) / (lq1 - lq0) * (W - L - R); };
    auto Y = [&](double t) { return H - B - (std::log10(t) - lt0) / (lt1 - lt0) * (H - T - B); };
    FILE* o = fopen(svg_path, "wb");
    if (!o) return set_error(BRMQ_EIO, "emit_plot: cannot write the SVG");
    fprintf(o, "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"%.0f\" height=\"%.0f\" "
               "font-family=\"sans-serif\" font-size=\"12\">\n", W, H);
    fprintf(o, "<rect width=\"100%%\" height=\"100%%\" fill=\"white\"/>\n");
    fprintf(o, "<text x=\"%.0f\" y=\"18\">batched RMQ, n = %llu: total time vs q</text>\n", L,
            (unsigned long long)n0);
    for (double d = lq0; d <= lq1 + 1e-9; d += 1) {
        fprintf(o, "<line x1=\"%.1f\" y1=\"%.1f\" x2=\"%.1f\" y2=\"%.1f\" stroke=\"#ddd\"/>\n", X(std::pow(10, d)), T,
                X(std::pow(10, d)), H - B);
        fprintf(o, "<text x=\"%.1f\" y=\"%.1f\" text-anchor=\"middle\">1e%.0f</text>\n", X(std::pow(10, d)),
                H - B + 16, d);
    }
    for (double d = lt0; d <= lt1 + 1e-9; d += 1) {
        fprintf(o, "<line x1=\"%.1f\" y1=\"%.1f\" x2=\"%.1f\" y2=\"%.1f\" stroke=\"#ddd\"/>\n", L, Y(std::pow(10, d)),
                W - R, Y(std::pow(10, d)));
        fprintf(o, "<text x=\"%.1f\" y=\"%.1f\" text-anchor=\"end\">1e%.0f ns</text>\n", L - 6,
                Y(std::pow(10, d)) + 4, d);
    }
    fprintf(o, "<text x=\"%.1f\" y=\"%.1f\" text-anchor=\"middle\">q (log scale)</text>\n", (L + W - R) / 2,
            H - 16);
    static const char* kColors[] = {"#1f77b4", "#d62728", "#2ca02c", "#9467bd", "#ff7f0e", "#8c564b",
                                    "#e377c2", "#17becf"};
    int si = 0;
    for (const auto& kv : series) {
        const char* c = kColors[si % 8];
        fprintf(o, "<polyline class=\"series\" fill=\"none\" stroke=\"%s\" stroke-width=\"2\" points=\"", c);
        for (const Pt& p : kv.second) fprintf(o, "%.1f,%.1f ", X(p.q), Y(p.t));
        fprintf(o, "\"/>\n");
        for (const Pt& p : kv.second)
            fprintf(o, "<circle cx=\"%.1f\" cy=\"%.1f\" r=\"3\" fill=\"%s\"/>\n", X(p.q), Y(p.t), c);
        fprintf(o, "<text x=\"%.1f\" y=\"%.1f\" fill=\"%s\">%s</text>\n", W - R + 12, T + 16 + 18.0 * si, c,
                kv.first.c_str());
        ++si;
    }
    fprintf(o, "</svg>\n");
    fclose(o);
    return BRMQ_OK;
}

}  // extern "C"
