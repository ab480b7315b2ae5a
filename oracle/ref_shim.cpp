// ref_shim.cpp -- extern "C" shim over the REFERENCE's own compiled code.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference sources where they lie (/root/reference/proj/core/src/*.cpp,
// headers from /root/reference/proj/core/include) into oracle/_ref/libbrmq_ref.so.
// No reference source is copied into this repository; this file only calls the
// reference's public functions (namespace batchrmq) and maps its exceptions to
// the C-ABI status codes of include/brmq.h.  It is used to pin oracle/oracle.c,
// to generate tests/golden fixtures, and as bench.py's "reference" CPU arm.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <span>
#include <stdexcept>
#include <vector>

#include "batchrmq/bits.hpp"
#include "batchrmq/contraction.hpp"
#include "batchrmq/element_sparse_table.hpp"
#include "batchrmq/naive.hpp"
#include "batchrmq/types.hpp"

using namespace batchrmq;

namespace {
int map_exc() {
    try {
        throw;
    } catch (const std::domain_error&) {
        return 1;
    } catch (const std::out_of_range&) {
        return 2;
    } catch (const std::invalid_argument&) {
        return 3;
    } catch (const std::logic_error&) {
        return 4;
    } catch (const std::bad_alloc&) {
        return 6;
    } catch (...) {
        return 4;
    }
}

QueryBatch to_batch(const uint64_t* Q, uint64_t q) {
    QueryBatch b;
    b.reserve(q);
    for (uint64_t i = 0; i < q; ++i) b.emplace_back(Q[2 * i], Q[2 * i + 1]);  // types.hpp:18 ctor
    return b;
}

std::vector<Endpoint> to_eps(const uint32_t* e, uint64_t m) {
    std::vector<Endpoint> v(m);
    for (uint64_t i = 0; i < m; ++i) v[i] = Endpoint{e[2 * i], e[2 * i + 1]};
    return v;
}
}  // namespace

extern "C" {

int ref_floor_log2(uint64_t x, uint32_t* out) {
    try {
        *out = floor_log2(x);
        return 0;
    } catch (...) {
        return map_exc();
    }
}

int ref_naive_rmq(const int32_t* A, uint64_t n, uint64_t l, uint64_t r, uint64_t* out) {
    try {
        *out = naive_rmq(std::span<const Value>(A, n), Query(l, r));
        return 0;
    } catch (...) {
        return map_exc();
    }
}

int ref_collect_endpoints(const uint64_t* Q, uint64_t q, uint32_t* eps) {
    try {
        auto v = collect_endpoints(to_batch(Q, q));
        for (uint64_t i = 0; i < v.size(); ++i) {
            eps[2 * i] = v[i].pos;
            eps[2 * i + 1] = v[i].origin;
        }
        return 0;
    } catch (...) {
        return map_exc();
    }
}

int ref_sort_endpoints(uint32_t* eps, uint64_t m, int kind) {
    try {
        auto v = to_eps(eps, m);
        sort_endpoints(v, kind == 0 ? SortKind::Radix : SortKind::Comparison);
        for (uint64_t i = 0; i < m; ++i) {
            eps[2 * i] = v[i].pos;
            eps[2 * i + 1] = v[i].origin;
        }
        return 0;
    } catch (...) {
        return map_exc();
    }
}

int ref_build_contracted(const int32_t* A, uint64_t n, const uint32_t* sorted_eps, uint64_t m,
                         unsigned threads, int32_t* aq_values, uint64_t* aq_origin,
                         uint64_t* boundary, uint64_t* nb, uint64_t* reads) {
    try {
        ContractionStats st;
        auto c = build_contracted(std::span<const Value>(A, n), to_eps(sorted_eps, m), threads,
                                  reads ? &st : nullptr);
        std::memcpy(aq_values, c.aq_values.data(), c.aq_values.size() * sizeof(int32_t));
        std::memcpy(aq_origin, c.aq_origin.data(), c.aq_origin.size() * sizeof(uint64_t));
        std::memcpy(boundary, c.boundary.data(), c.boundary.size() * sizeof(uint64_t));
        *nb = c.boundary.size();
        if (reads) *reads = st.array_reads;
        return 0;
    } catch (...) {
        return map_exc();
    }
}

int ref_remap_from_sorted(const uint32_t* sorted_eps, uint64_t m, const uint64_t* boundary,
                          uint64_t nb, uint64_t q, uint32_t* cl, uint32_t* cr, uint8_t* dg) {
    try {
        ContractedArray c;
        c.boundary.assign(boundary, boundary + nb);
        auto out = remap_queries_from_sorted(to_eps(sorted_eps, m), c, q);
        for (uint64_t i = 0; i < q; ++i) {
            cl[i] = out[i].cleft;
            cr[i] = out[i].cright;
            dg[i] = out[i].degenerate ? 1 : 0;
        }
        return 0;
    } catch (...) {
        return map_exc();
    }
}

int ref_remap_queries(const uint64_t* Q, uint64_t q, const uint64_t* boundary, uint64_t nb,
                      uint32_t* cl, uint32_t* cr, uint8_t* dg) {
    try {
        ContractedArray c;
        c.boundary.assign(boundary, boundary + nb);
        auto out = remap_queries(to_batch(Q, q), c);
        for (uint64_t i = 0; i < q; ++i) {
            cl[i] = out[i].cleft;
            cr[i] = out[i].cright;
            dg[i] = out[i].degenerate ? 1 : 0;
        }
        return 0;
    } catch (...) {
        return map_exc();
    }
}

void* ref_est_build(const int32_t* values, uint64_t n, int* rc) {
    try {
        *rc = 0;
        return new ElementSparseTable(std::span<const Value>(values, n));
    } catch (...) {
        *rc = map_exc();
        return nullptr;
    }
}

int ref_est_arg_min(const void* t, const int32_t* values, uint64_t n, uint64_t l, uint64_t r,
                    uint64_t* out) {
    try {
        *out = static_cast<const ElementSparseTable*>(t)->arg_min(std::span<const Value>(values, n),
                                                                  Query(l, r));
        return 0;
    } catch (...) {
        return map_exc();
    }
}

uint64_t ref_est_cell_count(const void* t) {
    return static_cast<const ElementSparseTable*>(t)->cell_count();
}
uint64_t ref_est_level_count(const void* t) {
    return static_cast<const ElementSparseTable*>(t)->level_count();
}
uint64_t ref_est_level(const void* t, uint64_t e, uint32_t* out) {
    const auto& row = static_cast<const ElementSparseTable*>(t)->level(e);
    std::memcpy(out, row.data(), row.size() * sizeof(uint32_t));
    return row.size();
}
void ref_est_free(void* t) { delete static_cast<ElementSparseTable*>(t); }

// The reference CPU path for the whole batch: every stage is the
// reference's own code; only build_contracted is multi-threaded (threads).
// stage_s (may be NULL) receives 5 wall-clock stage times in seconds:
// [collect+sort, build_contracted, remap, ElementSparseTable, answer].
int ref_solve_oracle(const int32_t* A, uint64_t n, const uint64_t* Q, uint64_t q,
                     unsigned threads, uint64_t* answers, double* stage_s) {
    using clk = std::chrono::steady_clock;
    try {
        if (q == 0) return 0;
        const QueryBatch batch = to_batch(Q, q);
        for (const Query& x : batch)
            if (x.right >= n) throw std::out_of_range("query exceeds array bounds");
        auto t0 = clk::now();
        auto eps = collect_endpoints(batch);
        sort_endpoints(eps, SortKind::Radix);
        auto t1 = clk::now();
        auto con = build_contracted(std::span<const Value>(A, n), eps, threads);
        auto t2 = clk::now();
        auto cq = remap_queries_from_sorted(eps, con, q);
        auto t3 = clk::now();
        ElementSparseTable est;
        if (con.size() > 0) est = ElementSparseTable(std::span<const Value>(con.aq_values));
        auto t4 = clk::now();
        const std::span<const Value> aq(con.aq_values);
        for (uint64_t i = 0; i < q; ++i) {
            if (cq[i].degenerate || con.size() == 0) {
                answers[i] = batch[i].left;
            } else {
                answers[i] = con.aq_origin[est.arg_min(aq, Query(cq[i].cleft, cq[i].cright))];
            }
        }
        auto t5 = clk::now();
        if (stage_s) {
            auto d = [](auto a, auto b) { return std::chrono::duration<double>(b - a).count(); };
            stage_s[0] = d(t0, t1);
            stage_s[1] = d(t1, t2);
            stage_s[2] = d(t2, t3);
            stage_s[3] = d(t3, t4);
            stage_s[4] = d(t4, t5);
        }
        return 0;
    } catch (...) {
        return map_exc();
    }
}

}  // extern "C"
