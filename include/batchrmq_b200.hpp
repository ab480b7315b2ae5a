// batchrmq_b200.hpp -- header-only C++ drop-in for the reference's `batchrmq`
// operator API, backed by the B200 engine through the C-ABI (brmq.h).
//
// A reference user replaces
//     #include "batchrmq/contraction.hpp"      (and types.hpp, bits.hpp)
// with
//     #include "batchrmq_b200.hpp"             (link -lbrmq)
// and keeps calling the same functions with the same types; the SPEC-level
// solves (SPEC.md:237 solve_batch_bbst_con, SPEC.md:302 solve_batch_bbst) are
// provided as well.  Errors are rethrown as the reference's std:: exception
// classes (brmq_status -> std::domain_error / out_of_range / invalid_argument
// / logic_error; CUDA failures -> std::runtime_error).
//
// Types are layout-identical to the reference (types.hpp:8-29,
// contraction.hpp:12-45), which is what lets the C-ABI take them by pointer.
#pragma once

#include <cstdint>
#include <new>
#include <span>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "brmq.h"

namespace batchrmq {

using Value = std::int32_t;  // types.hpp:8
using Index = std::uint64_t;  // types.hpp:9

struct Query {  // types.hpp:13-23
    Index left{0};
    Index right{0};
    Query() = default;
    Query(Index l, Index r) : left(l), right(r) {
        if (left > right) std::swap(left, right);
    }
    bool operator==(const Query&) const = default;
};
using QueryBatch = std::vector<Query>;  // types.hpp:26
using Answers = std::vector<Index>;     // types.hpp:29

struct Endpoint {  // contraction.hpp:12-21
    std::uint32_t pos{0};
    std::uint32_t origin{0};
    static std::uint32_t make_origin(std::uint32_t query_index, bool is_right) {
        return (query_index << 1) | (is_right ? 1u : 0u);
    }
    std::uint32_t query_index() const { return origin >> 1; }
    bool is_right() const { return (origin & 1u) != 0; }
};

enum class SortKind { Radix, Comparison };  // contraction.hpp:23

struct ContractionStats {  // contraction.hpp:47-49
    std::uint64_t array_reads{0};
};

struct ContractedArray {  // contraction.hpp:28-34
    std::vector<Value> aq_values;
    std::vector<Index> aq_origin;
    std::vector<Index> boundary;
    std::size_t size() const { return aq_values.size(); }
};

struct ContractedQuery {  // contraction.hpp:39-43
    std::uint32_t cleft{0};
    std::uint32_t cright{0};
    bool degenerate{false};
};
using ContractedQueryBatch = std::vector<ContractedQuery>;

struct BbstConParams {
    std::uint32_t k = 512;
    SortKind sort_kind = SortKind::Radix;
    unsigned thread_count = 1;  // accepted for source compatibility; the device decides
};

static_assert(sizeof(Query) == sizeof(brmq_query), "Query must match brmq_query");
static_assert(sizeof(Endpoint) == sizeof(brmq_endpoint), "Endpoint must match brmq_endpoint");

namespace b200 {

inline void check(int rc) {
    if (rc == BRMQ_OK) return;
    const std::string msg = brmq_last_error();
    switch (rc) {
        case BRMQ_EDOMAIN: throw std::domain_error(msg);
        case BRMQ_ERANGE: throw std::out_of_range(msg);
        case BRMQ_EINVAL: throw std::invalid_argument(msg);
        case BRMQ_ELOGIC: throw std::logic_error(msg);
        case BRMQ_ENOMEM: throw std::bad_alloc();
        default: throw std::runtime_error(msg);
    }
}

// One context (stream + workspace) per thread, device 0 unless set_device().
class Context {
public:
    explicit Context(int device = 0) { check(brmq_ctx_create(&ctx_, device)); }
    ~Context() { brmq_ctx_destroy(ctx_); }
    Context(const Context&) = delete;
    Context& operator=(const Context&) = delete;
    brmq_ctx* get() const { return ctx_; }

private:
    brmq_ctx* ctx_ = nullptr;
};

inline Context& context() {
    thread_local Context ctx(0);
    return ctx;
}

}  // namespace b200

// bits.hpp:10-13
inline std::uint32_t floor_log2(std::uint64_t x) {
    std::uint32_t out = 0;
    b200::check(brmq_floor_log2(x, &out));
    return out;
}

// contraction.hpp:51
inline std::vector<Endpoint> collect_endpoints(const QueryBatch& batch) {
    std::vector<Endpoint> eps(batch.size() * 2);
    b200::check(brmq_collect_endpoints(b200::context().get(),
                                       reinterpret_cast<const brmq_query*>(batch.data()), batch.size(),
                                       reinterpret_cast<brmq_endpoint*>(eps.data()), BRMQ_PTR_HOST));
    return eps;
}

// contraction.hpp:55
inline void sort_endpoints(std::vector<Endpoint>& endpoints, SortKind kind = SortKind::Radix) {
    b200::check(brmq_sort_endpoints(b200::context().get(),
                                    reinterpret_cast<brmq_endpoint*>(endpoints.data()), endpoints.size(),
                                    kind == SortKind::Radix ? BRMQ_SORT_RADIX : BRMQ_SORT_COMPARISON,
                                    BRMQ_PTR_HOST));
}

// contraction.hpp:61-64.  `threads` has no device meaning; `stats` receives the
// reads of `values` the device contraction counted (brmq_build_contracted_stats):
// every position of [b_0, b_last] once, the count of the reference's serial path
// (contraction.cpp:85-105, 133-139).
inline ContractedArray build_contracted(std::span<const Value> values,
                                        const std::vector<Endpoint>& sorted_endpoints,
                                        unsigned /*threads*/ = 1, ContractionStats* stats = nullptr) {
    const std::size_t m = sorted_endpoints.size();
    ContractedArray out;
    out.aq_values.resize(m);
    out.aq_origin.resize(m);
    out.boundary.resize(m);
    std::uint64_t nb = 0, reads = 0;
    b200::check(brmq_build_contracted_stats(b200::context().get(), values.data(), values.size(),
                                            reinterpret_cast<const brmq_endpoint*>(sorted_endpoints.data()), m,
                                            out.aq_values.data(), out.aq_origin.data(), out.boundary.data(),
                                            &nb, BRMQ_PTR_HOST, stats ? &reads : nullptr));
    const std::size_t areas = nb > 0 ? nb - 1 : 0;
    out.aq_values.resize(areas);
    out.aq_origin.resize(areas);
    out.boundary.resize(nb);
    if (stats) stats->array_reads += reads;
    return out;
}

// contraction.hpp:67 (contraction.cpp:152-171): binary search per query end
inline ContractedQueryBatch remap_queries(const QueryBatch& batch, const ContractedArray& contracted) {
    const std::size_t q = batch.size();
    std::vector<std::uint32_t> cl(q), cr(q);
    std::vector<std::uint8_t> dg(q);
    b200::check(brmq_remap_queries(b200::context().get(), reinterpret_cast<const brmq_query*>(batch.data()),
                                   q, contracted.boundary.data(), contracted.boundary.size(), cl.data(),
                                   cr.data(), dg.data(), BRMQ_PTR_HOST));
    ContractedQueryBatch out(q);
    for (std::size_t i = 0; i < q; ++i) out[i] = {cl[i], cr[i], dg[i] != 0};
    return out;
}

// contraction.hpp:71-73
inline ContractedQueryBatch remap_queries_from_sorted(const std::vector<Endpoint>& sorted_endpoints,
                                                      const ContractedArray& contracted,
                                                      std::size_t query_count) {
    std::vector<std::uint32_t> cl(query_count), cr(query_count);
    std::vector<std::uint8_t> dg(query_count);
    b200::check(brmq_remap_from_sorted(b200::context().get(),
                                       reinterpret_cast<const brmq_endpoint*>(sorted_endpoints.data()),
                                       sorted_endpoints.size(), contracted.boundary.data(),
                                       contracted.boundary.size(), query_count, cl.data(), cr.data(),
                                       dg.data(), BRMQ_PTR_HOST));
    ContractedQueryBatch out(query_count);
    for (std::size_t i = 0; i < query_count; ++i) out[i] = {cl[i], cr[i], dg[i] != 0};
    return out;
}

// SPEC.md:237-245
inline Answers solve_batch_bbst_con(std::span<const Value> array, const QueryBatch& batch,
                                    const BbstConParams& params = {}) {
    Answers out(batch.size());
    b200::check(brmq_solve_bbst_con(b200::context().get(), array.data(), array.size(),
                                    reinterpret_cast<const brmq_query*>(batch.data()), batch.size(),
                                    params.k,
                                    params.sort_kind == SortKind::Radix ? BRMQ_SORT_RADIX
                                                                        : BRMQ_SORT_COMPARISON,
                                    out.data(), BRMQ_PTR_HOST));
    return out;
}

// SPEC.md:302-310 with LevelConfig{[k]} (h = 1)
inline Answers solve_batch_bbst(std::span<const Value> array, const QueryBatch& batch,
                                std::uint32_t k = 512) {
    Answers out(batch.size());
    b200::check(brmq_solve_bbst(b200::context().get(), array.data(), array.size(),
                                reinterpret_cast<const brmq_query*>(batch.data()), batch.size(), k,
                                out.data(), BRMQ_PTR_HOST));
    return out;
}

// SPEC.md:331-377 solve_batch_st_rmq_con: the ST-RMQ_CON baseline
inline Answers solve_batch_st_rmq_con(std::span<const Value> array, const QueryBatch& batch) {
    Answers out(batch.size());
    b200::check(brmq_solve_st_rmq_con(b200::context().get(), array.data(), array.size(),
                                      reinterpret_cast<const brmq_query*>(batch.data()), batch.size(),
                                      out.data(), BRMQ_PTR_HOST));
    return out;
}

// naive.hpp:13-21 for every query (on the device)
inline Answers solve_batch_naive(std::span<const Value> array, const QueryBatch& batch) {
    Answers out(batch.size());
    b200::check(brmq_solve_naive(b200::context().get(), array.data(), array.size(),
                                 reinterpret_cast<const brmq_query*>(batch.data()), batch.size(),
                                 out.data(), BRMQ_PTR_HOST));
    return out;
}

// SPEC.md:266-310 with a LevelConfig chain (any dividing chain k_1 < ... < k_h, h <= 8)
struct LevelConfig {
    std::vector<std::uint32_t> block_sizes{512};
};
inline Answers solve_batch_bbst(std::span<const Value> array, const QueryBatch& batch,
                                const LevelConfig& cfg) {
    Answers out(batch.size());
    b200::check(brmq_solve_bbst_ml(b200::context().get(), array.data(), array.size(),
                                   reinterpret_cast<const brmq_query*>(batch.data()), batch.size(),
                                   cfg.block_sizes.data(), uint32_t(cfg.block_sizes.size()), out.data(),
                                   BRMQ_PTR_HOST));
    return out;
}

}  // namespace batchrmq
