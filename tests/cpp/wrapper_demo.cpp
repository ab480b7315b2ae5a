// Reference-style C++ caller of the B200 engine through include/batchrmq_b200.hpp:
// the same calls a user of the reference's batchrmq API makes (SPEC.md worked
// instance), plus the exception mapping.
#include <cstdio>
#include <stdexcept>
#include <vector>

#include "batchrmq_b200.hpp"

using namespace batchrmq;

#define CHECK(c)                                                        \
    do {                                                                \
        if (!(c)) {                                                     \
            std::fprintf(stderr, "FAILED %s:%d %s\n", __FILE__, __LINE__, #c); \
            return 1;                                                   \
        }                                                               \
    } while (0)

int main() {
    const std::vector<Value> A{5, 3, 8, 2, 7, 6, 9, 1};
    const QueryBatch batch{Query(1, 4), Query(6, 3)};  // reversed pair is normalised by the ctor
    auto eps = collect_endpoints(batch);
    CHECK(eps.size() == 4 && eps[0].pos == 1 && eps[3].pos == 6);
    sort_endpoints(eps);
    CHECK(eps[0].pos == 1 && eps[1].pos == 3 && eps[2].pos == 4 && eps[3].pos == 6);
    bool thrown = false;
    ContractionStats stats;
    auto con = build_contracted(A, eps, 1, &stats);
    CHECK(stats.array_reads == 6);  // positions 1..6 read once (contraction.cpp:85-105)
    CHECK((con.boundary == std::vector<Index>{1, 3, 4, 6}));
    CHECK((con.aq_values == std::vector<Value>{2, 2, 6}));
    CHECK((con.aq_origin == std::vector<Index>{3, 3, 5}));
    auto cq = remap_queries_from_sorted(eps, con, batch.size());
    CHECK(cq[0].cleft == 0 && cq[0].cright == 1 && cq[1].cleft == 1 && cq[1].cright == 2);
    auto bq = remap_queries(QueryBatch{Query(1, 4), Query(6, 3), Query(2, 2)}, con);  // contraction.cpp:152-171
    CHECK(bq[0].cleft == 0 && bq[0].cright == 1 && bq[1].cleft == 1 && bq[1].cright == 2);
    CHECK(bq[2].degenerate && bq[2].cleft == 0 && bq[2].cright == 0);
    thrown = false;
    try {
        remap_queries(QueryBatch{Query(0, 4)}, con);
    } catch (const std::logic_error&) {
        thrown = true;
    }
    CHECK(thrown);
    CHECK((solve_batch_bbst_con(A, batch) == Answers{3, 3}));
    CHECK((solve_batch_bbst_con(A, batch, BbstConParams{2, SortKind::Comparison, 4}) == Answers{3, 3}));
    CHECK((solve_batch_bbst(A, batch, 2) == Answers{3, 3}));
    CHECK((solve_batch_bbst(A, batch, LevelConfig{{32, 64}}) == Answers{3, 3}));
    CHECK((solve_batch_st_rmq_con(A, batch) == Answers{3, 3}));  // SPEC.md:359 worked instance
    CHECK((solve_batch_st_rmq_con(A, QueryBatch{Query(0, 7)}) == Answers{7}));
    CHECK((solve_batch_naive(A, batch) == Answers{3, 3}));
    CHECK(floor_log2(48829) == 15);
    thrown = false;
    try {
        solve_batch_bbst(A, QueryBatch{Query(0, 8)});
    } catch (const std::out_of_range&) {
        thrown = true;
    }
    CHECK(thrown);
    thrown = false;
    try {
        floor_log2(0);
    } catch (const std::domain_error&) {
        thrown = true;
    }
    CHECK(thrown);
    std::printf("wrapper_demo OK\n");
    return 0;
}
