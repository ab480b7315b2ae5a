// kernels.h -- host-side launchers of the sm_100a kernels (one .cu per stage).
// All launchers are asynchronous on the given stream and return the number of
// kernel launches they issued (for the bench's gpu_launches count).
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

namespace brmq {

// ---------------------------------------------------------------- launches
// Programmatic dependent launch (PDL) inside a solve: every kernel after the
// solve's first is launched with programmatic stream serialization, so its CTAs
// are scheduled while its predecessor drains (launch latency and the
// predecessor's tail overlap); each kernel opens with griddepcontrol.wait
// (common.cuh pdl_wait), which returns once the predecessor grid has completed
// and its memory is visible -- so the data dependences are unchanged, and since
// every kernel waits before it can complete, completion stays transitive along
// the chain.  Outside a PdlScope (stage entry points, timed stages) launches
// are plain stream-ordered launches.
struct PdlState {
    bool on = false;
    bool first = true;
};
inline PdlState& pdl_state() {
    static thread_local PdlState st;
    return st;
}
struct PdlScope {
    explicit PdlScope(bool on) { pdl_state() = PdlState{on, true}; }
    ~PdlScope() { pdl_state() = PdlState{}; }
    PdlScope(const PdlScope&) = delete;
    PdlScope& operator=(const PdlScope&) = delete;
};
// A kernel launch on `s`; launch errors surface through cudaGetLastError.
template <class... P, class... A>
inline void launch_k(void (*kern)(P...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     A&&... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    PdlState& st = pdl_state();
    if (st.on && !st.first) {
        at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
    }
    st.first = false;
    if (cudaLaunchKernelEx(&cfg, kern, static_cast<A&&>(args)...) != cudaSuccess) {
        // leave the error for the caller's cudaGetLastError (not consumed here)
    }
}
// A plain (non-PDL) launch point inside a scope: the next kernel after it is
// launched normally too (e.g. after a memcpy or an event record).
inline void pdl_break() { pdl_state().first = true; }

// End-of-solve publication of the control header into host-mapped memory: done
// by api.cu's k_publish after the final kernel (the kernels' `pub` arguments are
// unused since; kept so the launcher signatures stay stable).
struct CtlPublish {
    const uint32_t* ctl;  // device control header (u32 words)
    uint32_t* host;       // host-mapped mirror
    uint32_t* ticket;     // zeroed with the header at solve start
    uint32_t words;
    uint32_t reset_words; // leading words re-zeroed after the copy (for the next solve)
};

// ---------------------------------------------------------------- block_argmin.cu
// Level 0 of the block Sparse Table: keys[j] = packed leftmost-min key of block j
// (SPEC.md:199-203).
int launch_block_argmin_i32(const int32_t* A, uint64_t n, uint32_t k, uint64_t* keys,
                            cudaStream_t stream);
// Same over packed keys (A_Q) whose true length *len_dev <= len_max lives on the
// device; also stores *b_dev = ceil(len / k) for the later stages.
int launch_block_argmin_keys(const uint64_t* K, uint64_t len_max, const uint64_t* len_dev,
                             uint32_t k, uint64_t* keys, uint64_t* b_dev, cudaStream_t stream);

// Multi-level (k1 = 32) variant: also stores the leftmost-min key of every
// 32-element sub-block in sub[ceil(n/32)] (k must be a multiple of 32).
// A_Q keys: k-block keys + 32-key sub-block keys (k a multiple of 64, A_Q padded
// to an even count, 16-byte aligned), device-side length.
int launch_block_argmin_keys_ml(const uint64_t* K, uint64_t len_max, const uint64_t* len_dev,
                                uint32_t k, uint64_t* keys, uint64_t* sub, uint64_t* b_dev,
                                cudaStream_t stream);
int launch_block_argmin_ml(const int32_t* A, uint64_t n, uint32_t k, uint64_t* keys,
                           uint64_t* sub, cudaStream_t stream);
// ---------------------------------------------------------------- sparse_table.cu
// Levels 1..L-1 of the block Sparse Table, row e at ST + e*b (row 0 = level 0).
// b_dev (nullable) holds the true block count <= b (rows stay strided by b).
int launch_sparse_table(uint64_t* ST, uint64_t b, const uint64_t* b_dev, cudaStream_t stream);

// ---------------------------------------------------------------- query.cu
int launch_naive(const int32_t* A, uint64_t n, const uint64_t* Q, uint64_t q, uint64_t* answers,
                 uint32_t* err, cudaStream_t stream,
                    const CtlPublish& pub = CtlPublish{});
// scanned (nullable): += the cells of A inside the partial ranges scanned
// (the SPEC's instrumented speculation counter; one reduction per warp)
int launch_query_direct(const int32_t* A, uint64_t n, uint32_t k, const uint64_t* ST,
                        uint64_t b, const uint64_t* Q, uint64_t q, uint64_t* answers,
                        uint32_t* err, cudaStream_t stream,
                    const CtlPublish& pub = CtlPublish{}, uint64_t* scanned = nullptr);
// Multi-level BbST [32, k] answering: endpoint blocks resolved through the
// 32-element sub-block keys, raw A read only inside partial sub-blocks.
int launch_query_ml(const int32_t* A, uint64_t n, uint32_t k, const uint64_t* ST, uint64_t b,
                    const uint64_t* sub, const uint64_t* Q, uint64_t q, uint64_t* answers,
                    uint32_t* err, cudaStream_t stream,
                    const CtlPublish& pub = CtlPublish{});
// bitmap pipeline: contracted coordinates from the contraction's word_info
// BbST_CON answering with the sub-block level over A_Q (k a power of two in
// [64, 512]; launch_block_argmin_keys_ml built ST level 0 and `sub`).
int launch_query_con_flat(const uint64_t* AQ, uint32_t k, const uint64_t* ST, uint64_t b_max,
                          const uint64_t* sub, const uint64_t* Q, const uint2* word_info,
                          const uint32_t* cleft, const uint32_t* cright_raw, uint64_t n, uint64_t q,
                          uint64_t* answers, cudaStream_t stream, const CtlPublish& pub);
int launch_query_contracted_wi(const uint64_t* AQ, uint32_t k, const uint64_t* ST, uint64_t b_max,
                               const uint64_t* Q, const uint2* word_info, uint64_t n, uint64_t q,
                               uint64_t* answers, cudaStream_t stream,
                    const CtlPublish& pub = CtlPublish{});
int launch_query_contracted(const uint64_t* AQ, const uint64_t* aq_len_dev, uint32_t k,
                            const uint64_t* ST, uint64_t b_max, const uint64_t* Q,
                            const uint32_t* cleft, const uint32_t* cright_raw, uint64_t q,
                            uint64_t* answers, cudaStream_t stream,
                    const CtlPublish& pub = CtlPublish{});

// ---------------------------------------------------------------- query_chain.cu
// Multi-level BbST for any dividing chain ks[0] < ... < ks[h-1] (2 <= h <= kMaxChain):
// M[j] = ks[j]-block minima keys (j < h - 1), ST over the ks[h-1]-blocks.
constexpr uint32_t kMaxChain = 8;
int launch_query_chain(const int32_t* A, uint64_t n, const uint32_t* ks, uint32_t h,
                       const uint64_t* const* M, const uint64_t* ST, uint64_t stride,
                       const uint64_t* Q, uint64_t q, uint64_t* answers, uint32_t* err,
                       cudaStream_t stream, const CtlPublish& pub);
// ---------------------------------------------------------------- radix_sort.cu
size_t radix_sort_temp_bytes(uint64_t m, int bits);     // zeroed scratch (histograms, tickets)
size_t radix_sort_status_words(uint64_t m, int bits);   // epoch-tagged look-back words
int radix_sort_passes(int bits);
// Stable LSD sort of (key, value) u32 pairs by the low `bits` key bits; uses
// epochs *epoch_dev + epoch_off .. + passes - 1 (device counter, see api.cu).  *result_in_alt tells whether
// the sorted data ended in alt_keys / alt_vals.
int launch_radix_sort(uint32_t* keys, uint32_t* vals, uint32_t* alt_keys, uint32_t* alt_vals,
                      uint64_t m, int bits, void* tmp, uint64_t* status, cudaStream_t stream,
                      bool* result_in_alt, const uint32_t* epoch_dev, uint32_t epoch_off);
// The radix pipeline's sort + dedup as a two-level MSD radix sort: keys of 8..30
// bits, m >= 2^14 (radix_partition_shape; false: sort LSD with launch_radix_sort).
//   1. cudaMemsetAsync(tmp, 0, radix_sort_temp_bytes(m, bits))
//   2. launch_collect(..., span, ..., hist = radix_partition_hist(tmp), hshift = L,
//      hmask = 2^D - 1): the span and the top-digit histogram
//   3. launch_radix_partition_mark: the keys partitioned by their top D bits into
//      alt_keys (unstable: bucket order is all the next level needs), then per
//      bucket a counting digit over the low L bits in shared memory that dedups
//      and marks the (all-zero) boundary bitmap; err bit 2 as launch_mark_sorted.
bool radix_partition_shape(int bits, uint64_t m, uint64_t bitmap_words, int* D, int* L);
unsigned long long* radix_partition_hist(void* tmp);
int launch_radix_partition_mark(const uint32_t* keys, uint32_t* alt_keys, uint64_t m, int bits, uint64_t n,
                                void* tmp, uint32_t* bitmap, uint64_t bitmap_words, uint32_t* err,
                                cudaStream_t stream);

// ---------------------------------------------------------------- contract.cu
// The contraction partitions the tiles of A into G ranges of R tiles
// (contract_partition).  Its rank bases come either from the marked bitmap
// (k_collect, then k_piece_count: boundaries per piece and per range) or -- from
// sorted endpoints (k_unique) -- from the exclusive prefix rfirst[0..G] of the
// boundaries per range; launch_contract's `prefix` says which.
constexpr uint32_t kMaxContractRanges = 2048;
constexpr int kContractTileLog2 = 12;  // 4096-position tiles
void contract_partition(uint64_t n, uint32_t* G, uint32_t* R);
// fill0 / fill1 (nullable): ranges set to kNoKey on the way (ContractFuse's sub
// and table row 0)
// passes of k_collect's direct marking: 1, or one per 32 MiB slice of a bitmap
// larger than the L2 hit by at least one endpoint per 8 words
uint32_t collect_mark_slices(uint64_t n, uint64_t q);
int launch_collect(const uint64_t* Q, uint64_t q, uint64_t n, uint32_t* keys, uint32_t* vals,
                   uint32_t* bitmap, uint32_t* span, uint32_t* err, cudaStream_t s,
                   uint32_t* epoch_bump = nullptr, uint32_t epoch_by = 0,
                   uint64_t* fill0 = nullptr, uint64_t fill0_n = 0, uint64_t* fill1 = nullptr,
                   uint64_t fill1_n = 0, unsigned long long* hist = nullptr, uint32_t hshift = 0,
                   uint32_t hmask = 0);
// Boundaries per contraction piece (pcnt[g * 8 + w], 8 warps per range) and per
// range (rcnt[g]), popcounted from the bitmap.
#ifndef BRMQ_CWARPS
#define BRMQ_CWARPS 8
#endif
constexpr uint32_t kContractWarps = BRMQ_CWARPS;
int launch_piece_count(const uint32_t* bitmap, const uint32_t* span, uint64_t n, uint32_t* pcnt,
                       uint32_t* rcnt, cudaStream_t s);
size_t unique_status_words(uint64_t m);
// Sorted endpoint positions -> boundary bitmap + span (+ err bits 2: range, 4:
// unsorted); the ranks then come from the bitmap (launch_piece_count).
int launch_mark_sorted(const uint32_t* pos, uint64_t m, uint64_t n, uint32_t* bitmap, uint32_t* span,
                       uint32_t* err, cudaStream_t s);
int launch_unique(const uint32_t* pos, const uint32_t* org, uint64_t m, uint64_t n,
                  uint32_t* boundary, uint32_t* cleft, uint32_t* cright_raw, uint32_t* bitmap,
                  uint32_t* rcnt, uint32_t range_tiles, uint32_t* span, uint64_t* nb_out, uint32_t* err, uint64_t* status,
                  uint32_t* ticket, const uint32_t* epoch_dev, uint32_t epoch_off, cudaStream_t s);
size_t contract_tiles(uint64_t n);  // 8192-element tiles over A
size_t contract_bitmap_words(uint64_t n);  // bitmap words the contraction reads (whole tiles)
size_t contract_status_words();    // status-arena words the contraction needs
// Persistent cooperative contraction (contract.cu): bitmap of boundaries ->
// packed A_Q keys, |boundary| (nb_out) and |A_Q|; word_info (nullable) gets
// (rank prefix, bits) of every non-empty bitmap word, which is cleared.
// Small A_Q (BbST_CON, power-of-two k in [64, 512]): the contraction also
// yields the 32-key run minima (sub) and row 0 of the block Sparse Table (st) by
// reductions, and stores b = ceil(|A_Q| / k) in *b_dev.  sub[0 .. ceil(aq_max /
// 32)) and st[0 .. b_max) must hold kNoKey beforehand (k_collect fills them).
struct ContractFuse {
    uint64_t* sub;
    uint64_t* st;
    uint64_t b_max;
    uint32_t kshift;
    uint64_t* b_dev;
};
int launch_contract(const int32_t* A, uint64_t n, uint32_t* bitmap, const uint32_t* span,
                    const uint32_t* rcnt, bool prefix, uint64_t* aq, uint64_t* nb_out, uint64_t* aq_len, uint2* word_info,
                    uint64_t* status, const uint32_t* epoch_dev, uint32_t epoch_off,
                    cudaStream_t s, bool marked = false,
                    const uint32_t* pcnt = nullptr, uint64_t endpoints = 0,
                    const ContractFuse* fuse = nullptr, bool* fused = nullptr,
                    uint64_t* array_reads = nullptr);
int launch_remap_bitmap(const uint64_t* Q, uint64_t q, uint64_t n, const uint2* word_info,
                        uint32_t* cleft, uint32_t* cright_raw, cudaStream_t s);
// stage-API helpers (not on the solve path)
int launch_split_eps(const void* eps, uint64_t m, uint32_t* keys, uint32_t* vals, cudaStream_t s);
int launch_join_eps(const uint32_t* keys, const uint32_t* vals, uint64_t m, void* eps,
                    cudaStream_t s);
int launch_split_aq(const uint64_t* aq, const uint64_t* len, uint64_t len_max, int32_t* values,
                    uint64_t* origin, cudaStream_t s);
int launch_u32_to_u64(const uint32_t* a, const uint64_t* len, uint64_t len_max, uint64_t* out,
                      cudaStream_t s);
// remap_queries (contraction.cpp:152-171): binary search of both ends per query.
int launch_remap_queries(const uint64_t* Q, uint64_t q, const uint64_t* boundary, uint64_t nb,
                         uint32_t* cl, uint32_t* cr, uint8_t* dg, uint32_t* err, cudaStream_t s);
int launch_remap_search(const uint32_t* pos, const uint32_t* org, uint64_t m,
                        const uint64_t* boundary, uint64_t nb, uint64_t q, uint32_t* cl,
                        uint32_t* cr, uint8_t* dg, uint32_t* err, cudaStream_t s);
int launch_keys_to_pos(uint64_t* t, uint64_t count, cudaStream_t s);
// ST-RMQ_CON (SPEC.md "baseline"): marked entries + run fix-up, the two edge runs,
// and the element-Sparse-Table query over E (2m+1 keys, m = *m_dev boundaries).
int launch_marked_fill(const int32_t* A, const uint32_t* boundary, const uint64_t* m_dev,
                       uint64_t m_max, uint64_t* E, cudaStream_t s);
int launch_marked_edges(const int32_t* A, uint64_t n, const uint32_t* span, const uint64_t* m_dev,
                        uint64_t* E, cudaStream_t s);
int launch_query_st(const uint64_t* Q, const uint32_t* cleft, const uint32_t* cright_raw,
                    uint64_t q, const uint64_t* ST, uint64_t stride, uint64_t* answers,
                    cudaStream_t s,
                    const CtlPublish& pub = CtlPublish{});

}  // namespace brmq
