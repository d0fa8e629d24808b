// Host runtime of the B200 ABFT library: owns device buffers, tensor maps, the per-stream
// workspace and the launch decisions. The C ABI (capi.cpp) is a thin layer over this.
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include <vector>

#include "abft_internal.h"

namespace abftk {

struct Fault {
    bool active = false;
    int64_t row = 0, col = 0;
    uint32_t bit = 0;
};
// A C' fault of one problem of a batched call (grouped jobs carry several per launch).
struct BatchFault {
    int64_t batch = 0, row = 0, col = 0;
    uint32_t bit = 0;
};

// ---- GEMM (replaces P:src/gemm_abft.hpp:23-74)
// batch > 1: `batch` independent weights, weight b at d_b + b * b_bstride (batched GEMM).
GemmWeight* encode_weight(const int8_t* d_b, int64_t k, int64_t n, int64_t ldb, cudaStream_t st, int64_t batch = 1,
                          int64_t b_bstride = 0);
// Re-encode into an existing handle, growing its buffers only when needed (campaign scratch).
void encode_weight_into(GemmWeight& w, const int8_t* d_b, int64_t k, int64_t n, int64_t ldb, cudaStream_t st,
                        int64_t batch = 1, int64_t b_bstride = 0);
// Logical k x (n+1) [B | cs] matrix, row-major (PackedEncodedWeight::at contract).
void read_encoded(const GemmWeight& w, int8_t* d_out, cudaStream_t st);
void set_checksums(GemmWeight& w, const int8_t* d_cs, cudaStream_t st);
void free_weight(GemmWeight* w);
GemmTiling choose_tiling(int64_t m, int64_t n, int64_t k_pad, bool checked, bool c_tma_ok, bool fault);
// checked == false: plain GEMM (csum/flags/err_count ignored).
// Fused requantization of the GEMM output (P:src/quant.cpp:77-102): u8 out = requantize(C').
struct RequantArgs {
    const int32_t* row_sum_a = nullptr;  // [m]
    const int32_t* col_sum_b = nullptr;  // [n]
    RequantDev params{};
    uint8_t* out = nullptr;
    int64_t ld_out = 0;
};
void check_requant_params(const RequantDev& q);
// Batched GEMM: `batch` problems of one shape in one launch; problem b reads A at + b*a_bstride bytes and
// weight b of a batched weight (or weight 0 of a single one) and writes C/csum/flags at its strides and
// err_count[b]. Fault (if any) applies to problem fault_batch.
struct GemmBatch {
    int64_t batch = 1;
    int64_t a_bstride = 0;     // bytes
    int64_t c_bstride = 0;     // int32 elements
    int64_t csum_bstride = 0;  // int32 elements
    int64_t flags_bstride = 0; // bytes
    int64_t fault_batch = 0;            // problem of `fault` (single-fault form)
    const BatchFault* faults = nullptr;  // further C' faults; at most kMaxGemmFaults per call in total
    int64_t nfaults = 0;
    // (internal) row-stacked requests: batch == 1, m = requests * stack_rows; d_err_count has one entry per request
    int64_t stack_rows = 0;
};
void gemm(const uint8_t* d_a, int64_t m, int64_t lda, const GemmWeight& w, int32_t* d_c, int64_t ldc, bool checked,
          int32_t* d_csum, int64_t csum_ld, uint8_t* d_flags, uint32_t* d_err_count, const Fault* fault,
          cudaStream_t st, const GemmTiling* force = nullptr, const RequantArgs* rq = nullptr,
          const GemmBatch* batch = nullptr);
// Heterogeneous grouped GEMM: problems of different (m, n, k), each with its own A, encoded weight and outputs, in
// ONE persistent launch (the D5 MLP layers). Built once (tensor maps and per-problem parameters uploaded), run any
// number of times on one stream at a time (the per-row verdict scratch belongs to the group).
struct GemmProblem {
    const uint8_t* a = nullptr;
    int64_t m = 0, lda = 0;
    const GemmWeight* w = nullptr;
    int32_t* c = nullptr;
    int64_t ldc = 0;
    int32_t* csum = nullptr;  // checked only
    int64_t csum_ld = 1;
    uint8_t* flags = nullptr;
    uint32_t* err_count = nullptr;
};
struct GemmGroup {
    int n = 0, bn = 64, epi = kEpiTmaStore, ew = 4, pairs = 1;
    bool checked = true;
    std::vector<int> order;        // problem launched at group slot s
    GemmParams launch{};           // launch-wide fields: tile table and device pointers
    GemmParams* d_params = nullptr;
    CUtensorMap* d_maps = nullptr;
    unsigned long long* row_acc = nullptr;
    unsigned long long* err_pack = nullptr;
};
GemmGroup* gemm_group_create(const GemmProblem* probs, int n, bool checked);
void gemm_group_run(const GemmGroup& g, cudaStream_t st);
void gemm_group_free(GemmGroup* g);
// Dual-encoded locate / correct of a checked result (locate.cu): the flagged row from the mod-127 row checks plus the
// exact column checks against the column sums of A. status: 0 clean, 1 one cell located (corrected when asked),
// 2 the checksum column itself corrupted (recomputed when asked), 3 not locatable (several rows / columns),
// 4 column mismatch without a flagged row (an error the mod-127 row check aliases).
struct LocateResult {
    int status = 0;
    int64_t row = -1, col = -1, delta = 0;
    int64_t rows_flagged = 0, cols_mismatched = 0;
};
LocateResult gemm_locate(const uint8_t* d_a, int64_t m, int64_t lda, const GemmWeight& w, int32_t* d_c, int64_t ldc,
                         int32_t* d_csum, int64_t csum_ld, uint8_t* d_flags, bool correct, cudaStream_t st);
void requantize(const int32_t* d_c, int64_t ldc, int64_t m, int64_t n, const int32_t* d_row_sum_a,
                const int32_t* d_col_sum_b, const RequantDev& q, uint8_t* d_out, int64_t ld_out, cudaStream_t st);
void row_sums_u8(const uint8_t* d_a, int64_t m, int64_t k, int64_t lda, int32_t* d_out, cudaStream_t st);
void weight_col_sums(const GemmWeight& w, int32_t* d_out, cudaStream_t st);
void verify(const int32_t* d_c, int64_t ldc, const int32_t* d_csum, int64_t csum_ld, int64_t m, int64_t n,
            uint8_t* d_flags, uint32_t* d_err_count, cudaStream_t st);

// ---- EmbeddingBag (replaces P:src/embedding_abft.hpp:38-47)
EbTable* eb_table_create(int elem, const void* d_rows, int64_t rows, int64_t dim, int64_t row_stride, int scale_type,
                         const void* d_scales, const void* d_biases, const int32_t* d_given_sums, cudaStream_t st);
void eb_table_free(EbTable* t);
// Re-point an existing table at new rows/scales (reuses the metadata buffer when large enough).
void eb_table_rebuild(EbTable& t, int elem, const void* d_rows, int64_t rows, int64_t dim, int64_t row_stride,
                      int scale_type, const void* d_scales, const void* d_biases, const int32_t* d_given_sums,
                      cudaStream_t st);
void eb_row_sums(const EbTable& t, int32_t* d_out, cudaStream_t st);
// (Re)build the table's interleaved row+metadata copy from the caller's rows and the stored metadata
// (keeps the stored row sums: used after writing faults straight into the rows).
void eb_pack(EbTable& t, cudaStream_t st);
// Fault lab: flip table bits in the caller's rows and in the table's interleaved copy (if any).
void eb_flip_bit(EbTable& t, int64_t row, int64_t col, uint32_t bit, cudaStream_t st);
void eb_flip_bits(EbTable& t, const int64_t* d_rows, const int64_t* d_cols, const int32_t* d_bits, int64_t n,
                  int32_t* d_status, cudaStream_t st);
// Number of rows whose stored sum differs from the recomputed one (synchronizes `st`).
uint64_t eb_table_validate(const EbTable& t, const int32_t* d_given_sums, cudaStream_t st);
// Destination table of the scatter mode (see EbParams): device arrays of per-destination pointers.
struct EbScatter {
    float* const* out_dest = nullptr;
    uint8_t* const* flag_dest = nullptr;
    int64_t bags_per_dest = 0;
    int64_t flag_ld = 1;
};
void eb_run(const EbTable& t, const int64_t* d_offsets, const int64_t* d_indices, int64_t num_bags,
            const float* d_weights, float* d_out, int64_t ld_out, bool checked, uint8_t* d_flags, double* d_rsum,
            double* d_csum, uint32_t* d_flag_count, int32_t* d_status, cudaStream_t st,
            const EbScatter* scatter = nullptr);
int64_t eb_elem_row_bytes(int elem, int64_t dim);
// Grouped lookups: several tables of one element type, scale type and dim, each with its own bags (the same
// count per table), scatter destinations and optional weights, in ONE persistent launch (D5: a GPU's tables).
struct EbGroup {
    std::vector<const EbTable*> tables;
    std::vector<EbTableDesc> host;  // per-table descriptors (host copy)
    EbTableDesc* d_desc = nullptr;  // device copy of the per-table descriptors
    bool weighted = false;
    // fused: ONE persistent launch over all tables (every table's rows and metadata 16-byte aligned with equal
    // strides, dim % 32 == 0 -- the cp.async kernel's contract). Otherwise the group runs as one scatter launch
    // per table (any layout the single-table path takes) and d_counts gathers their flag counts.
    bool fused = true;
    uint32_t* d_counts = nullptr;
};
EbGroup* eb_group_create(const EbTable* const* tables, int64_t ntables, const int64_t* const* d_offsets,
                         const int64_t* const* d_indices, const float* const* d_weights, float* const* const* d_out_dest,
                         uint8_t* const* const* d_flag_dest);
void eb_group_free(EbGroup* g);
// Re-point the group's tables at new bags (CSR offsets / indices / optional weights) without rebuilding it: the
// device descriptors are rewritten with a stream-ordered copy, so later launches on `st` see the new bags.
void eb_group_set_bags(EbGroup& g, const int64_t* const* d_offsets, const int64_t* const* d_indices,
                       const float* const* d_weights, cudaStream_t st);
void eb_group_run(const EbGroup& g, int64_t bags_per_table, int64_t ld_out, int64_t flag_ld, int64_t bags_per_dest,
                  bool checked, uint32_t* d_flag_count, int32_t* d_status, cudaStream_t st);

// ---- fault lab
void flip_bit(void* d_base, uint64_t byte_offset, uint32_t bit, cudaStream_t st);
void set_random(void* d_cell, int width, uint64_t rng_state, cudaStream_t st);
void gen(void* d_out, int64_t count, uint64_t seed, uint64_t stream, uint64_t off, int kind, double lo, double hi,
         uint64_t bound, cudaStream_t st);
void l2_flush(void* d_buf, int64_t bytes, int salt, cudaStream_t st);

// ---- launchers implemented in the .cu files
cudaError_t launch_gemm_kernel(int bn, bool checked, int epi, int ew, int pairs, const CUtensorMap& a, const CUtensorMap& b,
                               const CUtensorMap& c, const GemmParams& p, cudaStream_t st);
cudaError_t launch_gemm_grouped(int bn, bool checked, int epi, int ew, int pairs, const GemmParams& p, cudaStream_t st);
cudaError_t launch_locate_colsum_a(const uint8_t* a, int64_t m, int64_t k, int64_t lda, uint32_t* out, int64_t k_pad,
                                   cudaStream_t st);
cudaError_t launch_locate_columns(const uint32_t* colsum_a, const GemmWeight& w, const int32_t* c, int64_t m, int64_t ldc,
                                  uint32_t* nbad, int64_t* bad_col, long long* bad_delta, int max_record, cudaStream_t st);
cudaError_t launch_locate_row_checksum(const uint8_t* a_row, int64_t k, const int8_t* cs, int32_t* out, cudaStream_t st);
cudaError_t launch_read_encoded(const GemmWeight& w, int8_t* out, cudaStream_t st);
cudaError_t launch_encode_weight(const int8_t* b, int64_t k, int64_t n, int64_t ldb, GemmWeight& w, cudaStream_t st);
cudaError_t launch_verify(const int32_t* c, int64_t ldc, const int32_t* csum, int64_t csum_ld, int64_t m, int64_t n,
                          uint8_t* flags, uint32_t* err_count, uint32_t* ws_acc, uint32_t* ws_blocks, cudaStream_t st);
cudaError_t launch_eb_bags(int elem, int scale, const EbParams& p, bool checked, cudaStream_t st);
constexpr int64_t kGemvMaxRows = 16;  // m <= this: the small-m (GEMV class) path
cudaError_t launch_gemv(const GemmParams& p, const GemmWeight& w, bool checked, cudaStream_t st);
cudaError_t launch_requantize(const int32_t* c, int64_t ldc, int64_t m, int64_t n, const int32_t* rs, const int32_t* cs,
                              const RequantDev& q, uint8_t* out, int64_t ld_out, cudaStream_t st);
cudaError_t launch_row_sums_u8(const uint8_t* a, int64_t m, int64_t k, int64_t lda, int32_t* out, cudaStream_t st);
cudaError_t launch_col_sums(const GemmWeight& w, int32_t* out, cudaStream_t st);
cudaError_t launch_eb_pack(const uint8_t* data, int64_t rows, int64_t row_bytes, int64_t row_stride, const void* meta,
                           int64_t meta_bytes, int64_t meta_off, int64_t rec_stride, uint8_t* packed, cudaStream_t st);
cudaError_t launch_flip_cells(uint8_t* a, int64_t sa, uint8_t* b, int64_t sb, const int64_t* rows, const int64_t* cols,
                              const int32_t* bits, int64_t n, int64_t nrows, int64_t dim, bool u4, int32_t* status,
                              cudaStream_t st);
cudaError_t launch_eb_meta(int elem, int scale, const uint8_t* data, int64_t rows, int64_t dim, int64_t row_stride,
                           const void* scales, const void* biases, const int32_t* given_sums, void* meta,
                           int32_t* sums_out, uint32_t* mismatch, cudaStream_t st);
cudaError_t launch_gen(void* out, int64_t count, uint64_t seed, uint64_t stream, uint64_t off, int kind, double lo,
                       double hi, uint64_t bound, cudaStream_t st);
cudaError_t launch_flip_bit(void* base, uint64_t byte_offset, uint32_t bit, cudaStream_t st);
cudaError_t launch_set_random(void* cell, int width, uint64_t state, cudaStream_t st);
cudaError_t launch_nonzero(const uint32_t* value, uint8_t* out, int64_t slot, cudaStream_t st);
cudaError_t launch_any_flag(const uint8_t* flags, int64_t n, uint8_t* out, int64_t slot, cudaStream_t st);
cudaError_t launch_flush(void* buf, int64_t bytes, int salt, cudaStream_t st);
cudaError_t launch_sum_u32(const uint32_t* src, int64_t n, uint32_t* dst, cudaStream_t st);
cudaError_t launch_gather_probe(const void* table, int64_t rec_bytes, const int64_t* idx, int64_t n, uint32_t* sink,
                                cudaStream_t st);

// Host SplitMix64, identical to P:src/rng.hpp:10-43 (drives fault placement on the host).
struct SplitMix64 {
    uint64_t state;
    static uint64_t mix(uint64_t z) {
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    SplitMix64(uint64_t seed, uint64_t stream) : state(mix(seed ^ mix(stream + 0x9e3779b97f4a7c15ULL))) {}
    uint64_t next() {
        state += 0x9e3779b97f4a7c15ULL;
        return mix(state);
    }
    uint64_t next_below(uint64_t bound) { return next() % bound; }
    // Value of draw `e` (0-based) of this stream without advancing (counter-based).
    static uint64_t draw_at(uint64_t seed, uint64_t stream, uint64_t e) {
        SplitMix64 r(seed, stream);
        return mix(r.state + (e + 1) * 0x9e3779b97f4a7c15ULL);
    }
};

int device_sm_count();
void set_gemm_trace(unsigned long long* d_trace);  // debug instrumentation (nullptr = off)
void set_eb_trace(unsigned long long* d_trace);

}  // namespace abftk
