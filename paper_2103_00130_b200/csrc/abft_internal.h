// Internal (non-exported) structures shared by the host runtime and the kernels.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <stdexcept>
#include <string>

namespace abftk {

// ------------------------------------------------------------------ errors
// Thrown by the host runtime, mapped to abftlp status codes in capi.cpp with the
// same exception classes as the reference's `guarded` (P:src/capi.cpp:28-41).
struct CudaError : std::exception {
    std::string msg;
    explicit CudaError(std::string m) : msg(std::move(m)) {}
    const char* what() const noexcept override { return msg.c_str(); }
};
void cuda_check(cudaError_t e, const char* what);
#define ABFT_CUDA(call) ::abftk::cuda_check((call), #call)

// ------------------------------------------------------------------ GEMM
constexpr int kBM = 128;  // rows of A per CTA tile (one UMMA M=128 accumulator)
constexpr int kBK = 128;  // K bytes per pipeline stage = one 128-byte swizzle span
constexpr int kCsRows = 16;  // checksum operand: row 0 = cs, rows 1..15 zero (UMMA N=16)

// Encoded weight B' = [B | cs] stored K-major: Bt[j][p] = B[p][j] for j < n,
// zero for n <= j < n_pad and p >= k. The checksum column lives in its own
// 16-row operand `cs_tile` so the MMA of the main tile never sees it.
struct GemmWeight {
    int64_t k = 0, n = 0;          // logical sizes (reference PackedEncodedWeight::k()/n())
    int64_t k_pad = 0, n_pad = 0;  // k_pad % 128 == 0, n_pad % 256 == 0
    int8_t* bt = nullptr;          // n_pad x k_pad
    int8_t* cs_tile = nullptr;     // 16 x k_pad
    int8_t* cs = nullptr;          // k  (WeightChecksum::values, each in [0,126])
    bool owns = true;
    size_t bt_cap = 0, kpad_cap = 0;  // allocation capacities (campaign scratch re-encodes in place)
    CUtensorMap map_b[3]{};        // box {128, BN} for BN = 64, 128, 256
    CUtensorMap map_cs{};          // box {128, 16}
};

struct GemmParams {
    int m, n;          // logical output size (n excludes the checksum column)
    int k_blocks;      // total 128-byte K blocks
    int kb_per_split;  // K blocks handled by one CTA
    int n_tiles, m_tiles, splits;
    int32_t* c;
    int64_t ldc;
    int32_t* csum;  // checksum column C'[:, n] (checked only)
    int64_t csum_ld;
    uint8_t* flags;      // per-row error flags (checked only)
    uint32_t* err_count; // number of flagged rows (checked only)
    // self-resetting per-stream workspace
    uint32_t* row_res;    // [m] sum of per-tile row residues (each < 127)
    int32_t* csum_acc;    // [m] split-K partial checksum column
    uint32_t* mtile_cnt;  // [m_tiles] arrival counters
    uint32_t* err_acc;    // [1]
    uint32_t* done_cnt;   // [1]
    uint32_t* tile_flag;  // [m_tiles * n_tiles] split-K zero-init epochs
    uint32_t epoch;
    // in-epilogue fault hook (P:src/fault_lab.cpp:192-195 semantics): flip `bit` of C'(row, col)
    int fault_active, fault_row, fault_col, fault_bit;
};

enum EpiMode { kEpiTmaStore = 0, kEpiTmaReduce = 1, kEpiDirect = 2 };

struct GemmTiling {
    int bn, splits, epi;
};

// ------------------------------------------------------------------ EmbeddingBag
enum EbElem { kEbS8 = 0, kEbU8 = 1, kEbU4 = 2 };
enum EbScale { kEbF32 = 0, kEbF16 = 1 };

struct EbMetaF32 {  // 16 B per row: one sector per lookup
    float scale;
    float bias;
    int32_t row_sum;
    int32_t pad;
};
struct EbMetaF16 {  // 8 B per row
    uint16_t scale;  // IEEE half bits
    uint16_t bias;
    int32_t row_sum;
};

struct EbTable {
    int elem = kEbS8;
    int scale_type = kEbF32;
    int64_t rows = 0, dim = 0;
    int64_t row_stride = 0;  // bytes between consecutive rows
    const uint8_t* data = nullptr;  // borrowed: caller keeps the rows alive
    void* meta = nullptr;           // owned: EbMetaF32[rows] or EbMetaF16[rows]
};

struct EbParams {
    const uint8_t* data;
    const void* meta;
    int64_t rows, dim, row_stride;
    const int64_t* offsets;  // [num_bags + 1]
    const int64_t* indices;
    const float* weights;    // nullable
    int64_t num_bags;
    float* out;
    int64_t ld_out;
    uint8_t* flags;
    double* rsum;
    double* csum;
    uint32_t* flag_count;  // nullable
    int32_t* status;       // nullable; bit 0 = index out of range
    uint32_t* ws_flag_acc;
    uint32_t* ws_block_cnt;
};

}  // namespace abftk
