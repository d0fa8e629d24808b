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

// Kernel attributes (dynamic shared-memory limit) and occupancy are per device; one process may drive several
// GPUs, so launchers remember them per device ordinal.
constexpr int kMaxDevices = 64;
inline int current_device() {
    int d = 0;
    if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
    return d;
}

// ------------------------------------------------------------------ GEMM
constexpr int kBM = 128;      // rows of A per CTA; a CTA pair covers 256 rows (tcgen05 cta_group::2, M=256)
constexpr int kPairM = 256;
constexpr int kBK = 128;      // K bytes per k-block = one 128-byte swizzle span
constexpr int kRowAlign = 256;  // B' rows are padded to a multiple of this

// Encoded weight: B stored transposed, K-block-major, for the mainloop's TMA requests:
//   bt[kb][j][kk] = B[kb*128 + kk][j]   for j < n, cs[kb*128 + kk] for j == n, zero for n < j < n_pad and
//                                       kb*128 + kk >= k.
// One k-block slab of a tile (rows j0..j0+R) is contiguous (R*128 bytes), so each TMA request is
// one long burst. The checksum column of the reference's [B | cs] (P:src/gemm_abft.cpp:73-85) is
// kept as the vector cs (k_pad bytes, zero beyond k): C'[:, n] = A*cs is a GEMV, computed exactly on
// CUDA cores by the epilogue warps (each N tile takes a K share), so it never costs an MMA tile.
struct GemmWeight {
    int64_t k = 0, n = 0;          // logical sizes (PackedEncodedWeight::k()/n())
    int64_t k_pad = 0, n_pad = 0;  // k_pad % 128 == 0, n_pad % 256 == 0, n_pad > n (column n = cs)
    int8_t* bt = nullptr;          // k_pad/128 x n_pad x 128
    int8_t* cs = nullptr;          // k_pad (WeightChecksum::values, each in [0,126]; zero pad)
    int32_t* cs_acc = nullptr;     // k_pad x batch encoder scratch: per-row sums of column-block residues (zeroed)
    bool owns = true;
    size_t bt_cap = 0, cs_cap = 0;  // allocation capacities (campaign scratch re-encodes in place)
    int64_t batch = 1;              // independent weights stored back to back (batched GEMM)
    int64_t bt_bstride = 0, cs_bstride = 0;  // bytes between consecutive weights' bt / cs
    CUtensorMap map_b[3]{};         // 4D {128 B, rows, k-blocks, batch}, box {128, BN/2, KS/NB, 1}, BN = 64, 128, 256
    // device pointer of logical element (i, j) of [B | cs], j <= n
    int8_t* element(int64_t i, int64_t j) const {
        return j == n ? cs + i : bt + ((i / kBK) * n_pad * kBK + j * kBK + (i % kBK));
    }
};

// Per-row accumulator of the checked epilogue: bits 63..32 = sum of the tiles' A*cs shares (the exact
// int32 checksum column, < 2^31 for k < 65793), 31..20 = tiles arrived (n_tiles <= 4095), 19..0 = sum
// of the tiles' row residues (each < 127, so < 2^20).
constexpr int kRowAccCountShift = 20;
constexpr unsigned long long kRowAccCountMask = 0xFFFull;
constexpr unsigned long long kRowAccResMask = (1ull << kRowAccCountShift) - 1;
constexpr int kMaxCheckedNTiles = 4095;

// RequantParams (P:src/quant.hpp:24-32) as the device sees it (k as a double, as the reference casts it).
struct RequantDev {
    double sA, bA, sB, bB, sC, bC, k;
};

constexpr int kMaxGemmFaults = 8;  // C' faults one launch can inject (grouped jobs)
constexpr int kMaxGemmGroup = 16;  // problems of different shapes in one grouped launch

struct GemmParams {
    int m, n, k;       // logical sizes (n excludes the checksum column)
    int k_blocks;      // 128-byte K blocks
    int n_tiles;       // N tiles of tile_w columns
    int tile_w;        // columns per N tile: BN, or (grouped launches) a multiple of 32 below it, the MMA's N
    int m_tiles;       // 256-row pair tiles
    int num_tiles;     // batch * m_tiles * n_tiles
    // batched GEMM (independent problems of one shape, one launch): tile t belongs to problem
    // t / (m_tiles * n_tiles); per-problem strides below (batch == 1: all zero)
    int batch;
    int b_shared;          // 1: every problem uses weight 0
    int64_t a_bstride;     // bytes
    int64_t cs_bstride;    // bytes (checksum vector of problem b)
    int64_t c_bstride;     // int32 elements
    int64_t csum_bstride;  // int32 elements
    int64_t flags_bstride; // bytes
    int a_exact;  // 1: A map is the exact-extent 3D {k, rows, batch} view (one k-block per request)
    // split-K over two units per tile (small-m shapes, one wave): unit u < num_tiles computes k-blocks
    // [kb_half, k_blocks) of tile u and publishes its partial tile; unit num_tiles + t computes
    // [0, kb_half) of tile t, adds the partial and runs the epilogue. split == 1: one unit per tile.
    int split;
    int kb_half;
    // checksum-column GEMV by the pairs the tile grid leaves idle (tall narrow shapes): tile epilogues then
    // contribute no GEMV share, and every row expects row_arrivals = n_tiles + 1 arrivals (n_tiles otherwise)
    int gemv_helpers;
    int row_arrivals;
    // checksum column on the tensor cores: B' column n holds cs, the tile covering column n reads C'[:, n]
    // from its accumulator, no GEMV share (n_tiles counts that tile)
    int cs_mma;
    int32_t* partial;     // [num_tiles][2 CTAs][BN/32][32][128] int32 (split only)
    uint32_t* part_flag;  // [num_tiles * 2], self-resetting
    int32_t* c;
    int64_t ldc;
    const uint8_t* a;  // A (u8, row-major, lda % 16 == 0) for the checksum GEMV
    int64_t lda;
    const int8_t* cs;  // checksum vector (k_pad bytes, zero pad)
    int32_t* csum;     // checksum column C'[:, n] (checked only)
    int64_t csum_ld;
    uint8_t* flags;      // per-row error flags (checked only)
    uint32_t* err_count; // number of flagged rows (checked only)
    // self-resetting per-stream workspace
    unsigned long long* row_acc;  // [m] see kRowAcc*: A*cs share sum | tile arrivals | residue sum
    unsigned long long* err_pack; // [1] (finished rows) << 32 | (flagged rows so far)
    // fused requantization (rq_out != nullptr): u8 C_I = requantize(C') with the checksum column excluded
    const int32_t* rq_row_sum_a;  // [m]
    const int32_t* rq_col_sum_b;  // [n]
    uint8_t* rq_out;
    int64_t rq_ld;
    RequantDev rq;
    // in-epilogue fault hook (P:src/fault_lab.cpp:192-195 semantics): fault f flips bit fault_bit[f] of
    // C'(fault_row[f], fault_col[f]) of problem fault_b[f] (col == n: the checksum column), before the check
    int nfaults;
    int fault_b[kMaxGemmFaults], fault_row[kMaxGemmFaults], fault_col[kMaxGemmFaults], fault_bit[kMaxGemmFaults];
    unsigned long long* trace;  // optional per-CTA phase timestamps (globaltimer ns), 16 per CTA
    // row-stacked requests (requests of one shape against one weight run as the row blocks of one tall GEMM): rows
    // per request; the flag count of request row / req_rows goes to err_count[row / req_rows] (0: one problem per b)
    int req_rows;
    // heterogeneous grouped launch (group_n > 0): problems of different (m, n, k) sharing one tile width; tile t
    // belongs to problem i with grp_tile_start[i] <= t < grp_tile_start[i + 1], whose fields (a single problem,
    // batch 1) are grp_params[i] and whose tensor maps (A, B', C) are grp_maps[3i .. 3i+2] in global memory
    int group_n;
    int grp_tile_start[kMaxGemmGroup + 1];
    const struct GemmParams* grp_params;
    const CUtensorMap* grp_maps;  // [3 * group_n] A, B', C per problem, then (grp_apf) [group_n] A L2-prefetch views
    int grp_apf;
};

// C' write-out: TMA store of 32x32 chunks; coalesced st.global.v4 after a swizzled smem transpose
// (keeps the SM's TMA engine free for the next tile's loads); scalar stores (unaligned C); none (bench).
enum EpiMode { kEpiTmaStore = 0, kEpiStg = 1, kEpiDirect = 2, kEpiNone = 4 };

struct GemmTiling {
    int bn, epi;
    int split = 1;  // 2: split-K over two co-resident units per tile (GemmParams::split)
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
    // owned interleaved copy (row bytes + metadata record in one 64-byte slot) when both fit: the
    // lookups read this instead of (data, meta); nullptr otherwise
    uint8_t* packed = nullptr;
    int64_t rec_stride = 0, meta_off = 0, packed_cap = 0;
};

// One table of a grouped EmbeddingBag launch (EbParams::tables): the per-table fields of EbParams.
struct EbTableDesc {
    const uint8_t* data;
    const void* meta;
    int64_t meta_stride, rows, row_stride;
    const int64_t* offsets;  // [bags_per_table + 1]
    const int64_t* indices;
    const float* weights;    // nullable
    float* const* out_dest;  // scatter destinations of this table (see EbParams)
    uint8_t* const* flag_dest;
};

struct EbParams {
    const uint8_t* data;
    const void* meta;
    int64_t meta_stride;  // bytes between consecutive metadata records
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
    unsigned long long* ws_bag_ctr;  // persistent kernels' next-bag counter (self-resetting)
    unsigned long long* trace;       // debug: per-warp timeline (16 slots), nullptr = off
    float neg_zero;                  // -0.0f, passed at run time (see f2_fma in eb.cu)
    int zero_rt;                     // 0, passed at run time (see the bag ticket in eb_bag_async_kernel)
    // scatter mode (table-wise sharded exchange fused into the lookups): when out_dest is set, bag b
    // writes out_dest[b / bags_per_dest] + (b % bags_per_dest) * ld_out and its flag to
    // flag_dest[b / bags_per_dest][(b % bags_per_dest) * flag_ld] (pointers may be NVLink peer memory)
    float* const* out_dest;
    uint8_t* const* flag_dest;
    int64_t bags_per_dest;
    int64_t flag_ld;
    // grouped tables (one launch over several tables of one element type, scale type and dim): when set,
    // num_bags counts the bags of ALL tables, bag g is bag g % bags_per_table of table g / bags_per_table, and
    // the per-table fields (data, meta, offsets, indices, weights, scatter destinations) come from tables[t]
    const EbTableDesc* tables;
    int64_t bags_per_table;
};

}  // namespace abftk
