/*
 * abftlp_b200.h -- device-pointer operator entry points of the B200 ABFT library.
 *
 * These are the hot-path operators the reference keeps as C++ functions
 * (P:src/gemm_abft.hpp:23-74, P:src/embedding_abft.hpp:38-52, P:src/fault_lab.hpp:98-106),
 * exposed in the same C conventions as abftlp.h: plain pointers and sizes, status codes,
 * thread-local abftlp_last_error(), explicit _free for every handle.
 *
 * All d_* pointers are device pointers; `stream` is a cudaStream_t (NULL = legacy default
 * stream). Calls are asynchronous on `stream` unless documented otherwise. Encoded weights
 * and tables are immutable after creation and may be shared by concurrent calls on different
 * streams; per-call scratch lives in a per-stream workspace inside the library.
 */
#ifndef ABFTLP_B200_H
#define ABFTLP_B200_H

#include "abftlp.h"

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

typedef void* abftlp_stream;

/* ------------------------------------------------------------------ int8 ABFT GEMM */
typedef struct abftlp_gemm_weight_s abftlp_gemm_weight;

/* Encode B (s8, k x n, row-major, leading dimension ldb >= n) once: mod-127 row checksums
 * cs[k] (each in [0,126]) plus B' in the GEMM's K-major TMA layout.
 * Replaces compute_row_checksums (P:src/gemm_abft.cpp:60-71) + PackedEncodedWeight
 * (P:src/gemm_abft.cpp:73-85). Empty B -> ABFTLP_ERR_INVALID_ARGUMENT. */
abftlp_status abftlp_gemm_encode(const int8_t* d_b, uint64_t k, uint64_t n, uint64_t ldb,
                                 abftlp_stream stream, abftlp_gemm_weight** out);
void abftlp_gemm_weight_free(abftlp_gemm_weight* w);
/* Re-encode a single-weight handle in place from a new B of the same k x n (e.g. after a weight update):
 * no allocation, asynchronous on `stream`; calls in flight on other streams must be ordered by the caller. */
abftlp_status abftlp_gemm_reencode(abftlp_gemm_weight* w, const int8_t* d_b, uint64_t ldb, abftlp_stream stream);
/* PackedEncodedWeight::k()/n() (P:src/gemm_abft.hpp:37-38). */
abftlp_status abftlp_gemm_weight_dims(const abftlp_gemm_weight* w, uint64_t* k, uint64_t* n);
/* Copies WeightChecksum::values (k int8) to d_cs. */
abftlp_status abftlp_gemm_weight_checksums(const abftlp_gemm_weight* w, int8_t* d_cs, abftlp_stream stream);
/* Replaces the stored checksum column with d_cs (k int8): PackedEncodedWeight(b, cs) with a
 * caller-supplied WeightChecksum (P:src/gemm_abft.cpp:73-85) -- e.g. checksums of the pristine
 * B packed next to a B corrupted after encoding (P:src/fault_lab.cpp:186-189). */
abftlp_status abftlp_gemm_weight_set_checksums(abftlp_gemm_weight* w, const int8_t* d_cs,
                                               abftlp_stream stream);
/* Reads the logical k x (n+1) encoded matrix [B | cs] to d_out (row-major, ld = n+1):
 * the PackedEncodedWeight::at(i, j) contract (P:src/gemm_abft.cpp:87-91). */
abftlp_status abftlp_gemm_weight_read(const abftlp_gemm_weight* w, int8_t* d_out, abftlp_stream stream);

/* In-epilogue fault hook: flip `bit` (0..31) of C'(row, col), col <= n (col == n hits the
 * checksum column), after the product and before verification -- the reference's
 * inject_intermediate_C point (P:src/fault_lab.cpp:192-195). */
typedef struct {
    int32_t active;
    uint64_t row;
    uint64_t col;
    uint32_t bit;
} abftlp_fault;

/* Checked GEMM: C = A x B (int32, m x n, ld ldc), csum[i] = C'[i][n] = sum_p A[i][p]*cs[p]
 * (stride csum_ld), row_flags[i] = mod127(sum_j C[i][j]) != mod127(csum[i]),
 * *d_err_count = number of flagged rows. A is u8 m x k (ld lda >= k).
 * Replaces abft_gemm + verify_checksums (P:src/gemm_abft.cpp:93-100, 113-124). The result is
 * returned even when rows are flagged. Pass d_c = C' and d_csum = C' + n, ldc = csum_ld = n+1
 * to obtain the reference's m x (n+1) cTemp layout directly. */
abftlp_status abftlp_gemm_checked(const uint8_t* d_a, uint64_t m, uint64_t lda,
                                  const abftlp_gemm_weight* w, int32_t* d_c, uint64_t ldc,
                                  int32_t* d_csum, uint64_t csum_ld, uint8_t* d_row_flags,
                                  uint32_t* d_err_count, const abftlp_fault* fault,
                                  abftlp_stream stream);
/* Same kernel with checking compiled out (no checksum MMA, no residue epilogue): the
 * apples-to-apples baseline. Replaces plain_gemm (P:src/gemm_abft.cpp:102-111). */
abftlp_status abftlp_gemm_unchecked(const uint8_t* d_a, uint64_t m, uint64_t lda,
                                    const abftlp_gemm_weight* w, int32_t* d_c, uint64_t ldc,
                                    abftlp_stream stream);
/* Standalone row check over an existing C and checksum column (faults injected after the
 * product). Replaces verify_checksums (P:src/gemm_abft.cpp:113-124). */
abftlp_status abftlp_gemm_verify(const int32_t* d_c, uint64_t ldc, const int32_t* d_csum,
                                 uint64_t csum_ld, uint64_t m, uint64_t n, uint8_t* d_row_flags,
                                 uint32_t* d_err_count, abftlp_stream stream);
/* Host-buffer convenience (the "e2e" path): copies A in, runs the checked GEMM, copies
 * C, csum, flags and the count out; synchronous. Any output pointer may be NULL. */
abftlp_status abftlp_gemm_checked_host(const uint8_t* a, uint64_t m, uint64_t lda,
                                       const abftlp_gemm_weight* w, int32_t* c, uint64_t ldc,
                                       int32_t* csum, uint8_t* row_flags, uint32_t* err_count,
                                       abftlp_stream stream);

/* Host-buffer job (the "e2e" path of a grouped job): `batch` checked GEMMs against one encoded weight, A_b at
 * a + b*stride_a (bytes, row pitch lda), C_b at c + b*stride_c (int32 elements, row pitch ldc), csum_b at
 * csum + b*stride_csum (m int32), flags_b at row_flags + b*stride_flags, err_count[b]. Internally pipelined:
 * chunks of runs are copied in on one stream, multiplied as grouped launches on `stream` and copied out on a
 * third, so host->device, compute and device->host overlap (pinned host buffers make the copies
 * asynchronous). Synchronous on return. Results are identical to abftlp_gemm_checked per run. */
abftlp_status abftlp_gemm_checked_host_batched(const uint8_t* a, uint64_t batch, uint64_t m, uint64_t lda,
                                               uint64_t stride_a, const abftlp_gemm_weight* w, int32_t* c,
                                               uint64_t ldc, uint64_t stride_c, int32_t* csum,
                                               uint64_t stride_csum, uint8_t* row_flags, uint64_t stride_flags,
                                               uint32_t* err_count, abftlp_stream stream);

/* ------------------------------------------------------------------ batched GEMM (many small problems) */
/* Encode `batch` independent weights of one shape: weight b is B_b = d_b + b*stride_b (k x n, ld ldb).
 * The batched handle serves abftlp_gemm_*_batched; per-weight accessors (checksums, read, flip, col sums)
 * need a single weight and return ABFTLP_ERR_INVALID_ARGUMENT on it. */
abftlp_status abftlp_gemm_encode_batched(const int8_t* d_b, uint64_t batch, uint64_t k, uint64_t n,
                                         uint64_t ldb, uint64_t stride_b, abftlp_stream stream,
                                         abftlp_gemm_weight** out);
typedef struct {
    int32_t active;
    uint64_t batch; /* problem index */
    uint64_t row;
    uint64_t col;   /* col == n: the checksum column */
    uint32_t bit;
} abftlp_batch_fault;
/* Corrupt B'(i, j) of problem `problem` of a batched weight after encoding (j == n hits its checksum column):
 * inject_weight_B (P:src/fault_lab.cpp:98-120) for one problem of a batched handle. */
abftlp_status abftlp_gemm_weight_flip_bit_batched(abftlp_gemm_weight* w, uint64_t problem, uint64_t i, uint64_t j,
                                                  uint32_t bit, abftlp_stream stream);
/* `batch` checked GEMMs of one shape in ONE launch (e.g. the reference's 100 seeded trials of config 0):
 * problem b multiplies A_b = d_a + b*stride_a (bytes; 16-byte multiple) by weight b of a batched weight
 * (or the single weight of a plain handle) and writes C_b = d_c + b*stride_c, csum at d_csum +
 * b*stride_csum (int32 elements), flags at d_row_flags + b*stride_flags and d_err_count[b]. Each problem's
 * result is bit-identical to abftlp_gemm_checked on it. */
abftlp_status abftlp_gemm_checked_batched(const uint8_t* d_a, uint64_t batch, uint64_t m, uint64_t lda,
                                          uint64_t stride_a, const abftlp_gemm_weight* w, int32_t* d_c,
                                          uint64_t ldc, uint64_t stride_c, int32_t* d_csum, uint64_t csum_ld,
                                          uint64_t stride_csum, uint8_t* d_row_flags, uint64_t stride_flags,
                                          uint32_t* d_err_count, const abftlp_batch_fault* fault,
                                          abftlp_stream stream);
/* Same, with a list of C' faults (entries with active == 0 are skipped; at most 8 active per call): the
 * form a grouped job uses when several of its runs carry an injected fault. */
abftlp_status abftlp_gemm_checked_batched_faults(const uint8_t* d_a, uint64_t batch, uint64_t m, uint64_t lda,
                                                 uint64_t stride_a, const abftlp_gemm_weight* w, int32_t* d_c,
                                                 uint64_t ldc, uint64_t stride_c, int32_t* d_csum, uint64_t csum_ld,
                                                 uint64_t stride_csum, uint8_t* d_row_flags, uint64_t stride_flags,
                                                 uint32_t* d_err_count, const abftlp_batch_fault* faults,
                                                 uint64_t nfaults, abftlp_stream stream);
abftlp_status abftlp_gemm_unchecked_batched(const uint8_t* d_a, uint64_t batch, uint64_t m, uint64_t lda,
                                            uint64_t stride_a, const abftlp_gemm_weight* w, int32_t* d_c,
                                            uint64_t ldc, uint64_t stride_c, abftlp_stream stream);

/* ------------------------------------------------------------------ requantization */
/* RequantParams (P:src/quant.hpp:24-32): out = clamp(round_half_away((cf - biasC) / scaleC), 0, 255) with
 * cf = scaleA*scaleB*C + scaleA*biasB*rowSumA[i] + scaleB*biasA*colSumB[j] + k*biasA*biasB, all in
 * double in the reference's order (P:src/quant.cpp:77-102); bit-identical results. */
typedef struct {
    double scaleA, biasA, scaleB, biasB, scaleC, biasC;
    uint64_t k;
} abftlp_requant_params;

/* Checked GEMM with the requantization fused into the epilogue: u8 d_out (m x n, ld_out) =
 * requantize(C') with the checksum column excluded, computed from the tile in TMEM after any injected C'
 * fault, plus the usual verdicts. d_c may be NULL (no int32 C' written; csum/flags still produced).
 * scaleC <= 0 -> ABFTLP_ERR_INVALID_ARGUMENT ("requantize: scaleC must be positive"). */
abftlp_status abftlp_gemm_checked_requant(const uint8_t* d_a, uint64_t m, uint64_t lda,
                                          const abftlp_gemm_weight* w, int32_t* d_c, uint64_t ldc,
                                          int32_t* d_csum, uint64_t csum_ld, uint8_t* d_row_flags,
                                          uint32_t* d_err_count, const abftlp_fault* fault,
                                          const int32_t* d_row_sum_a, const int32_t* d_col_sum_b,
                                          const abftlp_requant_params* params, uint8_t* d_out,
                                          uint64_t ld_out, abftlp_stream stream);
/* Standalone requantize over an existing C' (first n columns of each row; a checksum column is never
 * read). Replaces requantize (P:src/quant.cpp:77-102). */
abftlp_status abftlp_requantize(const int32_t* d_c, uint64_t ldc, uint64_t m, uint64_t n,
                                const int32_t* d_row_sum_a, const int32_t* d_col_sum_b,
                                const abftlp_requant_params* params, uint8_t* d_out, uint64_t ld_out,
                                abftlp_stream stream);
/* row_sums(A) for u8 A (P:src/quant.cpp:104-110) and col_sums(B) of an encoded weight (P:src/quant.cpp:112-118). */
abftlp_status abftlp_row_sums_u8(const uint8_t* d_a, uint64_t m, uint64_t k, uint64_t lda, int32_t* d_out,
                                 abftlp_stream stream);
abftlp_status abftlp_gemm_weight_col_sums(const abftlp_gemm_weight* w, int32_t* d_out, abftlp_stream stream);
/* Host-buffer job with the requantization fused (the DLRM layer as the pipeline uses it: u8 in, u8 out; replaces
 * abft_gemm + requantize, P:src/gemm_abft.cpp:93-100 + P:src/quant.cpp:77-102, per run): `batch` checked GEMMs against
 * one encoded weight, A_b at a + b*stride_a (bytes, row pitch lda); out_b = requantize(C'_b) at out + b*stride_out
 * (bytes, row pitch ld_out), csum_b = C'_b[:, n], flags_b and err_count[b] as abftlp_gemm_checked_host_batched. The
 * int32 product never leaves the GPU (it is not even written to HBM): row_sums(A_b) and col_sums(B) are computed on
 * the device, each chunk of runs is one row-stacked launch. Pipelined like abftlp_gemm_checked_host_batched;
 * synchronous on return; bit-identical to abftlp_gemm_checked_requant per run. */
abftlp_status abftlp_gemm_checked_requant_host_batched(const uint8_t* a, uint64_t batch, uint64_t m, uint64_t lda,
                                                       uint64_t stride_a, const abftlp_gemm_weight* w,
                                                       const abftlp_requant_params* params, uint8_t* out,
                                                       uint64_t ld_out, uint64_t stride_out, int32_t* csum,
                                                       uint64_t stride_csum, uint8_t* row_flags,
                                                       uint64_t stride_flags, uint32_t* err_count,
                                                       abftlp_stream stream);

/* ------------------------------------------------------------------ EmbeddingBag */
typedef struct abftlp_eb_table_s abftlp_eb_table;

#define ABFTLP_EB_S8 0  /* int8 rows (the reference's QuantEmbeddingTable) */
#define ABFTLP_EB_U8 1  /* uint8 rows */
#define ABFTLP_EB_U4 2  /* packed 4-bit rows: element j = (byte[j/2] >> 4*(j&1)) & 0xF */
#define ABFTLP_EB_SCALE_F32 0
#define ABFTLP_EB_SCALE_F16 1

/* Build a checked table over device rows (borrowed: the caller keeps them alive and
 * immutable) plus per-row scale/bias (f32 or f16). Row sums (int32) are computed on the
 * device -- precompute_row_sums (P:src/embedding_abft.cpp:39-45) -- unless d_row_sums is
 * given, in which case those are stored as-is (load_table(validate=false) semantics). */
abftlp_status abftlp_eb_table_create(int32_t elem_type, const void* d_rows, uint64_t rows,
                                     uint64_t dim, uint64_t row_stride_bytes, int32_t scale_type,
                                     const void* d_scales, const void* d_biases,
                                     const int32_t* d_row_sums, abftlp_stream stream,
                                     abftlp_eb_table** out);
void abftlp_eb_table_free(abftlp_eb_table* t);
/* Synchronous: number of rows whose d_row_sums entry differs from the recomputed sum
 * (load_table validation, P:src/embedding_abft.cpp:139-143). */
abftlp_status abftlp_eb_table_validate(const abftlp_eb_table* t, const int32_t* d_row_sums,
                                       abftlp_stream stream, uint64_t* mismatched_rows);
/* Device row sums of the table (int32[rows]). */
abftlp_status abftlp_eb_table_row_sums(const abftlp_eb_table* t, int32_t* d_out, abftlp_stream stream);

/* Checked pooled lookups over CSR bags: bag b = indices[offsets[b] .. offsets[b+1]),
 * optional per-lookup weights (NULL = unweighted). out[b][0..dim) (ld_out), flags[b],
 * rsum[b], csum[b] (nullable), *d_flag_count (nullable) = flagged bags. Indices >= rows set
 * bit 0 of *d_status (nullable) -- the reference's out_of_range (P:src/embedding_abft.cpp:16-22).
 * Replaces abft_embedding_bag / batch_abft_eb (P:src/embedding_abft.cpp:62-91). */
abftlp_status abftlp_eb_checked(const abftlp_eb_table* t, const int64_t* d_offsets,
                                const int64_t* d_indices, uint64_t num_bags,
                                const float* d_weights, float* d_out, uint64_t ld_out,
                                uint8_t* d_flags, double* d_rsum, double* d_csum,
                                uint32_t* d_flag_count, int32_t* d_status, abftlp_stream stream);
/* Same lookups without the check. Replaces embedding_bag (P:src/embedding_abft.cpp:47-60). */
abftlp_status abftlp_eb_unchecked(const abftlp_eb_table* t, const int64_t* d_offsets,
                                  const int64_t* d_indices, uint64_t num_bags,
                                  const float* d_weights, float* d_out, uint64_t ld_out,
                                  int32_t* d_status, abftlp_stream stream);

/* Checked pooled lookups that write straight into per-destination buffers: the table-wise sharded
 * DLRM exchange fused into the lookup kernel. Bag b's pooled vector goes to
 * d_out_dest[b / bags_per_dest] + (b % bags_per_dest) * ld_out and its flag to
 * d_flag_dest[b / bags_per_dest][(b % bags_per_dest) * flag_ld]. d_out_dest / d_flag_dest are DEVICE
 * arrays of pointers, which may point into peer GPUs' memory mapped over NVLink (CUDA IPC / symmetric
 * memory), so the all-to-all of pooled outputs overlaps the lookups instead of following them. Same
 * arithmetic and verdicts as abftlp_eb_checked. */
abftlp_status abftlp_eb_checked_scatter(const abftlp_eb_table* t, const int64_t* d_offsets,
                                        const int64_t* d_indices, uint64_t num_bags,
                                        const float* d_weights, float* const* d_out_dest,
                                        uint64_t ld_out, uint8_t* const* d_flag_dest, uint64_t flag_ld,
                                        uint64_t bags_per_dest, uint32_t* d_flag_count,
                                        int32_t* d_status, abftlp_stream stream);

/* Grouped checked lookups over several tables (one element type, scale type and dim; e.g. one GPU's tables of
 * the D5 DLRM step) in ONE persistent launch: table i has its own CSR bags (d_offsets[i], d_indices[i],
 * optional d_weights[i]), the same bag count per table, and scatter destinations d_out_dest[i] / d_flag_dest[i]
 * (device arrays of pointers, as in abftlp_eb_checked_scatter). The host arrays passed to _create are read
 * once; the group keeps a device copy. Results are identical to one abftlp_eb_checked_scatter per table. */
typedef struct abftlp_eb_group_s abftlp_eb_group;
abftlp_status abftlp_eb_group_create(const abftlp_eb_table* const* tables, uint32_t ntables,
                                     const int64_t* const* d_offsets, const int64_t* const* d_indices,
                                     const float* const* d_weights /* nullable */,
                                     float* const* const* d_out_dest, uint8_t* const* const* d_flag_dest,
                                     abftlp_eb_group** out);
void abftlp_eb_group_free(abftlp_eb_group* g);
abftlp_status abftlp_eb_group_checked_scatter(const abftlp_eb_group* g, uint64_t bags_per_table, uint64_t ld_out,
                                              uint64_t flag_ld, uint64_t bags_per_dest, uint32_t* d_flag_count,
                                              int32_t* d_status, abftlp_stream stream);
/* The same lookups without the check (embedding_bag, P:src/embedding_abft.cpp:47-60): the ABFT-overhead baseline. */
abftlp_status abftlp_eb_group_unchecked_scatter(const abftlp_eb_group* g, uint64_t bags_per_table, uint64_t ld_out,
                                                uint64_t bags_per_dest, int32_t* d_status, abftlp_stream stream);
/* Re-point a group at new bags (per table: device CSR offsets, indices, optional weights) without rebuilding it;
 * stream-ordered, so later launches on `stream` pool the new bags (a training step's fresh indices). */
abftlp_status abftlp_eb_group_set_bags(abftlp_eb_group* g, const int64_t* const* d_offsets,
                                       const int64_t* const* d_indices, const float* const* d_weights /* nullable */,
                                       abftlp_stream stream);

/* ------------------------------------------------------------------ dual-encoded locate / correct
 * After a checked GEMM flagged rows: the exact column checks of the dual encoding (column sums of A times B against
 * the column sums of C', P:tests/dual_check.hpp:23-73) find the corrupted column; with the single flagged row that is
 * the corrupted cell, and `correct` restores it (C -= delta) and re-runs the row check. status: 0 clean; 1 one cell
 * located (row, col, delta = corrupted - clean); 2 the checksum column C'[row][n] was hit (recomputed when
 * correcting); 3 not locatable (several errors); 4 a column mismatch with no flagged row (an error the mod-127 row
 * check aliases). Synchronizes `stream`. Correction is beyond the reference (it stops at detection). */
typedef struct {
    int32_t status;
    int64_t row, col, delta;
    uint64_t rows_flagged, cols_mismatched;
} abftlp_locate_result;
abftlp_status abftlp_gemm_locate(const uint8_t* d_a, uint64_t m, uint64_t lda, const abftlp_gemm_weight* w, int32_t* d_c,
                                 uint64_t ldc, int32_t* d_csum, uint64_t csum_ld, uint8_t* d_row_flags, int correct,
                                 abftlp_locate_result* out, abftlp_stream stream);

/* ------------------------------------------------------------------ heterogeneous grouped GEMM
 * Several checked (or plain) GEMMs of DIFFERENT shapes -- each its own A (u8, 16-byte aligned, lda % 16 == 0),
 * encoded weight, C', checksum column, row flags and count -- in ONE persistent launch (abft_gemm per problem,
 * P:src/gemm_abft.cpp:93-124; e.g. the layers of a DLRM MLP, BASELINE configs[4]). _create validates the problems,
 * picks one tile width for all of them and uploads their parameters and tensor maps once; _run launches (stream-
 * ordered, CUDA-graph capturable). Results are identical to one abftlp_gemm_checked / _unchecked call per problem.
 * A group is run on one stream at a time (its per-row verdict scratch is its own). At most 16 problems. */
typedef struct {
    const uint8_t* d_a;
    uint64_t m, lda;
    const abftlp_gemm_weight* w;
    int32_t* d_c;
    uint64_t ldc;
    int32_t* d_csum;      /* checked only: C'[:, n] (stride csum_ld) */
    uint64_t csum_ld;
    uint8_t* d_row_flags; /* checked only */
    uint32_t* d_err_count;/* checked only */
} abftlp_gemm_problem;
typedef struct abftlp_gemm_group_s abftlp_gemm_group;
abftlp_status abftlp_gemm_group_create(const abftlp_gemm_problem* problems, uint32_t count, int checked,
                                       abftlp_gemm_group** out);
abftlp_status abftlp_gemm_group_run(const abftlp_gemm_group* g, abftlp_stream stream);
void abftlp_gemm_group_free(abftlp_gemm_group* g);

/* ------------------------------------------------------------------ fault injection */
/* XOR bit `bit` of element `index` of an array of `elem_bytes`-wide integers
 * (flip_bit, P:src/fault_lab.hpp:87-93). */
abftlp_status abftlp_flip_bit(void* d_ptr, uint32_t elem_bytes, uint64_t index, uint32_t bit,
                              abftlp_stream stream);
/* Flip bit of encoded weight element B'(i, j), j < n (inject_weight_B after encoding,
 * P:src/fault_lab.cpp:98-115); j == n hits the checksum column. */
abftlp_status abftlp_gemm_weight_flip_bit(abftlp_gemm_weight* w, uint64_t i, uint64_t j,
                                          uint32_t bit, abftlp_stream stream);
/* Flip bit (< element width) of table element (row, col) after row sums were computed
 * (inject_eb_table, P:src/fault_lab.cpp:139-166). Mutates the caller's row buffer and the table's
 * device-resident interleaved copy (the lookups read the latter). Rows changed by other means after
 * abftlp_eb_table_create are not seen by the lookups: inject through these calls. */
abftlp_status abftlp_eb_table_flip_bit(abftlp_eb_table* t, uint64_t row, uint64_t col,
                                       uint32_t bit, abftlp_stream stream);
/* Batched table faults: flip bit d_bits[i] (< element width) of element (d_rows[i], d_cols[i]) for
 * i < count (device arrays); repeated coordinates compose like sequential flips. Out-of-range entries
 * are skipped and set bit 1 of *d_status (nullable). Same target as abftlp_eb_table_flip_bit. */
abftlp_status abftlp_eb_table_flip_bits(abftlp_eb_table* t, const int64_t* d_rows, const int64_t* d_cols,
                                        const int32_t* d_bits, uint64_t count, int32_t* d_status,
                                        abftlp_stream stream);
/* Seeded generators reproducing SplitMix64(seed, stream) draws off .. off+count-1
 * (P:src/rng.hpp:10-43): kind 0 = u8 next_below(256), 1 = s8 next_int(-128,127),
 * 2 = f32 (float)next_real(lo, hi), 3 = i64 next_below(bound). */
abftlp_status abftlp_generate(void* d_out, uint64_t count, uint64_t seed, uint64_t rng_stream,
                              uint64_t off, int32_t kind, double lo, double hi, uint64_t bound,
                              abftlp_stream stream);
/* Reads a buffer larger than L2 (benchmark cache flush). */
abftlp_status abftlp_l2_flush(void* d_buf, uint64_t bytes, int32_t salt, abftlp_stream stream);
/* Benchmark roof for the EmbeddingBag lines: reads record d_idx[i] (rec_bytes each, a multiple of 16 up to 512,
 * from d_table) for every i < n with maximal memory-level parallelism and no arithmetic -- the random-gather
 * floor of the same lookups. d_sink: one device uint32 (written practically never). */
abftlp_status abftlp_gather_probe(const void* d_table, uint64_t rec_bytes, const int64_t* d_idx, uint64_t n,
                                  uint32_t* d_sink, abftlp_stream stream);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif

#endif /* ABFTLP_B200_H */
