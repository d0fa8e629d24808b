/*
 * abft_oracle.c -- TEST INFRASTRUCTURE ONLY (the checker, never the product).
 *
 * Plain-C restatement of the reference's CPU algorithms for the ABFT hot path, used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg to check the CUDA library. Each
 * function cites the reference file:line it restates (P: = /root/reference/proj/).
 *
 * Parity pin: every function here is checked in tests/test_oracle.py against the reference's
 * own known answers (P:tests/*.cpp), against golden vectors produced by the real reference
 * compiled from its sources (oracle/_ref/libabftlp_ref.so, see oracle/Makefile and
 * oracle/make_golden.py -> tests/golden/), and -- when oracle/_ref is present -- against that
 * library directly on random inputs. The uint8 / int4 / fp16 EmbeddingBag variants (BASELINE
 * configs 3-4) have no reference implementation; they share the templated element decode with
 * the int8 path that is pinned bit-for-bit, which is their chain of trust.
 *
 * Build: make -C oracle  (gcc -O2 -ffp-contract=off: no FMA contraction, as the reference
 * build has none on baseline x86-64).
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------ SplitMix64 (P:src/rng.hpp:10-43) */
static uint64_t sm_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
typedef struct {
    uint64_t state;
} Rng;
static Rng rng_make(uint64_t seed, uint64_t stream) {
    Rng r;
    r.state = sm_mix(seed ^ sm_mix(stream + 0x9e3779b97f4a7c15ULL));
    return r;
}
static uint64_t rng_next(Rng* r) {
    r->state += 0x9e3779b97f4a7c15ULL;
    return sm_mix(r->state);
}
static uint64_t rng_below(Rng* r, uint64_t bound) { return rng_next(r) % bound; }
static int64_t rng_int(Rng* r, int64_t lo, int64_t hi) { return lo + (int64_t)rng_below(r, (uint64_t)(hi - lo + 1)); }
static double rng_double(Rng* r) { return (double)(rng_next(r) >> 11) * 0x1.0p-53; }
static double rng_real(Rng* r, double lo, double hi) { return lo + (hi - lo) * rng_double(r); }

void orc_splitmix64(uint64_t seed, uint64_t stream, uint64_t count, uint64_t* out) {
    Rng r = rng_make(seed, stream);
    for (uint64_t i = 0; i < count; ++i) out[i] = rng_next(&r);
}

/* Draw helpers used to build inputs exactly as the reference campaigns do
 * (P:src/fault_lab.cpp:75-85, 240-254). */
void orc_gen_u8(uint64_t seed, uint64_t stream, uint64_t skip, uint64_t count, uint8_t* out) {
    Rng r = rng_make(seed, stream);
    for (uint64_t i = 0; i < skip; ++i) rng_next(&r);
    for (uint64_t i = 0; i < count; ++i) out[i] = (uint8_t)rng_below(&r, 256);
}
void orc_gen_s8(uint64_t seed, uint64_t stream, uint64_t skip, uint64_t count, int8_t* out) {
    Rng r = rng_make(seed, stream);
    for (uint64_t i = 0; i < skip; ++i) rng_next(&r);
    for (uint64_t i = 0; i < count; ++i) out[i] = (int8_t)rng_int(&r, -128, 127);
}
void orc_gen_real_f32(uint64_t seed, uint64_t stream, uint64_t skip, uint64_t count, double lo, double hi,
                      float* out) {
    Rng r = rng_make(seed, stream);
    for (uint64_t i = 0; i < skip; ++i) rng_next(&r);
    for (uint64_t i = 0; i < count; ++i) out[i] = (float)rng_real(&r, lo, hi);
}
void orc_gen_below(uint64_t seed, uint64_t stream, uint64_t skip, uint64_t count, uint64_t bound, int64_t* out) {
    Rng r = rng_make(seed, stream);
    for (uint64_t i = 0; i < skip; ++i) rng_next(&r);
    for (uint64_t i = 0; i < count; ++i) out[i] = (int64_t)rng_below(&r, bound);
}

/* ------------------------------------------------------------ GEMM (P:src/gemm_abft.cpp) */
/* Least non-negative residue (P:src/gemm_abft.hpp:13-16). */
int32_t orc_mod127(int64_t v) {
    int64_t r = v % 127;
    return (int32_t)(r < 0 ? r + 127 : r);
}

/* compute_row_checksums (P:src/gemm_abft.cpp:60-71): int64 row sum -> mod127 -> int8. */
int orc_compute_row_checksums(const int8_t* b, size_t k, size_t n, int8_t* cs) {
    if (k == 0 || n == 0) return -1; /* "compute_row_checksums: empty matrix" */
    for (size_t i = 0; i < k; ++i) {
        int64_t s = 0;
        for (size_t j = 0; j < n; ++j) s += b[i * n + j];
        cs[i] = (int8_t)orc_mod127(s);
    }
    return 0;
}

/* pack_blocks + PackedEncodedWeight (P:src/gemm_abft.cpp:13-28, 73-85): logical k x (n+1)
 * [B | cs] stored block-major (rb x cb blocks, zero padded). Returns the buffer length. */
size_t orc_pack_len(size_t k, size_t n, size_t rb, size_t cb) {
    const size_t rbl = (k + rb - 1) / rb, cbl = (n + 1 + cb - 1) / cb;
    return rbl * cbl * rb * cb;
}
int orc_pack_encoded(const int8_t* b, const int8_t* cs, size_t k, size_t n, size_t rb, size_t cb, int8_t* buf) {
    if (rb == 0 || cb == 0) return -1;
    const size_t cols = n + 1, cbl = (cols + cb - 1) / cb;
    memset(buf, 0, orc_pack_len(k, n, rb, cb));
    for (size_t i = 0; i < k; ++i)
        for (size_t j = 0; j < cols; ++j) {
            const size_t blk = (i / rb) * cbl + j / cb;
            buf[blk * rb * cb + (i % rb) * cb + j % cb] = j < n ? b[i * n + j] : cs[i];
        }
    return 0;
}
/* PackedEncodedWeight::at (P:src/gemm_abft.cpp:87-91). */
int8_t orc_packed_at(const int8_t* buf, size_t n, size_t rb, size_t cb, size_t i, size_t j) {
    const size_t cbl = (n + 1 + cb - 1) / cb;
    return buf[((i / rb) * cbl + j / cb) * rb * cb + (i % rb) * cb + j % cb];
}

/* packed_gemm semantics (P:src/gemm_abft.cpp:30-56): C[i][j] = sum_p A[i][p] * B'[p][j] with
 * int32 accumulation (exact for k < 65793; two's-complement wrap otherwise). Per-element
 * integer sums are order independent, so a plain loop nest reproduces it. */
static void gemm_i32(const uint8_t* a, size_t m, size_t k, const int8_t* b, size_t ldb, size_t cols,
                     const int8_t* extra_col, int32_t* c, size_t ldc) {
    for (size_t i = 0; i < m; ++i) {
        uint32_t* crow = (uint32_t*)(c + i * ldc);
        for (size_t j = 0; j < cols + (extra_col ? 1 : 0); ++j) crow[j] = 0;
        for (size_t p = 0; p < k; ++p) {
            const int32_t av = a[i * k + p];
            if (av == 0) continue;
            const int8_t* brow = b + p * ldb;
            for (size_t j = 0; j < cols; ++j) crow[j] += (uint32_t)(av * (int32_t)brow[j]);
            if (extra_col) crow[cols] += (uint32_t)(av * (int32_t)extra_col[p]);
        }
    }
}

/* verify_checksums (P:src/gemm_abft.cpp:113-124): rows x (n+1) with the checksum column last. */
uint64_t orc_verify_checksums(const int32_t* c, size_t rows, size_t cols, uint8_t* flags) {
    const size_t n = cols - 1;
    uint64_t err = 0;
    for (size_t i = 0; i < rows; ++i) {
        int64_t s = 0;
        for (size_t j = 0; j < n; ++j) s += c[i * cols + j];
        const int f = orc_mod127(s) != orc_mod127(c[i * cols + n]);
        if (flags) flags[i] = (uint8_t)f;
        err += (uint64_t)f;
    }
    return err;
}

/* abft_gemm (P:src/gemm_abft.cpp:93-100): cTemp = A x [B | cs], m x (n+1), then verify.
 * cs == NULL -> compute_row_checksums(B). */
int orc_abft_gemm(const uint8_t* a, size_t m, size_t k, const int8_t* b, size_t n, const int8_t* cs_in,
                  int32_t* ctemp, uint8_t* flags, uint64_t* err_count) {
    if (k == 0 || n == 0) return -1;
    int8_t* cs = (int8_t*)cs_in;
    if (!cs) {
        cs = (int8_t*)malloc(k);
        orc_compute_row_checksums(b, k, n, cs);
    }
    gemm_i32(a, m, k, b, n, n, cs, ctemp, n + 1);
    *err_count = orc_verify_checksums(ctemp, m, n + 1, flags);
    if (!cs_in) free(cs);
    return 0;
}

/* plain_gemm (P:src/gemm_abft.cpp:102-111). */
int orc_plain_gemm(const uint8_t* a, size_t m, size_t k, const int8_t* b, size_t n, int32_t* c) {
    gemm_i32(a, m, k, b, n, n, NULL, c, n);
    return 0;
}

/* Dual-encoded test oracle (P:tests/dual_check.hpp:23-73): (m+1) x (n+1) int64 product with
 * exact checksum row/column. kind: 0 clean, 1 located (i, j), 2 multi_error. */
void orc_dual_encoded_product(const uint8_t* a, size_t m, size_t k, const int8_t* b, size_t n, int64_t* c) {
    const size_t N = n + 1;
    memset(c, 0, (m + 1) * N * sizeof(int64_t));
    for (size_t i = 0; i <= m; ++i)
        for (size_t p = 0; p < k; ++p) {
            int64_t av = 0;
            if (i < m)
                av = a[i * k + p];
            else
                for (size_t r = 0; r < m; ++r) av += a[r * k + p];
            int64_t bs = 0;
            for (size_t j = 0; j < n; ++j) {
                c[i * N + j] += av * b[p * n + j];
                bs += b[p * n + j];
            }
            c[i * N + n] += av * bs;
        }
}
int orc_dual_encoded_check(const int64_t* c, size_t m, size_t n, size_t* bi, size_t* bj) {
    const size_t N = n + 1;
    size_t nbr = 0, nbc = 0, r0 = 0, c0 = 0;
    for (size_t i = 0; i <= m; ++i) {
        int64_t s = 0;
        for (size_t j = 0; j < n; ++j) s += c[i * N + j];
        if (s != c[i * N + n]) {
            if (!nbr) r0 = i;
            ++nbr;
        }
    }
    for (size_t j = 0; j <= n; ++j) {
        int64_t s = 0;
        for (size_t i = 0; i < m; ++i) s += c[i * N + j];
        if (s != c[m * N + j]) {
            if (!nbc) c0 = j;
            ++nbc;
        }
    }
    if (!nbr && !nbc) return 0;
    if (nbr == 1 && nbc == 1) {
        *bi = r0;
        *bj = c0;
        return 1;
    }
    return 2;
}

/* ------------------------------------------------------------ EmbeddingBag (P:src/embedding_abft.cpp) */
enum { ELEM_S8 = 0, ELEM_U8 = 1, ELEM_U4 = 2 };
enum { SCALE_F32 = 0, SCALE_F16 = 1 };

float orc_half_to_float(uint16_t h) {
    const uint32_t sign = (uint32_t)(h >> 15) << 31;
    const int exp = (h >> 10) & 0x1F;
    const uint32_t man = h & 0x3FF;
    uint32_t bits;
    if (exp == 0) {
        if (man == 0) {
            bits = sign;
        } else { /* subnormal: value = man * 2^-24, exact in float */
            float v = (float)man * 0x1.0p-24f;
            memcpy(&bits, &v, 4);
            bits |= sign;
        }
    } else if (exp == 31) {
        bits = sign | 0x7F800000u | (man << 13);
    } else {
        bits = sign | ((uint32_t)(exp - 15 + 127) << 23) | (man << 13);
    }
    float f;
    memcpy(&f, &bits, 4);
    return f;
}

/* Element decode, templated on the storage type (s8 is the reference's; u8/u4 per SURVEY 8c). */
static float elem_at(int elem, const uint8_t* row, size_t j) {
    if (elem == ELEM_S8) return (float)(int8_t)row[j];
    if (elem == ELEM_U8) return (float)row[j];
    return (float)((row[j >> 1] >> (4 * (j & 1))) & 0xF);
}
static int32_t elem_int(int elem, const uint8_t* row, size_t j) {
    if (elem == ELEM_S8) return (int8_t)row[j];
    if (elem == ELEM_U8) return row[j];
    return (row[j >> 1] >> (4 * (j & 1))) & 0xF;
}
static void scale_bias(int st, const void* scales, const void* biases, size_t i, float* s, float* b) {
    if (st == SCALE_F32) {
        *s = ((const float*)scales)[i];
        *b = ((const float*)biases)[i];
    } else {
        *s = orc_half_to_float(((const uint16_t*)scales)[i]);
        *b = orc_half_to_float(((const uint16_t*)biases)[i]);
    }
}

/* precompute_row_sums (P:src/embedding_abft.cpp:39-45): int32 element sums. */
void orc_precompute_row_sums(int elem, const uint8_t* rows, size_t R, size_t d, size_t stride, int32_t* out) {
    for (size_t i = 0; i < R; ++i) {
        int32_t s = 0;
        for (size_t j = 0; j < d; ++j) s += elem_int(elem, rows + i * stride, j);
        out[i] = s;
    }
}

/* One bag: embedding_bag (P:src/embedding_abft.cpp:47-60) + abft_embedding_bag (62-83).
 * Returns -2 if an index is out of range (the reference throws out_of_range, 16-22). */
static int one_bag(int elem, int st, const uint8_t* rows, size_t R, size_t d, size_t stride, const void* scales,
                   const void* biases, const int32_t* row_sums, const int64_t* idx, const float* w, size_t L,
                   int checked, float* r, double* rsum, double* csum, uint8_t* err) {
    for (size_t t = 0; t < L; ++t)
        if ((uint64_t)idx[t] >= R) return -2;
    for (size_t j = 0; j < d; ++j) r[j] = 0.0f;
    for (size_t t = 0; t < L; ++t) {
        const size_t i = (size_t)idx[t];
        const float wt = w ? w[t] : 1.0f;
        float s, b;
        scale_bias(st, scales, biases, i, &s, &b);
        const uint8_t* row = rows + i * stride;
        for (size_t j = 0; j < d; ++j) {
            float x = s * elem_at(elem, row, j);
            x = x + b;
            x = wt * x;
            r[j] = r[j] + x;
        }
    }
    if (!checked) return 0;
    double rs = 0.0;
    for (size_t j = 0; j < d; ++j) rs += (double)r[j];
    const double dd = (double)d;
    double cs = 0.0;
    for (size_t t = 0; t < L; ++t) {
        const size_t i = (size_t)idx[t];
        const double wt = w ? (double)w[t] : 1.0;
        float s, b;
        scale_bias(st, scales, biases, i, &s, &b);
        const double term = (double)s * (double)row_sums[i] + dd * (double)b;
        cs += wt * term;
    }
    *rsum = rs;
    *csum = cs;
    double mx = fabs(rs) > fabs(cs) ? fabs(rs) : fabs(cs);
    if (mx < 1.0) mx = 1.0;
    *err = (uint8_t)(fabs(rs - cs) > 1e-5 * mx);
    return 0;
}

/* batch_abft_eb / embedding_bag over CSR bags (P:src/embedding_abft.cpp:85-91).
 * row_sums == NULL -> precomputed here. rsum/csum/err may be NULL when !checked. */
int orc_eb_bags(int elem, int scale_type, const uint8_t* rows, size_t R, size_t d, size_t stride, const void* scales,
                const void* biases, const int32_t* row_sums, const int64_t* offsets, const int64_t* indices,
                const float* weights, size_t nbags, int checked, float* r_out, double* rsum, double* csum,
                uint8_t* err) {
    int32_t* sums = (int32_t*)row_sums;
    if (checked && !sums) {
        sums = (int32_t*)malloc(R * sizeof(int32_t));
        orc_precompute_row_sums(elem, rows, R, d, stride, sums);
    }
    int rc = 0;
    for (size_t b = 0; b < nbags && rc == 0; ++b) {
        double rs = 0, cs = 0;
        uint8_t e = 0;
        rc = one_bag(elem, scale_type, rows, R, d, stride, scales, biases, sums, indices + offsets[b],
                     weights ? weights + offsets[b] : NULL, (size_t)(offsets[b + 1] - offsets[b]), checked,
                     r_out + b * d, &rs, &cs, &e);
        if (checked) {
            if (rsum) rsum[b] = rs;
            if (csum) csum[b] = cs;
            if (err) err[b] = e;
        }
    }
    if (checked && !row_sums) free(sums);
    return rc;
}

/* ------------------------------------------------------------ fault lab (P:src/fault_lab.cpp) */
enum { T_WEIGHT_B = 0, T_INTERMEDIATE_C = 1, T_EB_TABLE = 2, T_NONE = 3 };
enum { M_BITFLIP = 0, M_RANDOM = 1 };
enum { R_ALL = 0, R_HIGH4 = 1, R_LOW4 = 2 };

/* draw_bit_index (P:src/fault_lab.cpp:89-96). */
static unsigned draw_bit(Rng* r, int range, unsigned width) {
    if (range == R_HIGH4) return width - 4 + (unsigned)rng_below(r, 4);
    if (range == R_LOW4) return (unsigned)rng_below(r, 4);
    return (unsigned)rng_below(r, width);
}
unsigned orc_draw_bit_index(uint64_t seed, uint64_t stream, int range, unsigned width) {
    Rng r = rng_make(seed, stream);
    return draw_bit(&r, range, width);
}

/* inject_weight_B (P:src/fault_lab.cpp:98-115): rec = {injected, i, j, before, after}. */
int orc_inject_weight_B(int8_t* b, size_t k, size_t n, int target, int model, int range, uint64_t seed,
                        uint64_t trial, int64_t* rec) {
    rec[0] = 0;
    if (target == T_NONE) return 0;
    Rng r = rng_make(seed, trial * 4 + 1);
    const size_t i = (size_t)rng_below(&r, k), j = (size_t)rng_below(&r, n);
    int8_t* cell = &b[i * n + j];
    rec[0] = 1;
    rec[1] = (int64_t)i;
    rec[2] = (int64_t)j;
    rec[3] = *cell;
    if (model == M_BITFLIP) {
        *cell = (int8_t)((uint8_t)*cell ^ (uint8_t)(1u << draw_bit(&r, range, 8)));
    } else {
        int8_t nv;
        do nv = (int8_t)rng_int(&r, -128, 127);
        while (nv == *cell);
        *cell = nv;
    }
    rec[4] = *cell;
    return 0;
}

/* inject_intermediate_C (P:src/fault_lab.cpp:117-137): any column j <= n, 32-bit. */
int orc_inject_intermediate_C(int32_t* c, size_t rows, size_t cols, int target, int model, int range, uint64_t seed,
                              uint64_t trial, int64_t* rec) {
    rec[0] = 0;
    if (target == T_NONE) return 0;
    Rng r = rng_make(seed, trial * 4 + 1);
    const size_t i = (size_t)rng_below(&r, rows), j = (size_t)rng_below(&r, cols);
    int32_t* cell = &c[i * cols + j];
    rec[0] = 1;
    rec[1] = (int64_t)i;
    rec[2] = (int64_t)j;
    rec[3] = *cell;
    if (model == M_BITFLIP) {
        *cell = (int32_t)((uint32_t)*cell ^ (1u << draw_bit(&r, range, 32)));
    } else {
        int32_t nv;
        do nv = (int32_t)rng_next(&r);
        while (nv == *cell);
        *cell = nv;
    }
    rec[4] = *cell;
    return 0;
}

/* inject_eb_table (P:src/fault_lab.cpp:139-166): an element of a row pooled by a non-empty bag.
 * Works on any 8-bit table (s8 semantics for random_value). */
int orc_inject_eb_table(int8_t* rows, size_t R, size_t d, const int64_t* offsets, const int64_t* indices, size_t nbags,
                        int target, int model, int range, uint64_t seed, uint64_t trial, int64_t* rec) {
    (void)R;
    rec[0] = 0;
    if (target == T_NONE) return 0;
    Rng r = rng_make(seed, trial * 4 + 1);
    size_t nusable = 0;
    for (size_t b = 0; b < nbags; ++b) nusable += offsets[b + 1] > offsets[b];
    if (!nusable) return -1; /* "inject_eb_table: all bags empty" */
    size_t pick = (size_t)rng_below(&r, nusable), bag = 0;
    for (size_t b = 0; b < nbags; ++b)
        if (offsets[b + 1] > offsets[b]) {
            if (pick == 0) {
                bag = b;
                break;
            }
            --pick;
        }
    const size_t len = (size_t)(offsets[bag + 1] - offsets[bag]);
    const size_t row = (size_t)indices[offsets[bag] + (int64_t)rng_below(&r, len)];
    const size_t col = (size_t)rng_below(&r, d);
    int8_t* cell = &rows[row * d + col];
    rec[0] = 1;
    rec[1] = (int64_t)row;
    rec[2] = (int64_t)col;
    rec[3] = *cell;
    if (model == M_BITFLIP) {
        *cell = (int8_t)((uint8_t)*cell ^ (uint8_t)(1u << draw_bit(&r, range, 8)));
    } else {
        int8_t nv;
        do nv = (int8_t)rng_int(&r, -128, 127);
        while (nv == *cell);
        *cell = nv;
    }
    rec[4] = *cell;
    return 0;
}

/* ------------------------------------------------------------ campaigns (P:src/fault_lab.cpp:168-285) */
typedef struct {
    const uint64_t* shapes; /* m, n, k triples */
    size_t nshapes, per;
    int target, model, range;
    uint64_t seed;
    uint8_t* detected;
    size_t total, worker, workers;
} GemmJob;

static void* gemm_worker(void* arg) {
    GemmJob* j = (GemmJob*)arg;
    for (size_t t = j->worker; t < j->total; t += j->workers) {
        const uint64_t* s = j->shapes + 3 * (t / j->per);
        const size_t m = s[0], n = s[1], k = s[2];
        uint8_t* a = (uint8_t*)malloc(m * k);
        int8_t* b = (int8_t*)malloc(k * n);
        int8_t* cs = (int8_t*)malloc(k);
        int32_t* c = (int32_t*)malloc(m * (n + 1) * sizeof(int32_t));
        Rng r = rng_make(j->seed, t * 4 + 0);
        for (size_t e = 0; e < m * k; ++e) a[e] = (uint8_t)rng_below(&r, 256);
        for (size_t e = 0; e < k * n; ++e) b[e] = (int8_t)rng_int(&r, -128, 127);
        orc_compute_row_checksums(b, k, n, cs);
        int64_t rec[5];
        if (j->target == T_WEIGHT_B) orc_inject_weight_B(b, k, n, j->target, j->model, j->range, j->seed, t, rec);
        uint64_t err = 0;
        orc_abft_gemm(a, m, k, b, n, cs, c, NULL, &err);
        if (j->target == T_INTERMEDIATE_C) {
            orc_inject_intermediate_C(c, m, n + 1, j->target, j->model, j->range, j->seed, t, rec);
            err = orc_verify_checksums(c, m, n + 1, NULL);
        }
        j->detected[t] = err > 0;
        free(a);
        free(b);
        free(cs);
        free(c);
    }
    return NULL;
}

static void run_parallel(void* (*fn)(void*), void* jobs, size_t job_size, size_t workers) {
    pthread_t* th = (pthread_t*)malloc(workers * sizeof(pthread_t));
    for (size_t w = 0; w < workers; ++w) pthread_create(&th[w], NULL, fn, (char*)jobs + w * job_size);
    for (size_t w = 0; w < workers; ++w) pthread_join(th[w], NULL);
    free(th);
}

int orc_run_gemm_campaign(const uint64_t* shapes, size_t nshapes, size_t per, int target, int model, int range,
                          uint64_t seed, size_t workers, uint8_t* detected) {
    if (!nshapes || !per) return -1;
    if (target == T_EB_TABLE) return -1;
    const size_t total = nshapes * per;
    if (workers < 1) workers = 1;
    if (workers > total) workers = total;
    GemmJob* jobs = (GemmJob*)calloc(workers, sizeof(GemmJob));
    for (size_t w = 0; w < workers; ++w)
        jobs[w] = (GemmJob){shapes, nshapes, per, target, model, range, seed, detected, total, w, workers};
    run_parallel(gemm_worker, jobs, sizeof(GemmJob), workers);
    free(jobs);
    return 0;
}

typedef struct {
    size_t R, d, pool, batch, trials;
    int target, model, range;
    uint64_t seed;
    uint8_t* detected;
    size_t worker, workers;
} EbJob;

static void* eb_worker(void* arg) {
    EbJob* j = (EbJob*)arg;
    const size_t R = j->R, d = j->d, L = j->pool * j->batch;
    int8_t* rows = (int8_t*)malloc(R * d);
    float* sc = (float*)malloc(R * sizeof(float));
    float* bi = (float*)malloc(R * sizeof(float));
    int32_t* sums = (int32_t*)malloc(R * sizeof(int32_t));
    int64_t* idx = (int64_t*)malloc(L * sizeof(int64_t));
    int64_t* off = (int64_t*)malloc((j->batch + 1) * sizeof(int64_t));
    float* r = (float*)malloc(j->batch * d * sizeof(float));
    uint8_t* err = (uint8_t*)malloc(j->batch);
    for (size_t b = 0; b <= j->batch; ++b) off[b] = (int64_t)(b * j->pool);
    for (size_t t = j->worker; t < j->trials; t += j->workers) {
        Rng g = rng_make(j->seed, t * 4 + 0);
        for (size_t e = 0; e < R * d; ++e) rows[e] = (int8_t)rng_int(&g, -128, 127);
        for (size_t i = 0; i < R; ++i) sc[i] = (float)rng_real(&g, 0.005, 0.02);
        for (size_t i = 0; i < R; ++i) bi[i] = (float)rng_real(&g, -1.0, 1.0);
        orc_precompute_row_sums(ELEM_S8, (const uint8_t*)rows, R, d, d, sums);
        Rng bg = rng_make(j->seed, t * 4 + 2);
        for (size_t e = 0; e < L; ++e) idx[e] = (int64_t)rng_below(&bg, R);
        int64_t rec[5];
        if (j->target == T_EB_TABLE)
            orc_inject_eb_table(rows, R, d, off, idx, j->batch, j->target, j->model, j->range, j->seed, t, rec);
        orc_eb_bags(ELEM_S8, SCALE_F32, (const uint8_t*)rows, R, d, d, sc, bi, sums, off, idx, NULL, j->batch, 1, r,
                    NULL, NULL, err);
        uint8_t any = 0;
        for (size_t b = 0; b < j->batch; ++b) any |= err[b];
        j->detected[t] = any;
    }
    free(rows);
    free(sc);
    free(bi);
    free(sums);
    free(idx);
    free(off);
    free(r);
    free(err);
    return NULL;
}

int orc_run_eb_campaign(size_t R, size_t d, size_t pool, size_t batch, size_t trials, int target, int model, int range,
                        uint64_t seed, size_t workers, uint8_t* detected) {
    if (!trials || !R || !d || !pool || !batch) return -1;
    if (target == T_WEIGHT_B || target == T_INTERMEDIATE_C) return -1;
    if (workers < 1) workers = 1;
    if (workers > trials) workers = trials;
    EbJob* jobs = (EbJob*)calloc(workers, sizeof(EbJob));
    for (size_t w = 0; w < workers; ++w)
        jobs[w] = (EbJob){R, d, pool, batch, trials, target, model, range, seed, detected, w, workers};
    run_parallel(eb_worker, jobs, sizeof(EbJob), workers);
    free(jobs);
    return 0;
}

/* ------------------------------------------------------------ multi-threaded CPU baselines */
typedef struct {
    const uint8_t* a;
    size_t m, k;
    const int8_t* b;
    size_t n;
    const int8_t* cs;
    int32_t* c;
    uint64_t err;
} GemmRep;

static void* gemm_rep_worker(void* arg) {
    GemmRep* g = (GemmRep*)arg;
    orc_abft_gemm(g->a, g->m, g->k, g->b, g->n, g->cs, g->c, NULL, &g->err);
    return NULL;
}

/* `copies` independent checked GEMMs on `copies` threads (each writes its own cTemp). */
int orc_abft_gemm_parallel(const uint8_t* a, size_t m, size_t k, const int8_t* b, size_t n, const int8_t* cs,
                           size_t copies, int32_t* ctemp_scratch, uint64_t* err_out) {
    GemmRep* reps = (GemmRep*)calloc(copies, sizeof(GemmRep));
    for (size_t i = 0; i < copies; ++i)
        reps[i] = (GemmRep){a, m, k, b, n, cs, ctemp_scratch + i * m * (n + 1), 0};
    run_parallel(gemm_rep_worker, reps, sizeof(GemmRep), copies);
    uint64_t e = 0;
    for (size_t i = 0; i < copies; ++i) e += reps[i].err;
    *err_out = e;
    free(reps);
    return 0;
}

/* ------------------------------------------------------------ requantization (P:src/quant.cpp:10-14, 77-118)
 * params = {scaleA, biasA, scaleB, biasB, scaleC, biasC} (RequantParams, P:src/quant.hpp:24-32), k separate.
 * cf = sA*sB*c + sA*bB*rowSumA[i] + sB*bA*colSumB[j] + k*bA*bB in the reference's left-to-right double
 * order; out = clamp(round_half_away((cf - bC) / sC), 0, 255). Columns >= n (a checksum column) are never
 * read. Returns -1 (invalid_argument) when scaleC <= 0. */
static double round_half_away(double x) { return x >= 0.0 ? floor(x + 0.5) : ceil(x - 0.5); }
int orc_requantize(const int32_t* c, size_t ldc, size_t m, size_t n, const int32_t* row_sum_a,
                   const int32_t* col_sum_b, const double* prm, uint64_t k, uint8_t* out, size_t ld_out) {
    const double sA = prm[0], bA = prm[1], sB = prm[2], bB = prm[3], sC = prm[4], bC = prm[5];
    if (!(sC > 0.0)) return -1;
    for (size_t i = 0; i < m; ++i)
        for (size_t j = 0; j < n; ++j) {
            const double cf = sA * sB * (double)c[i * ldc + j] + sA * bB * (double)row_sum_a[i] +
                              sB * bA * (double)col_sum_b[j] + (double)k * bA * bB;
            double r = round_half_away((cf - bC) / sC);
            r = r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r);
            out[i * ld_out + j] = (uint8_t)r;
        }
    return 0;
}
void orc_row_sums_u8(const uint8_t* a, size_t m, size_t k, size_t lda, int32_t* out) {
    for (size_t i = 0; i < m; ++i) {
        int32_t s = 0;
        for (size_t p = 0; p < k; ++p) s += (int32_t)a[i * lda + p];
        out[i] = s;
    }
}
void orc_col_sums_i8(const int8_t* b, size_t k, size_t n, size_t ldb, int32_t* out) {
    for (size_t j = 0; j < n; ++j) out[j] = 0;
    for (size_t i = 0; i < k; ++i)
        for (size_t j = 0; j < n; ++j) out[j] += (int32_t)b[i * ldb + j];
}
