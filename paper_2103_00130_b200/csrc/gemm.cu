// ABFT int8 GEMM for sm_100a.
//
//   encode_weight_kernel  replaces compute_row_checksums + PackedEncodedWeight
//                         (P:src/gemm_abft.cpp:60-91): one pass over B producing the mod-127 row
//                         checksums cs and B^T in the K-block-major layout the mainloop streams
//                         (abft_internal.h: GemmWeight). The checksum column C'[:, n] = A*cs is a
//                         GEMV done by the epilogue warps while the tensor cores run the tile.
//   gemm_pair_kernel      replaces abft_gemm + verify_checksums / plain_gemm
//                         (P:src/gemm_abft.cpp:30-56, 93-124). Persistent CTA pairs
//                         (cluster of 2, tcgen05.mma.cta_group::2 kind::i8, M=256 x N=BN, A u8 x
//                         B s8 -> s32 in TMEM). Each CTA loads its 128 rows of A and half of the
//                         B' tile; one 3-D TMA request per operand brings KS k-blocks (few, large
//                         requests: the per-SM TMA engine completes requests ~serially, so bytes per
//                         request set the ingest rate). Two TMEM accumulators let the epilogue of
//                         tile i overlap the mainloop of tile i+1. The CHECKED epilogue reduces
//                         every output row mod 127 straight from TMEM, adds its K share of
//                         A*cs (exact int32, dp4a), and folds both plus an arrival count into one
//                         64-bit atomic per row; the thread that completes a row compares and
//                         publishes its flag -- no second pass over C, no fences or counters, and
//                         no extra MMA tile for the checksum column.
//   verify_kernel         replaces verify_checksums (P:src/gemm_abft.cpp:113-124) for post-hoc
//                         checks (faults injected into C after the product).
#include <cuda_runtime.h>

#include <cstdlib>
#include <cstring>

#include "abft_internal.h"
#include "ptx.cuh"
#include "requant.cuh"

namespace abftk {

// ============================================================ encoder
// Block handles a 64-row slab of B (64 consecutive p, inside one k-block) and walks all n_pad
// columns in 64-wide chunks, so the int64 row sums stay block-local (as the reference). Writes
// B'[kb][j][p % 128] (64 contiguous bytes per j) and cs[p] (zero for k <= p < k_pad).
__global__ void __launch_bounds__(256) encode_weight_kernel(const int8_t* __restrict__ b, int64_t k, int64_t n,
                                                            int64_t ldb, int8_t* __restrict__ bt, int64_t n_pad,
                                                            int8_t* __restrict__ cs) {
    __shared__ int8_t tile[64][64 + 4];
    __shared__ long long part[4][64];
    const int tid = threadIdx.x;
    const int64_t p0 = static_cast<int64_t>(blockIdx.x) * 64;
    int8_t* slab = bt + (p0 / kBK) * n_pad * kBK + (p0 % kBK);
    long long acc = 0;  // thread (tid & 63) accumulates row (tid & 63) for column quarter (tid >> 6)
    for (int64_t j0 = 0; j0 < n_pad; j0 += 64) {
        for (int idx = tid; idx < 64 * 64; idx += 256) {
            const int r = idx >> 6, c = idx & 63;
            const int64_t p = p0 + r, j = j0 + c;
            tile[r][c] = (p < k && j < n) ? b[p * ldb + j] : static_cast<int8_t>(0);
        }
        __syncthreads();
        {
            const int r = tid & 63, q = tid >> 6;
#pragma unroll
            for (int c = 0; c < 16; ++c) acc += tile[r][q * 16 + c];
        }
        for (int idx = tid; idx < 64 * 64; idx += 256) {
            const int c = idx >> 6, r = idx & 63;
            slab[(j0 + c) * kBK + r] = tile[r][c];
        }
        __syncthreads();
    }
    part[tid >> 6][tid & 63] = acc;
    __syncthreads();
    if (tid < 64) {
        const long long s = part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid];
        const int64_t p = p0 + tid;
        const int8_t v = p < k ? static_cast<int8_t>(mod127(s)) : static_cast<int8_t>(0);
        cs[p] = v;
        if (n < n_pad) slab[n * kBK + tid] = v;  // the checksum column as B' column n: C'[:, n] on the tensor cores
    }
}

// 2-D encoder (the one above walks every column of a 64-row slab in one block: 64 blocks for k = 4096, ~150 GB/s).
// One block per (k-block, 128-column) tile of B: its slab of B' -- bt[kb][j0 .. j0 + 127][0 .. 127] -- is one
// contiguous 16 KB run.
//   load       128 rows x 128 bytes as 16-byte pieces (8 consecutive threads per row segment, 4 pieces per thread in
//              flight), into shared memory with the 16-byte chunk index XOR-swizzled by the row's 16-row group, so
//              the transposing reads below are bank-conflict free;
//   row sums   dp4a over each piece, reduced over the row's 8 threads, residue mod 127 added to cs_acc[p] together
//              with one arrival (the residue of a sum is the sum of the residues: P:src/gemm_abft.cpp:60-71 reduces
//              the int64 row sum once). Atomics on one address are totally ordered, so the thread that brings the
//              last column tile's arrival holds the row's complete residue: it writes cs[p] and B' column n and
//              re-zeroes the scratch word -- no second kernel, no fence;
//   transpose  a thread owns 16 rows x 4 columns: 16 word reads, 4 x (4x4 byte transposes by PRMT), four 16-byte
//              stores (8 threads cover one column's 128 contiguous bytes).
// Column n (the checksum column's slot) is written by the rows' finalizing threads only; the tile that contains it
// zero-fills its rows past k.
constexpr int kEncCountShift = 20;  // cs_acc word: arrivals << 20 | residue sum (tiles <= 2047, residues < 127 each)
__device__ __forceinline__ void transpose4x4(uint32_t& a, uint32_t& b, uint32_t& c, uint32_t& d) {
    // rows a, b, c, d of a 4x4 byte matrix (byte i of a = a[i]) -> columns
    const uint32_t ab_lo = __byte_perm(a, b, 0x5140);  // a0 b0 a1 b1
    const uint32_t ab_hi = __byte_perm(a, b, 0x7362);  // a2 b2 a3 b3
    const uint32_t cd_lo = __byte_perm(c, d, 0x5140);  // c0 d0 c1 d1
    const uint32_t cd_hi = __byte_perm(c, d, 0x7362);  // c2 d2 c3 d3
    a = __byte_perm(ab_lo, cd_lo, 0x5410);             // a0 b0 c0 d0
    b = __byte_perm(ab_lo, cd_lo, 0x7632);             // a1 b1 c1 d1
    c = __byte_perm(ab_hi, cd_hi, 0x5410);             // a2 b2 c2 d2
    d = __byte_perm(ab_hi, cd_hi, 0x7632);             // a3 b3 c3 d3
}
__global__ void __launch_bounds__(256) encode_tiles_kernel(const int8_t* __restrict__ b, int64_t k, int64_t n,
                                                           int64_t ldb, int8_t* __restrict__ bt, int64_t n_pad,
                                                           int32_t* __restrict__ cs_acc, int8_t* __restrict__ cs,
                                                           int col_tiles) {
    __shared__ __align__(16) uint4 tile[128][8];  // [row][swizzled 16-byte chunk]
    const int tid = threadIdx.x;
    const int64_t kb = blockIdx.y, p0 = kb * kBK, j0 = static_cast<int64_t>(blockIdx.x) * 128;
    const bool fast = (ldb % 16) == 0 && (reinterpret_cast<uintptr_t>(b) % 16) == 0;
    // ---- load + row sums: piece = tid + 256 i -> row piece / 8, chunk piece % 8
    uint4 v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = (tid >> 3) + 32 * i, c = tid & 7;
        const int64_t p = p0 + r, j = j0 + 16 * c;
        const int8_t* src = b + p * ldb + j;
        if (p < k && j + 16 <= n && fast) {
            v[i] = __ldg(reinterpret_cast<const uint4*>(src));
        } else {
            alignas(16) int8_t tmp[16];
#pragma unroll
            for (int e = 0; e < 16; ++e) tmp[e] = (p < k && j + e < n) ? src[e] : static_cast<int8_t>(0);
            v[i] = *reinterpret_cast<const uint4*>(tmp);
        }
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = (tid >> 3) + 32 * i, c = tid & 7;
        tile[r][c ^ ((r >> 4) & 7)] = v[i];
        int s = __dp4a(static_cast<int>(v[i].x), 0x01010101, 0);
        s = __dp4a(static_cast<int>(v[i].y), 0x01010101, s);
        s = __dp4a(static_cast<int>(v[i].z), 0x01010101, s);
        s = __dp4a(static_cast<int>(v[i].w), 0x01010101, s);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        const int64_t p = p0 + r;
        if (c == 0 && p < k && j0 < n) {
            const int add = (1 << kEncCountShift) | mod127(s);
            const int tot = atomicAdd(&cs_acc[p], add) + add;
            if ((tot >> kEncCountShift) == col_tiles) {  // the row is complete
                const int8_t cv = static_cast<int8_t>((tot & ((1 << kEncCountShift) - 1)) % 127);
                cs[p] = cv;
                bt[kb * n_pad * kBK + n * kBK + r] = cv;  // checksum column as B' column n
                cs_acc[p] = 0;
            }
        }
    }
    __syncthreads();
    // ---- transpose: rows [16 q, 16 q + 16) x columns [4 g, 4 g + 4)
    const int q = tid & 7, g = tid >> 3;
    uint32_t w[4][4];  // w[h][e]: row 16 q + 4 h + e, columns 4 g .. 4 g + 3
#pragma unroll
    for (int h = 0; h < 4; ++h)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const int r = 16 * q + 4 * h + e;
            w[h][e] = reinterpret_cast<const uint32_t*>(&tile[r][(g >> 2) ^ q])[g & 3];
        }
#pragma unroll
    for (int h = 0; h < 4; ++h) transpose4x4(w[h][0], w[h][1], w[h][2], w[h][3]);  // w[h][c]: column 4 g + c, rows 16 q + 4 h ..
    int8_t* const slab = bt + kb * n_pad * kBK + j0 * kBK + 16 * q;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const int64_t j = j0 + 4 * g + c;
        int8_t* dst = slab + (4 * g + c) * kBK;
        if (j == n) {  // the checksum column's slot: only the padding rows past k are ours
#pragma unroll
            for (int e = 0; e < 16; ++e)
                if (p0 + 16 * q + e >= k) {
                    dst[e] = 0;
                    cs[p0 + 16 * q + e] = 0;
                }
            continue;
        }
        *reinterpret_cast<uint4*>(dst) = make_uint4(w[0][c], w[1][c], w[2][c], w[3][c]);
    }
}

// Replace the checksum vector with caller-supplied values.
__global__ void set_checksums_kernel(int8_t* __restrict__ cs, const int8_t* __restrict__ src, int64_t k,
                                     int8_t* __restrict__ bt, int64_t n, int64_t n_pad) {
    for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < k;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        cs[p] = src[p];
        if (n < n_pad) bt[(p / kBK) * n_pad * kBK + n * kBK + (p % kBK)] = src[p];  // B' column n mirrors cs
    }
}

// Logical k x (n+1) view [B | cs] of an encoded weight (PackedEncodedWeight::at contract).
__global__ void read_encoded_kernel(const int8_t* __restrict__ bt, const int8_t* __restrict__ cs, int64_t k,
                                    int64_t n, int64_t n_pad, int8_t* __restrict__ out) {
    const int64_t total = k * (n + 1);
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e / (n + 1), j = e - i * (n + 1);
        out[e] = j == n ? cs[i] : bt[(i / kBK) * n_pad * kBK + j * kBK + (i % kBK)];
    }
}

// ============================================================ checksum GEMV share
// sum_{p in [k0, k1)} A[row][p] * cs[p], exact in 32 bits (A <= 255, |cs| <= 128, k < 65793 as the
// reference's int32 accumulation). 16-byte loads (lda % 16 == 0), four u8 x s8 dot products per dp4a.
__device__ __forceinline__ uint32_t csum_share(const GemmParams& p, int b, int row, int k0, int k1) {
    const uint8_t* arow = p.a + b * p.a_bstride + static_cast<int64_t>(row) * p.lda;
    const int8_t* cs = p.cs + b * p.cs_bstride;
    uint32_t s = 0;
    int kk = k0;
    for (; kk + 128 <= k1; kk += 128) {
        uint4 av[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) av[u] = __ldg(reinterpret_cast<const uint4*>(arow + kk + 16 * u));
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint4 cv = __ldg(reinterpret_cast<const uint4*>(cs + kk + 16 * u));
            s = dp4a_us(av[u].x, cv.x, s);
            s = dp4a_us(av[u].y, cv.y, s);
            s = dp4a_us(av[u].z, cv.z, s);
            s = dp4a_us(av[u].w, cv.w, s);
        }
    }
    for (; kk < k1; ++kk) s += static_cast<uint32_t>(static_cast<int32_t>(arow[kk]) * static_cast<int32_t>(cs[kk]));
    return s;
}

// ============================================================ row verdicts
// One 64-bit atomic per row carries a contribution's GEMV share (high 32 bits), one arrival and its residue
// (kRowAcc* layout). Atomics on one address are totally ordered, so the thread whose add brings arrival
// p.row_arrivals holds the complete row: it applies the reference's comparison (P:src/gemm_abft.cpp:113-124),
// writes the flag and the checksum column (after any injected C'[:, n] fault) and resets the slot.
__device__ __forceinline__ void row_arrive(const GemmParams& p, int b, int row, unsigned long long add, int& fin,
                                           int& flag) {
    unsigned long long* racc = p.row_acc + static_cast<int64_t>(b) * p.m + row;
    // a row with one contribution (one N tile, checksum in the same tile) is complete here: no round trip
    const bool sole = p.row_arrivals == 1;
    const unsigned long long v = sole ? add : atomicAdd(racc, add) + add;
    if (((v >> kRowAccCountShift) & kRowAccCountMask) == static_cast<unsigned long long>(p.row_arrivals)) {
        fin = 1;
        int32_t csv = static_cast<int32_t>(static_cast<uint32_t>(v >> 32));
        for (int f = 0; f < p.nfaults; ++f)
            if (b == p.fault_b[f] && row == p.fault_row[f] && p.fault_col[f] == p.n)
                csv ^= static_cast<int32_t>(1u << p.fault_bit[f]);  // fault in C'[:, n]
        const uint32_t res = static_cast<uint32_t>(v & kRowAccResMask) % 127u;
        flag = static_cast<int32_t>(res) != mod127(csv);
        p.flags[b * p.flags_bstride + row] = static_cast<uint8_t>(flag);
        p.csum[b * p.csum_bstride + static_cast<int64_t>(row) * p.csum_ld] = csv;
        if (!sole) *racc = 0ull;  // self-resetting workspace (a sole arrival never touched it)
    }
}
// (finished rows) << 32 | (flagged rows) per warp on the problem's word; the call's last finished row publishes
// Row-stacked requests: the finished rows of a warp may belong to several requests -- lanes are grouped by request
// (match.any), each group's lowest lane adds (rows finished, rows flagged) to the request's word, and the add that
// completes a request's req_rows rows publishes its count.
__device__ __forceinline__ void warp_publish_stacked(const GemmParams& p, int row, int fin, int flag) {
    const uint32_t finmask = __ballot_sync(0xffffffffu, fin);
    const uint32_t flagmask = __ballot_sync(0xffffffffu, flag);
    if (!fin) return;
    const int req = row / p.req_rows;
    const uint32_t grp = __match_any_sync(finmask, req);
    if ((threadIdx.x & 31) == static_cast<unsigned>(__ffs(static_cast<int>(grp)) - 1)) {
        const unsigned long long nfin = __popc(grp), nflag = __popc(grp & flagmask);
        const unsigned long long prev = atomicAdd(p.err_pack + req, (nfin << 32) | nflag);
        if ((prev >> 32) + nfin == static_cast<unsigned long long>(p.req_rows)) {
            p.err_count[req] = static_cast<uint32_t>(prev) + static_cast<uint32_t>(nflag);
            p.err_pack[req] = 0ull;
        }
    }
}
__device__ __forceinline__ void warp_publish(const GemmParams& p, int b, int fin, int flag) {
    const uint32_t nfin = __popc(__ballot_sync(0xffffffffu, fin));
    const uint32_t nflag = __popc(__ballot_sync(0xffffffffu, flag));
    if ((threadIdx.x & 31) == 0 && nfin) {
        const unsigned long long prev = atomicAdd(p.err_pack + b, (static_cast<unsigned long long>(nfin) << 32) | nflag);
        if ((prev >> 32) + nfin == static_cast<unsigned long long>(p.m)) {
            p.err_count[b] = static_cast<uint32_t>(prev) + nflag;
            p.err_pack[b] = 0ull;
        }
    }
}

// GEMV helpers (GemmParams::gemv_helpers): when the tile grid leaves pairs idle and few N tiles would split
// K (tall, narrow shards such as the D5 MLP layers), the idle CTAs compute the whole checksum column
// C'[:, n] = A * cs and add it as one extra arrival per row. A warp takes 8 consecutive rows of a problem;
// rows are read coalesced (lane l: bytes [16 l + 512 c, +16) of chunk c), four rows x four 512-byte chunks
// of loads in flight per lane before any is consumed (the helpers are latency-bound otherwise), each row
// reduced with one redux.sync and kept by lane (row % 8), which then arrives for its row.
__device__ __forceinline__ uint4 ld_slot(const uint8_t* p, int valid) {
    if (valid >= 16) return __ldg(reinterpret_cast<const uint4*>(p));
    uint32_t w[4] = {0u, 0u, 0u, 0u};
    for (int e = 0; e < valid; ++e) w[e >> 2] |= static_cast<uint32_t>(p[e]) << (8 * (e & 3));
    return make_uint4(w[0], w[1], w[2], w[3]);
}
__device__ void gemv_helper(const GemmParams& p, int helper_cta, int helper_ctas) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int hw = helper_cta * (blockDim.x >> 5) + warp, nhw = helper_ctas * (blockDim.x >> 5);
    const int tasks_per_problem = (p.m + 7) / 8;
    const long long tasks = static_cast<long long>(tasks_per_problem) * p.batch;
    for (long long g = hw; g < tasks; g += nhw) {
        const int b = static_cast<int>(g / tasks_per_problem);
        const int r0 = static_cast<int>(g - static_cast<long long>(b) * tasks_per_problem) * 8;
        const uint8_t* abase = p.a + b * p.a_bstride;
        const uint8_t* cs = reinterpret_cast<const uint8_t*>(p.cs + b * p.cs_bstride);
        uint32_t mine = 0u;
#pragma unroll 1
        for (int j0 = 0; j0 < 8 && r0 + j0 < p.m; j0 += 4) {
            uint32_t part[4] = {0u, 0u, 0u, 0u};
#pragma unroll 1
            for (int k0 = 0; k0 < p.k; k0 += 2048) {
                uint4 av[4][4], cv[4];
#pragma unroll
                for (int c = 0; c < 4; ++c) {
                    const int kp = k0 + 512 * c + 16 * lane;
                    const int valid = min(16, max(0, p.k - kp));
                    cv[c] = valid > 0 ? ld_slot(cs + kp, valid) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        av[j][c] = (valid > 0 && r0 + j0 + j < p.m)
                                       ? ld_slot(abase + static_cast<int64_t>(r0 + j0 + j) * p.lda + kp, valid)
                                       : make_uint4(0u, 0u, 0u, 0u);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j)
#pragma unroll
                    for (int c = 0; c < 4; ++c) {
                        part[j] = dp4a_us(av[j][c].x, cv[c].x, part[j]);
                        part[j] = dp4a_us(av[j][c].y, cv[c].y, part[j]);
                        part[j] = dp4a_us(av[j][c].z, cv[c].z, part[j]);
                        part[j] = dp4a_us(av[j][c].w, cv[c].w, part[j]);
                    }
            }
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t tot = __reduce_add_sync(0xffffffffu, part[j]);
                if (lane == j0 + j) mine = tot;
            }
        }
        int fin = 0, flag = 0;
        const int row = r0 + lane;
        if (lane < 8 && row < p.m)
            row_arrive(p, b, row, (static_cast<unsigned long long>(mine) << 32) | (1ull << kRowAccCountShift), fin, flag);
        if (p.req_rows > 0)
            warp_publish_stacked(p, row, fin, flag);
        else
            warp_publish(p, b, fin, flag);
    }
}

// ============================================================ GEMM (CTA pairs)
#ifndef ABFT_EPI_WARPS
#define ABFT_EPI_WARPS 4
#endif
template <int BN, int EW = ABFT_EPI_WARPS>
struct PairCfg {
    // k-blocks per pipeline stage. Measured on B200: an SM's TMA requests pipeline (issue ~50 ns each,
    // completions ~100-200 ns apart under full load), so what sustains ingest is BYTES IN FLIGHT, not
    // bytes per request -- small stages, as many as shared memory holds.
#ifndef ABFT_KS64
#define ABFT_KS64 4
#endif
#ifndef ABFT_KS128
#define ABFT_KS128 2
#endif
#ifndef ABFT_KS256
#define ABFT_KS256 2
#endif
#ifndef ABFT_STAGING_BUFS
#define ABFT_STAGING_BUFS 2
#endif
    static constexpr int KS = BN == 64 ? ABFT_KS64 : BN == 128 ? ABFT_KS128 : ABFT_KS256;
    // per epilogue warp; one with 8 epilogue warps (a pipeline stage more: measured 44.5 -> 43.0 us on the D5 MLP share)
    static constexpr int kStagingBufs = EW == 8 ? 1 : ABFT_STAGING_BUFS;
#ifndef ABFT_NA64
#define ABFT_NA64 2
#endif
#ifndef ABFT_NB64
#define ABFT_NB64 1
#endif
#ifndef ABFT_NA
#define ABFT_NA 2
#endif
#ifndef ABFT_NB
#define ABFT_NB 1
#endif
    static constexpr int NA = BN == 64 ? ABFT_NA64 : ABFT_NA;  // TMA warps loading A (K split)
    static constexpr int NB = BN == 64 ? ABFT_NB64 : ABFT_NB;  // TMA warps loading B' (K split)
    static constexpr int kProducers = NA + NB;
    // epilogue warps: one group of 4 (one per TMEM lane quarter) or two groups splitting the tile's columns
    static constexpr int kEpiWarps = EW;
    static constexpr int kEpiGroups = kEpiWarps / 4;
    static_assert(kEpiWarps == 4 || kEpiWarps == 8, "4 or 8 epilogue warps");
    // warps: producer 0, MMA, epilogue group 0 (4), producers 1.., epilogue group 1 (4, optional)
    static constexpr int kThreads = 32 * (1 + 1 + kEpiWarps + (kProducers - 1));
    static constexpr int kEpiG1 = 5 + kProducers;  // first warp of epilogue group 1
    static_assert(KS % NA == 0 && KS % NB == 0, "producer warps split the stage's k-blocks evenly");
    static constexpr int kABytes = kBM * kBK;                // per CTA per k-block (its 128 rows of A)
    static constexpr int kBBytes = (BN / 2) * kBK;           // per CTA per k-block (its half of the B' tile)
    static constexpr int kStageBytes = KS * (kABytes + kBBytes);
    static constexpr int kStaging = kEpiWarps * kStagingBufs * 4096; // epilogue warps x bufs x (32 x 32 int32)
    static constexpr int kBarBytes = 512;
    static constexpr int kRawStages = (227 * 1024 - 1024 - kStaging - kBarBytes) / kStageBytes;
    static constexpr int kStages = kRawStages > 16 ? 16 : kRawStages;
    static constexpr uint32_t kTmemCols = 2 * BN <= 128 ? 128 : 2 * BN <= 256 ? 256 : 512;
    static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kStaging + kBarBytes;
    static_assert(kStages >= 2, "need a double-buffered ring");
    static_assert(kBBytes % 1024 == 0 && kABytes % 1024 == 0, "SW128 tiles must stay 1024-byte aligned");
};

template <int BN, bool CHECKED, int EPI, int EW, bool GROUPED = false>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PairCfg<BN, EW>::kThreads, 1)
    gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmC, const GemmParams p) {
    using Cfg = PairCfg<BN, EW>;
    constexpr int STAGES = Cfg::kStages;
    constexpr int KS = Cfg::KS;
    // Grouped launches with 8 epilogue warps: the two groups take alternate TILES (group g drains accumulator buffer
    // g), so the fixed per-tile latencies of the epilogue chain (parameter loads, accumulator hand-over, row verdict
    // round trips) of consecutive tiles overlap; elsewhere two groups split each tile's column chunks.
    // (batched launches of one shape measured the same either way: G1 20.7 us)
    constexpr bool TILE_ALT = GROUPED && EW == 8;
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment by pointer arithmetic on the __shared__ array (not through an integer round trip),
    // so the compiler keeps the shared state space: staging-buffer accesses compile to STS/LDS, not to
    // generic ST/LD
    uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    uint8_t* staging = smem + STAGES * Cfg::kStageBytes;
    uint64_t* full = reinterpret_cast<uint64_t*>(staging + Cfg::kStaging);
    uint64_t* empty = full + STAGES;
    uint64_t* tfull = empty + STAGES;
    uint64_t* tempty = tfull + 2;
    uint64_t* xbar = tempty + 2;  // split-K: the partner's partial tile landed in shared memory
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(xbar + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    const int pair = static_cast<int>(cluster_id_x()), npairs = static_cast<int>(nclusters_x());
    const int num_units = p.num_tiles * p.split;
    // unit -> (tile, k range); see GemmParams::split
    // b: the problem of a batched launch (coordinate of the 4-D maps, stride index) -- or, GROUPED, the problem
    // index into grp_params / grp_maps (each of those a single problem, batch coordinate 0)
    struct Unit {
        int tile, b, mt, nt, kh, kb0, steps;
        int tw;  // columns per N tile (BN unless GROUPED: the problem's tile_w)
    };
    const int tiles_per_problem = p.m_tiles * p.n_tiles;
    auto unit_of = [&](int u) {
        Unit x;
        if constexpr (GROUPED) {
            int i = 0;
            while (i + 1 < p.group_n && u >= p.grp_tile_start[i + 1]) ++i;
            const GemmParams& q = p.grp_params[i];
            const int tl = u - p.grp_tile_start[i];
            x.tile = u;
            x.b = i;
            x.kh = 0;
            x.kb0 = 0;
            x.mt = tl / q.n_tiles;
            x.nt = tl - x.mt * q.n_tiles;
            x.steps = (q.k_blocks + KS - 1) / KS;
            x.tw = q.tile_w;
            return x;
        }
        x.tw = p.tile_w;  // BN, or balanced narrower tiles (runtime: short-K problems whose n fills its tiles)
        x.kh = (p.split == 2 && u < p.num_tiles) ? 1 : 0;
        x.tile = p.split == 2 && !x.kh ? u - p.num_tiles : u;
        x.b = x.tile / tiles_per_problem;
        const int tl = x.tile - x.b * tiles_per_problem;
        x.mt = tl / p.n_tiles;
        x.nt = tl - x.mt * p.n_tiles;
        x.kb0 = x.kh ? p.kb_half : 0;
        const int cnt = p.split == 2 ? (x.kh ? p.k_blocks - p.kb_half : p.kb_half) : p.k_blocks;
        x.steps = (cnt + KS - 1) / KS;
        return x;
    };
    // the unit's problem parameters, tensor maps and batch coordinate
    auto prm = [&](const Unit& x) -> const GemmParams& {
        if constexpr (GROUPED) return p.grp_params[x.b];
        return p;
    };
    auto map_a = [&](const Unit& x) -> const CUtensorMap* {
        if constexpr (GROUPED) return p.grp_maps + 3 * x.b;
        return &tmA;
    };
    auto map_b = [&](const Unit& x) -> const CUtensorMap* {
        if constexpr (GROUPED) return p.grp_maps + 3 * x.b + 1;
        return &tmB;
    };
    auto map_c = [&](const Unit& x) -> const CUtensorMap* {
        if constexpr (GROUPED) return p.grp_maps + 3 * x.b + 2;
        return &tmC;
    };
    auto bcoord = [&](const Unit& x) { return GROUPED ? 0 : x.b; };
#ifdef ABFT_TRACE_TILES  // (debug: per-tile timestamps, 8 per tile for the CTA's first 8 tiles: MMA start / end,
    // epilogue loop top / accumulator ready / chunks done / accumulator released / row verdicts / published)
    unsigned long long* const tt = p.trace ? p.trace + 64ull * blockIdx.x : nullptr;
    unsigned long long* trace = nullptr;
#else
    unsigned long long* trace = p.trace ? p.trace + 16ull * blockIdx.x : nullptr;
#endif
    if (trace && threadIdx.x == 0) trace[0] = globaltimer();

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], Cfg::kProducers);  // one expect_tx arrival per producer warp (leader)
            mbar_init(&empty[s], 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(&tfull[a], 1);
            mbar_init(&tempty[a], TILE_ALT ? 2 * 4 : 2 * Cfg::kEpiWarps);  // draining epilogue warps x 2 CTAs
        }
        mbar_init(xbar, 1);
        fence_mbar_init();
    }
    if (warp == 0 && lane == 0) {
        griddep_launch_dependents();  // the next kernel's prologue may overlap this grid
        if constexpr (GROUPED) {  // the maps of this pair's first problem
            if (pair < num_units) {
                const Unit x0 = unit_of(pair);
                tma_prefetch(map_a(x0));
                tma_prefetch(map_b(x0));
                if (EPI == kEpiTmaStore) tma_prefetch(map_c(x0));
            }
        } else {
            tma_prefetch(&tmA);
            tma_prefetch(&tmB);
            if (EPI == kEpiTmaStore) tma_prefetch(&tmC);
        }
    }
    // Barriers must be visible to the peer before any TMA / commit targets them; TMEM is allocated
    // afterwards by the MMA warp so the producer's first loads overlap the allocation.
    cluster_sync();
    if (trace && threadIdx.x == 0) trace[1] = globaltimer();
    // warm L2 with this pair's first stages while the previous grid finishes (before griddep_wait:
    // prefetches only touch L2, the point of coherence); one producer warp per operand part
    const bool is_producer = warp == 0 || (warp >= 6 && warp < Cfg::kEpiG1);
    const bool is_epi = (warp >= 2 && warp <= 5) || warp >= Cfg::kEpiG1;
    if (is_producer && lane == 0 && pair < num_units) {
        const int role = warp == 0 ? 0 : warp - 5;
        const Unit x = unit_of(pair);
        const GemmParams& q = prm(x);
        const int pre = x.steps < STAGES ? x.steps : STAGES;
        const int rot = x.nt % x.steps;
        for (int ks0 = 0; ks0 < pre; ++ks0) {
            const int kb = x.kb0 + ((ks0 + rot) % x.steps) * KS;
            if (role < Cfg::NA && q.a_exact)
                tma_prefetch_l2_3d(map_a(x), (kb + role * (KS / Cfg::NA)) * kBK, x.mt * kPairM + static_cast<int>(rank) * kBM,
                                   bcoord(x));
            else if (role < Cfg::NA)
                tma_prefetch_l2_4d(map_a(x), 0, x.mt * kPairM + static_cast<int>(rank) * kBM, kb + role * (KS / Cfg::NA),
                                   bcoord(x));
            else
                tma_prefetch_l2_4d(map_b(x), 0, x.nt * x.tw + static_cast<int>(rank) * (x.tw / 2),
                                   kb + (role - Cfg::NA) * (KS / Cfg::NB), q.b_shared ? 0 : bcoord(x));
        }
    }
    uint32_t tmem = 0;
    if (warp == 1 || is_epi) {
        if (warp == 1) {
            tmem_alloc_pair<Cfg::kTmemCols>(tmem_holder);
            tc_fence_before();
        }
        named_bar_sync(2, 32 * (1 + Cfg::kEpiWarps));  // MMA warp + epilogue warps
        tc_fence_after();
        tmem = *tmem_holder;
    }

    // Everything above is independent of the preceding kernel's results; from here on global memory is
    // read and written (PDL: blocks until the previous grid on the stream has completed).
    griddep_wait();

    if (CHECKED && p.gemv_helpers && pair >= num_units) {
        // ---------------- idle pair: checksum-column GEMV for every row (see gemv_helper)
        gemv_helper(p, (pair - num_units) * 2 + static_cast<int>(rank), (npairs - num_units) * 2);
    } else if (is_producer) {
        // ---------------- TMA producers (both CTAs; completion counted on the leader's barrier). An SM
        // serves the TMA requests of ONE issuing warp one after another (~275-300 ns each under load,
        // scripts/pipe_bench9.cu), so the stage is split over three warps issuing in parallel:
        // A k-blocks [0, KS/2), A k-blocks [KS/2, KS), and the B' slab.
        if (lane == 0) {
            const int role = warp == 0 ? 0 : warp - 5;  // [0, NA): A k-block groups; [NA, NA+NB): B' groups
            const uint64_t pol = policy_evict_last();   // A is re-read by every N tile, B' by every call
            constexpr int KA = KS / Cfg::NA, KB = KS / Cfg::NB;
            const bool is_a = role < Cfg::NA;
            const int grp = is_a ? role : role - Cfg::NA;
            const uint32_t bytes = is_a ? KA * Cfg::kABytes : KB * Cfg::kBBytes;
            int it = 0;
            for (int u = pair; u < num_units; u += npairs) {
                const Unit x = unit_of(u);
                const GemmParams& q = prm(x);
                const CUtensorMap* mA = map_a(x);
                const CUtensorMap* mB = map_b(x);
                const int bc = bcoord(x);
                if constexpr (GROUPED) {
                    // A streams from HBM once per problem row block here (few N tiles share it): warm L2 with the
                    // whole slab of this unit (first unit) and of the next one in long per-row runs (1 KB boxes of
                    // the prefetch view grp_maps[3 * group_n + i]) -- DRAM-friendlier than the mainloop's 128-byte
                    // k-block pieces, and a unit ahead of them
                    if (rank == 0 && role == 0 && p.grp_apf) {
                        auto warm = [&](const Unit& y) {
                            const GemmParams& qy = prm(y);
                            const CUtensorMap* mp = p.grp_maps + 3 * p.group_n + y.b;
                            for (int c0 = 0; c0 < qy.k / 4; c0 += 256) tma_prefetch_l2_2d(mp, c0, y.mt * kPairM);
                        };
                        if (u == pair) warm(x);
                        if (u + npairs < num_units) warm(unit_of(u + npairs));
                    }
                }
                // Tiles of one M block read the same A rows; starting each tile at a different K step
                // spreads those reads over all of A's L2 lines instead of hammering one k-block's lines
                // (integer accumulation is exact, so the K order does not change the result).
                const int rot = x.nt % x.steps;
                // GROUPED: the problem's B' map boxes exactly the tw / 2 rows of this CTA's half tile (k-blocks land
                // tw / 2 * 128 bytes apart), so narrow tiles do not pull a full BN / 2-row slab through L2
                const uint32_t b_kstride = GROUPED ? static_cast<uint32_t>(x.tw / 2) * kBK : Cfg::kBBytes;
                const uint32_t tx_bytes = (GROUPED && !is_a) ? KB * b_kstride : bytes;
                for (int ks0 = 0; ks0 < x.steps; ++ks0, ++it) {
                    const int ks = ks0 + rot < x.steps ? ks0 + rot : ks0 + rot - x.steps;
                    const int kb = x.kb0 + ks * KS;
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    mbar_wait(&empty[s], ph ^ 1);
                    uint8_t* st = smem + s * Cfg::kStageBytes;
                    if (rank == 0) mbar_arrive_expect_tx(&full[s], 2 * tx_bytes);
                    if (is_a && q.a_exact) {
#pragma unroll
                        for (int qq = 0; qq < KA; ++qq)  // exact-extent view: one k-block per request
                            tma_load_3d_pair(st + (grp * KA + qq) * Cfg::kABytes, mA, &full[s], (kb + grp * KA + qq) * kBK,
                                             x.mt * kPairM + static_cast<int>(rank) * kBM, bc, pol);
                    } else if (is_a)
                        tma_load_4d_pair(st + grp * KA * Cfg::kABytes, mA, &full[s], 0,
                                         x.mt * kPairM + static_cast<int>(rank) * kBM, kb + grp * KA, bc, pol);
                    else
                        tma_load_4d_pair(st + KS * Cfg::kABytes + grp * KB * b_kstride, mB, &full[s], 0,
                                         x.nt * x.tw + static_cast<int>(rank) * (x.tw / 2), kb + grp * KB,
                                         q.b_shared ? 0 : bc, pol);
                }
            }
        }
    } else if (warp == 1) {
        // ---------------- MMA issuer: leader CTA, one thread, for the whole pair
        if (rank == 0 && lane == 0) {
            int it = 0, local = 0;
            for (int u = pair; u < num_units; u += npairs, ++local) {
                const Unit xu = unit_of(u);
                const int steps = xu.steps;
                // the MMA's N is the tile width: the pair's B' slabs hold tw / 2 rows each that matter
                const uint32_t idesc = idesc_u8s8(kPairM, static_cast<uint32_t>(xu.tw));
                const uint32_t b_kstride = GROUPED ? static_cast<uint32_t>(xu.tw / 2) * kBK : Cfg::kBBytes;
                const int acc = local & 1;
                const uint32_t aph = (local >> 1) & 1;
#ifdef ABFT_TRACE_STEADY  // (debug: steady-state tile 8: how long the MMA waits for its accumulator)
                if (trace && local == 8) trace[11] = globaltimer();
#endif
                mbar_wait(&tempty[acc], aph ^ 1);
#ifdef ABFT_TRACE_TILES
                if (tt && local < 8) tt[8 * local] = globaltimer();
#endif
#ifdef ABFT_TRACE_STEADY
                if (trace && local == 8) trace[12] = globaltimer();
#endif
                tc_fence_after();
                const uint32_t d = tmem + static_cast<uint32_t>(acc * BN);
                for (int ks = 0; ks < steps; ++ks, ++it) {
                    const int s = it % STAGES;
                    const uint32_t ph = (it / STAGES) & 1;
                    mbar_wait(&full[s], ph);
                    tc_fence_after();
                    if (trace && local == 0 && ks == 0) trace[2] = globaltimer();
#ifndef ABFT_TRACE_STEADY
                    if (trace && local == 0 && ks >= 1 && ks <= 3) trace[8 + ks] = globaltimer();  // stage arrivals
#endif
                    const uint32_t a0 = smem_u32(smem + s * Cfg::kStageBytes);
                    const uint32_t b0 = a0 + KS * Cfg::kABytes;
#pragma unroll
                    for (int j = 0; j < KS; ++j) {
                        const uint64_t da = umma_desc_sw128(a0 + j * Cfg::kABytes);
                        const uint64_t db = umma_desc_sw128(b0 + j * b_kstride);
#pragma unroll
                        for (int kk = 0; kk < kBK / 32; ++kk) {  // UMMA K = 32 bytes for 8-bit operands
#ifndef ABFT_NO_MMA  // (experiment switch: pure load pipeline)
                            mma_i8_pair(d, da + 2 * kk, db + 2 * kk, idesc, (ks | j | kk) != 0 ? 1u : 0u);
#endif
                        }
                    }
                    mma_commit_pair(&empty[s]);  // frees the slot in both CTAs once these MMAs read it
                }
                mma_commit_pair(&tfull[acc]);  // accumulator complete, both CTAs' epilogues may read
#ifdef ABFT_TRACE_TILES
                if (tt && local < 8) tt[8 * local + 1] = globaltimer();
#endif
                if (trace && local == 0) trace[3] = globaltimer();
            }
        }
    } else {
        // ---------------- epilogue: warps 2..5, thread <-> one row of this CTA's 128-row half
        const int q = warp & 3;                  // TMEM lane quarter this warp may access
        const int eg = warp >= Cfg::kEpiG1 ? 1 : 0;  // epilogue group: chunks c = eg, eg + kEpiGroups, ...
        const int eslot = eg * 4 + q;                // this warp's staging buffers
        const uint32_t tempty_leader = mapa_shared(smem_u32(tempty), 0);
        int local = 0, chunk_ctr = 0;
        for (int u = pair; u < num_units; u += npairs, ++local) {
            if (TILE_ALT && (local & 1) != eg) continue;  // the other group's tile
#ifdef ABFT_TRACE_TILES
            if (tt && local < 8 && (threadIdx.x == 64 || threadIdx.x == 32 * Cfg::kEpiG1)) tt[8 * local + 2] = globaltimer();
#endif
            const Unit x = unit_of(u);
            const int mt = x.mt, nt = x.nt;
            const GemmParams& pq = prm(x);  // this tile's problem (the launch's own fields unless GROUPED)
            const int bb = bcoord(x);
            // the tile's hot fields in registers (GROUPED: the problem's parameters live in global memory and would be
            // re-read after every memory clobber of the chunk loop)
            const int pn = pq.n, pm = pq.m;
            const int64_t pldc = pq.ldc;
            uint8_t* const prq = pq.rq_out;
            const int acc = local & 1;
            const uint32_t aph = (local >> 1) & 1;
            const int row0 = mt * kPairM + static_cast<int>(rank) * kBM + q * 32;  // first row of this warp
            const int row = row0 + lane;
            // This tile's share of the checksum column C'[row][n] = sum_p A[row][p]*cs[p]: K blocks
            // [kb0, kb1) of the GEMV, read from global while the tensor cores run the mainloop.
            uint32_t cs_part = 0;
            if (CHECKED && x.kh == 0 && !p.gemv_helpers && !pq.cs_mma) {
                const int t0 = static_cast<int>(static_cast<long long>(nt) * pq.k_blocks / pq.n_tiles);
                const int t1 = static_cast<int>(static_cast<long long>(nt + 1) * pq.k_blocks / pq.n_tiles);
                const int kb0 = TILE_ALT ? t0 : t0 + (t1 - t0) * eg / Cfg::kEpiGroups;  // the groups split the tile's share
                const int kb1 = TILE_ALT ? t1 : t0 + (t1 - t0) * (eg + 1) / Cfg::kEpiGroups;
                if (kb1 > kb0 && row < pm) cs_part = csum_share(pq, bb, row, kb0 * kBK, min(kb1 * kBK, pq.k));
            }
            mbar_wait(&tfull[acc], aph);
            tc_fence_after();
#ifdef ABFT_TRACE_TILES
            if (tt && local < 8 && (threadIdx.x == 64 || threadIdx.x == 32 * Cfg::kEpiG1)) tt[8 * local + 3] = globaltimer();
#endif
            if (trace && local == 0 && threadIdx.x == 64) trace[4] = globaltimer();
#ifdef ABFT_TRACE_STEADY
            if (trace && local == 8 && threadIdx.x == 64) trace[9] = globaltimer();
#endif
            const int tw = x.tw;
            const int n0 = nt * tw;
            const uint32_t t_row = tmem + (static_cast<uint32_t>(q * 32) << 16) + static_cast<uint32_t>(acc * BN);
            // split-K exchange slot of this CTA's half tile (BN*128 int32): [BN/32 chunks][8 column quads]
            // [128 rows][4], so a warp moves 512 contiguous bytes per 16-byte access, in global memory (the
            // upper-K unit's stores) and in shared memory (the lower-K unit's conflict-free reads)
            const int64_t part_base = (static_cast<int64_t>(x.tile) * 2 + rank) * (BN * kBM);
            uint32_t* pflag = p.split == 2 ? p.part_flag + x.tile * 2 + rank : nullptr;
            const int prow = q * 32 + lane;
            if (x.kh == 1) {
                // upper-K unit: publish the partial tile through L2 and hand the tile to its partner
                uint4* part = reinterpret_cast<uint4*>(p.partial + part_base);
#pragma unroll 1
                for (int c = eg; c < BN / 32; c += Cfg::kEpiGroups) {
                    uint32_t v[32];
                    tmem_ld_32x32b_x32(t_row + c * 32, v);
                    tmem_wait_ld();
#pragma unroll
                    for (int j4 = 0; j4 < 8; ++j4)
                        part[(c * 8 + j4) * kBM + prow] = make_uint4(v[4 * j4], v[4 * j4 + 1], v[4 * j4 + 2], v[4 * j4 + 3]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if (rank == 0)
                        mbar_arrive_local(&tempty[acc]);
                    else
                        mbar_arrive_cluster(tempty_leader + static_cast<uint32_t>(acc * 8));
                }
                __threadfence();
                named_bar_sync(1, 32 * Cfg::kEpiWarps);
                if (threadIdx.x == 64) {
                    st_release_gpu(pflag, 1u);
                    if (trace) trace[14] = globaltimer();
                }
                continue;
            }
            const uint4* spart = nullptr;
            if (p.split == 2) {
                // lower-K unit: wait for the partner's partial (it was scheduled first and never waits),
                // then pull it into the now idle pipeline buffers with bulk copies (one L2 round trip)
                if (threadIdx.x == 64) {
                    while (ld_acquire_gpu(pflag) == 0u) {
                    }
                    if (trace) trace[12] = globaltimer();
                    fence_proxy_async_global();
                    constexpr uint32_t kBytes = BN * kBM * 4;
                    mbar_arrive_expect_tx(xbar, kBytes);
                    const uint8_t* src = reinterpret_cast<const uint8_t*>(p.partial + part_base);
#pragma unroll
                    for (uint32_t o = 0; o < kBytes; o += 16384) bulk_load_1d(smem + o, src + o, 16384, xbar);
                }
                mbar_wait(xbar, 0);  // one split unit per CTA (units <= pairs), so phase 0
                if (trace && threadIdx.x == 64) trace[13] = globaltimer();
                spart = reinterpret_cast<const uint4*>(smem);
            }
            bool fault_here = false;  // some injected fault hits a data column of this row
            for (int f = 0; f < pq.nfaults; ++f)
                fault_here |= bb == pq.fault_b[f] && row == pq.fault_row[f] && pq.fault_col[f] < pn;
            int32_t* const cb = pq.c + bb * pq.c_bstride;  // this problem's C
            long long rsum = 0;
            // columns whose int32 sum cannot overflow (|C'| <= 255 * 128 * k): the row sum of a chunk is then plain
            // 32-bit adds (3-input IADD3) instead of a 64-bit tree
            const int sum32 = pq.k <= 2056 ? 32 : pq.k <= 4112 ? 16 : 0;
            // One 32-column chunk of this warp's rows, already in registers.
            auto chunk = [&](const int c, uint32_t (&v)[32]) {
                const int col0 = n0 + c * 32;
                if (spart != nullptr) {
#pragma unroll
                    for (int j4 = 0; j4 < 8; ++j4) {
                        const uint4 w = spart[(c * 8 + j4) * kBM + prow];
                        v[4 * j4] += w.x;
                        v[4 * j4 + 1] += w.y;
                        v[4 * j4 + 2] += w.z;
                        v[4 * j4 + 3] += w.w;
                    }
                }
                if (fault_here) {
                    for (int f = 0; f < pq.nfaults; ++f) {
                        if (bb != pq.fault_b[f] || row != pq.fault_row[f]) continue;
                        const int fc = pq.fault_col[f];
                        const uint32_t fm = 1u << pq.fault_bit[f];
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (fc == col0 + j) v[j] ^= fm;
                    }
                }
                if (prq != nullptr && row < pm) {
                    // fused requantization of this row's 32 columns (the checksum column is never part
                    // of C, so it is excluded by construction), after any injected C' fault
                    const RequantConsts rk = requant_consts(pq.rq);
                    const int32_t rsa = pq.rq_row_sum_a[row];
                    const RequantFast rf = requant_fast(rk, rsa);  // (two FMAs per element; exact path near a boundary)
                    uint32_t pk[8];
#pragma unroll
                    for (int q4 = 0; q4 < 8; ++q4) pk[q4] = 0u;
                    // the chunk's 32 column sums first (vector loads when the array allows), then one straight-line pass
                    // over the columns -- no per-column branch, so the 32 independent chains interleave; columns past n
                    // run on zeros and are never stored
                    int32_t csv[32];
                    const int32_t* const csp = pq.rq_col_sum_b + col0;
                    if (col0 + 32 <= pn && (reinterpret_cast<uintptr_t>(csp) & 15) == 0) {
#pragma unroll
                        for (int j4 = 0; j4 < 8; ++j4) {
                            const int4 t4 = __ldg(reinterpret_cast<const int4*>(csp) + j4);
                            csv[4 * j4] = t4.x;
                            csv[4 * j4 + 1] = t4.y;
                            csv[4 * j4 + 2] = t4.z;
                            csv[4 * j4 + 3] = t4.w;
                        }
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j) csv[j] = col0 + j < pn ? __ldg(csp + j) : 0;
                    }
                    uint32_t need = 0u;  // columns that take the reference-order sequence (near a rounding boundary)
#pragma unroll
                    for (int j = 0; j < 32; ++j) {  // fully unrolled: v[] and pk[] must stay in registers
                        bool exact;
                        pk[j >> 2] |= requant_try_fast(static_cast<int32_t>(v[j]), csv[j], rf, exact) << (8 * (j & 3));
                        need |= exact ? 1u << j : 0u;
                    }
                    if (col0 + 32 > pn) need &= (1u << (pn - col0)) - 1u;  // (1 <= pn - col0 < 32 here)
                    if (need != 0u) {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if ((need >> j) & 1u)
                                pk[j >> 2] = (pk[j >> 2] & ~(0xFFu << (8 * (j & 3)))) |
                                             (requant_one_cold(static_cast<int32_t>(v[j]), rsa, csv[j], rk.m1, rk.m2, rk.m3, rk.t4,
                                                               rk.bC, rk.sC)
                                              << (8 * (j & 3)));
                    }
                    uint8_t* dst = prq + static_cast<int64_t>(row) * pq.rq_ld + col0;
                    if (col0 + 32 <= pn && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
                        reinterpret_cast<uint4*>(dst)[0] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
                        reinterpret_cast<uint4*>(dst)[1] = make_uint4(pk[4], pk[5], pk[6], pk[7]);
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (col0 + j < pn) dst[j] = static_cast<uint8_t>(pk[j >> 2] >> (8 * (j & 3)));
                    }
                }
#ifdef ABFT_TRACE_CHUNKS
                if (trace && local == 0 && threadIdx.x == 64 && c == 0) trace[9] = globaltimer();
#endif
                if constexpr (CHECKED) {
                    if (col0 + 32 <= pn && sum32 == 32) {
                        int32_t t[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            t[j] = static_cast<int32_t>(v[4 * j]) + static_cast<int32_t>(v[4 * j + 1]) +
                                   static_cast<int32_t>(v[4 * j + 2]) + static_cast<int32_t>(v[4 * j + 3]);
                        rsum += ((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]));
                    } else if (col0 + 32 <= pn && sum32 == 16) {
                        int32_t t[8];
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            t[j] = static_cast<int32_t>(v[4 * j]) + static_cast<int32_t>(v[4 * j + 1]) +
                                   static_cast<int32_t>(v[4 * j + 2]) + static_cast<int32_t>(v[4 * j + 3]);
                        rsum += static_cast<long long>((t[0] + t[1]) + (t[2] + t[3])) + ((t[4] + t[5]) + (t[6] + t[7]));
                    } else if (col0 + 32 <= pn) {
                        // pairwise tree: 5 dependent int64 adds instead of a 32-long carry chain (exact in
                        // any order: |sum| < 32 * 2^31)
                        long long t[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j)
                            t[j] = static_cast<long long>(static_cast<int32_t>(v[2 * j])) + static_cast<int32_t>(v[2 * j + 1]);
#pragma unroll
                        for (int w2 = 8; w2 > 0; w2 >>= 1)
#pragma unroll
                            for (int j = 0; j < w2; ++j) t[j] += t[j + w2];
                        rsum += t[0];
                    } else {
#pragma unroll
                        for (int j = 0; j < 32; ++j)
                            if (col0 + j < pn) rsum += static_cast<int32_t>(v[j]);
                    }
                }
                if constexpr (EPI == kEpiTmaStore) {
                    constexpr int NB = Cfg::kStagingBufs;
                    uint8_t* buf = staging + (eslot * NB + (chunk_ctr % NB)) * 4096;
                    if (chunk_ctr >= NB) {
                        if (lane == 0) bulk_wait_read<NB - 1>();
                        __syncwarp();
                    }
#pragma unroll
                    for (int qq = 0; qq < 8; ++qq)
                        *reinterpret_cast<uint4*>(buf + lane * 128 + ((qq ^ (lane & 7)) << 4)) =
                            make_uint4(v[4 * qq], v[4 * qq + 1], v[4 * qq + 2], v[4 * qq + 3]);
#ifdef ABFT_TRACE_CHUNKS
                    if (trace && local == 0 && threadIdx.x == 64 && c == 0) trace[10] = globaltimer();
#endif
                    fence_proxy_async_smem();
                    __syncwarp();
#ifdef ABFT_TRACE_CHUNKS
                    if (trace && local == 0 && threadIdx.x == 64 && c == 0) trace[11] = globaltimer();
#endif
                    if (lane == 0) {
                        if (row0 < pm && col0 < pn) tma_store_3d(map_c(x), buf, col0, row0, bb);
                        bulk_commit();
                    }
                    ++chunk_ctr;
                } else if constexpr (EPI == kEpiStg) {
                    // transpose the warp's 32x32 chunk through its staging buffer so every store
                    // instruction writes four full 128-byte row segments
                    uint8_t* buf = staging + eslot * Cfg::kStagingBufs * 4096;
#pragma unroll
                    for (int qq = 0; qq < 8; ++qq)
                        *reinterpret_cast<uint4*>(buf + lane * 128 + ((qq ^ (lane & 7)) << 4)) =
                            make_uint4(v[4 * qq], v[4 * qq + 1], v[4 * qq + 2], v[4 * qq + 3]);
                    __syncwarp();
                    const int rsub = lane >> 3, cq = lane & 7;
                    const int gcol = col0 + cq * 4;
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int r = i * 4 + rsub;
                        const uint4 val = *reinterpret_cast<const uint4*>(buf + r * 128 + ((cq ^ (r & 7)) << 4));
                        const int grow = row0 + r;
                        if (grow < pm && gcol < pn) {
                            int32_t* dst = cb + static_cast<int64_t>(grow) * pldc + gcol;
                            if (gcol + 3 < pn) {
                                *reinterpret_cast<uint4*>(dst) = val;
                            } else {
                                const uint32_t e4[4] = {val.x, val.y, val.z, val.w};
                                for (int e = 0; e < 4 && gcol + e < pn; ++e) dst[e] = static_cast<int32_t>(e4[e]);
                            }
                        }
                    }
                    __syncwarp();
                } else if constexpr (EPI == kEpiDirect) {
                    // straight from the registers (no shared-memory staging, whose traffic competes with the
                    // mainloop's operand reads): 16-byte stores when the row segment is aligned
                    if (row < pm) {
                        int32_t* crow = cb + static_cast<int64_t>(row) * pldc + col0;
                        if (col0 + 32 <= pn && (reinterpret_cast<uintptr_t>(crow) & 31) == 0) {
#pragma unroll
                            for (int q8 = 0; q8 < 4; ++q8)  // 32-byte stores: full sectors (STG.256)
                                asm volatile("st.global.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(crow + 8 * q8),
                                             "r"(v[8 * q8]), "r"(v[8 * q8 + 1]), "r"(v[8 * q8 + 2]), "r"(v[8 * q8 + 3]),
                                             "r"(v[8 * q8 + 4]), "r"(v[8 * q8 + 5]), "r"(v[8 * q8 + 6]), "r"(v[8 * q8 + 7])
                                             : "memory");
                        } else if (col0 + 32 <= pn && (reinterpret_cast<uintptr_t>(crow) & 15) == 0) {
#pragma unroll
                            for (int q4 = 0; q4 < 8; ++q4)
                                reinterpret_cast<uint4*>(crow)[q4] =
                                    make_uint4(v[4 * q4], v[4 * q4 + 1], v[4 * q4 + 2], v[4 * q4 + 3]);
                        } else {
#pragma unroll
                            for (int j = 0; j < 32; ++j)
                                if (col0 + j < pn) crow[j] = static_cast<int32_t>(v[j]);
                        }
                    }
                }
            };
            // Chunks c = eg, eg + groups, ...: the TMEM load of the next chunk is in flight while the current one is
            // reduced, staged and stored (two register buffers; tcgen05.wait::ld waits for every load issued, so the
            // next load is issued right after the wait that completes the current one).
            {
                constexpr int G = TILE_ALT ? 1 : Cfg::kEpiGroups;
                uint32_t va[32], vb[32];
                int c = TILE_ALT ? 0 : eg;
                // (a warp whose 32 rows all lie past m -- small-m problems in 256-row tiles -- has nothing to drain)
                auto live = [&](int cc) { return row0 < pm && cc * 32 < tw && n0 + cc * 32 < pn; };  // warp-uniform
                if constexpr (Cfg::kThreads <= 256) {
                    if (live(c)) tmem_ld_32x32b_x32(t_row + c * 32, va);
#pragma unroll 1
                    while (live(c)) {
                        tmem_wait_ld_tie(va);
                        if (live(c + G)) tmem_ld_32x32b_x32(t_row + (c + G) * 32, vb);
                        chunk(c, va);
                        c += G;
                        if (!live(c)) break;
                        tmem_wait_ld_tie(vb);
                        if (live(c + G)) tmem_ld_32x32b_x32(t_row + (c + G) * 32, va);
                        chunk(c, vb);
                        c += G;
                    }
                } else {  // (384 threads: 168 registers per thread, one chunk buffer)
#pragma unroll 1
                    for (; live(c); c += G) {
                        tmem_ld_32x32b_x32(t_row + c * 32, va);
                        tmem_wait_ld();
                        chunk(c, va);
                    }
                }
            }
#ifdef ABFT_TRACE_TILES
            if (tt && local < 8 && (threadIdx.x == 64 || threadIdx.x == 32 * Cfg::kEpiG1)) tt[8 * local + 4] = globaltimer();
#endif
            if constexpr (CHECKED) {
                // C'[row][n] = A*cs computed by the tensor cores (B' column n) when this tile covers column n
                if (pq.cs_mma && (TILE_ALT || eg == 0) && n0 <= pn && pn < n0 + tw) {
                    cs_part = tmem_ld_32x32b_x1(t_row + static_cast<uint32_t>(pn - n0));
                    tmem_wait_ld();
                }
            }
            if (trace && local == 0 && threadIdx.x == 64) trace[7] = globaltimer();
#ifdef ABFT_TRACE_STEADY
            if (trace && local == 8 && threadIdx.x == 64) trace[10] = globaltimer();
            if (trace && local == 9 && threadIdx.x == 64) trace[13] = globaltimer();
#endif
            if (pflag != nullptr && threadIdx.x == 64) *pflag = 0u;  // self-resetting for the next call
            // accumulator drained: let the MMA warp reuse it
            tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (rank == 0)
                    mbar_arrive_local(&tempty[acc]);
                else
                    mbar_arrive_cluster(tempty_leader + static_cast<uint32_t>(acc * 8));
            }
#ifdef ABFT_TRACE_TILES
            if (tt && local < 8 && (threadIdx.x == 64 || threadIdx.x == 32 * Cfg::kEpiG1)) tt[8 * local + 5] = globaltimer();
#endif
            if constexpr (CHECKED) {
                // mod is a ring homomorphism: the residue of the int64 row sum equals the sum of the
                // per-tile residues mod 127 (P:src/gemm_abft.cpp:119-122 reduces the row sum once).
                // One 64-bit atomic per row carries this tile's GEMV share, one arrival and its residue
                // (kRowAcc* layout). Atomics on one address are totally ordered, so the thread that
                // brings arrival n_tiles holds the complete row and finalizes it -- no fences, no
                // counters, no second pass.
                int fin = 0, flag = 0;
                if (row < pm)
                    row_arrive(pq, bb, row,
                               (static_cast<unsigned long long>(p.gemv_helpers ? 0u : cs_part) << 32) |
                                   (1ull << kRowAccCountShift) | static_cast<unsigned long long>(mod127(rsum)),
                               fin, flag);
                if (trace && local == 0 && threadIdx.x == 64) trace[8] = globaltimer();
#ifdef ABFT_TRACE_TILES
                if (tt && local < 8 && (threadIdx.x == 64 || threadIdx.x == 32 * Cfg::kEpiG1)) tt[8 * local + 6] = globaltimer();
#endif
                if (!GROUPED && p.req_rows > 0)
                    warp_publish_stacked(p, row, fin, flag);
                else
                    warp_publish(pq, bb, fin, flag);
            }
#ifdef ABFT_TRACE_TILES
            if (tt && local < 8 && (threadIdx.x == 64 || threadIdx.x == 32 * Cfg::kEpiG1)) tt[8 * local + 7] = globaltimer();
#endif
        }
        if constexpr (EPI == kEpiTmaStore) {
            if (lane == 0) bulk_wait<0>();
            __syncwarp();
        }
        if (trace && threadIdx.x == 64) trace[5] = globaltimer();
    }
#ifdef ABFT_TRACE_ROLES  // (debug: when each non-epilogue warp reaches the final cluster barrier)
    if (trace && lane == 0 && (warp == 0 || warp == 1 || (warp >= 6 && warp <= 7)))
        trace[warp == 0 ? 9 : warp == 1 ? 10 : warp == 6 ? 11 : 12] = globaltimer();
#endif
    tc_fence_before();
#ifdef ABFT_END_RELAXED
    cluster_sync_relaxed();
#else
    cluster_sync();
#endif
    if (trace && threadIdx.x == 0) trace[6] = globaltimer();
    if (warp == 1) {
        tc_fence_after();
        tmem_dealloc_pair<Cfg::kTmemCols>(tmem);
    }
}

// ============================================================ standalone verify
// One warp per row: int64 row sum over the first n columns, compared mod 127 with csum[row].
// Flag count is reduced through a self-resetting workspace (last block publishes).
__global__ void __launch_bounds__(256) verify_kernel(const int32_t* __restrict__ c, int64_t ldc,
                                                     const int32_t* __restrict__ csum, int64_t csum_ld,
                                                     int64_t m, int64_t n, uint8_t* __restrict__ flags,
                                                     uint32_t* err_count, uint32_t* ws_acc, uint32_t* ws_blocks) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    __shared__ uint32_t block_count;
    __shared__ uint32_t is_last;
    if (threadIdx.x == 0) block_count = 0;
    __syncthreads();
    for (int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + warp; row < m; row += static_cast<int64_t>(gridDim.x) * 8) {
        const int32_t* crow = c + row * ldc;
        long long s = 0;
        for (int64_t j = lane; j < n; j += 32) s += crow[j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            const int flag = mod127(s) != mod127(csum[row * csum_ld]);
            if (flags) flags[row] = static_cast<uint8_t>(flag);
            if (flag) atomicAdd(&block_count, 1u);
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        if (block_count) atomicAdd(ws_acc, block_count);
        __threadfence();
        is_last = atomicAdd(ws_blocks, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (is_last && threadIdx.x == 0) {
        __threadfence();
        const uint32_t total = atomicExch(ws_acc, 0u);
        if (err_count) *err_count = total;
        atomicExch(ws_blocks, 0u);
    }
}

// ============================================================ host launchers
template <int BN, bool CHECKED, int EPI, int EW, bool GROUPED = false>
static cudaError_t launch_one(int pairs, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                              const GemmParams& p, cudaStream_t st) {
    using Cfg = PairCfg<BN, EW>;
    auto kern = gemm_pair_kernel<BN, CHECKED, EPI, EW, GROUPED>;
    static bool attr_done[kMaxDevices] = {};  // per device; benign race: idempotent attribute set
    const int dev = current_device();
    if (!attr_done[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
        if (e != cudaSuccess) return e;
        attr_done[dev] = true;
    }
    static const bool pdl = std::getenv("ABFTLP_NO_PDL") == nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * pairs);
    cfg.blockDim = dim3(Cfg::kThreads);
    cfg.dynamicSmemBytes = Cfg::kSmemBytes;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, a, b, c, p);
}

template <int BN, bool CHECKED>
static cudaError_t launch_epi(int epi, int ew, int pairs, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& c,
                              const GemmParams& p, cudaStream_t st) {
    switch (epi) {
        case kEpiTmaStore:  // 8 epilogue warps only with the TMA-store epilogue (short-K batched problems)
            return ew == 8 ? launch_one<BN, CHECKED, kEpiTmaStore, 8>(pairs, a, b, c, p, st)
                           : launch_one<BN, CHECKED, kEpiTmaStore, 4>(pairs, a, b, c, p, st);
        case kEpiNone:  // (requantized output only: 8 epilogue warps, the requantization is the long side of the tile)
            if constexpr (CHECKED)
                if (ew == 8) return launch_one<BN, true, kEpiNone, 8>(pairs, a, b, c, p, st);
            return launch_one<BN, CHECKED, kEpiNone, 4>(pairs, a, b, c, p, st);
        case kEpiStg: return launch_one<BN, CHECKED, kEpiStg, 4>(pairs, a, b, c, p, st);
        default: return launch_one<BN, CHECKED, kEpiDirect, 4>(pairs, a, b, c, p, st);
    }
}

cudaError_t launch_gemm_kernel(int bn, bool checked, int epi, int ew, int pairs, const CUtensorMap& a, const CUtensorMap& b,
                               const CUtensorMap& c, const GemmParams& p, cudaStream_t st) {
    if (checked) {
        if (bn == 256) return launch_epi<256, true>(epi, ew, pairs, a, b, c, p, st);
        if (bn == 128) return launch_epi<128, true>(epi, ew, pairs, a, b, c, p, st);
        return launch_epi<64, true>(epi, ew, pairs, a, b, c, p, st);
    }
    if (bn == 256) return launch_epi<256, false>(epi, ew, pairs, a, b, c, p, st);
    if (bn == 128) return launch_epi<128, false>(epi, ew, pairs, a, b, c, p, st);
    return launch_epi<64, false>(epi, ew, pairs, a, b, c, p, st);
}

// Heterogeneous grouped launch (GemmParams::group_n problems; tensor maps in p.grp_maps): TMA-store or direct
// epilogue, 4 epilogue warps.
template <int BN, bool CHECKED>
static cudaError_t launch_grouped_bn(int epi, int ew, int pairs, const GemmParams& p, cudaStream_t st) {
    CUtensorMap none;
    std::memset(&none, 0, sizeof(none));
    if (epi == kEpiTmaStore && ew == 8) return launch_one<BN, CHECKED, kEpiTmaStore, 8, true>(pairs, none, none, none, p, st);
    if (epi == kEpiTmaStore) return launch_one<BN, CHECKED, kEpiTmaStore, 4, true>(pairs, none, none, none, p, st);
    if (epi == kEpiStg) return launch_one<BN, CHECKED, kEpiStg, 4, true>(pairs, none, none, none, p, st);
    return launch_one<BN, CHECKED, kEpiDirect, 4, true>(pairs, none, none, none, p, st);
}
cudaError_t launch_gemm_grouped(int bn, bool checked, int epi, int ew, int pairs, const GemmParams& p, cudaStream_t st) {
    if (checked) {
        if (bn == 256) return launch_grouped_bn<256, true>(epi, ew, pairs, p, st);
        if (bn == 128) return launch_grouped_bn<128, true>(epi, ew, pairs, p, st);
        return launch_grouped_bn<64, true>(epi, ew, pairs, p, st);
    }
    if (bn == 256) return launch_grouped_bn<256, false>(epi, ew, pairs, p, st);
    if (bn == 128) return launch_grouped_bn<128, false>(epi, ew, pairs, p, st);
    return launch_grouped_bn<64, false>(epi, ew, pairs, p, st);
}

int gemm_ks(int bn) { return bn == 256 ? PairCfg<256>::KS : bn == 128 ? PairCfg<128>::KS : PairCfg<64>::KS; }
int gemm_box_a(int bn) {  // k-blocks per A request
    return bn == 256 ? PairCfg<256>::KS / PairCfg<256>::NA : bn == 128 ? PairCfg<128>::KS / PairCfg<128>::NA
                                                                    : PairCfg<64>::KS / PairCfg<64>::NA;
}
int gemm_box_b(int bn) {  // k-blocks per B' request
    return bn == 256 ? PairCfg<256>::KS / PairCfg<256>::NB : bn == 128 ? PairCfg<128>::KS / PairCfg<128>::NB
                                                                    : PairCfg<64>::KS / PairCfg<64>::NB;
}

cudaError_t launch_read_encoded(const GemmWeight& w, int8_t* out, cudaStream_t st) {
    int64_t blocks = (w.k * (w.n + 1) + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    read_encoded_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(w.bt, w.cs, w.k, w.n, w.n_pad, out);
    return cudaGetLastError();
}

cudaError_t launch_set_checksums(GemmWeight& w, const int8_t* src, cudaStream_t st) {
    set_checksums_kernel<<<static_cast<unsigned>((w.k + 255) / 256), 256, 0, st>>>(w.cs, src, w.k, w.bt, w.n, w.n_pad);
    return cudaGetLastError();
}

cudaError_t launch_encode_weight(const int8_t* b, int64_t k, int64_t n, int64_t ldb, GemmWeight& w, cudaStream_t st) {
    // column tiles of the tile encoder; beyond 2047 (n > 262 016) its 11-bit arrival field would overflow: such
    // weights, and handles without encoder scratch, take the one-block-per-row-slab encoder
    const int64_t col_tiles = (n + 127) / 128;
    if (!w.cs_acc || col_tiles >= (1 << (31 - kEncCountShift))) {
        encode_weight_kernel<<<static_cast<unsigned>(w.k_pad / 64), 256, 0, st>>>(b, k, n, ldb, w.bt, w.n_pad, w.cs);
        return cudaGetLastError();
    }
    const dim3 grid(static_cast<unsigned>(w.n_pad / 128), static_cast<unsigned>(w.k_pad / kBK));
    encode_tiles_kernel<<<grid, 256, 0, st>>>(b, k, n, ldb, w.bt, w.n_pad, w.cs_acc, w.cs, static_cast<int>(col_tiles));
    return cudaGetLastError();
}

cudaError_t launch_verify(const int32_t* c, int64_t ldc, const int32_t* csum, int64_t csum_ld, int64_t m, int64_t n,
                          uint8_t* flags, uint32_t* err_count, uint32_t* ws_acc, uint32_t* ws_blocks, cudaStream_t st) {
    int64_t blocks = (m + 7) / 8;
    if (blocks > 1184) blocks = 1184;
    if (blocks < 1) blocks = 1;
    verify_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(c, ldc, csum, csum_ld, m, n, flags, err_count, ws_acc,
                                                                ws_blocks);
    return cudaGetLastError();
}

}  // namespace abftk
