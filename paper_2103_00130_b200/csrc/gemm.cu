// ABFT int8 GEMM for sm_100a.
//
//   encode_weight_kernel  replaces compute_row_checksums + PackedEncodedWeight
//                         (P:src/gemm_abft.cpp:60-91): one pass over B producing the
//                         mod-127 row checksums and B' in the K-major, zero-padded layout
//                         the TMA/UMMA mainloop streams.
//   gemm_u8s8_kernel      replaces abft_gemm + verify_checksums / plain_gemm
//                         (P:src/gemm_abft.cpp:30-56, 93-124): TMA -> 128B-swizzled smem ring
//                         -> tcgen05.mma.kind::i8 (A u8 x B s8 -> s32 in TMEM) -> epilogue that
//                         stores C (TMA store, or TMA reduce-add for split-K) and, when CHECKED,
//                         reduces every output row mod 127 and compares it with the checksum
//                         column A*cs (an extra N=16 MMA on the checksum operand) -- per-row
//                         flags without a second pass over C.
//   verify_kernel         replaces verify_checksums (P:src/gemm_abft.cpp:113-124) for
//                         post-hoc checks (faults injected into C after the product).
#include <cuda_runtime.h>

#include "abft_internal.h"
#include "ptx.cuh"

namespace abftk {

// ============================================================ encoder
// Block handles a 64-row slab of B (k rows) and walks all n columns in 64-wide chunks, so the
// row sums stay block-local (int64, as the reference). Writes Bt[j][p] = B[p][j] (zero padded to
// n_pad x k_pad), cs[p] = mod127(sum_j B[p][j]) and row 0 of the 16-row checksum operand.
__global__ void __launch_bounds__(256) encode_weight_kernel(const int8_t* __restrict__ b, int64_t k, int64_t n,
                                                            int64_t ldb, int8_t* __restrict__ bt, int64_t k_pad,
                                                            int64_t n_pad, int8_t* __restrict__ cs_tile,
                                                            int8_t* __restrict__ cs) {
    __shared__ int8_t tile[64][64 + 4];
    __shared__ long long part[4][64];
    const int tid = threadIdx.x;
    const int64_t p0 = static_cast<int64_t>(blockIdx.x) * 64;
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
            bt[(j0 + c) * k_pad + p0 + r] = tile[r][c];
        }
        __syncthreads();
    }
    part[tid >> 6][tid & 63] = acc;
    __syncthreads();
    if (tid < 64) {
        const long long s = part[0][tid] + part[1][tid] + part[2][tid] + part[3][tid];
        const int64_t p = p0 + tid;
        const int8_t v = p < k ? static_cast<int8_t>(mod127(s)) : static_cast<int8_t>(0);
        cs_tile[p] = v;  // row 0 of the checksum operand; rows 1..15 stay zero
        if (p < k) cs[p] = v;
    }
}

// Logical k x (n+1) view [B | cs] of an encoded weight (PackedEncodedWeight::at contract).
__global__ void read_encoded_kernel(const int8_t* __restrict__ bt, const int8_t* __restrict__ cs, int64_t k, int64_t n,
                                    int64_t k_pad, int8_t* __restrict__ out) {
    const int64_t total = k * (n + 1);
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < total;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e / (n + 1), j = e - i * (n + 1);
        out[e] = j < n ? bt[j * k_pad + i] : cs[i];
    }
}

// ============================================================ GEMM
template <int BN, bool CHECKED>
struct GemmCfg {
    static constexpr int kABytes = kBM * kBK;
    static constexpr int kBBytes = BN * kBK;
    static constexpr int kCsBytes = CHECKED ? kCsRows * kBK : 0;
    static constexpr int kStageBytes = kABytes + kBBytes + kCsBytes;
    static constexpr int kStages = (200 * 1024) / kStageBytes > 8 ? 8 : (200 * 1024) / kStageBytes;
    static constexpr int kTmemNeed = BN + (CHECKED ? 16 : 0);
    static constexpr uint32_t kTmemCols = kTmemNeed <= 32 ? 32 : kTmemNeed <= 64 ? 64 : kTmemNeed <= 128 ? 128
                                                                : kTmemNeed <= 256 ? 256 : 512;
    static constexpr int kBarBytes = 256;
    static constexpr int kSmemBytes = 1024 + kStages * kStageBytes + kBarBytes;
    static_assert(kStageBytes % 1024 == 0, "stage buffers must keep 1024-byte alignment");
    static_assert(kStages * kStageBytes >= 4 * 2 * 4096, "epilogue staging reuses the stage ring");
};

template <int BN, bool CHECKED, int EPI>
__global__ void __launch_bounds__(192, 1)
    gemm_u8s8_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                     const __grid_constant__ CUtensorMap tmCS, const __grid_constant__ CUtensorMap tmC,
                     const GemmParams p) {
    using Cfg = GemmCfg<BN, CHECKED>;
    constexpr int STAGES = Cfg::kStages;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * Cfg::kStageBytes);
    uint64_t* empty = full + STAGES;
    uint64_t* tmem_full = empty + STAGES;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(tmem_full + 1);
    uint32_t* bcast = tmem_holder + 1;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nt = blockIdx.x, mt = blockIdx.y, sp = blockIdx.z;
    const int kb0 = sp * p.kb_per_split;
    const int kb1 = min(kb0 + p.kb_per_split, p.k_blocks);
    const int nkb = kb1 - kb0;
    const bool has_cs = CHECKED && nt == 0;

    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        mbar_init(tmem_full, 1);
        fence_mbar_init();
    }
    if (warp == 0) tmem_alloc<Cfg::kTmemCols>(tmem_holder);
    if (warp == 4 && lane == 0) {
        tma_prefetch(&tmA);
        tma_prefetch(&tmB);
        if (has_cs) tma_prefetch(&tmCS);
        if (EPI != kEpiDirect) tma_prefetch(&tmC);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_holder;

    if (warp == 4) {
        // ---------------- TMA producer (one elected lane)
        if (lane == 0) {
            const uint64_t pol_a = policy_evict_last();   // A is re-read by every N tile
            const uint64_t pol_b = policy_evict_first();  // B' is streamed once per call
            const uint32_t bytes = Cfg::kABytes + Cfg::kBBytes + (has_cs ? Cfg::kCsBytes : 0);
            for (int i = 0; i < nkb; ++i) {
                const int s = i % STAGES;
                const uint32_t ph = (i / STAGES) & 1;
                mbar_wait(&empty[s], ph ^ 1);
                uint8_t* st = smem + s * Cfg::kStageBytes;
                mbar_arrive_expect_tx(&full[s], bytes);
                const int kx = (kb0 + i) * kBK;
                tma_load_2d(st, &tmA, &full[s], kx, mt * kBM, pol_a);
                tma_load_2d(st + Cfg::kABytes, &tmB, &full[s], kx, nt * BN, pol_b);
                if (has_cs) tma_load_2d(st + Cfg::kABytes + Cfg::kBBytes, &tmCS, &full[s], kx, 0, pol_a);
            }
        }
    } else if (warp == 5) {
        // ---------------- MMA issuer (one thread issues for the whole CTA)
        if (lane == 0) {
            constexpr uint32_t id_main = idesc_u8s8(kBM, BN);
            constexpr uint32_t id_cs = idesc_u8s8(kBM, kCsRows);
            for (int i = 0; i < nkb; ++i) {
                const int s = i % STAGES;
                const uint32_t ph = (i / STAGES) & 1;
                mbar_wait(&full[s], ph);
                tc_fence_after();
                const uint32_t a_addr = smem_u32(smem + s * Cfg::kStageBytes);
                const uint64_t da = umma_desc_sw128(a_addr);
                const uint64_t db = umma_desc_sw128(a_addr + Cfg::kABytes);
                const uint64_t dc = umma_desc_sw128(a_addr + Cfg::kABytes + Cfg::kBBytes);
#pragma unroll
                for (int kk = 0; kk < kBK / 32; ++kk) {  // UMMA K = 32 bytes for 8-bit operands
                    const uint32_t acc = (i | kk) != 0;
                    mma_i8(tmem, da + 2 * kk, db + 2 * kk, id_main, acc);
                    if (has_cs) mma_i8(tmem + BN, da + 2 * kk, dc + 2 * kk, id_cs, acc);
                }
                mma_commit(&empty[s]);  // frees the smem slot once these MMAs have read it
            }
            mma_commit(tmem_full);  // accumulator complete
        }
    } else {
        // ---------------- epilogue: warps 0..3, thread <-> output row (TMEM lane)
        const int row = mt * kBM + warp * 32 + lane;
        const int n0 = nt * BN;
        uint32_t* my_flag = p.tile_flag + (mt * p.n_tiles + nt);
        if constexpr (EPI == kEpiTmaReduce) {
            if (sp == 0) {
                // Split 0 zero-fills this CTA's C tile while the mainloop runs; every split then
                // reduce-adds its partial product into it (int32 addition is exact).
                const int rows_here = min(kBM, p.m - mt * kBM);
                const int v4_per_row = min(BN, p.n - n0) >> 2;
                const int total = rows_here * v4_per_row;
                for (int idx = threadIdx.x; idx < total; idx += 128) {
                    const int r = idx / v4_per_row, q = idx - r * v4_per_row;
                    *reinterpret_cast<int4*>(p.c + static_cast<int64_t>(mt * kBM + r) * p.ldc + n0 + 4 * q) =
                        make_int4(0, 0, 0, 0);
                }
                __threadfence();
                named_bar_sync(1, 128);
                if (threadIdx.x == 0) st_release_gpu(my_flag, p.epoch);
            }
        }
        mbar_wait(tmem_full, 0);
        tc_fence_after();
        if constexpr (EPI == kEpiTmaReduce) {
            if (lane == 0) {
                while (static_cast<int32_t>(ld_acquire_gpu(my_flag) - p.epoch) < 0) {
                }
                fence_proxy_async_global();
            }
            __syncwarp();
        }
        fence_proxy_async_smem();
        const uint32_t t_row = tmem + (static_cast<uint32_t>(warp * 32) << 16);
        const int fault_here = p.fault_active && row == p.fault_row;
        long long rsum = 0;
#pragma unroll 1
        for (int c = 0; c < BN / 32; ++c) {
            const int col0 = n0 + c * 32;
            if (col0 >= p.n) break;  // warp-uniform
            uint32_t v[32];
            tmem_ld_32x32b_x32(t_row + c * 32, v);
            tmem_wait_ld();
            if (fault_here) {
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (p.fault_col == col0 + j) v[j] ^= 1u << p.fault_bit;
            }
            if constexpr (CHECKED) {
#pragma unroll
                for (int j = 0; j < 32; ++j) rsum += static_cast<int32_t>(v[j]);
            }
            if constexpr (EPI == kEpiDirect) {
                if (row < p.m) {
                    int32_t* crow = p.c + static_cast<int64_t>(row) * p.ldc;
#pragma unroll
                    for (int j = 0; j < 32; ++j)
                        if (col0 + j < p.n) crow[col0 + j] = static_cast<int32_t>(v[j]);
                }
            } else {
                uint8_t* buf = smem + (warp * 2 + (c & 1)) * 4096;
                if (c >= 2) {
                    if (lane == 0) bulk_wait_read<1>();
                    __syncwarp();
                }
#pragma unroll
                for (int q = 0; q < 8; ++q)
                    *reinterpret_cast<uint4*>(buf + lane * 128 + ((q ^ (lane & 7)) << 4)) =
                        make_uint4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) {
                    if (mt * kBM + warp * 32 < p.m) {
                        if constexpr (EPI == kEpiTmaStore)
                            tma_store_2d(&tmC, buf, col0, mt * kBM + warp * 32);
                        else
                            tma_reduce_add_2d(&tmC, buf, col0, mt * kBM + warp * 32);
                    }
                    bulk_commit();
                }
            }
        }
        if constexpr (EPI != kEpiDirect) {
            if (lane == 0) bulk_wait<0>();
            __syncwarp();
        }
        if constexpr (CHECKED) {
            int32_t csv = 0;
            if (has_cs) {
                csv = static_cast<int32_t>(tmem_ld_32x32b_x1(t_row + BN));
                tmem_wait_ld();
                if (fault_here && p.fault_col == p.n) csv ^= static_cast<int32_t>(1u << p.fault_bit);
            }
            if (row < p.m) {
                // mod is a ring homomorphism: the residue of the full int64 row sum equals the sum of
                // per-tile residues mod 127 (P:src/gemm_abft.cpp:119-122 reduces the int64 sum once).
                atomicAdd(&p.row_res[row], static_cast<uint32_t>(mod127(rsum)));
                if (has_cs) atomicAdd(&p.csum_acc[row], csv);
            }
            __threadfence();
            named_bar_sync(1, 128);
            if (threadIdx.x == 0) {
                const uint32_t prev = atomicAdd(&p.mtile_cnt[mt], 1u);
                *bcast = prev == static_cast<uint32_t>(p.n_tiles * p.splits - 1) ? 1u : 0u;
            }
            named_bar_sync(1, 128);
            if (*bcast) {
                // Last CTA of this M tile: every contribution is in; finalize the rows and clean the
                // workspace for the next call on this stream.
                __threadfence();
                int flag = 0;
                if (row < p.m) {
                    const uint32_t acc = atomicExch(&p.row_res[row], 0u);
                    const int32_t cs = atomicExch(&p.csum_acc[row], 0);
                    flag = static_cast<int32_t>(acc % 127u) != mod127(cs);
                    p.flags[row] = static_cast<uint8_t>(flag);
                    p.csum[static_cast<int64_t>(row) * p.csum_ld] = cs;
                }
                const uint32_t wcount = __popc(__ballot_sync(0xffffffffu, flag));
                if (lane == 0 && wcount) atomicAdd(p.err_acc, wcount);
                __threadfence();
                named_bar_sync(1, 128);
                if (threadIdx.x == 0) {
                    atomicExch(&p.mtile_cnt[mt], 0u);
                    const uint32_t prev = atomicAdd(p.done_cnt, 1u);
                    if (prev == static_cast<uint32_t>(p.m_tiles - 1)) {
                        __threadfence();
                        *p.err_count = atomicExch(p.err_acc, 0u);
                        atomicExch(p.done_cnt, 0u);
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        tmem_dealloc<Cfg::kTmemCols>(tmem);
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
template <int BN, bool CHECKED, int EPI>
static cudaError_t launch_one(dim3 grid, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& cs,
                              const CUtensorMap& c, const GemmParams& p, cudaStream_t st) {
    using Cfg = GemmCfg<BN, CHECKED>;
    auto kern = gemm_u8s8_kernel<BN, CHECKED, EPI>;
    static bool attr_done = false;  // benign race: idempotent attribute set
    if (!attr_done) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::kSmemBytes);
        if (e != cudaSuccess) return e;
        attr_done = true;
    }
    kern<<<grid, 192, Cfg::kSmemBytes, st>>>(a, b, cs, c, p);
    return cudaGetLastError();
}

template <int BN, bool CHECKED>
static cudaError_t launch_epi(int epi, dim3 grid, const CUtensorMap& a, const CUtensorMap& b, const CUtensorMap& cs,
                              const CUtensorMap& c, const GemmParams& p, cudaStream_t st) {
    switch (epi) {
        case kEpiTmaStore: return launch_one<BN, CHECKED, kEpiTmaStore>(grid, a, b, cs, c, p, st);
        case kEpiTmaReduce: return launch_one<BN, CHECKED, kEpiTmaReduce>(grid, a, b, cs, c, p, st);
        default: return launch_one<BN, CHECKED, kEpiDirect>(grid, a, b, cs, c, p, st);
    }
}

cudaError_t launch_gemm_kernel(int bn, bool checked, int epi, dim3 grid, const CUtensorMap& a, const CUtensorMap& b,
                               const CUtensorMap& cs, const CUtensorMap& c, const GemmParams& p, cudaStream_t st) {
    if (checked) {
        if (bn == 256) return launch_epi<256, true>(epi, grid, a, b, cs, c, p, st);
        if (bn == 128) return launch_epi<128, true>(epi, grid, a, b, cs, c, p, st);
        return launch_epi<64, true>(epi, grid, a, b, cs, c, p, st);
    }
    if (bn == 256) return launch_epi<256, false>(epi, grid, a, b, cs, c, p, st);
    if (bn == 128) return launch_epi<128, false>(epi, grid, a, b, cs, c, p, st);
    return launch_epi<64, false>(epi, grid, a, b, cs, c, p, st);
}

int gemm_stages(int bn, bool checked) {
    if (checked) return bn == 256 ? GemmCfg<256, true>::kStages : bn == 128 ? GemmCfg<128, true>::kStages
                                                                            : GemmCfg<64, true>::kStages;
    return bn == 256 ? GemmCfg<256, false>::kStages : bn == 128 ? GemmCfg<128, false>::kStages
                                                                : GemmCfg<64, false>::kStages;
}

cudaError_t launch_read_encoded(const GemmWeight& w, int8_t* out, cudaStream_t st) {
    int64_t blocks = (w.k * (w.n + 1) + 255) / 256;
    if (blocks > 4096) blocks = 4096;
    read_encoded_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(w.bt, w.cs, w.k, w.n, w.k_pad, out);
    return cudaGetLastError();
}

cudaError_t launch_encode_weight(const int8_t* b, int64_t k, int64_t n, int64_t ldb, GemmWeight& w, cudaStream_t st) {
    encode_weight_kernel<<<static_cast<unsigned>(w.k_pad / 64), 256, 0, st>>>(b, k, n, ldb, w.bt, w.k_pad, w.n_pad,
                                                                             w.cs_tile, w.cs);
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
