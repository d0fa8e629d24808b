// Small-m checked GEMM ("GEMV class"): m <= 16 rows of A against the encoded weight.
//
// For the activation-heavy DLRM shapes of P:data/shapes.txt (m in {1, 8, 32, 64}) the tensor-core pair
// kernel pays a full 256-row tile and its pipeline latency for a handful of rows; this path is bound by
// streaming B' once instead. Block = 32 output columns x 8 warps, each warp a contiguous K range; a lane
// owns one column and reads that column's 128-byte k-block slab of the K-block-major B' (the warp reads
// 4 KB contiguous), A (all m rows) is staged in shared memory and broadcast, products are u8 x s8 dp4a
// into int32 (exact). The 8 warps' partials are summed in shared memory; the block then runs the same
// checked epilogue as the pair kernel: per-row residue of its 32 columns + its K share of the checksum
// GEMV folded into one 64-bit atomic per row whose last arrival finalizes the row (gemm.cu).
#include <cuda_runtime.h>

#include "abft_internal.h"
#include "ptx.cuh"

namespace abftk {

constexpr int kGemvWarps = 8;

template <int MR, bool CHECKED>
__global__ void __launch_bounds__(32 * kGemvWarps) gemv_checked_kernel(const GemmParams p, const int8_t* __restrict__ bt,
                                                                       int64_t n_pad) {
    extern __shared__ __align__(16) uint8_t gsm[];
    uint8_t* As = gsm;                                             // [MR][k_pad] u8
    int32_t* red = reinterpret_cast<int32_t*>(gsm + MR * p.k_blocks * kBK);  // [warps][MR][32]
    int32_t* xin = red + kGemvWarps * MR * 32;                     // [cluster][MR][32] (leader)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // A cluster of `ks` blocks along K shares one column group when the column groups alone cannot fill
    // the GPU; the partials meet in the leader's shared memory (DSMEM).
    uint32_t ks_n;
    asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(ks_n));
    const int ks = static_cast<int>(ks_n), kr = static_cast<int>(cluster_ctarank());
    const int ncg = static_cast<int>(gridDim.x) / ks;
    const int cg = static_cast<int>(blockIdx.x) / ks;  // column group
    const int j = cg * 32 + lane;
    const int kpad = p.k_blocks * kBK;
    const int bkb0 = kr * p.k_blocks / ks, bkb1 = (kr + 1) * p.k_blocks / ks;  // this block's k-blocks

    griddep_wait();
    // stage A (all of it: the leader's checksum share may span any k range; rows >= m and columns >= k
    // are zero)
    for (int e = threadIdx.x * 16; e < MR * kpad; e += blockDim.x * 16) {
        const int i = e / kpad, c = e - i * kpad;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (i < p.m) {
            const uint8_t* src = p.a + static_cast<int64_t>(i) * p.lda + c;
            if (c + 16 <= p.k && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
                v = *reinterpret_cast<const uint4*>(src);
            } else {
                alignas(16) uint8_t t[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) t[q] = c + q < p.k ? src[q] : 0;
                v = *reinterpret_cast<const uint4*>(t);
            }
        }
        *reinterpret_cast<uint4*>(As + e) = v;
    }
    __syncthreads();

    uint32_t acc[MR];
#pragma unroll
    for (int i = 0; i < MR; ++i) acc[i] = 0u;
    const int kb0 = bkb0 + warp * (bkb1 - bkb0) / kGemvWarps, kb1 = bkb0 + (warp + 1) * (bkb1 - bkb0) / kGemvWarps;
    const int8_t* col = bt + static_cast<int64_t>(j) * kBK;  // + kb * n_pad * 128
    for (int kb = kb0; kb < kb1; ++kb) {
        uint4 w[8];
        const uint4* src = reinterpret_cast<const uint4*>(col + static_cast<int64_t>(kb) * n_pad * kBK);
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = __ldg(src + u);  // padded columns read zeros (n_pad >= n)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int i = 0; i < MR; ++i) {
                const uint4 a = *reinterpret_cast<const uint4*>(As + i * kpad + kb * kBK + u * 16);
                acc[i] = dp4a_us(a.x, w[u].x, acc[i]);
                acc[i] = dp4a_us(a.y, w[u].y, acc[i]);
                acc[i] = dp4a_us(a.z, w[u].z, acc[i]);
                acc[i] = dp4a_us(a.w, w[u].w, acc[i]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < MR; ++i) red[(warp * MR + i) * 32 + lane] = static_cast<int32_t>(acc[i]);
    __syncthreads();
    // block partial of every row -> the cluster leader's slot kr (its own slot 0 stays local)
    for (int e = threadIdx.x; e < MR * 32; e += blockDim.x) {
        uint32_t v = 0u;
#pragma unroll
        for (int w8 = 0; w8 < kGemvWarps; ++w8) v += static_cast<uint32_t>(red[w8 * MR * 32 + e]);
        if (ks == 1 || kr == 0) {
            xin[kr * MR * 32 + e] = static_cast<int32_t>(v);
        } else {
            const uint32_t dst = mapa_shared(smem_u32(&xin[kr * MR * 32 + e]), 0);
            asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(dst), "r"(v) : "memory");
        }
    }
    if (ks > 1) cluster_sync();
    else __syncthreads();
    if (kr != 0) return;  // the leader finishes the column group

    // warp i (< MR) finishes row i: column sums over the cluster's K ranges, C store, fault hook, residue
    for (int i = warp; i < MR && i < p.m; i += kGemvWarps) {
        uint32_t v = 0u;
        for (int r = 0; r < ks; ++r) v += static_cast<uint32_t>(xin[(r * MR + i) * 32 + lane]);
        for (int f = 0; f < p.nfaults; ++f)
            if (i == p.fault_row[f] && p.fault_col[f] == j && j < p.n) v ^= 1u << p.fault_bit[f];
        if (j < p.n && p.c) p.c[static_cast<int64_t>(i) * p.ldc + j] = static_cast<int32_t>(v);
        if constexpr (CHECKED) {
            long long rs = j < p.n ? static_cast<int32_t>(v) : 0;
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) rs += __shfl_xor_sync(0xffffffffu, rs, o);
            // this block's K share of the checksum GEMV C'[i][n] = sum_p A[i][p]*cs[p]
            const int s0 = static_cast<int>(static_cast<long long>(cg) * p.k_blocks / ncg) * kBK;
            const int s1 = min(static_cast<int>(static_cast<long long>(cg + 1) * p.k_blocks / ncg) * kBK, p.k);
            uint32_t cs_part = 0u;
            for (int q = s0 + lane * 4; q < s1; q += 128) {
                const uint32_t a4 = *reinterpret_cast<const uint32_t*>(As + i * kpad + q);
                uint32_t c4 = 0u;
                if (q + 4 <= p.k) {
                    c4 = *reinterpret_cast<const uint32_t*>(p.cs + q);
                } else {
                    for (int e = 0; e < 4 && q + e < p.k; ++e) c4 |= static_cast<uint32_t>(static_cast<uint8_t>(p.cs[q + e])) << (8 * e);
                }
                cs_part = dp4a_us(a4, c4, cs_part);  // cs is s8 (negative after a sign-bit flip)
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) cs_part += __shfl_xor_sync(0xffffffffu, cs_part, o);
            if (lane == 0) {
                const unsigned long long add = (static_cast<unsigned long long>(cs_part) << 32) |
                                               (1ull << kRowAccCountShift) |
                                               static_cast<unsigned long long>(mod127(rs));
                const unsigned long long acc64 = atomicAdd(&p.row_acc[i], add) + add;
                if (((acc64 >> kRowAccCountShift) & kRowAccCountMask) == static_cast<unsigned long long>(ncg)) {
                    int32_t csv = static_cast<int32_t>(static_cast<uint32_t>(acc64 >> 32));
                    for (int f = 0; f < p.nfaults; ++f)
                        if (i == p.fault_row[f] && p.fault_col[f] == p.n)
                            csv ^= static_cast<int32_t>(1u << p.fault_bit[f]);  // fault in C'[:, n]
                    const uint32_t res = static_cast<uint32_t>(acc64 & kRowAccResMask) % 127u;
                    const int flag = static_cast<int32_t>(res) != mod127(csv);
                    p.flags[i] = static_cast<uint8_t>(flag);
                    p.csum[static_cast<int64_t>(i) * p.csum_ld] = csv;
                    p.row_acc[i] = 0ull;
                    if (p.m == 1) {  // the only row: its finisher publishes the count (no second round trip)
                        *p.err_count = static_cast<uint32_t>(flag);
                    } else {
                        const unsigned long long prev =
                            atomicAdd(p.err_pack, (1ull << 32) | static_cast<unsigned>(flag));
                        if ((prev >> 32) + 1 == static_cast<unsigned long long>(p.m)) {
                            *p.err_count = static_cast<uint32_t>(prev) + static_cast<uint32_t>(flag);
                            *p.err_pack = 0ull;
                        }
                    }
                }
            }
        }
    }
}

template <int MR, bool CK>
static cudaError_t launch_gemv_mr(const GemmParams& p, const GemmWeight& w, cudaStream_t st) {
    // K split across a cluster when the column groups alone cannot fill ~2 blocks per SM
    const int ncg = (p.n + 31) / 32;
    int ks = 1;
    while (ks < 8 && ncg * ks * 2 <= 2 * 148 && p.k_blocks >= ks * 2) ks *= 2;
    const int smem = MR * p.k_blocks * kBK + kGemvWarps * MR * 32 * 4 + ks * MR * 32 * 4;
    auto kern = gemv_checked_kernel<MR, CK>;
    static int attr_smem[kMaxDevices] = {};  // per device; benign race: idempotent
    const int dev = current_device();
    if (smem > 48 * 1024 && smem > attr_smem[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_smem[dev] = smem;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(ncg * ks));
    cfg.blockDim = dim3(32 * kGemvWarps);
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = static_cast<unsigned>(ks);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p, static_cast<const int8_t*>(w.bt), static_cast<int64_t>(w.n_pad));
}

// Row capacity of the small-m path; the runtime routes m <= kGemvMaxRows here.
cudaError_t launch_gemv(const GemmParams& p, const GemmWeight& w, bool checked, cudaStream_t st) {
    const int m = p.m;
    if (checked) {
        if (m <= 1) return launch_gemv_mr<1, true>(p, w, st);
        if (m <= 2) return launch_gemv_mr<2, true>(p, w, st);
        if (m <= 4) return launch_gemv_mr<4, true>(p, w, st);
        if (m <= 8) return launch_gemv_mr<8, true>(p, w, st);
        return launch_gemv_mr<16, true>(p, w, st);
    }
    if (m <= 1) return launch_gemv_mr<1, false>(p, w, st);
    if (m <= 2) return launch_gemv_mr<2, false>(p, w, st);
    if (m <= 4) return launch_gemv_mr<4, false>(p, w, st);
    if (m <= 8) return launch_gemv_mr<8, false>(p, w, st);
    return launch_gemv_mr<16, false>(p, w, st);
}

}  // namespace abftk
