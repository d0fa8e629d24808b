// Requantization kernels: the standalone requantize over an existing C'
// (P:src/quant.cpp:77-102), and the row / column sums it consumes (P:src/quant.cpp:104-118). The fused
// variant lives in the GEMM epilogue (gemm.cu, GemmParams::rq_out).
#include <cuda_runtime.h>

#include "abft_internal.h"
#include "requant.cuh"

namespace abftk {

// One thread per output element; C' columns >= n (the checksum column) are never read.
__global__ void requantize_kernel(const int32_t* __restrict__ c, int64_t ldc, int64_t m, int64_t n,
                                  const int32_t* __restrict__ rs, const int32_t* __restrict__ cs, RequantDev q,
                                  uint8_t* __restrict__ out, int64_t ld_out) {
    const RequantConsts k = requant_consts(q);
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < m * n;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t i = e / n, j = e - i * n;
        out[i * ld_out + j] = static_cast<uint8_t>(requant_one(c[i * ldc + j], rs[i], cs[j], k));
    }
}

// rowSum(A)[i] = sum_p A[i][p] (u8), one warp per row, dp4a on 16-byte loads when aligned.
__global__ void row_sums_u8_kernel(const uint8_t* __restrict__ a, int64_t m, int64_t k, int64_t lda,
                                   int32_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < m;
         r += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
        const uint8_t* row = a + r * lda;
        uint32_t s = 0;
        int64_t p = 0;
        if ((reinterpret_cast<uintptr_t>(row) & 15) == 0) {
            for (; p + 512 <= k; p += 512) {
                const uint4 v = __ldg(reinterpret_cast<const uint4*>(row + p) + lane);
                s = __dp4a(v.x, 0x01010101u, s);
                s = __dp4a(v.y, 0x01010101u, s);
                s = __dp4a(v.z, 0x01010101u, s);
                s = __dp4a(v.w, 0x01010101u, s);
            }
        }
        for (int64_t q = p + lane; q < k; q += 32) s += row[q];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[r] = static_cast<int32_t>(s);
    }
}

// colSum(B)[j] = sum_i B[i][j] from the encoded weight (bt[kb][j][kk], zero padded past k): one warp per
// column, 4 bytes per lane per k-block.
__global__ void col_sums_kernel(const int8_t* __restrict__ bt, int64_t k_blocks, int64_t n, int64_t n_pad,
                                int32_t* __restrict__ out) {
    const int lane = threadIdx.x & 31;
    for (int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; j < n;
         j += (static_cast<int64_t>(gridDim.x) * blockDim.x) >> 5) {
        int s = 0;
        for (int64_t kb = 0; kb < k_blocks; ++kb) {
            const int w = __ldg(reinterpret_cast<const int*>(bt + (kb * n_pad + j) * kBK) + lane);
            s = __dp4a(w, 0x01010101, s);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) out[j] = s;
    }
}

static unsigned grid_for(int64_t items, int per_block) {
    int64_t b = (items + per_block - 1) / per_block;
    if (b > 148 * 16) b = 148 * 16;
    return static_cast<unsigned>(b < 1 ? 1 : b);
}

cudaError_t launch_requantize(const int32_t* c, int64_t ldc, int64_t m, int64_t n, const int32_t* rs, const int32_t* cs,
                              const RequantDev& q, uint8_t* out, int64_t ld_out, cudaStream_t st) {
    if (m <= 0 || n <= 0) return cudaSuccess;
    requantize_kernel<<<grid_for(m * n, 256), 256, 0, st>>>(c, ldc, m, n, rs, cs, q, out, ld_out);
    return cudaGetLastError();
}

cudaError_t launch_row_sums_u8(const uint8_t* a, int64_t m, int64_t k, int64_t lda, int32_t* out, cudaStream_t st) {
    if (m <= 0) return cudaSuccess;
    row_sums_u8_kernel<<<grid_for(m, 8), 256, 0, st>>>(a, m, k, lda, out);
    return cudaGetLastError();
}

cudaError_t launch_col_sums(const GemmWeight& w, int32_t* out, cudaStream_t st) {
    if (w.n <= 0) return cudaSuccess;
    col_sums_kernel<<<grid_for(w.n, 8), 256, 0, st>>>(w.bt, w.k_pad / kBK, w.n, w.n_pad, out);
    return cudaGetLastError();
}

}  // namespace abftk
