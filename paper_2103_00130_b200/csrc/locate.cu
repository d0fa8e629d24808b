// Dual-encoded locate / correct of a checked GEMM result on the GPU (the reference keeps the
// dual-encoded check as a test oracle, P:tests/dual_check.hpp:23-73).
//
// The product path carries one mod-127 row checksum per row (P:src/gemm_abft.cpp:113-124): it says WHICH row is
// wrong, not which column. The dual encoding adds the column check: with a = the column sums of A
// (a[p] = sum_i A[i][p]), the exact column sums of a clean C are  colref[j] = sum_p a[p] * B[p][j]  (int64, no
// modulus). Comparing them with the actual column sums  colact[j] = sum_i C[i][j]  gives the corrupted column j*
// and the exact error delta = colact[j*] - colref[j*]; with the flagged row i* the corrupted cell is (i*, j*) and
// C[i*][j*] -= delta restores it. A flagged row with no column mismatch means the checksum column itself was hit;
// it is recomputed exactly (A[i*] . cs).
#include <cuda_runtime.h>

#include <cstdint>

#include "abft_internal.h"
#include "ptx.cuh"

namespace abftk {

// a[p] = sum_i A[i][p] (u32: m <= 2^24). One thread per column p, rows strided by lda.
__global__ void locate_colsum_a_kernel(const uint8_t* __restrict__ a, int64_t m, int64_t k, int64_t lda,
                                       uint32_t* __restrict__ out, int64_t k_pad) {
    for (int64_t p = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; p < k_pad;
         p += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        uint32_t s = 0;
        if (p < k)
            for (int64_t i = 0; i < m; ++i) s += a[i * lda + p];
        out[p] = s;
    }
}

// One warp per column j < n: colref[j] (B' K-major: bt[kb][j][kk], 128 contiguous bytes per k-block) and colact[j];
// mismatching columns are counted and the first ones recorded (column, delta).
__global__ void locate_columns_kernel(const uint32_t* __restrict__ colsum_a, const int8_t* __restrict__ bt, int64_t k_pad,
                                      int64_t n, int64_t n_pad, const int32_t* __restrict__ c, int64_t m, int64_t ldc,
                                      uint32_t* __restrict__ nbad, int64_t* __restrict__ bad_col,
                                      long long* __restrict__ bad_delta, int max_record) {
    const int lane = threadIdx.x & 31;
    const int64_t warps = static_cast<int64_t>(gridDim.x) * (blockDim.x >> 5);
    for (int64_t j = static_cast<int64_t>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5); j < n; j += warps) {
        long long ref = 0, act = 0;
        for (int64_t kb = 0; kb < k_pad / kBK; ++kb) {
            const int8_t* col = bt + (kb * n_pad + j) * kBK;
            const uint32_t w = *reinterpret_cast<const uint32_t*>(col + 4 * lane);
            const int64_t p0 = kb * kBK + 4 * lane;
#pragma unroll
            for (int e = 0; e < 4; ++e)
                ref += static_cast<long long>(colsum_a[p0 + e]) * static_cast<int8_t>(static_cast<uint8_t>(w >> (8 * e)));
        }
        for (int64_t i = lane; i < m; i += 32) act += c[i * ldc + j];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            ref += __shfl_xor_sync(0xffffffffu, ref, o);
            act += __shfl_xor_sync(0xffffffffu, act, o);
        }
        if (lane == 0 && ref != act) {
            const uint32_t slot = atomicAdd(nbad, 1u);
            if (static_cast<int>(slot) < max_record) {
                bad_col[slot] = j;
                bad_delta[slot] = act - ref;
            }
        }
    }
}

// Exact checksum column of one row: sum_p A[row][p] * cs[p] (int32, as the reference's C'[:, n]).
__global__ void locate_row_checksum_kernel(const uint8_t* __restrict__ a, int64_t k, const int8_t* __restrict__ cs,
                                           int32_t* __restrict__ out) {
    int32_t s = 0;
    for (int64_t p = threadIdx.x; p < k; p += blockDim.x) s += static_cast<int32_t>(a[p]) * cs[p];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ int32_t part[8];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        int32_t t = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += part[w];
        *out = t;
    }
}

cudaError_t launch_locate_colsum_a(const uint8_t* a, int64_t m, int64_t k, int64_t lda, uint32_t* out, int64_t k_pad,
                                   cudaStream_t st) {
    int64_t blocks = (k_pad + 255) / 256;
    if (blocks > 1184) blocks = 1184;
    locate_colsum_a_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(a, m, k, lda, out, k_pad);
    return cudaGetLastError();
}

cudaError_t launch_locate_columns(const uint32_t* colsum_a, const GemmWeight& w, const int32_t* c, int64_t m, int64_t ldc,
                                  uint32_t* nbad, int64_t* bad_col, long long* bad_delta, int max_record,
                                  cudaStream_t st) {
    int64_t blocks = (w.n + 7) / 8;
    if (blocks > 148 * 16) blocks = 148 * 16;
    if (blocks < 1) blocks = 1;
    locate_columns_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(colsum_a, w.bt, w.k_pad, w.n, w.n_pad, c, m, ldc,
                                                                        nbad, bad_col, bad_delta, max_record);
    return cudaGetLastError();
}

cudaError_t launch_locate_row_checksum(const uint8_t* a_row, int64_t k, const int8_t* cs, int32_t* out, cudaStream_t st) {
    locate_row_checksum_kernel<<<1, 256, 0, st>>>(a_row, k, cs, out);
    return cudaGetLastError();
}

}  // namespace abftk
