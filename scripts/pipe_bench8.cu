// Microbenchmark 8: completion timeline of R back-to-back TMA requests issued by one thread into distinct
// smem slots (one mbarrier per request), all CTAs at once or a single CTA. Tells whether an SM's TMA
// requests overlap (completions bunched) or are served one after another (completions evenly spaced).
//   usage: pipe_bench8 box_rows kbs R ctas layout   (layout 0: A-style row-major, 1: k-block-major)
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "ptx.cuh"
using namespace abftk;

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(
            smem_u32(dst)),
        "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

__global__ void __launch_bounds__(32, 1) timeline(const __grid_constant__ CUtensorMap tm, int rows, int kbs, int R,
                                                  unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    const int rb = rows * 128 * kbs;
    uint64_t* bars = (uint64_t*)(smem + R * rb);
    if (threadIdx.x == 0) {
        for (int r = 0; r < R; ++r) mbar_init(&bars[r], 1);
        fence_mbar_init();
        tma_prefetch(&tm);
    }
    __syncwarp();
    if (threadIdx.x == 0) {
        const int region = blockIdx.x % 32;
        const unsigned long long t0 = globaltimer();
        for (int r = 0; r < R; ++r) {
            mbar_arrive_expect_tx(&bars[r], rb);
            tma3d(smem + r * rb, &tm, &bars[r], 0, region * 256 % (8192 - rows), (r * kbs) % 32);
        }
        const unsigned long long t_issue = globaltimer();
        out[blockIdx.x * 66 + 0] = t_issue - t0;
        for (int r = 0; r < R; ++r) {
            mbar_wait(&bars[r], 0);
            out[blockIdx.x * 66 + 1 + r] = globaltimer() - t0;
        }
    }
}

int main(int argc, char** argv) {
    const int rows = atoi(argv[1]), kbs = atoi(argv[2]), R = atoi(argv[3]), ctas = atoi(argv[4]), layout = atoi(argv[5]);
    EncodeFn fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
    uint8_t* buf;
    const size_t rows_total = 8192, kbt = 32;
    cudaMalloc(&buf, rows_total * kbt * 128);
    cudaMemset(buf, 1, rows_total * kbt * 128);
    unsigned long long* d;
    cudaMalloc(&d, 148 * 66 * 8);
    CUtensorMap m;
    memset(&m, 0, sizeof m);
    cuuint64_t dims[3] = {128, rows_total, kbt}, str[2] = {kbt * 128, 128};
    if (layout == 1) {
        str[0] = 128;
        str[1] = rows_total * 128;
    }
    cuuint32_t box[3] = {128, (cuuint32_t)rows, (cuuint32_t)kbs}, es[3] = {1, 1, 1};
    fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
       CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const int smem = 2048 + R * rows * 128 * kbs + 64 * 8;
    cudaFuncSetAttribute(timeline, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    for (int rep = 0; rep < 3; ++rep) timeline<<<ctas, 32, smem>>>(m, rows, kbs, R, d);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148 * 66];
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    printf("box %d rows x %d kb = %d B, R=%d, ctas=%d, layout %d (%s): issue %llu ns; completions (CTA 0):", rows, kbs,
           rows * 128 * kbs, R, ctas, layout, cudaGetErrorString(e), h[0]);
    for (int r = 0; r < R; ++r) printf(" %llu", h[1 + r]);
    double last = 0;
    for (int c = 0; c < ctas; ++c) last += h[c * 66 + R];
    printf("  | mean last %.0f ns -> %.1f GB/s/SM\n", last / ctas, (double)R * rows * 128 * kbs / (last / ctas));
    return 0;
}
