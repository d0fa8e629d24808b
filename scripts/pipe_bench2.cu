// Microbenchmark 2: per-SM load throughput of different async-copy shapes through a stage ring.
// mode 0: one 2D tensor box per stage (rows x 128 B, SW128)
// mode 1: `nbox` 2D boxes per stage (rows/nbox each)
// mode 2: one 1D cp.async.bulk of stage_bytes per stage (pre-laid-out, contiguous)
// mode 3: nbox 1D bulk copies per stage
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

#include "ptx.cuh"
using namespace abftk;

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}

__global__ void __launch_bounds__(64, 1) ring(const __grid_constant__ CUtensorMap tm, const uint8_t* src, int mode,
                                              int rows, int nbox, int kb, int stages, uint64_t ld,
                                              unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    const int sb = rows * 128;
    uint64_t* full = (uint64_t*)(smem + stages * sb);
    uint64_t* empty = full + 16;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    unsigned long long t0 = globaltimer();
    if (threadIdx.x == 0) {
        for (int i = 0; i < kb; ++i) {
            int s = i % stages;
            uint32_t ph = (i / stages) & 1;
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], sb);
            uint8_t* dst = smem + s * sb;
            if (mode <= 1) {
                const int r = rows / nbox;
                for (int b = 0; b < nbox; ++b)
                    tma_load_2d(dst + b * r * 128, &tm, &full[s], i * 128, blockIdx.x * rows + b * r, 0);
            } else {
                const uint8_t* base = src + ((uint64_t)blockIdx.x * kb + i) * sb;
                const int chunk = sb / nbox;
                for (int b = 0; b < nbox; ++b) bulk_load(dst + b * chunk, base + b * chunk, chunk, &full[s]);
            }
        }
    } else if (threadIdx.x == 32) {
        for (int i = 0; i < kb; ++i) {
            int s = i % stages;
            uint32_t ph = (i / stages) & 1;
            mbar_wait(&full[s], ph);
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
        }
        out[blockIdx.x] = globaltimer() - t0;
    }
}

int main() {
    EncodeFn fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
    const uint64_t ld = 4096;
    uint8_t* buf;
    const size_t bytes = 512ull << 20;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    unsigned long long* d;
    cudaMalloc(&d, 4096 * 8);
    struct Cfg {
        int mode, rows, nbox, stages, ctas;
    };
    Cfg cfgs[] = {{0, 128, 1, 8, 1}, {0, 256, 1, 6, 1}, {0, 64, 1, 12, 1}, {1, 256, 2, 6, 1}, {1, 256, 4, 6, 1},
                  {2, 128, 1, 8, 1}, {2, 256, 1, 6, 1}, {3, 256, 4, 6, 1}, {3, 256, 16, 6, 1},
                  {0, 128, 1, 8, 148}, {0, 256, 1, 6, 148}, {2, 128, 1, 8, 148}, {2, 256, 1, 6, 148},
                  {3, 256, 4, 6, 148}, {0, 128, 1, 3, 1}, {2, 128, 1, 3, 1}, {2, 384, 1, 4, 148}};
    for (Cfg c : cfgs) {
        CUtensorMap tm;
        memset(&tm, 0, sizeof tm);
        const uint64_t outer = bytes / ld;
        cuuint64_t dim[2] = {ld, outer}, str[1] = {ld};
        cuuint32_t box[2] = {128, (cuuint32_t)(c.rows / c.nbox)}, es[2] = {1, 1};
        fn(&tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, buf, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int kb = 32;
        int smem = 2048 + c.stages * c.rows * 128 + 512;
        cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        for (int rep = 0; rep < 2; ++rep) ring<<<c.ctas, 64, smem>>>(tm, buf, c.mode, c.rows, c.nbox, kb, c.stages, ld, d);
        cudaDeviceSynchronize();
        unsigned long long h[256];
        cudaMemcpy(h, d, c.ctas * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < c.ctas; ++i) avg += h[i];
        avg /= c.ctas;
        double sb = c.rows * 128.0;
        printf("mode=%d rows=%3d nbox=%2d stages=%2d ctas=%3d: %.0f ns/stage, %.1f GB/s per SM, %.2f TB/s total  %s\n",
               c.mode, c.rows, c.nbox, c.stages, c.ctas, avg / kb, sb * kb / avg, sb * kb * c.ctas / avg / 1e3,
               cudaGetErrorString(cudaGetLastError()));
    }
    return 0;
}
