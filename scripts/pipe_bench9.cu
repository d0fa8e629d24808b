// Microbenchmark 9 (derived from 7): P independent producer/consumer lanes per CTA (each lane its own
// warp pair, stage ring and barriers) -- does a second issuing warp raise an SM's TMA ingest?
// Old header of 7: aggregate L2 -> SMEM TMA throughput vs bytes per request, requests per stage and
// stages in flight (argv-driven sweep of pipe_bench5's unicast kernel; nreq requests of rows/nreq rows).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

#include "ptx.cuh"
using namespace abftk;

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

__device__ __forceinline__ void tma3d(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                 ::"r"(smem_u32(dst)), "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2) : "memory");
}
__device__ __forceinline__ void tma3d_mc(void* dst, const CUtensorMap* m, uint64_t* bar, int c0, int c1, int c2,
                                         uint16_t mask) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes.multicast::cluster"
                 " [%0], [%1, {%3, %4, %5}], [%2], %6;"
                 ::"r"(smem_u32(dst)), "l"((uint64_t)m), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "h"(mask)
                 : "memory");
}

__global__ void __launch_bounds__(512, 1) stream(const __grid_constant__ CUtensorMap tm, int rows, int kbs, int stages,
                                                 int iters, int lanes, int nreq, int spin, int same, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem0 = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    const int sb = rows * 128 * kbs;
    const int lane_id = threadIdx.x / 64;
    uint8_t* smem = smem0 + lane_id * stages * sb;
    uint64_t* bars = (uint64_t*)(smem0 + lanes * stages * sb);
    uint64_t* full = bars + lane_id * 32;
    uint64_t* empty = full + 16;
    if (threadIdx.x % 64 == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    unsigned long long t0 = globaltimer();
    const int region = same ? lane_id % 4 : (blockIdx.x * lanes + lane_id) % 32;
    if (threadIdx.x % 64 == 0) {
        for (int i = 0; i < iters; ++i) {
            const int s = i % stages;
            const uint32_t ph = (i / stages) & 1;
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], sb);
            const int kb = (i * kbs) % 32;
            const int r0 = region * 256;
            const int pr = rows / nreq;
            for (int q = 0; q < nreq; ++q) tma3d(smem + s * sb + q * pr * 128 * kbs, &tm, &full[s], 0, r0 + q * pr, kb);
        }
    } else if (threadIdx.x % 64 == 32) {
        for (int i = 0; i < iters; ++i) {
            const int s = i % stages;
            const uint32_t ph = (i / stages) & 1;
            if (spin) {
                uint32_t ok = 0;
                while (!ok)
                    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
                                 : "=r"(ok) : "r"(smem_u32(&full[s])), "r"(ph) : "memory");
            } else {
                mbar_wait(&full[s], ph);
            }
            mbar_arrive_local(&empty[s]);
        }
        if (lane_id == 0) out[blockIdx.x] = globaltimer() - t0;
    }
    __syncthreads();
}

int main(int argc, char** argv) {
    EncodeFn fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
    uint8_t* buf;
    const size_t rows_total = 32 * 256, kbt = 32;
    cudaMalloc(&buf, rows_total * kbt * 128);
    cudaMemset(buf, 1, rows_total * kbt * 128);
    unsigned long long* d;
    cudaMalloc(&d, 4096 * 8);
    for (int ai = 1; ai + 4 < argc + 1 && ai < argc; ai += 5) {
        const int rows = atoi(argv[ai]), kbs = atoi(argv[ai + 1]), stages = atoi(argv[ai + 2]), lanes = atoi(argv[ai + 3]),
                  nreq = atoi(argv[ai + 4]) % 10, spin = (atoi(argv[ai + 4]) / 10) % 10, same = atoi(argv[ai + 4]) / 100;
        CUtensorMap m;
        memset(&m, 0, sizeof m);
        cuuint64_t dims[3] = {128, rows_total, kbt}, str[2] = {128, rows_total * 128};
        cuuint32_t box[3] = {128, (cuuint32_t)(rows / nreq), (cuuint32_t)kbs}, es[3] = {1, 1, 1};
        fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int sb = rows * 128 * kbs;
        const int smem = 2048 + lanes * stages * sb + lanes * 256;
        const int ctas = 148;
        cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int iters = 1024 * 1024 * 16 / sb;
        for (int rep = 0; rep < 2; ++rep) stream<<<ctas, 64 * lanes, smem>>>(m, rows, kbs, stages, iters, lanes, nreq, spin, same, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[256];
        cudaMemcpy(h, d, ctas * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < ctas; ++i) avg += h[i];
        avg /= ctas;
        const double per_sm = (double)sb * iters * lanes / avg;
        printf("same %d spin %d lanes %d req %6d B x %d per stage, stages %d: %5.0f ns/stage/lane, %6.1f GB/s/SM, %5.2f TB/s  %s\n", same, spin, lanes,
               sb / nreq, nreq, stages, avg / iters, per_sm, per_sm * ctas / 1e3, cudaGetErrorString(e));
    }
}
