// Microbenchmark 7: aggregate L2 -> SMEM TMA throughput vs bytes per request, requests per stage and
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

// Each "stage" = box {128, rows, kbs} = rows*128*kbs bytes. Cluster of cs CTAs: CTA r loads rows
// [r*rows/cs, (r+1)*rows/cs) and multicasts to all; every CTA's full barrier expects the full stage.
// Empty barriers: a stage slot may be refilled only when all cs CTAs released it.
__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap tm, int rows, int kbs, int stages,
                                                int iters, int cs, int distinct, int nreq, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    const int sb = rows * 128 * kbs;
    uint64_t* full = (uint64_t*)(smem + stages * sb);
    uint64_t* empty = full + 8;
    const uint32_t rank = cluster_ctarank();
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], cs);
        }
        fence_mbar_init();
    }
    cluster_sync();
    unsigned long long t0 = globaltimer();
    const int cluster = blockIdx.x / cs;
    const int region = distinct ? cluster % 32 : 0;
    if (threadIdx.x == 0) {
        for (int i = 0; i < iters; ++i) {
            const int s = i % stages;
            const uint32_t ph = (i / stages) & 1;
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], sb);
            const int kb = (i * kbs) % 32;
            const int r0 = region * 256;
            if (cs == 1) {
                const int pr = rows / nreq;
                for (int q = 0; q < nreq; ++q) tma3d(smem + s * sb + q * pr * 128 * kbs, &tm, &full[s], 0, r0 + q * pr, kb);
            } else {
                const int part = rows / cs;
                // a part of rows: box rows == rows/cs (tensor map built with that box)
                tma3d_mc(smem + s * sb + rank * part * 128, &tm, &full[s], 0, r0 + rank * part, kb,
                         (uint16_t)((1u << cs) - 1));
            }
        }
    } else if (threadIdx.x == 32) {
        for (int i = 0; i < iters; ++i) {
            const int s = i % stages;
            const uint32_t ph = (i / stages) & 1;
            mbar_wait(&full[s], ph);
            // release the slot in every CTA of the cluster
            if (cs == 1) mbar_arrive_local(&empty[s]);
            else for (int r = 0; r < cs; ++r) mbar_arrive_cluster(mapa_shared(smem_u32(&empty[s]), r));
        }
        out[blockIdx.x] = globaltimer() - t0;
    }
    __syncwarp();
    cluster_sync();
}

int main(int argc, char** argv) {
    EncodeFn fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
    uint8_t* buf;
    const size_t rows_total = 32 * 256, kbt = 32;  // 32 MB, L2-resident
    cudaMalloc(&buf, rows_total * kbt * 128);
    cudaMemset(buf, 1, rows_total * kbt * 128);
    unsigned long long* d;
    cudaMalloc(&d, 4096 * 8);
    for (int ai = 1; ai + 4 < argc + 1 && ai < argc; ai += 5) {
        const int rows = atoi(argv[ai]), kbs = atoi(argv[ai + 1]), stages = atoi(argv[ai + 2]), nreq = atoi(argv[ai + 3]), layout = atoi(argv[ai + 4]);
        const int cs = 1, distinct = 1;
        CUtensorMap m;
        memset(&m, 0, sizeof m);
        cuuint64_t dims[3] = {128, rows_total, kbt}, str[2] = {kbt * 128, 128};
        if (layout == 1) {  // K-block-major (B' style): rows contiguous inside a k-block
            str[0] = 128;
            str[1] = rows_total * 128;
        }
        cuuint32_t box[3] = {128, (cuuint32_t)(rows / nreq), (cuuint32_t)kbs}, es[3] = {1, 1, 1};
        fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int sb = rows * 128 * kbs;
        const int smem = 2048 + stages * sb + 256;
        cudaLaunchConfig_t cfg = {};
        const int ctas = 148;
        cfg.gridDim = dim3(ctas);
        cfg.blockDim = dim3(64);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 1;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int iters = 2 * 1024 * 1024 * 16 / sb;  // ~32 MB per CTA
        for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, stream, m, rows, kbs, stages, iters, cs, distinct, nreq, d);
        cudaError_t e = cudaDeviceSynchronize();
        unsigned long long h[256];
        cudaMemcpy(h, d, ctas * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < ctas; ++i) avg += h[i];
        avg /= ctas;
        const double per_sm = (double)sb * iters / avg;
        printf("layout %d req %6d B x %d per stage, stages %d (%6d B in flight max): %5.0f ns/stage, %6.1f GB/s/SM, %5.2f TB/s  %s\n",
               layout, sb / nreq, nreq, stages, sb * stages, avg / iters, per_sm, per_sm * ctas / 1e3, cudaGetErrorString(e));
    }
}
