// Microbenchmark 5: aggregate L2 -> SMEM throughput with all SMs streaming L2-resident data,
// unicast vs TMA multicast across a cluster (cs CTAs share every box; each issues 1/cs of it).
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
                                                int iters, int cs, int distinct, unsigned long long* out) {
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
                tma3d(smem + s * sb, &tm, &full[s], 0, r0, kb);
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
            for (int r = 0; r < cs; ++r) mbar_arrive_cluster(mapa_shared(smem_u32(&empty[s]), r));
        }
        out[blockIdx.x] = globaltimer() - t0;
    }
    __syncwarp();
    cluster_sync();
}

int main() {
    EncodeFn fn;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
    uint8_t* buf;
    const size_t rows_total = 32 * 256, kbt = 32;  // 32 regions x 256 rows x 32 k-blocks = 32 MB (L2-resident)
    cudaMalloc(&buf, rows_total * kbt * 128);
    cudaMemset(buf, 1, rows_total * kbt * 128);
    unsigned long long* d;
    cudaMalloc(&d, 4096 * 8);
    struct C {
        int rows, kbs, stages, cs, distinct;
    } cfgs[] = {{128, 2, 4, 1, 1}, {128, 4, 2, 1, 1}, {256, 2, 2, 1, 1}, {128, 2, 4, 2, 1}, {128, 2, 4, 4, 1},
                {128, 2, 4, 8, 1}, {128, 4, 2, 4, 1}, {128, 2, 4, 1, 0}, {128, 2, 4, 4, 0}};
    for (auto c : cfgs) {
        CUtensorMap m;
        memset(&m, 0, sizeof m);
        cuuint64_t dims[3] = {128, rows_total, kbt}, str[2] = {kbt * 128, 128};
        cuuint32_t box[3] = {128, (cuuint32_t)(c.rows / c.cs), (cuuint32_t)c.kbs}, es[3] = {1, 1, 1};
        fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, buf, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int sb = c.rows * 128 * c.kbs;
        const int smem = 2048 + c.stages * sb + 256;
        cudaLaunchConfig_t cfg = {};
        const int ctas = 144;  // multiple of 1,2,4,8 (and 16)
        cfg.gridDim = dim3(ctas);
        cfg.blockDim = dim3(64);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = c.cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        const int iters = 64;
        for (int rep = 0; rep < 2; ++rep) cudaLaunchKernelEx(&cfg, stream, m, c.rows, c.kbs, c.stages, iters, c.cs, c.distinct, d);
        cudaDeviceSynchronize();
        unsigned long long h[256];
        cudaMemcpy(h, d, ctas * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < ctas; ++i) avg += h[i];
        avg /= ctas;
        const double per_sm = (double)sb * iters / avg;
        printf("stage %6d B (rows %3d x kbs %d) stages %d cluster %d distinct %d: %.0f ns/stage, %.1f GB/s/SM recv, "
               "%.2f TB/s recv total, %.2f TB/s from L2  %s\n",
               sb, c.rows, c.kbs, c.stages, c.cs, c.distinct, avg / iters, per_sm, per_sm * ctas / 1e3,
               per_sm * ctas / 1e3 / c.cs, cudaGetErrorString(cudaGetLastError()));
    }
}
