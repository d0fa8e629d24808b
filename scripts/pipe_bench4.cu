// Microbenchmark 4: TMA store / reduce-add throughput per SM vs request size, and whether a 3D
// tensor map with non-monotonic strides (K-blocks of a row-major A) encodes and loads correctly.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>
#include <vector>

#include "ptx.cuh"
using namespace abftk;

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeFn fn;

__global__ void __launch_bounds__(32, 1) stores(const __grid_constant__ CUtensorMap tm, int mode, int nreq, int bw,
                                                int bh, int reps, unsigned long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    for (int i = threadIdx.x; i < 128 * 1024 / 4; i += 32) ((int*)smem)[i] = i;
    fence_proxy_async_smem();
    __syncwarp();
    unsigned long long t0 = globaltimer();
    if (threadIdx.x == 0) {
        for (int r = 0; r < reps; ++r) {
            for (int q = 0; q < nreq; ++q) {
                const int c0 = (q * bw) % 4096, c1 = blockIdx.x * 128 + ((q * bw) / 4096) * bh;
                if (mode == 0)
                    tma_store_2d(&tm, smem + (size_t)q * bw * bh * 4 % (96 * 1024), c0, c1);
                else
                    tma_reduce_add_2d(&tm, smem + (size_t)q * bw * bh * 4 % (96 * 1024), c0, c1);
            }
            bulk_commit();
            bulk_wait<0>();
        }
        out[blockIdx.x] = globaltimer() - t0;
    }
}

__global__ void load3d(const __grid_constant__ CUtensorMap tm, uint8_t* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(&bar, 128 * 8 * 4);
        asm volatile(
            "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
            ::"r"(smem_u32(smem)), "l"((uint64_t)&tm), "r"(smem_u32(&bar)), "r"(0), "r"(0), "r"(1) : "memory");
        mbar_wait(&bar, 0);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < 128 * 8 * 4; i += blockDim.x) out[i] = smem[i];
}

int main() {
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
    // ---- 3D non-monotonic map over a row-major 8 x 1024 byte matrix: {128 B, rows, kblocks}
    {
        uint8_t* A;
        cudaMalloc(&A, 8 * 1024);
        std::vector<uint8_t> h(8 * 1024);
        for (int r = 0; r < 8; ++r)
            for (int c = 0; c < 1024; ++c) h[r * 1024 + c] = (uint8_t)(r * 7 + c);
        cudaMemcpy(A, h.data(), h.size(), cudaMemcpyHostToDevice);
        CUtensorMap m;
        memset(&m, 0, sizeof m);
        cuuint64_t dim[3] = {128, 8, 8}, str[2] = {1024, 128};
        cuuint32_t box[3] = {128, 8, 4}, es[3] = {1, 1, 1};
        CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, A, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        printf("3D non-monotonic encode: %d\n", (int)r);
        if (r == 0) {
            uint8_t* o;
            cudaMalloc(&o, 4096);
            load3d<<<1, 128, 8192>>>(m, o);
            std::vector<uint8_t> g(4096);
            cudaMemcpy(g.data(), o, 4096, cudaMemcpyDeviceToHost);
            int bad = 0;
            for (int kb = 0; kb < 4; ++kb)
                for (int r2 = 0; r2 < 8; ++r2)
                    for (int c = 0; c < 128; ++c)
                        bad += g[(kb * 8 + r2) * 128 + c] != h[r2 * 1024 + (kb + 1) * 128 + c];
            printf("3D load check: %d mismatches (%s)\n", bad, cudaGetErrorString(cudaGetLastError()));
        }
    }
    // ---- stores / reduces
    int* C;
    cudaMalloc(&C, 148ull * 128 * 4096 * 4);
    unsigned long long* d;
    cudaMalloc(&d, 4096 * 8);
    cudaFuncSetAttribute(stores, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Cf {
        int mode, bw, bh, sw, ctas;
    } cfs[] = {{0, 32, 32, 1, 1}, {0, 32, 128, 1, 1}, {0, 128, 128, 0, 1}, {0, 256, 64, 0, 1}, {1, 32, 32, 1, 1},
               {1, 32, 128, 1, 1}, {1, 128, 128, 0, 1}, {0, 32, 32, 1, 148}, {0, 32, 128, 1, 148},
               {0, 128, 128, 0, 148}, {1, 32, 32, 1, 148}, {1, 32, 128, 1, 148}, {1, 128, 128, 0, 148}};
    for (auto c : cfs) {
        CUtensorMap m;
        memset(&m, 0, sizeof m);
        cuuint64_t dim[2] = {4096, 148ull * 128}, str[1] = {4096 * 4};
        cuuint32_t box[2] = {(cuuint32_t)c.bw, (cuuint32_t)c.bh}, es[2] = {1, 1};
        CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_INT32, 2, C, dim, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        c.sw ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        const int tile_bytes = 128 * 1024 * 4 / 4;  // 128 KB tile per rep
        const int req_bytes = c.bw * c.bh * 4;
        const int nreq = tile_bytes / req_bytes;
        const int reps = 8;
        for (int w = 0; w < 2; ++w) stores<<<c.ctas, 32, 200 * 1024>>>(m, c.mode, nreq, c.bw, c.bh, reps, d);
        cudaDeviceSynchronize();
        std::vector<unsigned long long> h(c.ctas);
        cudaMemcpy(h.data(), d, c.ctas * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (auto x : h) avg += x;
        avg /= c.ctas;
        printf("%s box %3dx%3d (%6d B, %2d req/tile) ctas=%3d enc=%d: %.0f ns per 128KB tile, %.1f GB/s/SM, %.2f TB/s  %s\n",
               c.mode ? "reduce" : "store ", c.bw, c.bh, req_bytes, nreq, c.ctas, (int)r, avg / reps,
               (double)tile_bytes * reps / avg, (double)tile_bytes * reps * c.ctas / avg / 1e3,
               cudaGetErrorString(cudaGetLastError()));
    }
}
