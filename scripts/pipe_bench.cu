// Microbenchmark: TMA load pipeline throughput per SM (no MMA), to separate TMA/L2 limits from
// the MMA. Each CTA streams `kb` k-blocks of an A-like tile (rows x 128 B, row stride = ld bytes)
// plus a B-like tile through a ring of `stages` buffers; the consumer releases immediately (or
// after issuing MMAs when mma=1).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2103_00130_b200/csrc scripts/pipe_bench.cu -o scripts/bin/pipe_bench
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <cstring>

#include "ptx.cuh"
using namespace abftk;

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static CUtensorMap mk(void* base, uint64_t inner, uint64_t outer, uint64_t ld, uint32_t bi, uint32_t bo,
                      CUtensorMapL2promotion promo) {
    static EncodeFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void**)&fn, cudaEnableDefault, &q);
    }
    CUtensorMap m;
    memset(&m, 0, sizeof m);
    cuuint64_t d[2] = {inner, outer}, s[1] = {ld};
    cuuint32_t b[2] = {bi, bo}, e[2] = {1, 1};
    CUresult r = fn(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, base, d, s, b, e, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, promo, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r) printf("encode failed %d\n", (int)r);
    return m;
}

template <int BN>
__global__ void __launch_bounds__(128, 1) pipe(const __grid_constant__ CUtensorMap ta, const __grid_constant__ CUtensorMap tb,
                                               int kb, int stages, int mma, int a_rows_per_cta, long long* out) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    const int stage_bytes = 128 * 128 + BN * 128;
    uint64_t* full = (uint64_t*)(smem + stages * stage_bytes);
    uint64_t* empty = full + 8;
    __shared__ uint32_t holder;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    if (threadIdx.x < 32) tmem_alloc<256>(&holder);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = holder;
    long long t0 = clock64();
    const int arow = (blockIdx.x * a_rows_per_cta) % 2048;
    if (threadIdx.x == 32) {
        for (int i = 0; i < kb; ++i) {
            int s = i % stages;
            uint32_t ph = (i / stages) & 1;
            mbar_wait(&empty[s], ph ^ 1);
            mbar_arrive_expect_tx(&full[s], stage_bytes);
            tma_load_2d(smem + s * stage_bytes, &ta, &full[s], i * 128, arow, 0);
            tma_load_2d(smem + s * stage_bytes + 128 * 128, &tb, &full[s], i * 128, blockIdx.x * BN, 0);
        }
    } else if (threadIdx.x == 64) {
        for (int i = 0; i < kb; ++i) {
            int s = i % stages;
            uint32_t ph = (i / stages) & 1;
            mbar_wait(&full[s], ph);
            tc_fence_after();
            if (mma) {
                uint32_t a = smem_u32(smem + s * stage_bytes);
                uint64_t da = umma_desc_sw128(a), db = umma_desc_sw128(a + 128 * 128);
                for (int kk = 0; kk < 4; ++kk) mma_i8(tmem, da + 2 * kk, db + 2 * kk, idesc_u8s8(128, BN), (i | kk) != 0);
                mma_commit(&empty[s]);
            } else {
                asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
            }
        }
        if (mma) {
            mma_commit(&full[7]);
        }
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

template <int BN>
void run(uint8_t* A, uint8_t* B, uint64_t k, int ctas, int stages, int mma, int a_rows_per_cta,
         CUtensorMapL2promotion promo, const char* tag) {
    CUtensorMap ta = mk(A, k, 2048, k, 128, 128, promo);
    CUtensorMap tb = mk(B, k, 8192, k, 128, BN, promo);
    long long* d;
    cudaMalloc(&d, 1024 * 8);
    int smem = 1024 + stages * (128 * 128 + BN * 128) + 256;
    cudaFuncSetAttribute(pipe<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int kb = (int)(k / 128);
    pipe<BN><<<ctas, 128, smem>>>(ta, tb, kb, stages, mma, a_rows_per_cta, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    pipe<BN><<<ctas, 128, smem>>>(ta, tb, kb, stages, mma, a_rows_per_cta, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[1024];
    cudaMemcpy(h, d, ctas * 8, cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < ctas; ++i) avg += h[i];
    avg /= ctas;
    double bytes = (double)kb * (128 * 128 + BN * 128);
    printf("%-10s BN=%3d k=%5llu ctas=%3d stages=%d mma=%d promo=%d: %.0f cyc/kblock, %.1f B/clk/SM, kernel %.2f us "
           "(%.1f TB/s total) %s\n",
           tag, BN, (unsigned long long)k, ctas, stages, mma, (int)promo, avg / kb, bytes / avg * 1.0, ms * 1e3,
           bytes * ctas / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    uint8_t *A, *B;
    cudaMalloc(&A, 2048ull * 16384);
    cudaMalloc(&B, 8192ull * 16384);
    cudaMemset(A, 1, 2048ull * 16384);
    cudaMemset(B, 1, 8192ull * 16384);
    auto P256 = CU_TENSOR_MAP_L2_PROMOTION_L2_256B, PNONE = CU_TENSOR_MAP_L2_PROMOTION_NONE;
    for (uint64_t k : {2048ull, 4096ull, 8192ull}) {
        run<64>(A, B, k, 128, 7, 0, 128, P256, "tma-only");
        run<256>(A, B, k, 128, 4, 0, 128, P256, "tma-only");
        run<64>(A, B, k, 128, 7, 1, 128, P256, "tma+mma");
        run<256>(A, B, k, 128, 4, 1, 128, P256, "tma+mma");
    }
    run<64>(A, B, 4096, 128, 7, 0, 128, PNONE, "nopromo");
    run<256>(A, B, 4096, 128, 4, 0, 128, PNONE, "nopromo");
    run<64>(A, B, 4096, 128, 2, 0, 128, P256, "2stage");
    run<64>(A, B, 4096, 128, 4, 0, 128, P256, "4stage");
    run<64>(A, B, 4096, 1, 7, 0, 128, P256, "1cta");
    run<256>(A, B, 4096, 1, 4, 0, 128, P256, "1cta");
    run<256>(A, B, 4096, 148, 4, 1, 128, P256, "148");
    return 0;
}
