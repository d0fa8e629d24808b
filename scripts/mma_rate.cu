// Microbenchmark: sustained tcgen05.mma issue rate per SM for int8 / f16 kinds and several N.
// One CTA per SM, one thread issues `iters` MMAs on the same smem operands, commit, wait.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I paper_2103_00130_b200/csrc scripts/mma_rate.cu
#include <cstdio>
#include <cuda_runtime.h>

#include "ptx.cuh"
using namespace abftk;

template <int KIND, int N>  // KIND 0 = i8 (K=32 B), 1 = f16 (K=16 elems = 32 B)
__global__ void __launch_bounds__(128, 1) mma_rate(int iters, long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
    for (int i = threadIdx.x; i < (128 + 256) * 128; i += blockDim.x) base[i] = 1;
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) tmem_alloc<256>(&holder);
    asm volatile("fence.proxy.async.shared::cta;");
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = holder;
    if (threadIdx.x == 0) {
        const uint32_t a = smem_u32(base), b = a + 128 * 128;
        const uint64_t da = umma_desc_sw128(a), db = umma_desc_sw128(b);
        uint32_t idesc;
        if (KIND == 0)
            idesc = idesc_u8s8(128, N);
        else  // kind::f16: D f32 (bit 4 = 1), A/B f16 (0), K-major
            idesc = (1u << 4) | ((N >> 3) << 17) | ((128 >> 4) << 24);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int kk = i & 3;
            if (KIND == 0)
                mma_i8(tmem, da + 2 * kk, db + 2 * kk, idesc, 1);
            else
                asm volatile(
                    "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                    "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                    "l"(da + 2 * kk), "l"(db + 2 * kk), "r"(idesc), "r"(1)
                    : "memory");
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    tc_fence_before();
    __syncthreads();
    if (threadIdx.x < 32) {
        tc_fence_after();
        tmem_dealloc<256>(tmem);
    }
}

template <int KIND, int N>
void run(int sms) {
    long long* d;
    cudaMalloc(&d, sms * sizeof(long long));
    auto k = mma_rate<KIND, N>;
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int iters = 4096;
    k<<<sms, 128, 100 * 1024>>>(64, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<sms, 128, 100 * 1024>>>(iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h[256];
    cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
    double macs_per_mma = 128.0 * N * (KIND == 0 ? 32 : 16);
    double cyc = (double)h[0] / iters;
    double tot = macs_per_mma * iters * sms * 2 / (ms * 1e-3);
    printf("kind=%s N=%d: %.1f cycles/MMA -> %.0f MAC/clk/SM ; grid=%d wall %.3f ms -> %.1f T(FL)OPS  err=%s\n",
           KIND == 0 ? "i8 " : "f16", N, cyc, macs_per_mma / cyc, sms, ms, tot / 1e12,
           cudaGetErrorString(cudaGetLastError()));
    cudaFree(d);
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    run<0, 256>(sms);
    run<0, 128>(sms);
    run<0, 64>(sms);
    run<1, 256>(sms);
    run<1, 128>(sms);
    run<0, 256>(1);
    run<1, 256>(1);
    return 0;
}
