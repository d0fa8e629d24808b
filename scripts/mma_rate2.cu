// Microbenchmark: tcgen05.mma.cta_group::2 (CTA pair, M=256) kind::i8 issue rate vs N.
#include <cuda_runtime.h>

#include <cstdio>

#include "ptx.cuh"
using namespace abftk;

__device__ __forceinline__ uint32_t cluster_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma2(int iters, long long* cycles) {
    extern __shared__ __align__(1024) uint8_t smem[];
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem) + 1023) & ~uintptr_t(1023));
    for (int i = threadIdx.x; i < (128 + 256) * 128; i += blockDim.x) base[i] = 1;
    const uint32_t rank = cluster_rank();
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&holder)),
                     "n"(256) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem = holder;
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t a = smem_u32(base), b = a + 128 * 128;
        const uint64_t da = umma_desc_sw128(a), db = umma_desc_sw128(b);
        const uint32_t idesc = idesc_u8s8(256, N);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            const int kk = i & 3;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                "l"(da + 2 * kk), "l"(db + 2 * kk), "r"(idesc), "r"(1)
                : "memory");
        }
        asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                     ::"r"(smem_u32(&bar)), "h"((uint16_t)3) : "memory");
        mbar_wait(&bar, 0);
        cycles[blockIdx.x / 2] = clock64() - t0;
    }
    if (rank == 1 && threadIdx.x == 0) mbar_wait(&bar, 0);
    tc_fence_before();
    cluster_sync();
    if (threadIdx.x < 32) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256) : "memory");
    }
}

template <int N>
void run(int pairs) {
    long long* d;
    cudaMalloc(&d, pairs * 8);
    cudaFuncSetAttribute(mma2<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024);
    const int iters = 4096;
    mma2<N><<<2 * pairs, 128, 100 * 1024>>>(64, d);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    mma2<N><<<2 * pairs, 128, 100 * 1024>>>(iters, d);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    long long h;
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    const double cyc = (double)h / iters;
    const double macs_sm = 128.0 * N * 32;  // per SM per instruction
    printf("cta_group::2 i8 M=256 N=%3d pairs=%2d: %.1f cycles/MMA -> %.0f MAC/clk/SM; %.0f TOPS  %s\n", N, pairs, cyc,
           macs_sm / cyc, 2.0 * 256 * N * 32 * iters * pairs / (ms * 1e-3) / 1e12, cudaGetErrorString(cudaGetLastError()));
}

int main() {
    run<32>(74);
    run<64>(74);
    run<128>(74);
    run<256>(74);
    run<64>(1);
}
