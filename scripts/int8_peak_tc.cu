// Measured int8 tensor roof of this B200: tcgen05.mma.cta_group::2.kind::i8 (M=256, N=256, K=32) issued
// back to back by one thread per CTA pair on all 74 pairs, operands random bytes resident in shared memory
// (no memory traffic: the tensor pipe's own rate, under the power cap the data pattern implies).
//   burst:     one launch of ~5 ms, CUDA events
//   sustained: launches back to back for >= 4 s, total ops / total time
// Output: one JSON line. Used by scripts/int8_peak.py (which adds cuBLASLt int8) -> profiles/r02/int8_peak.json.
#include <cuda_runtime.h>

#include <chrono>
#include <cstdio>

#include "ptx.cuh"
using namespace abftk;

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) mma_loop(int iters, uint32_t seed, int* sink) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ uint64_t bar;
    __shared__ uint32_t holder;
    uint8_t* base = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    // random operand bytes (A: 128 rows x 128 B, B: 128 rows x 128 B per CTA), xorshift per thread
    uint32_t x = seed ^ (threadIdx.x * 0x9E3779B9u) ^ (blockIdx.x * 0x85EBCA6Bu);
    for (int i = threadIdx.x; i < (128 + 128) * 128 / 4; i += blockDim.x) {
        x ^= x << 13;
        x ^= x >> 17;
        x ^= x << 5;
        reinterpret_cast<uint32_t*>(base)[i] = x;
    }
    uint32_t rank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (threadIdx.x < 32) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&holder)),
                     "n"(256)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    asm volatile("fence.proxy.async.shared::cta;");
    tc_fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    tc_fence_after();
    const uint32_t tmem = holder;
    if (rank == 0 && threadIdx.x == 0) {
        const uint32_t a = smem_u32(base), b = a + 128 * 128;
        const uint64_t da = umma_desc_sw128(a), db = umma_desc_sw128(b);
        constexpr uint32_t idesc = idesc_u8s8(256, 256);
        for (int i = 0; i < iters; ++i) {
            const int kk = i & 3;
            asm volatile(
                "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
                "tcgen05.mma.cta_group::2.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
                "l"(da + 2 * kk), "l"(db + 2 * kk), "r"(idesc), "r"(i & 1023)
                : "memory");
        }
        asm volatile(
            "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
                smem_u32(&bar)),
            "h"((uint16_t)3)
            : "memory");
        mbar_wait(&bar, 0);
    }
    if (rank == 1 && threadIdx.x == 0) mbar_wait(&bar, 0);
    tc_fence_before();
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x < 32) {
        tc_fence_after();
        uint32_t v;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(v) : "r"(tmem));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (v == 0x7fffffffu) atomicAdd(sink, 1);  // keep the accumulator live
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(256) : "memory");
    }
}

int main() {
    int dev = 0, sms = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int pairs = sms / 2;
    int* sink;
    cudaMalloc(&sink, 4);
    const int smem = 1024 + 2 * 128 * 128;
    cudaFuncSetAttribute(mma_loop, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const double ops_per_mma = 2.0 * 256 * 256 * 32;  // per pair instruction
    auto launch = [&](int iters, uint32_t seed) { mma_loop<<<2 * pairs, 128, smem>>>(iters, seed, sink); };
    launch(1024, 1);
    cudaDeviceSynchronize();
    // burst: one ~5 ms launch after an idle second (the GPU starts cool / uncapped)
    const int burst_iters = 60000;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    double burst = 0;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(e0);
        launch(burst_iters, 7 + r);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double t = ops_per_mma * burst_iters * pairs / (ms * 1e-3) / 1e12;
        if (t > burst) burst = t;
    }
    // sustained: back-to-back launches for >= 4 s
    const auto w0 = std::chrono::steady_clock::now();
    cudaEventRecord(e0);
    long long total = 0;
    int launches = 0;
    while (std::chrono::duration<double>(std::chrono::steady_clock::now() - w0).count() < 4.0) {
        for (int q = 0; q < 20; ++q) launch(burst_iters, 100 + launches++);
        total += 20ll * burst_iters;
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
    }
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double sustained = ops_per_mma * total * pairs / (ms * 1e-3) / 1e12;
    printf("{\"tcgen05_i8_burst_tops\": %.1f, \"tcgen05_i8_sustained_tops\": %.1f, \"sustained_s\": %.2f, "
           "\"pairs\": %d, \"shape\": \"cta_group::2 M=256 N=256 K=32, random smem operands\", \"err\": \"%s\"}\n",
           burst, sustained, ms * 1e-3, pairs, ops_per_mma > 0 ? cudaGetErrorString(cudaGetLastError()) : "");
    return 0;
}
