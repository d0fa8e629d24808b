// Microbenchmark 3: where does the ~325 ns/stage single-CTA floor come from?
// wait 0: mbarrier.try_wait loop; 1: mbarrier.test_wait spin; 2: try_wait with suspend hint 0
// upfront 1: all loads issued at once into distinct buffers (no ring reuse), timestamps per arrival.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "ptx.cuh"
using namespace abftk;

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     smem_u32(dst)),
                 "l"(src), "r"(bytes), "r"(smem_u32(bar))
                 : "memory");
}
__device__ __forceinline__ bool test_wait(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(parity) : "memory");
    return ok;
}
__device__ __forceinline__ bool try_wait_hint(uint32_t bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n\tselp.u32 %0,1,0,p;\n\t}"
                 : "=r"(ok) : "r"(bar), "r"(parity), "r"(0) : "memory");
    return ok;
}
__device__ __forceinline__ void wait(uint64_t* b, uint32_t ph, int mode) {
    uint32_t a = smem_u32(b);
    if (mode == 0) while (!mbar_try_wait(a, ph)) {}
    else if (mode == 1) while (!test_wait(a, ph)) {}
    else while (!try_wait_hint(a, ph)) {}
}

__global__ void __launch_bounds__(64, 1) k(const uint8_t* src, int sb, int kb, int stages, int wmode, int upfront,
                                           unsigned long long* out, unsigned long long* stamps) {
    extern __shared__ uint8_t raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)raw + 1023) & ~uintptr_t(1023));
    uint64_t* full = (uint64_t*)(smem + stages * sb);
    uint64_t* empty = full + 32;
    if (threadIdx.x == 0) {
        for (int s = 0; s < stages; ++s) {
            mbar_init(&full[s], 1);
            mbar_init(&empty[s], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    unsigned long long t0 = globaltimer();
    const uint8_t* base = src + (uint64_t)blockIdx.x * kb * sb;
    if (threadIdx.x == 0) {
        for (int i = 0; i < kb; ++i) {
            int s = i % stages;
            uint32_t ph = (i / stages) & 1;
            if (!upfront) wait(&empty[s], ph ^ 1, wmode);
            mbar_arrive_expect_tx(&full[s], sb);
            bulk_load(smem + s * sb, base + (uint64_t)i * sb, sb, &full[s]);
        }
    } else if (threadIdx.x == 32) {
        for (int i = 0; i < kb; ++i) {
            int s = i % stages;
            uint32_t ph = (i / stages) & 1;
            wait(&full[s], ph, wmode);
            if (stamps && blockIdx.x == 0 && i < 64) stamps[i] = globaltimer() - t0;
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
        }
        out[blockIdx.x] = globaltimer() - t0;
    }
}

int main() {
    uint8_t* buf;
    const size_t bytes = 1024ull << 20;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    unsigned long long *d, *st;
    cudaMalloc(&d, 4096 * 8);
    cudaMalloc(&st, 64 * 8);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024);
    struct C {
        int sb, kb, stages, wmode, upfront, ctas;
    } cs[] = {{32768, 32, 6, 0, 0, 1}, {32768, 32, 6, 1, 0, 1}, {32768, 32, 6, 2, 0, 1}, {32768, 6, 6, 0, 1, 1},
              {16384, 12, 12, 0, 1, 1}, {8192, 24, 24, 0, 1, 1}, {32768, 6, 6, 1, 1, 1}, {49152, 4, 4, 0, 1, 1},
              {65536, 3, 3, 0, 1, 1}, {32768, 32, 6, 1, 0, 148}, {32768, 32, 6, 0, 0, 148}};
    for (auto c : cs) {
        for (int r = 0; r < 2; ++r)
            k<<<c.ctas, 64, 220 * 1024>>>(buf + (r ? 0 : (512ull << 20)), c.sb, c.kb, c.stages, c.wmode, c.upfront, d,
                                        r ? st : nullptr);
        cudaDeviceSynchronize();
        unsigned long long h[256], s[64];
        cudaMemcpy(h, d, c.ctas * 8, cudaMemcpyDeviceToHost);
        cudaMemcpy(s, st, 64 * 8, cudaMemcpyDeviceToHost);
        double avg = 0;
        for (int i = 0; i < c.ctas; ++i) avg += h[i];
        avg /= c.ctas;
        printf("sb=%6d kb=%2d stages=%2d wait=%d upfront=%d ctas=%3d: %.0f ns/stage %.1f GB/s/SM  arrivals(ns):", c.sb,
               c.kb, c.stages, c.wmode, c.upfront, c.ctas, avg / c.kb, (double)c.sb * c.kb / avg);
        for (int i = 0; i < (c.kb < 8 ? c.kb : 8); ++i) printf(" %llu", s[i]);
        printf("  %s\n", cudaGetErrorString(cudaGetLastError()));
    }
}
