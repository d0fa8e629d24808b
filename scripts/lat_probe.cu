// Dependent-chain latency of DADD / FADD2-style FP32 add / LDS on one warp (clock64).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(double* out, float* outf, long long* cyc, double x, float y) {
    __shared__ float sm[64];
    sm[threadIdx.x & 63] = y;
    __syncthreads();
    double a = x;
    long long t0 = clock64();
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) a = __dadd_rn(a, x);
    long long t1 = clock64();
    float f = y;
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) f = __fadd_rn(f, y);
    long long t2 = clock64();
    int idx = threadIdx.x & 31;
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) idx = __float_as_int(sm[idx]) & 31;
    long long t3 = clock64();
    out[threadIdx.x] = a;
    outf[threadIdx.x] = f + idx;
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; }
}
int main() {
    double* o; float* of; long long* c;
    cudaMalloc(&o, 256 * 8); cudaMalloc(&of, 256 * 4); cudaMalloc(&c, 64);
    for (int r = 0; r < 2; ++r) k<<<1, 32>>>(o, of, c, 1.000001, 0.0f);
    long long h[3];
    cudaMemcpy(h, c, 24, cudaMemcpyDeviceToHost);
    printf("DADD chain %.1f cyc/op, FADD chain %.1f cyc/op, LDS chain %.1f cyc/op\n", h[0] / 1024.0, h[1] / 1024.0, h[2] / 1024.0);
}
