// Pipelined random-row gather floor: each warp keeps S chunks of 32 rows (128 B each) in flight, via TMA
// tile::gather4 (one instruction per 4 rows, mbarrier completion) or cp.async (16 B per lane-op, group
// waits). usage: gather4_probe2 rows n stages blocks_per_sm
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

template <int S>
__global__ void __launch_bounds__(128) g4_kernel(const __grid_constant__ CUtensorMap m, const int* __restrict__ idx,
                                                 long long n, unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char dyn[];
    __shared__ __align__(8) unsigned long long bar[4][S];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* buf = dyn + w * S * 4096;
    if (lane < S) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[w][lane])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    unsigned long long acc = 0;
    const long long gw = (long long)blockIdx.x * 4 + w, nw = (long long)gridDim.x * 4;
    const long long nch = (n + 31) / 32;
    auto issue = [&](long long ch, int slot) {
        const long long c = ch * 32;
        const int ix = c + lane < n ? idx[c + lane] : 0;
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[w][slot])), "r"(32 * 128)
                         : "memory");
        int rr[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) rr[q] = __shfl_sync(0xffffffffu, ix, (lane & ~3) + q);
        __syncwarp();
        if ((lane & 3) == 0)
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, "
                "%4, %5, %6}], [%7];" ::"r"(smem_u32(buf + slot * 4096 + (lane >> 2) * 512)),
                "l"(&m), "r"(0), "r"(rr[0]), "r"(rr[1]), "r"(rr[2]), "r"(rr[3]), "r"(smem_u32(&bar[w][slot]))
                : "memory");
    };
    long long ch = gw;
    int k = 0;
    for (int s = 0; s < S - 1; ++s)
        if (gw + s * nw < nch) issue(gw + s * nw, s);
    unsigned phases = 0;
    for (; ch < nch; ch += nw, ++k) {
        const long long nx = ch + (S - 1) * nw;
        if (nx < nch) issue(nx, (k + S - 1) % S);
        const int slot = k % S;
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(
                         smem_u32(&bar[w][slot])),
                     "r"((phases >> slot) & 1u)
                     : "memory");
        phases ^= 1u << slot;
        const unsigned char* row = buf + slot * 4096 + lane * 128;
        unsigned s = 0;
        for (int e = 0; e < 128; e += 4) s += *reinterpret_cast<const unsigned*>(row + ((e + 4 * lane) & 127)) & 0xFFu;
        if (ch * 32 + lane < n) acc += s;
        __syncwarp();
    }
    atomicAdd(out, acc);
}

template <int S>
__global__ void __launch_bounds__(128) cpa_kernel(const unsigned char* __restrict__ tab, const int* __restrict__ idx,
                                                  long long n, unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char dyn[];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* buf = dyn + w * S * 4096;
    unsigned long long acc = 0;
    const long long gw = (long long)blockIdx.x * 4 + w, nw = (long long)gridDim.x * 4;
    const long long nch = (n + 31) / 32;
    auto issue = [&](long long ch, int slot) {
        if (ch < nch) {
            const long long c = ch * 32;
            const int ix = c + lane < n ? idx[c + lane] : 0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const int piece = lane + 32 * i, r = piece >> 3, q = piece & 7;
                const int rix = __shfl_sync(0xffffffffu, ix, r);
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(buf + slot * 4096 + r * 128 + q * 16)),
                             "l"(tab + (long long)rix * 128 + q * 16)
                             : "memory");
            }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int k = 0;
    for (int s = 0; s < S - 1; ++s) issue(gw + s * nw, s);
    for (long long ch = gw; ch < nch; ch += nw, ++k) {
        issue(ch + (S - 1) * nw, (k + S - 1) % S);
        asm volatile("cp.async.wait_group %0;" ::"n"(S - 1) : "memory");
        __syncwarp();
        const unsigned char* row = buf + (k % S) * 4096 + lane * 128;
        unsigned s = 0;
        for (int e = 0; e < 128; e += 4) s += *reinterpret_cast<const unsigned*>(row + ((e + 4 * lane) & 127)) & 0xFFu;
        if (ch * 32 + lane < n) acc += s;
        __syncwarp();
    }
    atomicAdd(out, acc);
}


template <int S>
__global__ void __launch_bounds__(128) bulk_kernel(const unsigned char* __restrict__ tab, const int* __restrict__ idx,
                                                   long long n, unsigned long long* out) {
    extern __shared__ __align__(1024) unsigned char dyn[];
    __shared__ __align__(8) unsigned long long bar[4][S];
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    unsigned char* buf = dyn + w * S * 4096;
    if (lane < S) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_u32(&bar[w][lane])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    unsigned long long acc = 0;
    const long long gw = (long long)blockIdx.x * 4 + w, nw = (long long)gridDim.x * 4;
    const long long nch = (n + 31) / 32;
    auto issue = [&](long long ch, int slot) {
        const long long c = ch * 32;
        const int ix = c + lane < n ? idx[c + lane] : 0;
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[w][slot])), "r"(32 * 128)
                         : "memory");
        __syncwarp();
        asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 128, [%2];"
                     ::"r"(smem_u32(buf + slot * 4096 + lane * 128)), "l"(tab + (long long)ix * 128),
                       "r"(smem_u32(&bar[w][slot]))
                     : "memory");
    };
    int k = 0;
    for (int s = 0; s < S - 1; ++s)
        if (gw + s * nw < nch) issue(gw + s * nw, s);
    unsigned phases = 0;
    for (long long ch = gw; ch < nch; ch += nw, ++k) {
        const long long nx = ch + (S - 1) * nw;
        if (nx < nch) issue(nx, (k + S - 1) % S);
        const int slot = k % S;
        asm volatile("{ .reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1; @!p bra W; }" ::"r"(
                         smem_u32(&bar[w][slot])),
                     "r"((phases >> slot) & 1u)
                     : "memory");
        phases ^= 1u << slot;
        const unsigned char* row = buf + slot * 4096 + lane * 128;
        unsigned s = 0;
        for (int e = 0; e < 128; e += 4) s += *reinterpret_cast<const unsigned*>(row + ((e + 4 * lane) & 127)) & 0xFFu;
        if (ch * 32 + lane < n) acc += s;
        __syncwarp();
    }
    atomicAdd(out, acc);
}

template <int S>
void run(const CUtensorMap& m, unsigned char* tab, int* idx, long long n, unsigned long long* out, int bps,
         unsigned long long ref) {
    const int smem = 4 * S * 4096;
    cudaFuncSetAttribute(g4_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(cpa_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(bulk_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int kind = 0; kind < 3; ++kind) {
        float best = 1e30f; unsigned long long got = 0;
        for (int rep = 0; rep < 4; ++rep) {
            cudaMemset(out, 0, 8);
            cudaEventRecord(e0);
            if (kind == 0) g4_kernel<S><<<148 * bps, 128, smem>>>(m, idx, n, out);
            else if (kind == 1) cpa_kernel<S><<<148 * bps, 128, smem>>>(tab, idx, n, out);
            else bulk_kernel<S><<<148 * bps, 128, smem>>>(tab, idx, n, out);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms; cudaEventElapsedTime(&ms, e0, e1);
            if (rep && ms < best) best = ms;
            cudaMemcpy(&got, out, 8, cudaMemcpyDeviceToHost);
        }
        printf("S=%d bps=%d %s: %.2f us %.2f TB/s %s (%s)\n", S, bps, kind == 0 ? "gather4" : kind == 1 ? "cp.async" : "bulk1d", best * 1e3,
               n * 128.0 / (best * 1e-3) / 1e12, got == ref ? "OK" : "MISMATCH", cudaGetErrorString(cudaGetLastError()));
    }
}

int main(int argc, char** argv) {
    const long long R = atoll(argv[1]), n = atoll(argv[2]);
    std::vector<unsigned char> h(R * 128);
    unsigned long long x = 88172645463325252ull;
    for (auto& v : h) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; v = (unsigned char)x; }
    std::vector<int> hi(n);
    const int zipf = argc > 3 ? atoi(argv[3]) : 0;  // D5-like: 8 tables of R/8 rows, Zipf(1.05) ranks, permuted
    if (!zipf) {
        for (auto& v : hi) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; v = (int)(x % R); }
    } else {
        const long long T = 8, Rt = R / T;
        std::vector<double> cdf(Rt);
        double acc = 0;
        for (long long r = 0; r < Rt; ++r) cdf[r] = (acc += std::pow((double)(r + 1), -1.05));
        std::vector<int> perm(Rt);
        for (long long r = 0; r < Rt; ++r) perm[r] = (int)r;
        for (long long r = Rt - 1; r > 0; --r) { x ^= x << 13; x ^= x >> 7; x ^= x << 17; std::swap(perm[r], perm[x % (r + 1)]); }
        for (long long i = 0; i < n; ++i) {
            x ^= x << 13; x ^= x >> 7; x ^= x << 17;
            const double u = (double)(x >> 11) / 9007199254740992.0 * acc;
            const long long r = std::lower_bound(cdf.begin(), cdf.end(), u) - cdf.begin();
            hi[i] = (int)((i * T / n) * Rt + perm[std::min(r, Rt - 1)]);
        }
    }
    unsigned long long ref = 0;
    for (long long i = 0; i < n; ++i)
        for (int e = 0; e < 128; e += 4) ref += h[(long long)hi[i] * 128 + e];
    unsigned char* tab; int* idx; unsigned long long* out;
    cudaMalloc(&tab, R * 128); cudaMalloc(&idx, n * 4); cudaMalloc(&out, 8);
    cudaMemcpy(tab, h.data(), R * 128, cudaMemcpyHostToDevice);
    cudaMemcpy(idx, hi.data(), n * 4, cudaMemcpyHostToDevice);
    CUtensorMap m;
    cuuint64_t dims[2] = {128, (cuuint64_t)R};
    cuuint64_t strides[1] = {128};
    cuuint32_t box[2] = {128, 1};
    cuuint32_t es[2] = {1, 1};
    cuTensorMapEncodeTiled(&m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, tab, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    for (int bps : {2, 4, 8}) {
        run<2>(m, tab, idx, n, out, bps, ref);
        run<4>(m, tab, idx, n, out, bps, ref);
        if (bps <= 4) run<8>(m, tab, idx, n, out, bps, ref);
    }
    return 0;
}
