// Microbenchmark 6: DSMEM exchange throughput inside a cluster (split-K partial reduction model).
// Every CTA of a cluster of cs sends `per_peer` bytes to each of its cs-1 peers per iteration.
//   mode 0: st.shared::cluster.v4 from registers (all threads), cluster barrier per iteration
//   mode 1: cp.async.bulk smem -> peer smem (one thread issues), mbarrier complete_tx at the receiver
// Grid fills the GPU with clusters. Prints the median per-SM send rate (bytes / ns).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ptx.cuh"
using namespace abftk;

__device__ __forceinline__ void st_cluster_v4(uint32_t addr, uint4 v) {
    asm volatile("st.shared::cluster.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w)
                 : "memory");
}
__device__ __forceinline__ void bulk_s2c(uint32_t dst_cluster, uint32_t src, uint32_t bytes, uint32_t bar_cluster) {
    asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                     dst_cluster),
                 "r"(src), "r"(bytes), "r"(bar_cluster)
                 : "memory");
}

__global__ void __launch_bounds__(256, 1) xchg(int mode, int per_peer, int iters, unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint32_t csize;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(csize));
    const uint32_t rank = cluster_ctarank();
    // layout: [send buffer per_peer][recv slots (csize-1) * per_peer][barrier]
    uint8_t* send = smem;
    uint8_t* recv = smem + per_peer;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + per_peer * csize);
    if (threadIdx.x == 0) {
        mbar_init(bar, 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x * 16; i < per_peer; i += 256 * 16)
        *reinterpret_cast<uint4*>(send + i) = make_uint4(i, rank, 1, 2);
    __syncthreads();
    cluster_sync();
    const unsigned long long t0 = globaltimer();
    for (int it = 0; it < iters; ++it) {
        if (mode == 0) {
            for (uint32_t d = 1; d < csize; ++d) {
                const uint32_t peer = (rank + d) % csize;
                const uint32_t slot = (rank + csize - peer - 1) % csize;  // distinct slot per sender at receiver
                const uint32_t base = mapa_shared(smem_u32(recv + slot * per_peer), peer);
                for (int i = threadIdx.x * 16; i < per_peer; i += 256 * 16)
                    st_cluster_v4(base + i, *reinterpret_cast<const uint4*>(send + i));
            }
            cluster_sync();
        } else {
            if (threadIdx.x == 0) mbar_arrive_expect_tx(bar, per_peer * (csize - 1));
            cluster_sync();  // expectations are armed everywhere
            if (threadIdx.x == 0) {
                for (uint32_t d = 1; d < csize; ++d) {
                    const uint32_t peer = (rank + d) % csize;
                    const uint32_t slot = (rank + csize - peer - 1) % csize;
                    const uint32_t dst = mapa_shared(smem_u32(recv + slot * per_peer), peer);
                    const uint32_t pbar = mapa_shared(smem_u32(bar), peer);
                    for (int off = 0; off < per_peer; off += 32768) {
                        const int b = min(32768, per_peer - off);
                        bulk_s2c(dst + off, smem_u32(send + off), b, pbar);
                    }
                }
            }
            mbar_wait(bar, it & 1);
        }
    }
    cluster_sync();
    const unsigned long long t1 = globaltimer();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}

int main(int argc, char** argv) {
    const int cs = argc > 1 ? atoi(argv[1]) : 4;
    const int per_peer = argc > 2 ? atoi(argv[2]) : 32768;
    const int iters = argc > 3 ? atoi(argv[3]) : 20;
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int smem = per_peer * cs + 1024;
    cudaFuncSetAttribute(xchg, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    if (cs > 8) cudaFuncSetAttribute(xchg, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    int nclusters = 0;
    cfg.gridDim = dim3(cs);
    cudaOccupancyMaxActiveClusters(&nclusters, xchg, &cfg);
    const int grid = nclusters * cs;
    cfg.gridDim = dim3(grid);
    unsigned long long* d;
    cudaMalloc(&d, grid * 8);
    for (int mode = 0; mode < 2; ++mode) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaLaunchKernelEx(&cfg, xchg, mode, per_peer, iters, d);
            cudaError_t e = cudaDeviceSynchronize();
            if (e != cudaSuccess) {
                printf("error %s\n", cudaGetErrorString(e));
                return 1;
            }
        }
        std::vector<unsigned long long> h(grid);
        cudaMemcpy(h.data(), d, grid * 8, cudaMemcpyDeviceToHost);
        std::sort(h.begin(), h.end());
        const double ns = double(h[grid / 2]);
        const double bytes = double(per_peer) * (cs - 1) * iters;
        printf("cs=%d clusters=%d (%d SMs of %d) per_peer=%d mode=%d: %.2f us/iter, %.1f B/ns per SM sent (%.1f B/clk @1.965GHz)\n",
               cs, nclusters, grid, sms, per_peer, mode, ns / iters / 1e3, bytes / ns, bytes / ns / 1.965);
    }
    return 0;
}
