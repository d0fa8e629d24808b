// Small-m checked GEMM ("GEMV class"): m <= 16 rows of A against the encoded weight.
//
// For the activation-heavy DLRM shapes of P:data/shapes.txt (m in {1, 8, 32, 64}) the tensor-core pair
// kernel pays a full 256-row tile and its pipeline latency for a handful of rows; this path is bound by
// streaming B' once instead. Block = 32 output columns x 8 warps, each warp a contiguous K range; a lane
// owns one column and reads that column's 128-byte k-block slab of the K-block-major B' (the warp reads
// 4 KB contiguous), A (all m rows) is staged in shared memory and broadcast, products are u8 x s8 dp4a
// into int32 (exact). The 8 warps' partials are summed in shared memory; the block then runs the same
// checked epilogue as the pair kernel: per-row residue of its 32 columns + its K share of the checksum
// GEMV folded into one 64-bit atomic per row whose last arrival finalizes the row (gemm.cu).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>

#include "abft_internal.h"
#include "ptx.cuh"

namespace abftk {

constexpr int kGemvWarps = 8;

template <int MR, bool CHECKED>
__global__ void __launch_bounds__(32 * kGemvWarps) gemv_checked_kernel(const GemmParams p, const int8_t* __restrict__ bt,
                                                                       int64_t n_pad) {
    extern __shared__ __align__(16) uint8_t gsm[];
    uint8_t* As = gsm;                                             // [MR][k_pad] u8
    int8_t* csS = reinterpret_cast<int8_t*>(gsm + MR * p.k_blocks * kBK);   // [k_pad] the checksum vector
    int32_t* red = reinterpret_cast<int32_t*>(gsm + (MR + 1) * p.k_blocks * kBK);  // [warps][MR][32]
    int32_t* xin = red + kGemvWarps * MR * 32;                     // [cluster][MR][32] (leader)
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    // A cluster of `ks` blocks along K shares one column group when the column groups alone cannot fill
    // the GPU; the partials meet in the leader's shared memory (DSMEM).
    uint32_t ks_n;
    asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(ks_n));
    const int ks = static_cast<int>(ks_n), kr = static_cast<int>(cluster_ctarank());
    const int ncg = static_cast<int>(gridDim.x) / ks;
    const int cg = static_cast<int>(blockIdx.x) / ks;  // column group
    const int j = cg * 32 + lane;
    const int kpad = p.k_blocks * kBK;
    const int bkb0 = kr * p.k_blocks / ks, bkb1 = (kr + 1) * p.k_blocks / ks;  // this block's k-blocks

    griddep_wait();
    // The flag count (rows 2..16): the leader of column group 0 zeroes it before any of its row contributions --
    // every row's verdict needs that contribution, so each finisher's later add lands on the zeroed count (one
    // round trip fewer on the critical path than publishing it through a finished-rows counter)
    if (CHECKED && p.m > 1 && cg == 0 && kr == 0 && threadIdx.x == 0) {
        *p.err_count = 0u;
        __threadfence();
    }
    // the checksum vector next to A in shared memory (the leader's checksum share reads it at the end, off the
    // global-memory critical path)
    // (loaded now, stored after A's staging loop: the two global round trips overlap)
    constexpr int kCsPer = 4;  // 16-byte pieces per thread: k_pad <= 256 threads * 16 B * 4
    uint4 csv_pre[kCsPer];
    if (CHECKED && kr == 0)
#pragma unroll
        for (int u = 0; u < kCsPer; ++u) {
            const int e = (threadIdx.x + u * blockDim.x) * 16;
            csv_pre[u] = e < kpad ? *reinterpret_cast<const uint4*>(p.cs + e) : make_uint4(0u, 0u, 0u, 0u);
        }
    // stage A (all of it: the leader's checksum share may span any k range; rows >= m and columns >= k
    // are zero)
    for (int e = threadIdx.x * 16; e < MR * kpad; e += blockDim.x * 16) {
        const int i = e / kpad, c = e - i * kpad;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (i < p.m) {
            const uint8_t* src = p.a + static_cast<int64_t>(i) * p.lda + c;
            if (c + 16 <= p.k && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
                v = *reinterpret_cast<const uint4*>(src);
            } else {
                alignas(16) uint8_t t[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) t[q] = c + q < p.k ? src[q] : 0;
                v = *reinterpret_cast<const uint4*>(t);
            }
        }
        *reinterpret_cast<uint4*>(As + e) = v;
    }
    if (CHECKED && kr == 0) {
#pragma unroll
        for (int u = 0; u < kCsPer; ++u) {
            const int e = (threadIdx.x + u * blockDim.x) * 16;
            if (e < kpad) *reinterpret_cast<uint4*>(csS + e) = csv_pre[u];
        }
        for (int e = (threadIdx.x + kCsPer * blockDim.x) * 16; e < kpad; e += blockDim.x * 16)  // (k_pad > 16 KB)
            *reinterpret_cast<uint4*>(csS + e) = *reinterpret_cast<const uint4*>(p.cs + e);
    }
    __syncthreads();

    uint32_t acc[MR];
#pragma unroll
    for (int i = 0; i < MR; ++i) acc[i] = 0u;
    const int kb0 = bkb0 + warp * (bkb1 - bkb0) / kGemvWarps, kb1 = bkb0 + (warp + 1) * (bkb1 - bkb0) / kGemvWarps;
    const int8_t* col = bt + static_cast<int64_t>(j) * kBK;  // + kb * n_pad * 128
    for (int kb = kb0; kb < kb1; ++kb) {
        uint4 w[8];
        const uint4* src = reinterpret_cast<const uint4*>(col + static_cast<int64_t>(kb) * n_pad * kBK);
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = __ldg(src + u);  // padded columns read zeros (n_pad >= n)
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int i = 0; i < MR; ++i) {
                const uint4 a = *reinterpret_cast<const uint4*>(As + i * kpad + kb * kBK + u * 16);
                acc[i] = dp4a_us(a.x, w[u].x, acc[i]);
                acc[i] = dp4a_us(a.y, w[u].y, acc[i]);
                acc[i] = dp4a_us(a.z, w[u].z, acc[i]);
                acc[i] = dp4a_us(a.w, w[u].w, acc[i]);
            }
        }
    }
#pragma unroll
    for (int i = 0; i < MR; ++i) red[(warp * MR + i) * 32 + lane] = static_cast<int32_t>(acc[i]);
    __syncthreads();
    // block partial of every row -> the cluster leader's slot kr (its own slot 0 stays local)
    for (int e = threadIdx.x; e < MR * 32; e += blockDim.x) {
        uint32_t v = 0u;
#pragma unroll
        for (int w8 = 0; w8 < kGemvWarps; ++w8) v += static_cast<uint32_t>(red[w8 * MR * 32 + e]);
        if (ks == 1 || kr == 0) {
            xin[kr * MR * 32 + e] = static_cast<int32_t>(v);
        } else {
            const uint32_t dst = mapa_shared(smem_u32(&xin[kr * MR * 32 + e]), 0);
            asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(dst), "r"(v) : "memory");
        }
    }
    if (ks > 1) cluster_sync();
    else __syncthreads();
    if (kr != 0) return;  // the leader finishes the column group

    // warp i (< MR) finishes row i: column sums over the cluster's K ranges, C store, fault hook, residue
    for (int i = warp; i < MR && i < p.m; i += kGemvWarps) {
        uint32_t v = 0u;
        for (int r = 0; r < ks; ++r) v += static_cast<uint32_t>(xin[(r * MR + i) * 32 + lane]);
        for (int f = 0; f < p.nfaults; ++f)
            if (i == p.fault_row[f] && p.fault_col[f] == j && j < p.n) v ^= 1u << p.fault_bit[f];
        if (j < p.n && p.c) p.c[static_cast<int64_t>(i) * p.ldc + j] = static_cast<int32_t>(v);
        if constexpr (CHECKED) {
            const uint32_t rs = __reduce_add_sync(0xffffffffu, j < p.n ? mod127_i32(static_cast<int32_t>(v)) : 0u);
            // this block's K share of the checksum GEMV C'[i][n] = sum_p A[i][p]*cs[p]
            const int s0 = static_cast<int>(static_cast<long long>(cg) * p.k_blocks / ncg) * kBK;
            const int s1 = min(static_cast<int>(static_cast<long long>(cg + 1) * p.k_blocks / ncg) * kBK, p.k);
            uint32_t cs_part = 0u;
            for (int q = s0 + lane * 4; q < s1; q += 128) {  // (A and cs are zero past k)
                const uint32_t a4 = *reinterpret_cast<const uint32_t*>(As + i * kpad + q);
                const uint32_t c4 = *reinterpret_cast<const uint32_t*>(csS + q);
                cs_part = dp4a_us(a4, c4, cs_part);  // cs is s8 (negative after a sign-bit flip)
            }
            cs_part = __reduce_add_sync(0xffffffffu, cs_part);
            if (lane == 0) {
                const unsigned long long add = (static_cast<unsigned long long>(cs_part) << 32) |
                                               (1ull << kRowAccCountShift) |
                                               static_cast<unsigned long long>(rs % 127u);
                const unsigned long long acc64 = atomicAdd(&p.row_acc[i], add) + add;
                if (((acc64 >> kRowAccCountShift) & kRowAccCountMask) == static_cast<unsigned long long>(ncg)) {
                    int32_t csv = static_cast<int32_t>(static_cast<uint32_t>(acc64 >> 32));
                    for (int f = 0; f < p.nfaults; ++f)
                        if (i == p.fault_row[f] && p.fault_col[f] == p.n)
                            csv ^= static_cast<int32_t>(1u << p.fault_bit[f]);  // fault in C'[:, n]
                    const uint32_t res = static_cast<uint32_t>(acc64 & kRowAccResMask) % 127u;
                    const int flag = static_cast<int32_t>(res) != mod127(csv);
                    p.flags[i] = static_cast<uint8_t>(flag);
                    p.csum[static_cast<int64_t>(i) * p.csum_ld] = csv;
                    p.row_acc[i] = 0ull;
                    if (p.m == 1) {  // the only row: its finisher publishes the count (no second round trip)
                        *p.err_count = static_cast<uint32_t>(flag);
                    } else if (flag) {  // onto the count zeroed before this row's first contribution
                        __threadfence();
                        atomicAdd(p.err_count, 1u);
                    }
                }
            }
        }
    }
}

// Single-cluster small GEMV (m <= 16, B' of at most a few MB): the whole problem runs on ONE thread-block cluster of
// CS <= 16 blocks, so the row verdicts need no global atomics: every block reduces its columns' row residues and
// its K share of the checksum column in shared memory, sends them to the leader over DSMEM, and after one cluster
// barrier the leader compares them (P:src/gemm_abft.cpp:113-124) and writes flags, the checksum column and the
// count. Block b owns column groups b, b + CS, ... (32 columns each); its 8 warps take (column group, k-block)
// items round-robin, two in flight, and add their partial dot products into shared memory.
constexpr int kGcMaxGroups = 8;  // column groups per block (n <= 16 * 8 * 32 = 4096)
template <int MR, bool CHECKED>
__global__ void __launch_bounds__(32 * kGemvWarps) gemv_cluster_kernel(const GemmParams p, const int8_t* __restrict__ bt,
                                                                       int64_t n_pad) {
    extern __shared__ __align__(16) uint8_t gsm[];
    const int kpad = p.k_blocks * kBK;
    uint8_t* As = gsm;                                                // [MR][kpad]
    int8_t* csS = reinterpret_cast<int8_t*>(gsm + MR * kpad);         // [kpad]
    int32_t* colacc = reinterpret_cast<int32_t*>(gsm + (MR + 1) * kpad);  // [kGcMaxGroups][MR][32]
    uint32_t* rowres = reinterpret_cast<uint32_t*>(colacc + kGcMaxGroups * MR * 32);  // [MR]
    uint32_t* share = rowres + MR;                                    // [MR]
    uint32_t* xin = share + MR;                                       // [16][MR][2] (leader)
    __shared__ __align__(8) uint64_t gbar;  // leader: completes when every block's rows have landed in xin
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    uint32_t cs_n;
    asm("mov.u32 %0, %%cluster_nctarank;" : "=r"(cs_n));
    const int CS = static_cast<int>(cs_n), b = static_cast<int>(cluster_ctarank());
    const int ncg = (p.n + 31) / 32;
    const int ngl = (ncg - b + CS - 1) / CS;  // this block's column groups
    griddep_wait();
    constexpr int kCsPer = 4;  // the checksum vector's 16-byte pieces, loaded before A's staging loop (overlap)
    uint4 csv_pre[kCsPer];
    if (CHECKED)
#pragma unroll
        for (int u = 0; u < kCsPer; ++u) {
            const int e = (threadIdx.x + u * blockDim.x) * 16;
            csv_pre[u] = e < kpad ? *reinterpret_cast<const uint4*>(p.cs + e) : make_uint4(0u, 0u, 0u, 0u);
        }
    for (int e = threadIdx.x * 16; e < MR * kpad; e += blockDim.x * 16) {
        const int i = e / kpad, c = e - i * kpad;
        uint4 v = make_uint4(0u, 0u, 0u, 0u);
        if (i < p.m) {
            const uint8_t* src = p.a + static_cast<int64_t>(i) * p.lda + c;
            if (c + 16 <= p.k && (reinterpret_cast<uintptr_t>(src) & 15) == 0) {
                v = *reinterpret_cast<const uint4*>(src);
            } else {
                alignas(16) uint8_t t[16];
#pragma unroll
                for (int q = 0; q < 16; ++q) t[q] = c + q < p.k ? src[q] : 0;
                v = *reinterpret_cast<const uint4*>(t);
            }
        }
        *reinterpret_cast<uint4*>(As + e) = v;
    }
    if (CHECKED) {
#pragma unroll
        for (int u = 0; u < kCsPer; ++u) {
            const int e = (threadIdx.x + u * blockDim.x) * 16;
            if (e < kpad) *reinterpret_cast<uint4*>(csS + e) = csv_pre[u];
        }
        for (int e = (threadIdx.x + kCsPer * blockDim.x) * 16; e < kpad; e += blockDim.x * 16)
            *reinterpret_cast<uint4*>(csS + e) = *reinterpret_cast<const uint4*>(p.cs + e);
    }
    for (int e = threadIdx.x; e < kGcMaxGroups * MR * 32; e += blockDim.x) colacc[e] = 0;
    if (threadIdx.x < 2 * MR) rowres[threadIdx.x] = 0u;  // (rowres and share are adjacent)
    if (CHECKED && b == 0 && threadIdx.x == 0) {
        mbar_init(&gbar, 1);
        fence_mbar_init();
        mbar_arrive_expect_tx(&gbar, static_cast<uint32_t>(CS * p.m * 8));
    }
    // the leader's barrier is visible cluster-wide before any block sends to it (no global stores are in flight
    // yet, so this release is cheap; the verdict hand-over itself is one st.async per row, no cluster barrier)
#ifdef GC_PROBE_NO_CSYNC
    __syncthreads();
#else
    if (CHECKED) cluster_sync();
    else __syncthreads();
#endif

    // (column group, k-block) items, round-robin over the warps, two in flight
    const int kbt = p.k_blocks, items = ngl * kbt;
    auto load = [&](int t, uint4 (&w)[8]) {
        const int gl = t / kbt, kb = t - gl * kbt;
        const int j = (b + gl * CS) * 32 + lane;
        const uint4* src = reinterpret_cast<const uint4*>(bt + static_cast<int64_t>(j) * kBK +
                                                          static_cast<int64_t>(kb) * n_pad * kBK);
#pragma unroll
        for (int u = 0; u < 8; ++u) w[u] = __ldg(src + u);  // columns past n read the zero padding
    };
    auto consume = [&](int t, const uint4 (&w)[8]) {
        const int gl = t / kbt, kb = t - gl * kbt;
        uint32_t acc[MR];
#pragma unroll
        for (int i = 0; i < MR; ++i) acc[i] = 0u;
#pragma unroll
        for (int u = 0; u < 8; ++u) {
#pragma unroll
            for (int i = 0; i < MR; ++i) {
                const uint4 a = *reinterpret_cast<const uint4*>(As + i * kpad + kb * kBK + u * 16);
                acc[i] = dp4a_us(a.x, w[u].x, acc[i]);
                acc[i] = dp4a_us(a.y, w[u].y, acc[i]);
                acc[i] = dp4a_us(a.z, w[u].z, acc[i]);
                acc[i] = dp4a_us(a.w, w[u].w, acc[i]);
            }
        }
#pragma unroll
        for (int i = 0; i < MR; ++i)
            if (i < p.m) atomicAdd(&colacc[(gl * MR + i) * 32 + lane], static_cast<int32_t>(acc[i]));
    };
    int t = warp;
    for (; t + kGemvWarps < items; t += 2 * kGemvWarps) {
        uint4 w0[8], w1[8];
        load(t, w0);
        load(t + kGemvWarps, w1);
        consume(t, w0);
        consume(t + kGemvWarps, w1);
    }
    if (t < items) {
        uint4 w0[8];
        load(t, w0);
        consume(t, w0);
    }
    // the checksum column: this block's K share of A*cs for every row (blocks split K)
    if (CHECKED) {
        const int q0 = static_cast<int>(static_cast<long long>(b) * p.k_blocks / CS) * kBK;
        const int q1 = static_cast<int>(static_cast<long long>(b + 1) * p.k_blocks / CS) * kBK;
        for (int i = warp; i < MR && i < p.m; i += kGemvWarps) {
            uint32_t sh = 0u;
            for (int q = q0 + lane * 4; q < q1; q += 128)  // (A and cs are zero past k)
                sh = dp4a_us(*reinterpret_cast<const uint32_t*>(As + i * kpad + q),
                             *reinterpret_cast<const uint32_t*>(csS + q), sh);
            sh = __reduce_add_sync(0xffffffffu, sh);
            if (lane == 0) share[i] = sh;
        }
    }
    __syncthreads();
    // columns: store C (after any injected C' fault) and fold each row's residue over this block's columns
    for (int r = warp; r < ngl * MR; r += kGemvWarps) {
        const int gl = r / MR, i = r - gl * MR;
        if (i >= p.m) continue;
        const int j = (b + gl * CS) * 32 + lane;
        uint32_t v = static_cast<uint32_t>(colacc[r * 32 + lane]);
        for (int f = 0; f < p.nfaults; ++f)
            if (i == p.fault_row[f] && p.fault_col[f] == j && j < p.n) v ^= 1u << p.fault_bit[f];
        if (j < p.n && p.c) p.c[static_cast<int64_t>(i) * p.ldc + j] = static_cast<int32_t>(v);
        if constexpr (CHECKED) {
            // residues add up (mod 127): each lane reduces its column, one redux sums the warp's 32 (< 4064)
            const uint32_t rs = __reduce_add_sync(0xffffffffu, j < p.n ? mod127_i32(static_cast<int32_t>(v)) : 0u);
            if (lane == 0) atomicAdd(&rowres[i], rs);
        }
    }
    if constexpr (!CHECKED) return;
#ifdef GC_PROBE_NO_TAIL
    return;
#endif
    __syncthreads();
    // (residue sum, checksum share) of every row into the leader's shared memory: st.async completing bytes on the
    // leader's mbarrier (fire-and-forget for the sender; no release of this block's C stores is waited for)
    if (threadIdx.x < p.m) {
        const uint32_t dst = mapa_shared(smem_u32(&xin[(b * MR + threadIdx.x) * 2]), 0);
        const uint32_t bar = mapa_shared(smem_u32(&gbar), 0);
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.u32 [%0], {%1, %2}, [%3];" ::"r"(dst),
                     "r"(rowres[threadIdx.x]), "r"(share[threadIdx.x]), "r"(bar)
                     : "memory");
    }
    if (b != 0 || warp != 0) return;
    mbar_wait(&gbar, 0);
    int flag = 0;
    if (lane < p.m) {
        uint32_t res = 0u, sh = 0u;
        for (int r = 0; r < CS; ++r) {
            res += xin[(r * MR + lane) * 2];
            sh += xin[(r * MR + lane) * 2 + 1];
        }
        int32_t csv = static_cast<int32_t>(sh);
        for (int f = 0; f < p.nfaults; ++f)
            if (lane == p.fault_row[f] && p.fault_col[f] == p.n) csv ^= static_cast<int32_t>(1u << p.fault_bit[f]);
        flag = static_cast<int32_t>(res % 127u) != mod127(csv);
        p.flags[lane] = static_cast<uint8_t>(flag);
        p.csum[static_cast<int64_t>(lane) * p.csum_ld] = csv;
    }
    const uint32_t nflag = __popc(__ballot_sync(0xffffffffu, flag));
    if (lane == 0) *p.err_count = nflag;
}

template <int MR, bool CK>
static cudaError_t launch_gemv_cluster_mr(const GemmParams& p, const GemmWeight& w, int cs, cudaStream_t st) {
    const int smem = (MR + 1) * p.k_blocks * kBK + kGcMaxGroups * MR * 32 * 4 + 2 * MR * 4 + 16 * MR * 2 * 4;
    auto kern = gemv_cluster_kernel<MR, CK>;
    static int attr_smem[kMaxDevices] = {};  // per device; benign race: idempotent
    const int dev = current_device();
    if (!attr_smem[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
        if (e != cudaSuccess) return e;
    }
    if (smem > attr_smem[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_smem[dev] = smem;
    }
    static const bool pdl = std::getenv("ABFTLP_NO_PDL") == nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(cs));
    cfg.blockDim = dim3(32 * kGemvWarps);
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cfg.stream = st;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = static_cast<unsigned>(cs);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 2 : 1;
    return cudaLaunchKernelEx(&cfg, kern, p, static_cast<const int8_t*>(w.bt), static_cast<int64_t>(w.n_pad));
}

// One-cluster path for small GEMV-class problems: the cluster size (<= 16 blocks) or 0 when the problem does not fit
// (more than 16 * kGcMaxGroups column groups, or more B' than a cluster streams in about a microsecond).
int gemv_cluster_size(const GemmParams& p, int64_t n_pad) {
    if (const char* e = std::getenv("ABFTLP_GEMV_CLUSTER"))
        if (std::atoi(e) == 0) return 0;
    const int ncg = (p.n + 31) / 32;
    const int64_t bytes = static_cast<int64_t>(p.k_blocks) * kBK * ncg * 32;  // the B' columns the kernel streams
    (void)n_pad;
    const int64_t limit = std::getenv("ABFTLP_GEMV_CLUSTER_BYTES") ? std::atoll(std::getenv("ABFTLP_GEMV_CLUSTER_BYTES"))
                                                                   : (int64_t{256} << 10);
    if (bytes > limit) return 0;
    int maxcs = 16;
    if (const char* e = std::getenv("ABFTLP_GEMV_CLUSTER_MAX")) maxcs = std::max(1, std::min(16, std::atoi(e)));
    int cs = ncg < maxcs ? ncg : maxcs;
    while ((ncg + cs - 1) / cs > kGcMaxGroups && cs < 16) ++cs;  // at most kGcMaxGroups column groups per block
    if ((ncg + cs - 1) / cs > kGcMaxGroups) return 0;
    return cs;
}

template <int MR, bool CK>
static cudaError_t launch_gemv_mr(const GemmParams& p, const GemmWeight& w, cudaStream_t st) {
    // K split across a cluster when the column groups alone cannot fill ~2 blocks per SM
    const int ncg = (p.n + 31) / 32;
    int ks = 1;
    while (ks < 8 && ncg * ks * 2 <= 2 * 148 && p.k_blocks >= ks * 2) ks *= 2;
    const int smem = (MR + 1) * p.k_blocks * kBK + kGemvWarps * MR * 32 * 4 + ks * MR * 32 * 4;
    auto kern = gemv_checked_kernel<MR, CK>;
    static int attr_smem[kMaxDevices] = {};  // per device; benign race: idempotent
    const int dev = current_device();
    if (smem > 48 * 1024 && smem > attr_smem[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr_smem[dev] = smem;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(static_cast<unsigned>(ncg * ks));
    cfg.blockDim = dim3(32 * kGemvWarps);
    cfg.dynamicSmemBytes = static_cast<size_t>(smem);
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = static_cast<unsigned>(ks);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kern, p, static_cast<const int8_t*>(w.bt), static_cast<int64_t>(w.n_pad));
}

// Row capacity of the small-m path; the runtime routes m <= kGemvMaxRows here.
cudaError_t launch_gemv(const GemmParams& p, const GemmWeight& w, bool checked, cudaStream_t st) {
    const int m = p.m;
    if (const int cs = gemv_cluster_size(p, w.n_pad)) {
        if (checked) {
            if (m <= 1) return launch_gemv_cluster_mr<1, true>(p, w, cs, st);
            if (m <= 2) return launch_gemv_cluster_mr<2, true>(p, w, cs, st);
            if (m <= 4) return launch_gemv_cluster_mr<4, true>(p, w, cs, st);
            if (m <= 8) return launch_gemv_cluster_mr<8, true>(p, w, cs, st);
            return launch_gemv_cluster_mr<16, true>(p, w, cs, st);
        }
        if (m <= 1) return launch_gemv_cluster_mr<1, false>(p, w, cs, st);
        if (m <= 2) return launch_gemv_cluster_mr<2, false>(p, w, cs, st);
        if (m <= 4) return launch_gemv_cluster_mr<4, false>(p, w, cs, st);
        if (m <= 8) return launch_gemv_cluster_mr<8, false>(p, w, cs, st);
        return launch_gemv_cluster_mr<16, false>(p, w, cs, st);
    }
    if (checked) {
        if (m <= 1) return launch_gemv_mr<1, true>(p, w, st);
        if (m <= 2) return launch_gemv_mr<2, true>(p, w, st);
        if (m <= 4) return launch_gemv_mr<4, true>(p, w, st);
        if (m <= 8) return launch_gemv_mr<8, true>(p, w, st);
        return launch_gemv_mr<16, true>(p, w, st);
    }
    if (m <= 1) return launch_gemv_mr<1, false>(p, w, st);
    if (m <= 2) return launch_gemv_mr<2, false>(p, w, st);
    if (m <= 4) return launch_gemv_mr<4, false>(p, w, st);
    if (m <= 8) return launch_gemv_mr<8, false>(p, w, st);
    return launch_gemv_mr<16, false>(p, w, st);
}

}  // namespace abftk
