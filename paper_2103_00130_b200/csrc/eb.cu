// ABFT EmbeddingBag for sm_100a: checked / unchecked pooled lookups and the row-sum encoder.
//
//   eb_meta_kernel  replaces precompute_row_sums (P:src/embedding_abft.cpp:39-45) and packs the
//                   per-row (scale, bias, rowSum) into one 16-B (fp32) or 8-B (fp16) record so a
//                   lookup touches one metadata sector.
//   eb_bag_kernel   replaces embedding_bag / abft_embedding_bag / batch_abft_eb
//                   (P:src/embedding_abft.cpp:47-91). A bag is processed by WPB warps, each owning
//                   a contiguous slice of the columns; lane l of a warp owns CPL columns of the slice.
//                   Every output column is therefore accumulated sequentially in bag order with the
//                   reference's exact fp32 operation order (scale*q, +bias, *w, +=; no FMA), which is
//                   what makes the pooled vector bit-identical. Lookups are processed in chunks of 32:
//                   the chunk's row offsets / scale / bias / weight are staged in shared memory
//                   (broadcast reads), the 32 row gathers are issued before any is consumed, the
//                   next chunk's indices are prefetched while the current one accumulates, and the
//                   cSum terms w*(scale*rowSum + d*bias) are formed lane-parallel so only the fp64
//                   additions stay sequential (as in the reference, P:src/embedding_abft.cpp:69-76).
//                   rSum is computed order-free when every partial sum is provably exact in fp64 and
//                   in the reference's sequential order otherwise -- bit-identical either way.
#include <cuda_fp16.h>
#include <cstdlib>
#include <type_traits>
#include <cuda_runtime.h>

#include "abft_internal.h"
#include "ptx.cuh"

namespace abftk {
int device_sm_count();

// Output row / flag slot of a bag: local buffers, or a destination table (sharded exchange, EbParams).
// (bag ids below 2^32 divide in 32 bits: a 64-bit divide is a ~40-instruction sequence on the per-bag path)
__device__ __forceinline__ void dest_of(const EbParams& p, int64_t bag, int64_t& dest, int64_t& slot) {
    if (bag <= 0xFFFFFFFFll && p.bags_per_dest <= 0xFFFFFFFFll) {
        const uint32_t d = static_cast<uint32_t>(bag) / static_cast<uint32_t>(p.bags_per_dest);
        dest = d;
        slot = static_cast<uint32_t>(bag) - d * static_cast<uint32_t>(p.bags_per_dest);
    } else {
        dest = bag / p.bags_per_dest;
        slot = bag - dest * p.bags_per_dest;
    }
}
__device__ __forceinline__ float* out_row(const EbParams& p, int64_t bag) {
    if (p.out_dest) {
        int64_t d, sl;
        dest_of(p, bag, d, sl);
        return p.out_dest[d] + sl * p.ld_out;
    }
    return p.out + bag * p.ld_out;
}
__device__ __forceinline__ uint8_t* flag_slot(const EbParams& p, int64_t bag) {
    if (p.flag_dest) {
        int64_t d, sl;
        dest_of(p, bag, d, sl);
        return p.flag_dest[d] + sl * p.flag_ld;
    }
    return p.flags ? p.flags + bag : nullptr;
}

namespace {

template <int BPL>
struct LaneWord {
    using T = uint32_t;
};
template <>
struct LaneWord<8> {
    using T = uint64_t;
};

template <int BPL>
__device__ __forceinline__ typename LaneWord<BPL>::T load_row_word(const uint8_t* ptr) {
    if constexpr (BPL == 1) {
        uint16_t v;
        asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(v) : "l"(ptr));
        return v;
    } else if constexpr (BPL == 2) {
        uint16_t v;
        asm volatile("ld.global.nc.L1::no_allocate.u16 %0, [%1];" : "=h"(v) : "l"(ptr));
        return v;
    } else if constexpr (BPL == 4) {
        uint32_t v;
        asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(v) : "l"(ptr));
        return v;
    } else {
        uint64_t v;
        asm volatile("ld.global.nc.L1::no_allocate.u64 %0, [%1];" : "=l"(v) : "l"(ptr));
        return v;
    }
}

// Decode element c (0-based within the lane's slice) of a lane word.
template <int ELEM, typename W>
__device__ __forceinline__ float decode(W w, int c) {
    if constexpr (ELEM == kEbS8) {
        return static_cast<float>(static_cast<int8_t>(static_cast<uint8_t>(w >> (8 * c))));
    } else if constexpr (ELEM == kEbU8) {
        return static_cast<float>(static_cast<uint8_t>(w >> (8 * c)));
    } else {  // u4: element j = (byte[j/2] >> 4*(j&1)) & 0xF, low nibble = even column
        return static_cast<float>(static_cast<uint32_t>(w >> (4 * c)) & 0xFu);
    }
}

template <int SCALE>
__device__ __forceinline__ void load_meta(const void* meta, int64_t i, int64_t stride, float& s, float& b, int32_t& rs) {
    const uint8_t* rec = reinterpret_cast<const uint8_t*>(meta) + i * stride;
    if constexpr (SCALE == kEbF32) {
        const uint4 v = __ldg(reinterpret_cast<const uint4*>(rec));
        s = __uint_as_float(v.x);
        b = __uint_as_float(v.y);
        rs = static_cast<int32_t>(v.z);
    } else {
        const uint2 v = __ldg(reinterpret_cast<const uint2*>(rec));
        s = __half2float(__ushort_as_half(static_cast<unsigned short>(v.x & 0xFFFFu)));
        b = __half2float(__ushort_as_half(static_cast<unsigned short>(v.x >> 16)));
        rs = static_cast<int32_t>(v.y);
    }
}

// Exponent range of a float's set bits: msb/lsb exponents (value = sum of 2^e over set bits).
__device__ __forceinline__ void bit_span(float v, int& emax, int& umin) {
    const uint32_t bits = __float_as_uint(v) & 0x7FFFFFFFu;
    if (!bits) return;
    const int ex = static_cast<int>(bits >> 23);
    const uint32_t mant = bits & 0x7FFFFFu;
    int lo, hi;
    if (ex == 0) {
        lo = -149 + (__ffs(static_cast<int>(mant)) - 1);
        hi = -149 + (31 - __clz(static_cast<int>(mant)));
    } else {
        const uint32_t sig = mant | 0x800000u;
        lo = ex - 150 + (__ffs(static_cast<int>(sig)) - 1);
        hi = ex - 127;
    }
    emax = max(emax, hi);
    umin = min(umin, lo);
}

__device__ __forceinline__ double csum_term(float s, float b, int32_t rs, float w, double dd, bool weighted) {
    double term = __dadd_rn(__dmul_rn(static_cast<double>(s), static_cast<double>(rs)), __dmul_rn(dd, static_cast<double>(b)));
    if (weighted) term = __dmul_rn(static_cast<double>(w), term);
    return term;
}

}  // namespace

// Block completion without fences: one 64-bit atomic per block on the per-stream word {flags (low 32),
// finished blocks (high 32)} (ws_flag_acc / ws_block_cnt, adjacent and 8-byte aligned). Atomics on one
// address are totally ordered, so the block whose add brings the count to gridDim.x sees every other
// block's flags in the returned value; it publishes the call's flag count and resets the per-stream words
// (the bag counter's last use by any block returned its value before that block arrived here).
__device__ __forceinline__ void eb_block_done(const EbParams& p, uint32_t blk_flags, bool reset_bag_ctr) {
    unsigned long long* pack = reinterpret_cast<unsigned long long*>(p.ws_flag_acc);
    const unsigned long long prev = atomicAdd(pack, (1ull << 32) | blk_flags);
    if ((prev >> 32) == gridDim.x - 1) {
        if (p.flag_count) *p.flag_count = static_cast<uint32_t>(prev) + blk_flags;
        *pack = 0ull;
        if (reset_bag_ctr) *p.ws_bag_ctr = 0ull;
    }
}

constexpr int kGenericSlots = 8;
constexpr int kChunk = 32;  // lookups gathered per round

struct ChunkStage {      // per warp
    int64_t off[kChunk];  // row byte offset, -1 = skipped (out of range / past the bag)
    float2 sb[kChunk];    // scale, bias
    float w[kChunk];
};

// Fast path: d == 32 * CPL * WPB, rows 8-byte aligned. Block = 8 warps = 8 / WPB bags.
template <int ELEM, int SCALE, int CPL, int WPB, bool WEIGHTED, bool CHECKED>
// 4 blocks/SM (<= 64 regs, 32 warps/SM) spills 0.5-0.9 KB per thread at 8 columns per lane; 2 blocks/SM does not.
__global__ void __launch_bounds__(256, CPL >= 8 ? 2 : 4) eb_bag_kernel(const EbParams p, int log2d) {
    constexpr int BPL = ELEM == kEbU4 ? CPL / 2 : CPL;  // bytes per lane per row
    constexpr int BAGS = 8 / WPB;
    using Word = typename LaneWord<BPL>::T;
    __shared__ ChunkStage stage[8];
    __shared__ double part_sum[8];
    __shared__ int part_emax[8], part_umin[8];
    __shared__ uint32_t blk_flags;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int bag_local = warp / WPB, slice = warp % WPB;
    const int64_t bag = static_cast<int64_t>(blockIdx.x) * BAGS + bag_local;
    const int64_t lane_byte = static_cast<int64_t>(slice) * 32 * BPL + lane * BPL;
    const double dd = static_cast<double>(p.dim);
    ChunkStage& cs = stage[warp];
    if (threadIdx.x == 0) blk_flags = 0;

    float acc[CPL];
#pragma unroll
    for (int c = 0; c < CPL; ++c) acc[c] = 0.0f;
    double csum = 0.0;
    bool oob = false;
    if (bag < p.num_bags) {
        const int64_t beg = p.offsets[bag], end = p.offsets[bag + 1];
        int64_t nidx = (beg + lane < end) ? p.indices[beg + lane] : -1;
        for (int64_t base = beg; base < end; base += kChunk) {
            const int cnt = static_cast<int>(min(static_cast<int64_t>(kChunk), end - base));
            const int64_t my_idx = nidx;
            const bool valid = lane < cnt && static_cast<uint64_t>(my_idx) < static_cast<uint64_t>(p.rows);
            if (lane < cnt && !valid) oob = true;
            cs.off[lane] = valid ? my_idx * p.row_stride : -1;
            __syncwarp();
            // gather the chunk's rows (independent of everything but the indices)
            // Every slot issues its load (skipped slots read row 0, masked below): a conditional on the
            // loaded value would make each load wait for the previous one.
            Word data[kChunk];
#pragma unroll
            for (int t = 0; t < kChunk; ++t) {
                const int64_t o = cs.off[t];
                data[t] = load_row_word<BPL>(p.data + ((t < cnt && o >= 0) ? o : 0) + lane_byte);
            }
            // metadata of lookup (base + lane), overlapping the row gathers
            float my_s = 0.f, my_b = 0.f, my_w = 1.f;
            int32_t my_rs = 0;
            if (valid) load_meta<SCALE>(p.meta, my_idx, p.meta_stride, my_s, my_b, my_rs);
            if constexpr (WEIGHTED) {
                if (lane < cnt) my_w = p.weights[base + lane];
            }
            // prefetch the next chunk's indices
            nidx = (base + kChunk + lane < end) ? p.indices[base + kChunk + lane] : -1;
            cs.sb[lane] = make_float2(my_s, my_b);
            if constexpr (WEIGHTED) cs.w[lane] = my_w;
            double my_term = 0.0;
            if constexpr (CHECKED) {
                if (slice == 0 && valid) my_term = csum_term(my_s, my_b, my_rs, my_w, dd, WEIGHTED);
            }
            __syncwarp();
#pragma unroll
            for (int t = 0; t < kChunk; ++t) {
                if (t < cnt && cs.off[t] >= 0) {  // warp-uniform
                    const float2 sb = cs.sb[t];
                    const float w = WEIGHTED ? cs.w[t] : 1.0f;
#pragma unroll
                    for (int c = 0; c < CPL; ++c) {
                        float x = __fadd_rn(__fmul_rn(sb.x, decode<ELEM>(data[t], c)), sb.y);
                        if constexpr (WEIGHTED) x = __fmul_rn(w, x);
                        acc[c] = __fadd_rn(acc[c], x);
                    }
                }
            }
            if constexpr (CHECKED) {
                if (slice == 0) {
                    for (int t = 0; t < cnt; ++t) {
                        const double term = __shfl_sync(0xffffffffu, my_term, t);
                        if (cs.off[t] >= 0) csum = __dadd_rn(csum, term);
                    }
                }
            }
            __syncwarp();
        }
        if (__any_sync(0xffffffffu, oob) && lane == 0 && p.status) atomicOr(p.status, 1);
        // pooled output: this warp's slice
        float* dst = out_row(p, bag) + slice * 32 * CPL + lane * CPL;
        if constexpr (CPL % 4 == 0) {
            if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
                for (int c = 0; c < CPL; c += 4)
                    *reinterpret_cast<float4*>(dst + c) = make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
            } else {
#pragma unroll
                for (int c = 0; c < CPL; ++c) dst[c] = acc[c];
            }
        } else if constexpr (CPL == 2) {
            if ((reinterpret_cast<uintptr_t>(dst) & 7) == 0)
                *reinterpret_cast<float2*>(dst) = make_float2(acc[0], acc[1]);
            else {
                dst[0] = acc[0];
                dst[1] = acc[1];
            }
        } else {
#pragma unroll
            for (int c = 0; c < CPL; ++c) dst[c] = acc[c];
        }
    }
    if constexpr (CHECKED) {
        // ---- per-slice exactness statistics and order-free partial sum
        int emax = -100000, umin = 100000;
#pragma unroll
        for (int c = 0; c < CPL; ++c) bit_span(acc[c], emax, umin);
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < CPL; ++c) s = __dadd_rn(s, static_cast<double>(acc[c]));
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
            umin = min(umin, __shfl_xor_sync(0xffffffffu, umin, o));
            s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
        }
        if (lane == 0) {
            part_sum[warp] = s;
            part_emax[warp] = emax;
            part_umin[warp] = umin;
        }
        __syncthreads();  // slices of a bag (and their global outputs) are complete
        if (slice == 0 && bag < p.num_bags) {
            int E = -100000, U = 100000;
            double exact = 0.0;
#pragma unroll
            for (int s2 = 0; s2 < WPB; ++s2) {
                E = max(E, part_emax[warp + s2]);
                U = min(U, part_umin[warp + s2]);
                exact = __dadd_rn(exact, part_sum[warp + s2]);
            }
            double rsum;
            if (E == -100000) {
                rsum = 0.0;
            } else if (E + 1 + log2d - U <= 53) {
                rsum = exact;  // every partial sum is an exact multiple of 2^U below 2^53 ulps: order-free
            } else {
                // the reference's order: j = 0 .. d-1 (P:src/embedding_abft.cpp:66-67)
                rsum = 0.0;
                const float* row = out_row(p, bag);
                for (int j0 = 0; j0 < p.dim; j0 += 32) {
                    const float v = (j0 + lane < p.dim) ? row[j0 + lane] : 0.0f;
                    for (int l = 0; l < 32 && j0 + l < p.dim; ++l)
                        rsum = __dadd_rn(rsum, static_cast<double>(__shfl_sync(0xffffffffu, v, l)));
                }
            }
            // ---- err = |rSum - cSum| > 1e-5 * max(|rSum|, |cSum|, 1)   (P:src/embedding_abft.cpp:80-81)
            const double diff = fabs(__dsub_rn(rsum, csum));
            const double mx = fmax(fmax(fabs(rsum), fabs(csum)), 1.0);
            const int flag = diff > __dmul_rn(1e-5, mx);
            if (lane == 0) {
                if (uint8_t* fs = flag_slot(p, bag)) *fs = static_cast<uint8_t>(flag);
                if (p.rsum) p.rsum[bag] = rsum;
                if (p.csum) p.csum[bag] = csum;
                if (flag) atomicAdd(&blk_flags, 1u);
            }
        }
        if (p.flag_count) {
            __syncthreads();
            if (threadIdx.x == 0) eb_block_done(p, blk_flags, false);
        }
    }
}

// ------------------------------------------------------------------ async-copy pipeline (main path)
// Same column ownership and accumulation order as eb_bag_kernel, but the 32 row slices and the 32
// metadata records of a chunk land in shared memory through cp.async (16-B copies, L1 bypass), double
// buffered per warp: while chunk c is accumulated from shared memory, chunk c+1's gathers are in flight
// and chunk c+2's indices are being loaded. Needs 16-byte aligned row slices.
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
// L1-allocating variant for row data: Zipf-hot rows are then served by the SM's L1 instead of
// hammering one L2 slice.
__device__ __forceinline__ void cp_async16_l1(void* smem, const void* gmem) {
#ifdef ABFT_EB_ROWS_CG  // (experiment switch: rows through L2 only)
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
#elif defined(ABFT_EB_ROWS_256B)  // (experiment switch: L2 prefetch hint for row pieces)
    asm volatile("cp.async.ca.shared.global.L2::256B [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
#else
    asm volatile("cp.async.ca.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
#endif
}
// base + a * b with a, b unsigned 32-bit (one IMAD.WIDE.U32)
__device__ __forceinline__ const uint8_t* mad_wide_u32(uint32_t a, uint32_t b, const uint8_t* base) {
    unsigned long long r;
    asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(reinterpret_cast<unsigned long long>(base)));
    return reinterpret_cast<const uint8_t*>(r);
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(smem_u32(smem)), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// Chunk slots in flight per warp: deep enough that a whole E4-sized bag (<= 160 lookups) is gathered in
// one round trip; fewer for wide slices (shared memory).
template <int BPL>
struct AsyncRing {
    static constexpr int SLICE = 32 * BPL;
#ifndef ABFT_EB_NST32
#define ABFT_EB_NST32 6
#endif
#ifndef ABFT_EB_NST64
#define ABFT_EB_NST64 4
#endif
#ifndef ABFT_EB_NST128
#define ABFT_EB_NST128 2  // measured: occupancy beats ring depth for 128-B slices (D5, E3)
#endif
    static constexpr int NST = SLICE <= 32 ? ABFT_EB_NST32 : SLICE <= 64 ? ABFT_EB_NST64 : SLICE <= 128 ? ABFT_EB_NST128 : 2;
};
// Per-lookup constants of the chunk being consumed, formed lane-parallel once per chunk (lane l: lookup l) so the
// column loop reads them with two 16-byte shared loads and does no conversion work:
//   s_lo/s_hi and c_lo/c_hi  the "splice" multipliers: a column value v (< 2^8) spliced into the mantissa of 2^23
//                            as the float 2^23 + v' gives s*v in ONE rounding as fma(2^23 + v', s', -s'*2^23) when
//                            s'*2^23 is exact (u8: v' = v, s' = s; u4 high nibble: v' = 16 v taken in place,
//                            s' = s/16); s8 uses the magic subtraction instead (see the column loop)
//   b, w                     bias and bag weight (1 when unweighted)
//   term                     the lookup's cSum term (P:src/embedding_abft.cpp:69-76)
struct __align__(16) LookupConst {
    float s_lo, s_hi, c_lo, c_hi;
    float b, w;
    double term;
};
// K16: s8 rows without bag weights need only (scale, bias, cSum term) per lookup -- 16 bytes, written over the
// lookup's landed metadata record, so such kernels carry no separate constant array (three resident blocks per SM
// at 128-byte slices instead of two).
template <int BPL, bool K16, bool WEIGHTED>
struct AsyncStage {
    static constexpr int NST = AsyncRing<BPL>::NST;
    uint8_t rows[NST][kChunk][32 * BPL];  // this warp's column slice of each gathered row
    uint4 meta[NST][kChunk];              // EbMetaF32 (16 B) or EbMetaF16 (first 8 B); zero = neutral slot
    float w[NST][WEIGHTED ? kChunk : 1];
    LookupConst k[K16 ? 1 : kChunk];      // constants of the chunk being consumed (K16: in place in meta[])
};

// The splice multiplication is exact when s*2^23 and s/16 are exact normal floats (and s is finite); a zero scale
// is fine too (every product is then +-0, and a signed zero term never changes a sum that starts at +0).
__device__ __forceinline__ bool splice_safe(float s) {
    const float a = fabsf(s);
    return a == 0.0f || (a >= 0x1p-100f && a <= 0x1p100f);
}
// Columns c, c+1 of a lane word spliced for the FMA form (u4: low nibble v, high nibble 16 v in place; u8: bytes).
template <int ELEM, typename W>
__device__ __forceinline__ unsigned long long splice_pair_bits(W w, int c) {
    if constexpr (ELEM == kEbU4) {
        const uint32_t byte = static_cast<uint32_t>(w >> (4 * c)) & 0xFFu;
        return static_cast<unsigned long long>(0x4B000000u | (byte & 0x0Fu)) |
               (static_cast<unsigned long long>(0x4B000000u | (byte & 0xF0u)) << 32);
    } else {
        const uint32_t half = (sizeof(W) == 8 && c >= 4) ? static_cast<uint32_t>(static_cast<uint64_t>(w) >> 32)
                                                         : static_cast<uint32_t>(w);
        const uint32_t bsel = static_cast<uint32_t>(c & 3);
        return static_cast<unsigned long long>(__byte_perm(half, 0x4B000000u, 0x7540u | bsel)) |
               (static_cast<unsigned long long>(__byte_perm(half, 0x4B000000u, 0x7540u | (bsel + 1))) << 32);
    }
}

template <int SCALE>
__device__ __forceinline__ void smem_meta(const uint4& m, float& s, float& b, int32_t& rs) {
    if constexpr (SCALE == kEbF32) {
        s = __uint_as_float(m.x);
        b = __uint_as_float(m.y);
        rs = static_cast<int32_t>(m.z);
    } else {
        s = __half2float(__ushort_as_half(static_cast<unsigned short>(m.x & 0xFFFFu)));
        b = __half2float(__ushort_as_half(static_cast<unsigned short>(m.x >> 16)));
        rs = static_cast<int32_t>(m.y);
    }
}

template <int BPL>
__device__ __forceinline__ typename LaneWord<BPL>::T lds_word(const uint8_t* p) {
    if constexpr (BPL == 1) return *p;
    else if constexpr (BPL == 2) return *reinterpret_cast<const uint16_t*>(p);
    else if constexpr (BPL == 4) return *reinterpret_cast<const uint32_t*>(p);
    else return *reinterpret_cast<const uint64_t*>(p);
}

// Small unsigned integer -> float without the (quarter-rate) I2F: splice v into the mantissa of 2^23 and
// subtract 2^23 -- exact for v < 2^23. `bias` folds a constant offset into the same subtraction.
__device__ __forceinline__ float splice_u2f(uint32_t v, float bias) {
    return __fsub_rn(__uint_as_float(0x4B000000u | v), bias);
}
template <int ELEM, typename W>
__device__ __forceinline__ float decode_fast(W w, int c) {
    if constexpr (ELEM == kEbS8)  // int8 = (u8 ^ 0x80) - 128
        return splice_u2f((static_cast<uint32_t>(w >> (8 * c)) & 0xFFu) ^ 0x80u, 8388608.0f + 128.0f);
    else if constexpr (ELEM == kEbU8)
        return splice_u2f(static_cast<uint32_t>(w >> (8 * c)) & 0xFFu, 8388608.0f);
    else
        return splice_u2f(static_cast<uint32_t>(w >> (4 * c)) & 0xFu, 8388608.0f);
}

// Packed fp32x2 arithmetic (Blackwell FFMA2 / FADD2): two columns per instruction with IEEE round-to-
// nearest on each lane, i.e. bit-identical to the scalar ops. A product is formed as fma(a, b, nz) with nz
// = -0.0 supplied at RUN time: round(a*b + -0) == round(a*b) for every a, b, and because ptxas cannot see
// that nz is -0 it cannot contract the product with the following add (it does contract a plain
// mul.rn.f32x2 + add.rn.f32x2 pair into one FFMA2, which would change the rounding).
__device__ __forceinline__ unsigned long long f2_pack(float lo, float hi) {
    unsigned long long r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ void f2_unpack(unsigned long long v, float& lo, float& hi) {
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ unsigned long long f2_fma(unsigned long long a, unsigned long long b, unsigned long long c) {
    unsigned long long d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ unsigned long long f2_add(unsigned long long a, unsigned long long b) {
    unsigned long long d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// Columns c, c+1 of a lane word as spliced floats (before the magic subtraction).
template <int ELEM, typename W>
__device__ __forceinline__ unsigned long long decode_pair_bits(W w, int c) {
    if constexpr (ELEM == kEbU4) {
        const uint32_t lo = static_cast<uint32_t>(w >> (4 * c)) & 0xFu;
        const uint32_t hi = static_cast<uint32_t>(w >> (4 * c + 4)) & 0xFu;
        return static_cast<unsigned long long>(0x4B000000u | lo) |
               (static_cast<unsigned long long>(0x4B000000u | hi) << 32);
    } else {
        // one PRMT per element: byte c of the lane word under the 0x4B0000 mantissa splice (s8: the sign flip
        // is one XOR per 32-bit half, shared by its four elements)
        uint32_t half = (sizeof(W) == 8 && c >= 4) ? static_cast<uint32_t>(static_cast<uint64_t>(w) >> 32)
                                                   : static_cast<uint32_t>(w);
        if constexpr (ELEM == kEbS8) half ^= 0x80808080u;
        const uint32_t bsel = static_cast<uint32_t>(c & 3);  // selector nibbles [byte, 4, 5, 7] -> 0x4B0000bb
        return static_cast<unsigned long long>(__byte_perm(half, 0x4B000000u, 0x7540u | bsel)) |
               (static_cast<unsigned long long>(__byte_perm(half, 0x4B000000u, 0x7540u | (bsel + 1))) << 32);
    }
}

#ifndef ABFT_EB_MINB_SMALL
#define ABFT_EB_MINB_SMALL 2  // resident blocks per SM asked of ptxas for 32-byte slices (E4-class rows)
#endif
template <int ELEM, int SCALE, int CPL, int WPB, bool WEIGHTED, bool CHECKED>
#ifndef ABFT_EB_MINB_K16
#define ABFT_EB_MINB_K16 3  // s8 unweighted 128-byte slices (D5): the in-place constants leave room for a third block
#endif
__global__ void __launch_bounds__(256, (ELEM == kEbU4 ? CPL / 2 : CPL) <= 1 ? ABFT_EB_MINB_SMALL
                                       : (ELEM == kEbS8 && !WEIGHTED && CPL == 4) ? ABFT_EB_MINB_K16 : 2)
    eb_bag_async_kernel(const EbParams p, int log2d) {
    constexpr int BPL = ELEM == kEbU4 ? CPL / 2 : CPL;
    constexpr int SLICE = 32 * BPL;        // bytes of a row this warp needs
    constexpr int PIECES = SLICE / 16;     // 16-B copies per row slice
    constexpr int PER_LANE = kChunk * PIECES / 32;
    constexpr int GROUPS = 8 / WPB;        // bag groups (WPB warps each) per block
    constexpr bool K16 = ELEM == kEbS8 && !WEIGHTED;  // per-lookup constants fit the landed metadata slot
    using Stage = AsyncStage<BPL, K16, WEIGHTED>;
    extern __shared__ __align__(16) uint8_t eb_smem[];
    Stage& S = reinterpret_cast<Stage*>(eb_smem)[threadIdx.x >> 5];
    __shared__ double part_sum[8];
    __shared__ int part_emax[8], part_umin[8];
    __shared__ long long grp_bag[GROUPS];
    __shared__ uint32_t blk_flags;

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int grp = warp / WPB, slice = warp % WPB;
    const int64_t slice_byte = static_cast<int64_t>(slice) * SLICE;
    const double dd = static_cast<double>(p.dim);
    if (threadIdx.x == 0) blk_flags = 0;
    griddep_launch_dependents();  // the next kernel on the stream may start its prologue
    __syncthreads();
    griddep_wait();  // inputs and the per-stream words are those the preceding grid left
    auto group_sync = [&]() {
        if constexpr (WPB > 1)
            named_bar_sync(1 + grp, 32 * WPB);
        else
            __syncwarp();
    };

    // Persistent bag groups: each takes the next bag from a global counter, so long and short bags
    // balance across SMs (the work per bag varies 150x in E4). The next bag id is requested while the
    // current one is processed, hiding the atomic's round trip.
    constexpr int NST = Stage::NST;
    // The first bag of every group is static (its global group id); later ones come from the counter,
    // offset by the number of groups -- 2k simultaneous atomics on one address at launch cost ~2.5 us.
    const unsigned long long n_groups = static_cast<unsigned long long>(gridDim.x) * GROUPS;
    // (inline PTX: with atomicAdd the compiler aggregates the warp's request and shuffles the RESULT out right
    // after the atomic, which stalls the bag's start on the atomic's round trip; the ticket is only needed when
    // the bag is done)
    auto fetch = [&]() -> unsigned long long {
        // (atom.inc on the counter's low word; bag ids fit 32 bits -- the launcher refuses larger batches. The address
        // carries laneid * zero_rt, zero at run time: on an address it can prove warp-uniform ptxas aggregates the
        // atomic -- also an inline-PTX one -- and shuffles the result out at once, which stalls the bag's start on the
        // atomic's round trip)
        uint32_t ticket = 0;
        if (slice == 0 && lane == 0) {
            uint32_t lid;  // (read here: inside this branch the compiler knows `lane` is 0)
            asm volatile("mov.u32 %0, %%laneid;" : "=r"(lid));
            asm volatile("atom.global.inc.u32 %0, [%1], 0xffffffff;"
                         : "=r"(ticket)
                         : "l"(reinterpret_cast<uint32_t*>(p.ws_bag_ctr) + 2 * lid * p.zero_rt));
        }
        return ticket;
    };
    auto share = [&](unsigned long long ticket) -> int64_t {  // broadcast lane 0 / slice 0's id to the group
        const unsigned long long b0 = n_groups + ticket;
        if constexpr (WPB == 1) {
            return static_cast<int64_t>(__shfl_sync(0xffffffffu, b0, 0));
        } else {
            if (slice == 0 && lane == 0) grp_bag[grp] = static_cast<long long>(b0);
            group_sync();
            const int64_t v = grp_bag[grp];
            group_sync();
            return v;
        }
    };
    unsigned long long* tr = p.trace ? p.trace + 16ull * (blockIdx.x * 8 + warp) : nullptr;
    if (tr && lane == 0) tr[0] = globaltimer();
    int nb_done = 0;
    // first bags strided over the blocks (group g of block b: bag g * blocks + b), so a batch smaller than the grid's
    // bag groups spreads evenly over the SMs instead of filling the first blocks
    int64_t bag = static_cast<int64_t>(grp) * gridDim.x + blockIdx.x;
    while (bag < p.num_bags) {
        if (tr && lane == 0 && nb_done < 4) tr[1 + 3 * nb_done] = globaltimer();
        // the bag's table view: the launch's own fields, or (grouped tables) its table's descriptor
        EbParams tv = p;
        int64_t lb = bag;  // bag index within its table
        if (p.tables) {
            // 32-bit division: bag ids fit (the launcher refuses larger batches), and a 64-bit divide is a
            // ~40-instruction sequence on the per-bag path
            const int64_t t = static_cast<int64_t>(static_cast<uint32_t>(bag) / static_cast<uint32_t>(p.bags_per_table));
            lb = bag - t * p.bags_per_table;
            const EbTableDesc& dsc = p.tables[t];
            tv.data = dsc.data;
            tv.meta = dsc.meta;
            tv.meta_stride = dsc.meta_stride;
            tv.rows = dsc.rows;
            tv.row_stride = dsc.row_stride;
            tv.offsets = dsc.offsets;
            tv.indices = dsc.indices;
            tv.weights = dsc.weights;
            tv.out_dest = dsc.out_dest;
            tv.flag_dest = dsc.flag_dest;
        }

        float acc[CPL];
#pragma unroll
        for (int c = 0; c < CPL; ++c) acc[c] = 0.0f;
        unsigned long long acc2[CPL / 2 > 0 ? CPL / 2 : 1];  // packed column pairs (CPL >= 2)
#pragma unroll
        for (int c = 0; c < (CPL / 2 > 0 ? CPL / 2 : 1); ++c) acc2[c] = 0ull;  // (+0.0, +0.0)
        const unsigned long long nz2 = f2_pack(p.neg_zero, p.neg_zero);
        const unsigned long long magic2 = f2_pack(-8388608.0f - (ELEM == kEbS8 ? 128.0f : 0.0f),
                                                  -8388608.0f - (ELEM == kEbS8 ? 128.0f : 0.0f));
        double csum = 0.0;
        bool oob = false;
        const int64_t beg = tv.offsets[lb], end = tv.offsets[lb + 1];
        // bag length in 32 bits; a table without rows (every lookup out of range) or an absurd length (corrupt
        // offsets) reports out_of_range and pools nothing
        int len = 0;
        if (end > beg) {
            if (tv.rows <= 0 || end - beg > (int64_t{1} << 30))
                oob = true;
            else
                len = static_cast<int>(end - beg);
        }
        const int nchunks = (len + kChunk - 1) / kChunk;
        const int64_t* const idx0 = tv.indices + beg + lane;
        const float* const w0 = WEIGHTED ? tv.weights + beg + lane : nullptr;
        const uint32_t meta_stride32 = static_cast<uint32_t>(tv.meta_stride);
        // this lane's 16-byte part of a row slice (row 0) and the row stride (< 2^32: checked by the launcher)
        const uint8_t* const src0 = tv.data + slice_byte + (lane % PIECES) * 16;
        const uint32_t stride32 = static_cast<uint32_t>(tv.row_stride);
        // Issue the gathers of chunk `ch` (indices `ix`, one per lane) into ring slot ch % NST. Slots past
        // the bag or out of range get a neutral record (scale = bias = 0, weight 1): they add +0.0, an
        // exact no-op on the running sums (which start at +0.0 and never become -0.0 in round-to-nearest),
        // so the consumer needs no per-lookup branch. Row pieces, metadata and weights all land through
        // cp.async; one commit group per chunk (empty groups keep the count uniform).
        auto issue = [&](int ch, int64_t ix) {
            if (ch < nchunks) {
                const int sl = ch % NST;
                const int cnt = min(kChunk, len - ch * kChunk);
                const bool valid = lane < cnt && static_cast<uint64_t>(ix) < static_cast<uint64_t>(tv.rows);
                if (lane < cnt && !valid) oob = true;
                // an out-of-range lookup gathers row 0 under its neutral record (a table without rows has no chunks)
                const uint32_t rid = valid ? static_cast<uint32_t>(ix) : 0u;
                if (valid) {
                    const uint8_t* const mrec = mad_wide_u32(rid, meta_stride32, reinterpret_cast<const uint8_t*>(tv.meta));
                    if constexpr (SCALE == kEbF32)
                        cp_async16(&S.meta[sl][lane], mrec);
                    else
                        cp_async8(&S.meta[sl][lane], mrec);
                    if constexpr (WEIGHTED) cp_async4(&S.w[sl][lane], w0 + ch * kChunk);
                } else {
                    S.meta[sl][lane] = make_uint4(0u, 0u, 0u, 0u);
                    if constexpr (WEIGHTED) S.w[sl][lane] = 1.0f;
                }
                // row pieces: piece = lane + 32 i covers row piece / PIECES, 16-byte part piece % PIECES; the row id
                // comes from the lane that holds the lookup (one shuffle, one 32 x 32 -> 64-bit multiply-add)
                uint8_t* const dst0 = &S.rows[sl][0][0] + lane * 16;
#pragma unroll
                for (int i = 0; i < PER_LANE; ++i) {
                    const int r = (lane + 32 * i) / PIECES;
                    const uint32_t rr = __shfl_sync(0xffffffffu, rid, r);
                    if (r < cnt) cp_async16_l1(dst0 + 512 * i, mad_wide_u32(rr, stride32, src0));
                }
            }
            cp_async_commit();
        };
        auto index_of = [&](int ch) -> int64_t { return ch * kChunk + lane < len ? idx0[ch * kChunk] : -1; };
        // prologue: NST-1 chunks in flight, the index of the next one loaded ahead
        {
            int64_t ixs[NST - 1];
#pragma unroll
            for (int c = 0; c < NST - 1; ++c) ixs[c] = c < nchunks ? index_of(c) : -1;
#pragma unroll
            for (int c = 0; c < NST - 1; ++c) issue(c, ixs[c]);
        }
        int64_t ix_ahead = NST - 1 < nchunks ? index_of(NST - 1) : -1;
        // the next bag id is requested once this bag's first gathers are in flight (at launch every group
        // requests at once: on one address those atomics serialise for ~1 us, which must not delay the
        // first loads) and is only consumed when this bag is done
        const unsigned long long next_req = fetch();
        for (int ch = 0; ch < nchunks; ++ch) {
            const int sl = ch % NST;
            issue(ch + NST - 1, ix_ahead);
            ix_ahead = ch + NST < nchunks ? index_of(ch + NST) : -1;
            cp_async_wait<NST - 1>();  // chunk ch has landed
            __syncwarp();
#ifdef ABFT_EB_TRACE  // (debug build: when the bag's first chunk landed)
            if (tr && lane == 0 && ch == 0 && nb_done < 4) tr[2 + 3 * nb_done] = globaltimer();
#endif
            const int cnt = min(kChunk, len - ch * kChunk);
            // the chunk's per-lookup constants, lane-parallel (a neutral slot has s = b = 0, w = 1: term +0.0)
            bool fast;
            {
                float s, b;
                int32_t rs;
                smem_meta<SCALE>(S.meta[sl][lane], s, b, rs);
                const float w = WEIGHTED ? S.w[sl][lane] : 1.0f;
                const double term = (CHECKED && slice == 0) ? csum_term(s, b, rs, w, dd, WEIGHTED) : 0.0;
                if constexpr (K16) {
                    S.meta[sl][lane] = make_uint4(__float_as_uint(s), __float_as_uint(b),
                                                  static_cast<uint32_t>(__double2loint(term)),
                                                  static_cast<uint32_t>(__double2hiint(term)));
                } else {
                    LookupConst kc;
                    kc.s_lo = s;
                    kc.s_hi = ELEM == kEbU4 ? s * 0.0625f : s;
                    kc.c_lo = -(kc.s_lo * 8388608.0f);
                    kc.c_hi = -(kc.s_hi * 8388608.0f);
                    kc.b = b;
                    kc.w = w;
                    kc.term = term;
                    S.k[lane] = kc;
                }
                // u8 / u4 chunks whose every scale admits the exact splice FMA take the short column path
                fast = ELEM != kEbS8 && __all_sync(0xffffffffu, splice_safe(s));
                __syncwarp();
            }
            const int tmax = (cnt + 3) & ~3;  // slots cnt..tmax-1 are neutral
            // Four lookups per step with the instruction-level parallelism spelled out: every shared-memory
            // load of the four first, then their (independent) column values, then the accumulations in
            // lookup order -- the only loop-carried chains are the per-column fp32 adds and the cSum DADD.
            // Per column, in the reference's rounding: x = s*q (one rounding), x += b, x *= w (weighted), r += x.
            using Word = typename LaneWord<BPL>::T;
            constexpr int NP = CPL >= 2 ? CPL / 2 : 1;
            auto column_loop = [&](auto fast_tag) {
                constexpr bool FAST = decltype(fast_tag)::value;
#pragma unroll 1
                for (int t0 = 0; t0 < tmax; t0 += 4) {
                    Word wd[4];
                    float4 ka[4];   // s_lo, s_hi, c_lo, c_hi
                    float4 kb[4];   // b, w, term
#pragma unroll
                    for (int u = 0; u < 4; ++u) {
                        wd[u] = lds_word<BPL>(&S.rows[sl][t0 + u][lane * BPL]);
                        if constexpr (K16) {  // (s, b, term) in the metadata slot
                            const uint4 m = S.meta[sl][t0 + u];
                            ka[u] = make_float4(__uint_as_float(m.x), 0.f, 0.f, 0.f);
                            kb[u] = make_float4(__uint_as_float(m.y), 1.0f, __uint_as_float(m.z), __uint_as_float(m.w));
                        } else {
                            ka[u] = *reinterpret_cast<const float4*>(&S.k[t0 + u].s_lo);
                            kb[u] = *reinterpret_cast<const float4*>(&S.k[t0 + u].b);
                        }
                    }
                    if constexpr (CPL >= 2) {
                        unsigned long long xv[4][NP];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const unsigned long long b2 = f2_pack(kb[u].x, kb[u].x);
                            const unsigned long long w2 = f2_pack(kb[u].y, kb[u].y);
#pragma unroll
                            for (int c = 0; c < CPL; c += 2) {
                                unsigned long long x2;
                                if constexpr (FAST) {  // s*q in one FMA on the spliced column values
                                    x2 = f2_fma(splice_pair_bits<ELEM>(wd[u], c), f2_pack(ka[u].x, ka[u].y),
                                                f2_pack(ka[u].z, ka[u].w));
                                } else {  // exact q by the magic subtraction, then s*q (fma with -0: no contraction)
                                    const unsigned long long q2 = f2_add(decode_pair_bits<ELEM>(wd[u], c), magic2);
                                    x2 = f2_fma(f2_pack(ka[u].x, ka[u].x), q2, nz2);
                                }
                                x2 = f2_add(x2, b2);
                                if constexpr (WEIGHTED) x2 = f2_fma(w2, x2, nz2);
                                xv[u][c / 2] = x2;
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u)
#pragma unroll
                            for (int c = 0; c < NP; ++c) acc2[c] = f2_add(acc2[c], xv[u][c]);
                    } else {
                        float xv[4][CPL];
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
#pragma unroll
                            for (int c = 0; c < CPL; ++c) {
                                float x;
                                if constexpr (FAST)
                                    x = __fmaf_rn(__uint_as_float(static_cast<uint32_t>(splice_pair_bits<ELEM>(wd[u], c))),
                                                  ka[u].x, ka[u].z);
                                else
                                    x = __fmul_rn(ka[u].x, decode_fast<ELEM>(wd[u], c));
                                x = __fadd_rn(x, kb[u].x);
                                if constexpr (WEIGHTED) x = __fmul_rn(kb[u].y, x);
                                xv[u][c] = x;
                            }
                        }
#pragma unroll
                        for (int u = 0; u < 4; ++u)
#pragma unroll
                            for (int c = 0; c < CPL; ++c) acc[c] = __fadd_rn(acc[c], xv[u][c]);
                    }
                    // cSum in the reference's sequential fp64 order (P:src/embedding_abft.cpp:69-76), kept by every
                    // lane of the slice-0 warp (same terms, same order, same value). A neutral slot's +0.0 term is
                    // an exact no-op (cSum starts at +0.0 and never becomes -0.0 in round-to-nearest).
                    if constexpr (CHECKED)
                        if (slice == 0) {
#pragma unroll
                            for (int u = 0; u < 4; ++u)
                                csum = __dadd_rn(csum, __hiloint2double(__float_as_int(kb[u].w), __float_as_int(kb[u].z)));
                        }
                }
            };
            if constexpr (ELEM != kEbS8) {
                if (fast)
                    column_loop(std::true_type{});
                else
                    column_loop(std::false_type{});
            } else {
                column_loop(std::false_type{});
            }
            __syncwarp();  // slot `sl` may be refilled by a later issue
        }
        cp_async_wait<0>();  // drain the (empty) trailing groups before the ring is reused
        if constexpr (CPL >= 2) {
#pragma unroll
            for (int c = 0; c < CPL; c += 2) f2_unpack(acc2[c / 2], acc[c], acc[c + 1]);
        }
        csum = __shfl_sync(0xffffffffu, csum, 0);
        if (__any_sync(0xffffffffu, oob) && lane == 0 && p.status) atomicOr(p.status, 1);
        float* dst = out_row(tv, lb) + slice * 32 * CPL + lane * CPL;
        if (CPL % 4 == 0 && (reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
#pragma unroll
            for (int c = 0; c + 3 < CPL; c += 4)
                *reinterpret_cast<float4*>(dst + c) = make_float4(acc[c], acc[c + 1], acc[c + 2], acc[c + 3]);
        } else {
#pragma unroll
            for (int c = 0; c < CPL; ++c) dst[c] = acc[c];
        }
        if constexpr (CHECKED) {
            // Exactness of the order-free fp64 sum from the outputs' biased exponents alone: every nonzero output is a
            // multiple of its ulp 2^(e - 150) and below 2^(e - 126) (denormals: e = 1), so with emax / emin over the
            // bag's outputs every partial sum of the d values is a multiple of 2^(emin - 150) below
            // 2^(emax - 126 + log2 d): exact in fp64 when emax - emin + 24 + log2 d <= 53.
            uint32_t emax = 0u, emin = 255u;
#pragma unroll
            for (int c = 0; c < CPL; ++c) {
                const uint32_t bits = __float_as_uint(acc[c]) & 0x7FFFFFFFu;
                const uint32_t e = max(bits >> 23, 1u);
                if (bits) {
                    emax = max(emax, e);
                    emin = min(emin, e);
                }
            }
            double sm = 0.0;
#pragma unroll
            for (int c = 0; c < CPL; ++c) sm = __dadd_rn(sm, static_cast<double>(acc[c]));
            emax = __reduce_max_sync(0xffffffffu, emax);
            emin = __reduce_min_sync(0xffffffffu, emin);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) sm = __dadd_rn(sm, __shfl_xor_sync(0xffffffffu, sm, o));
            if constexpr (WPB > 1) {
                if (lane == 0) {
                    part_sum[warp] = sm;
                    part_emax[warp] = static_cast<int>(emax);
                    part_umin[warp] = static_cast<int>(emin);
                }
            }
            // only the WPB warps of this bag synchronise (their slices and outputs are complete)
            group_sync();
            if (slice == 0) {
                int E = static_cast<int>(emax), U = static_cast<int>(emin);  // WPB == 1: the warp's own reduction
                double exact = sm;
                if constexpr (WPB > 1) {
                    E = 0;
                    U = 255;
                    exact = 0.0;
#pragma unroll
                    for (int s2 = 0; s2 < WPB; ++s2) {
                        E = max(E, part_emax[warp + s2]);
                        U = min(U, part_umin[warp + s2]);
                        exact = __dadd_rn(exact, part_sum[warp + s2]);
                    }
                }
                double rsum;
                if (E == 0) {
                    rsum = 0.0;
                } else if (E - U + 24 + log2d <= 53) {
                    rsum = exact;  // every partial sum is exact, so any order gives the reference's value
                } else {
                    rsum = 0.0;  // the reference's sequential order over the stored outputs
                    const float* row = out_row(tv, lb);
                    for (int j0 = 0; j0 < p.dim; j0 += 32) {
                        const float v = (j0 + lane < p.dim) ? row[j0 + lane] : 0.0f;
                        for (int l = 0; l < 32 && j0 + l < p.dim; ++l)
                            rsum = __dadd_rn(rsum, static_cast<double>(__shfl_sync(0xffffffffu, v, l)));
                    }
                }
                const double diff = fabs(__dsub_rn(rsum, csum));
                const double mx = fmax(fmax(fabs(rsum), fabs(csum)), 1.0);
                const int flag = diff > __dmul_rn(1e-5, mx);
                if (lane == 0) {
                    if (uint8_t* fs = flag_slot(tv, lb)) *fs = static_cast<uint8_t>(flag);
                    if (p.rsum) p.rsum[bag] = rsum;
                    if (p.csum) p.csum[bag] = csum;
                    if (flag) atomicAdd(&blk_flags, 1u);
                }
            }
            group_sync();  // part_* may be rewritten by the group's next bag
        }
        if (tr && lane == 0 && nb_done < 4) tr[3 + 3 * nb_done] = globaltimer();
        ++nb_done;
        bag = share(next_req);
    }
    if (tr && lane == 0) {
        tr[13] = globaltimer();
        tr[14] = nb_done;
    }
    // last block out publishes the flag count and resets the per-stream counters
    __syncthreads();
    if (threadIdx.x == 0) eb_block_done(p, CHECKED ? blk_flags : 0u, true);
}

// Generic path (any d <= 256, unaligned rows): warp per bag, lane owns columns lane + 32*c, byte loads.
template <int ELEM, int SCALE, bool WEIGHTED, bool CHECKED>
__global__ void __launch_bounds__(256) eb_bag_generic_kernel(const EbParams p, int log2d) {
    constexpr int NC = kGenericSlots;
    constexpr int R = 8;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t bag = static_cast<int64_t>(blockIdx.x) * 8 + warp;
    __shared__ uint32_t blk_flags;
    if (threadIdx.x == 0) blk_flags = 0;
    __syncthreads();
    if (bag < p.num_bags) {
        const int64_t beg = p.offsets[bag], end = p.offsets[bag + 1];
        float acc[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) acc[c] = 0.0f;
        double csum = 0.0;
        bool oob = false;
        const double dd = static_cast<double>(p.dim);
        for (int64_t base = beg; base < end; base += R) {
            const int cnt = static_cast<int>(min(static_cast<int64_t>(R), end - base));
            int64_t my_idx = -1;
            float my_s = 0.f, my_b = 0.f, my_w = 1.f;
            int32_t my_rs = 0;
            if (lane < cnt) {
                const int64_t ix = p.indices[base + lane];
                if (static_cast<uint64_t>(ix) >= static_cast<uint64_t>(p.rows)) {
                    oob = true;
                } else {
                    my_idx = ix;
                    load_meta<SCALE>(p.meta, ix, p.meta_stride, my_s, my_b, my_rs);
                }
                if constexpr (WEIGHTED) my_w = p.weights[base + lane];
            }
            uint32_t data[R][NC];
#pragma unroll
            for (int t = 0; t < R; ++t) {
                const int64_t it = __shfl_sync(0xffffffffu, my_idx, t);
#pragma unroll
                for (int c = 0; c < NC; ++c) {
                    const int64_t j = lane + 32 * c;
                    // unconditional load at a safe address (row 0, byte 0 for skipped slots); decode at use
                    const bool ok = t < cnt && it >= 0 && j < p.dim;
                    const int64_t byte = ELEM == kEbU4 ? (j >> 1) : j;
                    data[t][c] = __ldg(p.data + (ok ? it * p.row_stride + byte : 0));
                }
            }
#pragma unroll
            for (int t = 0; t < R; ++t) {
                if (t < cnt) {
                    const int64_t it = __shfl_sync(0xffffffffu, my_idx, t);
                    const float s = __shfl_sync(0xffffffffu, my_s, t);
                    const float b = __shfl_sync(0xffffffffu, my_b, t);
                    const float w = WEIGHTED ? __shfl_sync(0xffffffffu, my_w, t) : 1.0f;
                    const int32_t rs = __shfl_sync(0xffffffffu, my_rs, t);
                    if (it >= 0) {
#pragma unroll
                        for (int c = 0; c < NC; ++c) {
                            const uint32_t raw = data[t][c];
                            const uint32_t jj = static_cast<uint32_t>(lane + 32 * c);
                            const float q = ELEM == kEbS8   ? static_cast<float>(static_cast<int8_t>(raw))
                                            : ELEM == kEbU8 ? static_cast<float>(raw & 0xFFu)
                                                            : static_cast<float>((raw >> (4 * (jj & 1))) & 0xFu);
                            float x = __fadd_rn(__fmul_rn(s, q), b);
                            if constexpr (WEIGHTED) x = __fmul_rn(w, x);
                            if (lane + 32 * c < p.dim) acc[c] = __fadd_rn(acc[c], x);
                        }
                        if constexpr (CHECKED) csum = __dadd_rn(csum, csum_term(s, b, rs, w, dd, WEIGHTED));
                    }
                }
            }
        }
        if (__any_sync(0xffffffffu, oob) && lane == 0 && p.status) atomicOr(p.status, 1);
        float* dst = out_row(p, bag);
#pragma unroll
        for (int c = 0; c < NC; ++c)
            if (lane + 32 * c < p.dim) dst[lane + 32 * c] = acc[c];
        if constexpr (CHECKED) {
            int emax = -100000, umin = 100000;
#pragma unroll
            for (int c = 0; c < NC; ++c)
                if (lane + 32 * c < p.dim) bit_span(acc[c], emax, umin);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) {
                emax = max(emax, __shfl_xor_sync(0xffffffffu, emax, o));
                umin = min(umin, __shfl_xor_sync(0xffffffffu, umin, o));
            }
            double rsum = 0.0;
            if (emax != -100000 && emax + 1 + log2d - umin <= 53) {
                double s = 0.0;
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    if (lane + 32 * c < p.dim) s = __dadd_rn(s, static_cast<double>(acc[c]));
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
                rsum = s;
            } else if (emax != -100000) {
#pragma unroll
                for (int c = 0; c < NC; ++c)
                    for (int l = 0; l < 32; ++l) {
                        const float v = __shfl_sync(0xffffffffu, acc[c], l);
                        if (l + 32 * c < p.dim) rsum = __dadd_rn(rsum, static_cast<double>(v));
                    }
            }
            const double diff = fabs(__dsub_rn(rsum, csum));
            const double mx = fmax(fmax(fabs(rsum), fabs(csum)), 1.0);
            const int flag = diff > __dmul_rn(1e-5, mx);
            if (lane == 0) {
                if (uint8_t* fs = flag_slot(p, bag)) *fs = static_cast<uint8_t>(flag);
                if (p.rsum) p.rsum[bag] = rsum;
                if (p.csum) p.csum[bag] = csum;
                if (flag) atomicAdd(&blk_flags, 1u);
            }
        }
    }
    if constexpr (CHECKED) {
        if (p.flag_count) {
            __syncthreads();
            if (threadIdx.x == 0) eb_block_done(p, blk_flags, false);
        }
    }
}

// Row sums + metadata packing. One warp per row. If `given_sums` is non-null the stored sums are
// taken from it (stale sums survive, as load_table(validate=false)); `mismatch` counts rows whose
// given sum differs from the recomputed one (load_table validation, P:src/embedding_abft.cpp:139-143).
template <int ELEM, int SCALE>
__global__ void __launch_bounds__(256) eb_meta_kernel(const uint8_t* __restrict__ data, int64_t rows, int64_t dim,
                                                      int64_t row_stride, const void* __restrict__ scales,
                                                      const void* __restrict__ biases,
                                                      const int32_t* __restrict__ given_sums, void* __restrict__ meta,
                                                      int32_t* __restrict__ sums_out, uint32_t* mismatch) {
    const int lane = threadIdx.x & 31;
    for (int64_t r = (static_cast<int64_t>(blockIdx.x) * 256 + threadIdx.x) >> 5; r < rows;
         r += (static_cast<int64_t>(gridDim.x) * 256) >> 5) {
        const uint8_t* row = data + r * row_stride;
        int32_t s = 0;
        for (int64_t j = lane; j < dim; j += 32) {
            if (ELEM == kEbS8)
                s += static_cast<int8_t>(row[j]);
            else if (ELEM == kEbU8)
                s += row[j];
            else
                s += (row[j >> 1] >> (4 * (j & 1))) & 0xF;
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) {
            int32_t stored = s;
            if (given_sums) {
                stored = given_sums[r];
                if (mismatch && stored != s) atomicAdd(mismatch, 1u);
            }
            if (sums_out) sums_out[r] = s;
            if (meta) {
                if constexpr (SCALE == kEbF32) {
                    EbMetaF32 mrec;
                    mrec.scale = reinterpret_cast<const float*>(scales)[r];
                    mrec.bias = reinterpret_cast<const float*>(biases)[r];
                    mrec.row_sum = stored;
                    mrec.pad = 0;
                    reinterpret_cast<EbMetaF32*>(meta)[r] = mrec;
                } else {
                    EbMetaF16 mrec;
                    mrec.scale = reinterpret_cast<const uint16_t*>(scales)[r];
                    mrec.bias = reinterpret_cast<const uint16_t*>(biases)[r];
                    mrec.row_sum = stored;
                    reinterpret_cast<EbMetaF16*>(meta)[r] = mrec;
                }
            }
        }
    }
}

// ------------------------------------------------------------------ host launchers
template <int ELEM, int SCALE, int CPL, int WPB>
static cudaError_t launch_bag_fast(const EbParams& p, bool checked, int log2d, cudaStream_t st) {
    const unsigned blocks = static_cast<unsigned>((p.num_bags + (8 / WPB) - 1) / (8 / WPB));
    const bool w = p.weights != nullptr;
    if (checked) {
        if (w)
            eb_bag_kernel<ELEM, SCALE, CPL, WPB, true, true><<<blocks, 256, 0, st>>>(p, log2d);
        else
            eb_bag_kernel<ELEM, SCALE, CPL, WPB, false, true><<<blocks, 256, 0, st>>>(p, log2d);
    } else {
        if (w)
            eb_bag_kernel<ELEM, SCALE, CPL, WPB, true, false><<<blocks, 256, 0, st>>>(p, log2d);
        else
            eb_bag_kernel<ELEM, SCALE, CPL, WPB, false, false><<<blocks, 256, 0, st>>>(p, log2d);
    }
    return cudaGetLastError();
}

template <int ELEM, int SCALE, int CPL, int WPB, bool W, bool CK>
static cudaError_t launch_async_one(const EbParams& p, int log2d, cudaStream_t st) {
    constexpr int BPL = ELEM == kEbU4 ? CPL / 2 : CPL;
    constexpr int smem = 8 * static_cast<int>(sizeof(AsyncStage<BPL, ELEM == kEbS8 && !W, W>));
    auto kern = eb_bag_async_kernel<ELEM, SCALE, CPL, WPB, W, CK>;
    static bool attr[kMaxDevices] = {};  // per device
    static int per_sm_dev[kMaxDevices] = {};
    const int dev = current_device();
    if (!attr[dev]) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        if (e != cudaSuccess) return e;
        attr[dev] = true;
    }
    int& per_sm = per_sm_dev[dev];
    if (!per_sm) {
        int o = 0;
        cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, kern, 256, smem);
        per_sm = (e != cudaSuccess || o < 1) ? 1 : o;
    }
    if (p.num_bags >= (int64_t{1} << 31)) return cudaErrorInvalidValue;  // 32-bit bag tickets
    // every resident block slot gets work before any block gets a second bag group (one bag per block at least)
    const int64_t cap = static_cast<int64_t>(per_sm) * device_sm_count();
    const unsigned blocks = static_cast<unsigned>(p.num_bags < cap ? p.num_bags : cap);
    // programmatic dependent launch: consecutive batches overlap launch and prologue with the tail
    static const bool pdl = std::getenv("ABFTLP_NO_PDL") == nullptr;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(blocks);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl ? 1 : 0;
    return cudaLaunchKernelEx(&cfg, kern, p, log2d);
}

template <int ELEM, int SCALE, int CPL, int WPB>
static cudaError_t launch_bag_async(const EbParams& p, bool checked, int log2d, cudaStream_t st) {
    const bool w = p.weights != nullptr;
    if (checked)
        return w ? launch_async_one<ELEM, SCALE, CPL, WPB, true, true>(p, log2d, st)
                 : launch_async_one<ELEM, SCALE, CPL, WPB, false, true>(p, log2d, st);
    return w ? launch_async_one<ELEM, SCALE, CPL, WPB, true, false>(p, log2d, st)
             : launch_async_one<ELEM, SCALE, CPL, WPB, false, false>(p, log2d, st);
}

template <int ELEM, int SCALE>
static cudaError_t launch_bag_generic(const EbParams& p, bool checked, int log2d, cudaStream_t st) {
    const unsigned blocks = static_cast<unsigned>((p.num_bags + 7) / 8);
    const bool w = p.weights != nullptr;
    if (checked) {
        if (w)
            eb_bag_generic_kernel<ELEM, SCALE, true, true><<<blocks, 256, 0, st>>>(p, log2d);
        else
            eb_bag_generic_kernel<ELEM, SCALE, false, true><<<blocks, 256, 0, st>>>(p, log2d);
    } else {
        if (w)
            eb_bag_generic_kernel<ELEM, SCALE, true, false><<<blocks, 256, 0, st>>>(p, log2d);
        else
            eb_bag_generic_kernel<ELEM, SCALE, false, false><<<blocks, 256, 0, st>>>(p, log2d);
    }
    return cudaGetLastError();
}

// Warps per bag: enough warps to keep ~32 resident per SM when the batch is small.
static int pick_wpb(int64_t num_bags, int64_t d_over_32, bool u4) {
    if (const char* e = std::getenv("ABFTLP_EB_WPB")) {  // tuning override (1, 2 or 4; must divide d/32)
        const int f = std::atoi(e);
        if ((f == 1 || f == 2 || f == 4) && d_over_32 % f == 0 && (!u4 || d_over_32 / f >= 2)) return f;
    }
    // Split a bag over several warps only for small batches: a warp that owns the whole row amortises the
    // per-lookup metadata work over more columns, and occupancy (not per-bag latency) bounds the rest.
    const int64_t target = 148 * 8;
    int wpb = 1;
    while (wpb < 4 && num_bags * wpb * 2 <= target && (d_over_32 % (wpb * 2)) == 0 &&
           (!u4 || (d_over_32 / (wpb * 2)) >= 2))
        wpb *= 2;
    return wpb;
}

template <int ELEM, int SCALE>
static cudaError_t launch_bag_elem(const EbParams& p, bool checked, int log2d, cudaStream_t st) {
    const int64_t d = p.dim;
    const bool aligned_rows = (p.row_stride % 8) == 0 && (reinterpret_cast<uintptr_t>(p.data) % 8) == 0;
    if (aligned_rows && d % 32 == 0) {
        const int64_t d32 = d / 32;  // columns per lane when one warp owns the whole row
        const int wpb = pick_wpb(p.num_bags, d32, ELEM == kEbU4);
        const int64_t cpl = d32 / wpb;
        // (the gather kernel forms row addresses as a 32 x 32 -> 64-bit multiply-add)
        const bool async_ok = (p.tables || (p.row_stride < (int64_t{1} << 32) && p.rows <= (int64_t{1} << 32))) &&
                              (p.row_stride % 16) == 0 && (reinterpret_cast<uintptr_t>(p.data) % 16) == 0 &&
                              (reinterpret_cast<uintptr_t>(p.meta) % 16) == 0 && !std::getenv("ABFTLP_EB_SYNC");
        if (p.tables && !async_ok) return cudaErrorNotSupported;  // grouped tables: async kernel only
        if (async_ok) {
#define ABFT_ASYNC(CPL_, WPB_) \
    if (cpl == CPL_ && wpb == WPB_) return launch_bag_async<ELEM, SCALE, CPL_, WPB_>(p, checked, log2d, st)
            if constexpr (ELEM != kEbU4) {
                ABFT_ASYNC(1, 1);
                ABFT_ASYNC(1, 2);
                ABFT_ASYNC(1, 4);
            }
            ABFT_ASYNC(2, 1);
            ABFT_ASYNC(2, 2);
            ABFT_ASYNC(2, 4);
            ABFT_ASYNC(4, 1);
            ABFT_ASYNC(4, 2);
            ABFT_ASYNC(4, 4);
            ABFT_ASYNC(8, 1);
            ABFT_ASYNC(8, 2);
#undef ABFT_ASYNC
        }
#define ABFT_FAST(CPL_, WPB_) \
    if (cpl == CPL_ && wpb == WPB_) return launch_bag_fast<ELEM, SCALE, CPL_, WPB_>(p, checked, log2d, st)
        if constexpr (ELEM != kEbU4) {
            ABFT_FAST(1, 1);
            ABFT_FAST(1, 2);
            ABFT_FAST(1, 4);
        }
        ABFT_FAST(2, 1);
        ABFT_FAST(2, 2);
        ABFT_FAST(2, 4);
        ABFT_FAST(4, 1);
        ABFT_FAST(4, 2);
        ABFT_FAST(4, 4);
        ABFT_FAST(8, 1);
        ABFT_FAST(8, 2);
#undef ABFT_FAST
    }
    if (p.tables) return cudaErrorNotSupported;  // grouped tables: async kernel only
    if (d > 32 * kGenericSlots) return cudaErrorInvalidValue;
    return launch_bag_generic<ELEM, SCALE>(p, checked, log2d, st);
}

cudaError_t launch_eb_bags(int elem, int scale, const EbParams& p, bool checked, cudaStream_t st) {
    if (p.num_bags <= 0) return cudaSuccess;
    int log2d = 0;
    while ((int64_t{1} << log2d) < p.dim) ++log2d;
#ifdef ABFT_EB_DEV  // (development: compile one element / scale type only, for quick SASS inspection)
    return launch_bag_elem<ABFT_EB_DEV, kEbF32>(p, checked, log2d, st);
#endif
    if (scale == kEbF32) {
        if (elem == kEbS8) return launch_bag_elem<kEbS8, kEbF32>(p, checked, log2d, st);
        if (elem == kEbU8) return launch_bag_elem<kEbU8, kEbF32>(p, checked, log2d, st);
        return launch_bag_elem<kEbU4, kEbF32>(p, checked, log2d, st);
    }
    if (elem == kEbS8) return launch_bag_elem<kEbS8, kEbF16>(p, checked, log2d, st);
    if (elem == kEbU8) return launch_bag_elem<kEbU8, kEbF16>(p, checked, log2d, st);
    return launch_bag_elem<kEbU4, kEbF16>(p, checked, log2d, st);
}

cudaError_t launch_eb_meta(int elem, int scale, const uint8_t* data, int64_t rows, int64_t dim, int64_t row_stride,
                           const void* scales, const void* biases, const int32_t* given_sums, void* meta,
                           int32_t* sums_out, uint32_t* mismatch, cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    int64_t blocks = (rows + 7) / 8;
    if (blocks > 148 * 16) blocks = 148 * 16;
    const unsigned g = static_cast<unsigned>(blocks);
#define ABFT_META(E, S) \
    eb_meta_kernel<E, S><<<g, 256, 0, st>>>(data, rows, dim, row_stride, scales, biases, given_sums, meta, sums_out, mismatch)
    if (scale == kEbF32) {
        if (elem == kEbS8) ABFT_META(kEbS8, kEbF32);
        else if (elem == kEbU8) ABFT_META(kEbU8, kEbF32);
        else ABFT_META(kEbU4, kEbF32);
    } else {
        if (elem == kEbS8) ABFT_META(kEbS8, kEbF16);
        else if (elem == kEbU8) ABFT_META(kEbU8, kEbF16);
        else ABFT_META(kEbU4, kEbF16);
    }
#undef ABFT_META
    return cudaGetLastError();
}

// Interleaved record layout (EbTable::packed): row bytes, then the metadata record, in one 64-byte
// slot per row, so a lookup is one 64-byte DRAM access instead of two scattered ones. One thread per
// 16-byte piece of the record.
__global__ void eb_pack_kernel(const uint8_t* __restrict__ data, int64_t rows, int64_t row_bytes, int64_t row_stride,
                               const uint8_t* __restrict__ meta, int64_t meta_bytes, int64_t meta_off,
                               int64_t rec_stride, uint8_t* __restrict__ packed) {
    const int64_t pieces = rec_stride / 16;
    for (int64_t e = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < rows * pieces;
         e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = e / pieces, q = e - r * pieces;
        alignas(16) uint8_t buf[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) {
            const int64_t o = q * 16 + i;
            uint8_t v = 0;
            if (o < row_bytes) v = data[r * row_stride + o];
            else if (o >= meta_off && o < meta_off + meta_bytes) v = meta[r * meta_bytes + (o - meta_off)];
            buf[i] = v;
        }
        *reinterpret_cast<uint4*>(packed + r * rec_stride + q * 16) = *reinterpret_cast<const uint4*>(buf);
    }
}

cudaError_t launch_eb_pack(const uint8_t* data, int64_t rows, int64_t row_bytes, int64_t row_stride, const void* meta,
                           int64_t meta_bytes, int64_t meta_off, int64_t rec_stride, uint8_t* packed, cudaStream_t st) {
    if (rows <= 0) return cudaSuccess;
    int64_t blocks = (rows * (rec_stride / 16) + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    eb_pack_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(data, rows, row_bytes, row_stride,
                                                                  reinterpret_cast<const uint8_t*>(meta), meta_bytes,
                                                                  meta_off, rec_stride, packed);
    return cudaGetLastError();
}

// Sum of n per-launch counters into *dst (grouped tables run as one launch per table).
__global__ void sum_u32_kernel(const uint32_t* __restrict__ src, int64_t n, uint32_t* __restrict__ dst) {
    uint32_t s = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) s += src[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    __shared__ uint32_t part[8];
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t t = 0;
        for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) t += part[w];
        *dst = t;
    }
}

cudaError_t launch_sum_u32(const uint32_t* src, int64_t n, uint32_t* dst, cudaStream_t st) {
    sum_u32_kernel<<<1, 256, 0, st>>>(src, n, dst);
    return cudaGetLastError();
}

// Batched table faults (fault lab): flip bit bits[i] (< element width) of element (rows[i], cols[i]) in
// buffer a (row stride sa) and, when set, in buffer b (stride sb) -- 32-bit atomic XORs, so repeated
// coordinates compose exactly as sequential flips. Out-of-range entries set bit 1 of *status.
__global__ void flip_cells_kernel(uint8_t* a, int64_t sa, uint8_t* b, int64_t sb, const int64_t* __restrict__ rows,
                                  const int64_t* __restrict__ cols, const int32_t* __restrict__ bits, int64_t n,
                                  int64_t nrows, int64_t dim, int u4, int32_t* status) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int64_t r = rows[i], c = cols[i];
        const int32_t bt = bits[i];
        if (r < 0 || r >= nrows || c < 0 || c >= dim || bt < 0 || bt >= (u4 ? 4 : 8)) {
            if (status) atomicOr(status, 2);
            continue;
        }
        const int64_t cb = u4 ? c / 2 : c;
        const uint32_t bitpos = static_cast<uint32_t>(bt) + (u4 ? 4u * static_cast<uint32_t>(c & 1) : 0u);
        const uint64_t oa = static_cast<uint64_t>(r * sa + cb);
        atomicXor(reinterpret_cast<unsigned int*>(a + (oa & ~uint64_t{3})), (1u << bitpos) << (8 * (oa & 3)));
        if (b) {
            const uint64_t ob = static_cast<uint64_t>(r * sb + cb);
            atomicXor(reinterpret_cast<unsigned int*>(b + (ob & ~uint64_t{3})), (1u << bitpos) << (8 * (ob & 3)));
        }
    }
}

cudaError_t launch_flip_cells(uint8_t* a, int64_t sa, uint8_t* b, int64_t sb, const int64_t* rows, const int64_t* cols,
                              const int32_t* bits, int64_t n, int64_t nrows, int64_t dim, bool u4, int32_t* status,
                              cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    int64_t blocks = (n + 255) / 256;
    if (blocks > 1184) blocks = 1184;
    flip_cells_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(a, sa, b, sb, rows, cols, bits, n, nrows, dim,
                                                                     u4 ? 1 : 0, status);
    return cudaGetLastError();
}

}  // namespace abftk
