// Device side of the fault lab: counter-based SplitMix64 generators that reproduce the
// reference's host draw streams element for element (P:src/rng.hpp:10-43; stream roles
// P:src/fault_lab.cpp:16-21), single-element bit flips / random-value rewrites
// (P:src/fault_lab.cpp:89-166), and an L2 flush used by the benchmark.
#include <cuda_runtime.h>

#include <cstdint>

#include "abft_internal.h"

namespace abftk {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;

__host__ __device__ __forceinline__ uint64_t sm_mix(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
// State after construction; draw e (0-based) of the stream is mix(state0 + (e+1)*gamma).
__host__ __device__ __forceinline__ uint64_t sm_state0(uint64_t seed, uint64_t stream) {
    return sm_mix(seed ^ sm_mix(stream + kGamma));
}
__device__ __forceinline__ uint64_t sm_draw(uint64_t s0, uint64_t e) { return sm_mix(s0 + (e + 1) * kGamma); }

// kind: 0 = u8 next_below(256), 1 = s8 next_int(-128,127), 2 = f32 next_real(lo,hi),
//       3 = i64 next_below(bound)
__global__ void gen_kernel(void* out, int64_t count, uint64_t s0, uint64_t off, int kind, double lo, double hi,
                           uint64_t bound) {
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const uint64_t x = sm_draw(s0, off + static_cast<uint64_t>(i));
        switch (kind) {
            case 0: reinterpret_cast<uint8_t*>(out)[i] = static_cast<uint8_t>(x % 256u); break;
            case 1: reinterpret_cast<int8_t*>(out)[i] = static_cast<int8_t>(-128 + static_cast<int64_t>(x % 256u)); break;
            case 2: {
                const double u = static_cast<double>(x >> 11) * 0x1.0p-53;
                reinterpret_cast<float*>(out)[i] = __double2float_rn(__dadd_rn(lo, __dmul_rn(__dsub_rn(hi, lo), u)));
                break;
            }
            default: reinterpret_cast<int64_t*>(out)[i] = static_cast<int64_t>(x % bound); break;
        }
    }
}

__global__ void flip_bit_kernel(uint8_t* base, uint64_t byte_offset, uint32_t bit) {
    base[byte_offset + (bit >> 3)] ^= static_cast<uint8_t>(1u << (bit & 7));
}

// random_value model: redraw from the continuing inject stream until the value changes
// (P:src/fault_lab.cpp:109-114, 128-133). width: 8 (int8) or 32 (int32).
__global__ void set_random_kernel(void* cell, int width, uint64_t state) {
    if (width == 8) {
        int8_t* p = reinterpret_cast<int8_t*>(cell);
        int8_t nv;
        do {
            state += kGamma;
            nv = static_cast<int8_t>(-128 + static_cast<int64_t>(sm_mix(state) % 256u));
        } while (nv == *p);
        *p = nv;
    } else {
        int32_t* p = reinterpret_cast<int32_t*>(cell);
        int32_t nv;
        do {
            state += kGamma;
            nv = static_cast<int32_t>(sm_mix(state));
        } while (nv == *p);
        *p = nv;
    }
}

// Sets out[slot] = (value != 0) ? 1 : 0 -- collects a per-trial detection bit from a count.
__global__ void nonzero_kernel(const uint32_t* value, uint8_t* out, int64_t slot) { out[slot] = *value != 0u; }

// Any flagged bag in [0, n) -> out[slot].
__global__ void any_flag_kernel(const uint8_t* flags, int64_t n, uint8_t* out, int64_t slot) {
    __shared__ int any;
    if (threadIdx.x == 0) any = 0;
    __syncthreads();
    int mine = 0;
    for (int64_t i = threadIdx.x; i < n; i += blockDim.x) mine |= flags[i];
    if (mine) any = 1;
    __syncthreads();
    if (threadIdx.x == 0) out[slot] = static_cast<uint8_t>(any);
}

// L2 flush by READING a buffer larger than L2: it evicts the previous working set without leaving
// dirty lines whose write-back would otherwise land inside the next (timed) kernel.
__global__ void flush_kernel(int4* buf, int64_t n16, int salt) {
    int acc = 0;
    for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n16;
         i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
        const int4 v = __ldcg(buf + i);
        acc ^= v.x ^ v.y ^ v.z ^ v.w;
    }
    if (acc == salt + 0x5F3759DF) buf[0] = make_int4(acc, 0, 0, 0);  // practically never; keeps the loads live
}

cudaError_t launch_gen(void* out, int64_t count, uint64_t seed, uint64_t stream, uint64_t off, int kind, double lo,
                       double hi, uint64_t bound, cudaStream_t st) {
    if (count <= 0) return cudaSuccess;
    int64_t blocks = (count + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    gen_kernel<<<static_cast<unsigned>(blocks), 256, 0, st>>>(out, count, sm_state0(seed, stream), off, kind, lo, hi,
                                                             bound);
    return cudaGetLastError();
}

cudaError_t launch_flip_bit(void* base, uint64_t byte_offset, uint32_t bit, cudaStream_t st) {
    flip_bit_kernel<<<1, 1, 0, st>>>(reinterpret_cast<uint8_t*>(base), byte_offset, bit);
    return cudaGetLastError();
}

cudaError_t launch_set_random(void* cell, int width, uint64_t state, cudaStream_t st) {
    set_random_kernel<<<1, 1, 0, st>>>(cell, width, state);
    return cudaGetLastError();
}

cudaError_t launch_nonzero(const uint32_t* value, uint8_t* out, int64_t slot, cudaStream_t st) {
    nonzero_kernel<<<1, 1, 0, st>>>(value, out, slot);
    return cudaGetLastError();
}

cudaError_t launch_any_flag(const uint8_t* flags, int64_t n, uint8_t* out, int64_t slot, cudaStream_t st) {
    any_flag_kernel<<<1, 256, 0, st>>>(flags, n, out, slot);
    return cudaGetLastError();
}

// Random-record gather floor (benchmark roof for the EmbeddingBag lines): record idx[i] (rec16 16-byte pieces,
// one lane each) for every i, eight records per lane group in flight, no arithmetic beyond keeping the loads live.
template <int U>
__global__ void __launch_bounds__(256) gather_probe_kernel(const uint4* __restrict__ tab, const int64_t* __restrict__ idx,
                                                           int64_t n, int rec16, uint32_t* sink) {
    const int64_t lanes_total = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t groups = lanes_total / rec16;
    const int64_t g0 = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) / rec16;
    const int part = threadIdx.x % rec16;
    if (g0 >= groups) return;
    uint32_t acc = 0;
    for (int64_t base = g0; base < n; base += groups * U) {
        int64_t r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int64_t e = base + u * groups;
            r[u] = e < n ? idx[e] : -1;
        }
        uint4 v[U];
#pragma unroll
        for (int u = 0; u < U; ++u) v[u] = r[u] >= 0 ? __ldg(tab + r[u] * rec16 + part) : make_uint4(0u, 0u, 0u, 0u);
#pragma unroll
        for (int u = 0; u < U; ++u) acc ^= v[u].x ^ v[u].w;
    }
    if (acc == 0x9E3779B9u) *sink = acc;  // practically never; keeps the loads live
}

cudaError_t launch_gather_probe(const void* table, int64_t rec_bytes, const int64_t* idx, int64_t n, uint32_t* sink,
                                cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    gather_probe_kernel<8><<<148 * 8, 256, 0, st>>>(reinterpret_cast<const uint4*>(table), idx, n,
                                                    static_cast<int>(rec_bytes / 16), sink);
    return cudaGetLastError();
}

cudaError_t launch_flush(void* buf, int64_t bytes, int salt, cudaStream_t st) {
    flush_kernel<<<148 * 8, 256, 0, st>>>(reinterpret_cast<int4*>(buf), bytes / 16, salt);
    return cudaGetLastError();
}

}  // namespace abftk
