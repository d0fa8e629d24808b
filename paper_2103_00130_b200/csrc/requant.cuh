// Requantization of the int32 product to u8 (P:src/quant.cpp:10-14, 77-102), shared by the fused GEMM
// epilogue and the standalone kernel. Same double operations in the same order as the reference
// (built with -ffp-contract=off): cf = sA*sB*c + sA*bB*rowSumA + sB*bA*colSumB + k*bA*bB, then
// clamp(round_half_away((cf - bC) / sC), 0, 255) -- explicit __d*_rn intrinsics, so no contraction.
#pragma once
#include <cstdint>

#include "abft_internal.h"

namespace abftk {

struct RequantConsts {
    double m1, m2, m3, t4, bC, sC;  // sA*sB, sA*bB, sB*bA, k*bA*bB, biasC, scaleC
};

__device__ __forceinline__ RequantConsts requant_consts(const RequantDev& q) {
    RequantConsts r;
    r.m1 = __dmul_rn(q.sA, q.sB);
    r.m2 = __dmul_rn(q.sA, q.bB);
    r.m3 = __dmul_rn(q.sB, q.bA);
    r.t4 = __dmul_rn(__dmul_rn(q.k, q.bA), q.bB);
    r.bC = q.bC;
    r.sC = q.sC;
    return r;
}

__device__ __forceinline__ uint32_t requant_one(int32_t c, int32_t rs, int32_t cs, const RequantConsts& k) {
    const double cf = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(k.m1, static_cast<double>(c)),
                                                    __dmul_rn(k.m2, static_cast<double>(rs))),
                                          __dmul_rn(k.m3, static_cast<double>(cs))),
                                k.t4);
    const double x = __ddiv_rn(__dsub_rn(cf, k.bC), k.sC);
    double r = x >= 0.0 ? floor(__dadd_rn(x, 0.5)) : ceil(__dsub_rn(x, 0.5));
    r = r < 0.0 ? 0.0 : (r > 255.0 ? 255.0 : r);
    return static_cast<uint32_t>(r);
}

// Fast path of the fused epilogue. The reference's value x (seven rounded double operations, one a division) decides
// the output only through clamp(round_half_away(x), 0, 255), so any q with |q - x| < e gives the same byte unless q
// lies within e of a rounding boundary (j + 0.5). q is formed in fp32 with two FMAs from per-launch / per-row
// constants (the division by scaleC folded into them); e = 2^-21 * (|c a1| + |cs a3| + |rowt|) + 2^-14 bounds its
// distance from x: the fp32 side rounds c, cs, the three constants and two FMAs (each <= 2^-24 of a magnitude inside
// that sum, < 2^-21 together), forming t = q + 1/2 below 258 adds < 2^-15, and the double-precision differences
// between the folded constants and the reference's own order are < 2^-40 of the same sum (the constants are accepted
// only while that is so). An element within e of a boundary takes the reference-order sequence, and so does every
// element when the parameters are not finite or too large for fp32: the bytes are the reference's in every case.
struct RequantFast {
    float a1, a3, rowt;
    bool ok;
};

__device__ __forceinline__ RequantFast requant_fast(const RequantConsts& k, int32_t rs) {
    RequantFast f;
    const double inv = __ddiv_rn(1.0, k.sC);
    const double a1 = k.m1 * inv, a3 = k.m3 * inv;
    const double rowt = ((k.m2 * static_cast<double>(rs) + k.t4) - k.bC) * inv;
    f.a1 = static_cast<float>(a1);
    f.a3 = static_cast<float>(a3);
    f.rowt = static_cast<float>(rowt);
    // every magnitude the reference adds, over scaleC, must sit inside the fast sum's own magnitude up to 2^19 (then
    // cancellation among the row term's parts costs < 2^-53 * 2^19 * 8 < 2^-30 of it), and fp32 must hold the constants
    const double parts = (fabs(k.m2 * static_cast<double>(rs)) + fabs(k.t4) + fabs(k.bC)) * fabs(inv);
    f.ok = parts <= fabs(rowt) * 524288.0 + 1.0 && fabs(a1) < 1e28 && fabs(a3) < 1e28 && fabs(rowt) < 1e28 &&
           (fabs(a1) > 1e-30 || a1 == 0.0) && (fabs(a3) > 1e-30 || a3 == 0.0);
    return f;
}

// (one out-of-line copy: inlined at each of the epilogue's 32 unrolled columns the division sequence made the
// epilogue's code larger than the instruction cache)
static __device__ __noinline__ uint32_t requant_one_cold(int32_t c, int32_t rs, int32_t cs, double m1, double m2, double m3,
                                                  double t4, double bC, double sC) {
    RequantConsts k;
    k.m1 = m1;
    k.m2 = m2;
    k.m3 = m3;
    k.t4 = t4;
    k.bC = bC;
    k.sC = sC;
    return requant_one(c, rs, cs, k);
}

// Branch-free: the byte of the fast path and whether the element needs the reference-order sequence instead (the
// caller collects those in a mask and handles them after the straight-line pass over its columns -- a call inside
// the unrolled column loop kept the compiler from interleaving the columns' independent chains: 4x slower).
__device__ __forceinline__ uint32_t requant_try_fast(int32_t c, int32_t cs, const RequantFast& f, bool& exact) {
#ifdef ABFT_RQ_TRIVIAL  // (diagnostic build: the epilogue without the requantization arithmetic)
    exact = false;
    return static_cast<uint32_t>(c + cs) & 255u;
#endif
    const float cf = static_cast<float>(c), csf = static_cast<float>(cs);
    const float q = fmaf(csf, f.a3, fmaf(cf, f.a1, f.rowt));
    const float mag = fmaf(fabsf(csf), fabsf(f.a3), fmaf(fabsf(cf), fabsf(f.a1), fabsf(f.rowt)));
    const float e = fmaf(mag, 0x1p-21f, 0x1p-14f);
    const float t = fminf(fmaxf(q, 0.0f), 257.0f) + 0.5f;  // (beyond the clamp the byte is 0 / 255 whatever the distance)
    const float u = __fadd_rd(t, 8388608.0f);             // 2^23 + floor(t): the integer sits in the low mantissa bits
    const float dist = t - (u - 8388608.0f);              // t - floor(t) in [0, 1)
    exact = !(f.ok && dist > e && dist < 1.0f - e);
    return min(__float_as_uint(u) & 0x3FFu, 255u);
}

}  // namespace abftk
