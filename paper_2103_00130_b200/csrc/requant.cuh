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

}  // namespace abftk
