// optim.cuh — the element-wise optimizer updates shared by the fused reconstruction epilogue
// (recon_tc.cu) and the unfused kernels (pack_sgd.cu), so both round identically (one RN rounding
// per basic operation, no FMA contraction, the same SFU sqrt / reciprocal): fused == unfused bit
// for bit.
#pragma once
#include <cuda_runtime.h>

// EXP_ADAM_MATH (diagnostics builds only): 1 = IEEE round-to-nearest sqrt and division (the
// round-1 product), 2 = neither (a bound: what the Adam epilogue costs without them).
#ifndef EXP_ADAM_MATH
#define EXP_ADAM_MATH 0
#endif

namespace tag {

// Adam (DESIGN R22, torch.optim.Adam semantics): per-call constants from the host —
// omb = fl32(1 - beta), lr_t = fl32(lr / (1 - b1^t)), isbc2 = fl32(1 / sqrt(1 - b2^t)).
struct AdamConsts {
    float b1, omb1, b2, omb2, eps, lr_t, isbc2, wd;
};

__device__ __forceinline__ void adam_update(float dw, float& w, float& m, float& v,
                                            const AdamConsts& c) {
    const float g = __fadd_rn(dw, __fmul_rn(c.wd, w));
    m = __fadd_rn(__fmul_rn(c.b1, m), __fmul_rn(c.omb1, g));
    v = __fadd_rn(__fmul_rn(c.b2, v), __fmul_rn(c.omb2, __fmul_rn(g, g)));
#if EXP_ADAM_MATH == 2
    w = __fsub_rn(w, __fmul_rn(__fmul_rn(c.lr_t, m), __fadd_rn(__fmul_rn(v, c.isbc2), c.eps)));
#elif EXP_ADAM_MATH == 1
    const float den = __fadd_rn(__fmul_rn(__fsqrt_rn(v), c.isbc2), c.eps);
    w = __fsub_rn(w, __fdiv_rn(__fmul_rn(c.lr_t, m), den));
#else
    // the square root and the reciprocal on the SFU (sqrt.approx / rcp.approx, ~1 ulp): the
    // correctly rounded __fsqrt_rn / __fdiv_rn carry slow-path branches whose registers and
    // instructions cost the fused epilogue ~20 % (R22); den >= eps > 0, v >= 0
    float sv, rd;
    asm("sqrt.approx.f32 %0, %1;" : "=f"(sv) : "f"(v));
    const float den = __fadd_rn(__fmul_rn(sv, c.isbc2), c.eps);
    asm("rcp.approx.f32 %0, %1;" : "=f"(rd) : "f"(den));
    w = __fsub_rn(w, __fmul_rn(__fmul_rn(c.lr_t, m), rd));
#endif
}

}  // namespace tag
