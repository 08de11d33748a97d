// optim.cuh — the element-wise optimizer updates shared by the fused reconstruction epilogue
// (recon_tc.cu) and the unfused kernels (pack_sgd.cu), so both round identically (one RN rounding
// per operation, no FMA contraction): fused == unfused bit for bit.
#pragma once
#include <cuda_runtime.h>

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
    const float den = __fadd_rn(__fmul_rn(__fsqrt_rn(v), c.isbc2), c.eps);
    w = __fsub_rn(w, __fdiv_rn(__fmul_rn(c.lr_t, m), den));
}

}  // namespace tag
