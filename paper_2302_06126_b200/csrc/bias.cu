// bias.cu — bias gradient of a replicated Dense layer from the gathered factors (DESIGN R17).
//
// y = x W + b: the bias is the weight of a constant input 1, so its gradient is the outer product
// of the ones vector with dY, i.e. the column sums of dY. SFB already broadcasts dY
// (P:520-526), so every replica gets the identical global-batch bias gradient
//     db[j] = alpha * sum_{k < K} dY_all[k][j],   alpha = 1/(nB)
// with no communication at all. HBM-bound and tiny (K x N reads, N writes).
//
// CTA = 256 threads = 32 column slots (8 columns each: 256 columns) x 8 row phases. Phase t sums
// rows t, t+8, t+16, ... of its 8 columns in fp32, then the 8 phase partials are added in phase
// order through shared memory — a fixed summation order, so the result is bit-identical on
// every replica (no atomics). One launch covers a whole bucket of layers (blockIdx.y = layer).
#include <algorithm>

#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "tag_internal.h"

namespace tag {
namespace {

constexpr int COLS = 256;   // columns per CTA
constexpr int PHASES = 8;   // row phases per CTA

struct BiasGroup {
    BiasArgs a[MAX_GROUP];
};

template <typename T>
__device__ __forceinline__ float ld_f(const T* p) {
    if constexpr (sizeof(T) == 2) return __bfloat162float(*reinterpret_cast<const __nv_bfloat16*>(p));
    else return *reinterpret_cast<const float*>(p);
}

template <typename T>
__device__ __forceinline__ void accumulate(const BiasArgs& a, int64_t col0, int phase, float (&acc)[8]) {
    // a window source: the buffer of the latest gather (device state, see tag_internal.h)
    const T* dy = static_cast<const T*>(((load_calls(a.ctr) - 1u) & 1u) ? a.dy1 : a.dy);
    const bool vec = sizeof(T) == 2 && a.N % 8 == 0 && col0 + 8 <= a.N;
    for (int64_t k = phase; k < a.K; k += PHASES) {
        const T* row = dy + k * a.N + col0;
        if (vec) {   // 8 bf16 = one 16-byte load (rows are 16-byte aligned when N % 8 == 0)
            const uint4 v = __ldg(reinterpret_cast<const uint4*>(row));
            const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&v);
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                const float2 f = __bfloat1622float2(h[e]);
                acc[2 * e] = __fadd_rn(acc[2 * e], f.x);
                acc[2 * e + 1] = __fadd_rn(acc[2 * e + 1], f.y);
            }
        } else {
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (col0 + e < a.N) acc[e] = __fadd_rn(acc[e], ld_f(row + e));
        }
    }
}

__global__ void __launch_bounds__(COLS)
bias_grad_kernel(const __grid_constant__ BiasGroup g) {
    const BiasArgs& a = g.a[blockIdx.y];
    const int64_t blk0 = static_cast<int64_t>(blockIdx.x) * COLS;
    if (blk0 >= a.N) return;                                   // uniform for the whole CTA
    __shared__ float part[PHASES][COLS];
    const int slot = threadIdx.x & 31, phase = threadIdx.x >> 5;
    const int64_t col0 = blk0 + slot * 8;
    float acc[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
    if (col0 < a.N) {
        if (a.wire == TAG_BF16) accumulate<__nv_bfloat16>(a, col0, phase, acc);
        else accumulate<float>(a, col0, phase, acc);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) part[phase][slot * 8 + e] = acc[e];
    __syncthreads();
    const int c = threadIdx.x;                                 // one output column per thread
    const int64_t col = blk0 + c;
    if (col >= a.N) return;
    float s = part[0][c];
#pragma unroll
    for (int t = 1; t < PHASES; ++t) s = __fadd_rn(s, part[t][c]);
    const float v = __fmul_rn(s, a.alpha);                     // one rounding, as for dW
    if (a.out == TAG_BF16) static_cast<__nv_bfloat16*>(a.db)[col] = __float2bfloat16_rn(v);
    else static_cast<float*>(a.db)[col] = v;
}

}  // namespace

tag_status_t launch_bias_grad(const BiasArgs* a, int count, cudaStream_t s) {
    if (count < 1 || count > MAX_GROUP) return fail(TAG_ERR_INVALID_ARG, "bias group size");
    BiasGroup g;
    int64_t blocks = 1;
    for (int i = 0; i < count; ++i) {
        g.a[i] = a[i];
        blocks = std::max<int64_t>(blocks, (a[i].N + COLS - 1) / COLS);
    }
    if (blocks > 65535 * 64) return fail(TAG_ERR_UNSUPPORTED, "bias: N too large");
    bias_grad_kernel<<<dim3(static_cast<unsigned>(blocks), static_cast<unsigned>(count)), COLS, 0, s>>>(g);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "launch bias_grad_kernel");
    count_launch();
    return TAG_OK;
}

}  // namespace tag
