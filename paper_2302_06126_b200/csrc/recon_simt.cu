// recon_simt.cu — CUDA-core (FFMA) form of step a3+a4 for shapes the TMA/tensor-core path does
// not take: fp32 wire factors (the toy config, where single-pass TF32 misses the 1e-5 gate,
// DESIGN R10) and rows that are not 16-byte multiples (odd M or N). Same math as recon_tc.cu:
//   dW[m][j] = alpha * sum_{k<K} A[k][m] * Bm[k][j]     (alpha = 1/(nB), R1)
// accumulated in fp32 in k order (rank-major, then row: R12), then one fp32 multiply by alpha.
// Optional fused SGD-momentum epilogue (R14).
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "tag_internal.h"

namespace tag {
namespace {

constexpr int TM = 64, TN = 64, TK = 16;

template <typename T>
__device__ __forceinline__ float to_f(T v);
template <>
__device__ __forceinline__ float to_f<float>(float v) { return v; }
template <>
__device__ __forceinline__ float to_f<__nv_bfloat16>(__nv_bfloat16 v) { return __bfloat162float(v); }

template <typename T, bool OUT_BF16, bool SGD>
__global__ void __launch_bounds__(256)
recon_simt_kernel(const T* __restrict__ A0, const T* __restrict__ B0, const T* __restrict__ A1,
                  const T* __restrict__ B1, const uint32_t* ctr, void* __restrict__ C,
                  int M, int N, int K, int64_t lda, float alpha, float* __restrict__ W,
                  float* __restrict__ V, float lr, float mu, float wd)
{
    // window operands: the buffer of the latest gather (device state, see tag_internal.h)
    const bool one = (load_calls(ctr) - 1u) & 1u;
    const T* __restrict__ A = one ? A1 : A0;
    const T* __restrict__ Bm = one ? B1 : B0;
    __shared__ float As[TK][TM];
    __shared__ float Bs[TK][TN];
    const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
    const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
    float acc[4][4] = {};
    for (int k0 = 0; k0 < K; k0 += TK) {
        for (int i = threadIdx.x; i < TK * TM; i += 256) {
            const int kk = i / TM, mm = i % TM;
            const int k = k0 + kk, m = m0 + mm;
            As[kk][mm] = (k < K && m < M) ? to_f(A[static_cast<int64_t>(k) * lda + m]) : 0.f;
        }
        for (int i = threadIdx.x; i < TK * TN; i += 256) {
            const int kk = i / TN, nn = i % TN;
            const int k = k0 + kk, n = n0 + nn;
            Bs[kk][nn] = (k < K && n < N) ? to_f(Bm[static_cast<int64_t>(k) * N + n]) : 0.f;
        }
        __syncthreads();
        const int kmax = min(TK, K - k0);
        for (int kk = 0; kk < kmax; ++kk) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float a = As[kk][ty + 16 * i];
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = __fmaf_rn(a, Bs[kk][tx + 16 * j], acc[i][j]);
            }
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int m = m0 + ty + 16 * i;
        if (m >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int n = n0 + tx + 16 * j;
            if (n >= N) continue;
            const int64_t o = static_cast<int64_t>(m) * N + n;
            const float d = __fmul_rn(acc[i][j], alpha);
            if constexpr (SGD) {
                const float g = __fadd_rn(d, __fmul_rn(wd, W[o]));
                const float vn = __fadd_rn(__fmul_rn(mu, V[o]), g);
                V[o] = vn;
                W[o] = __fsub_rn(W[o], __fmul_rn(lr, vn));
            }
            if (C) {
                if constexpr (OUT_BF16) static_cast<__nv_bfloat16*>(C)[o] = __float2bfloat16_rn(d);
                else static_cast<float*>(C)[o] = d;
            }
        }
    }
}

template <typename T, bool OUT_BF16, bool SGD>
tag_status_t launch_t(const ReconArgs& a, cudaStream_t s) {
    dim3 grid(static_cast<unsigned>((a.N + TN - 1) / TN), static_cast<unsigned>((a.M + TM - 1) / TM));
    if (grid.y > 65535) return fail(TAG_ERR_UNSUPPORTED, "recon_simt: M too large");
    recon_simt_kernel<T, OUT_BF16, SGD><<<grid, 256, 0, s>>>(
        static_cast<const T*>(a.A), static_cast<const T*>(a.Bm), static_cast<const T*>(a.A1),
        static_cast<const T*>(a.Bm1), a.ctr_mode == 1 ? a.ctr : nullptr, a.C, static_cast<int>(a.M),
        static_cast<int>(a.N), static_cast<int>(a.K), a.lda ? a.lda : a.M, a.alpha, a.W, a.V, a.lr,
        a.mu, a.wd);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "launch recon_simt_kernel");
    count_launch();
    return TAG_OK;
}

template <typename T>
tag_status_t dispatch_out(const ReconArgs& a, cudaStream_t s) {
    if (a.sgd) return a.out == TAG_BF16 ? launch_t<T, true, true>(a, s) : launch_t<T, false, true>(a, s);
    return a.out == TAG_BF16 ? launch_t<T, true, false>(a, s) : launch_t<T, false, false>(a, s);
}

}  // namespace

tag_status_t launch_recon_simt(const ReconArgs& a, cudaStream_t s) {
    if (a.M > INT32_MAX || a.N > INT32_MAX || a.K > INT32_MAX)
        return fail(TAG_ERR_UNSUPPORTED, "recon_simt: dimension exceeds int32");
    if (a.M == 0 || a.N == 0) return TAG_OK;
    return a.wire == TAG_BF16 ? dispatch_out<__nv_bfloat16>(a, s) : dispatch_out<float>(a, s);
}

}  // namespace tag
