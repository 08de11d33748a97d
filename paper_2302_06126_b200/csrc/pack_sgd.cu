// pack_sgd.cu — the two element-wise kernels of the path (both HBM-bound).
//
// pack (step a1, north_star subsystem 1): cast this replica's sufficient factors X_r (B x M) and
// dY_r (B x N) to the wire dtype into its slot of the gather buffers. One launch covers both
// factors; 16-byte vector stores, 32-byte vector loads, grid = a multiple of the SM count with a
// grid-stride loop. fp32 -> bf16 uses round-to-nearest-even (DESIGN R11).
//
// sgd (unfused optimizer of the dense baseline, P:543-545 ApplyGradient; R14):
//   g = dW + wd*W ; v <- mu*v + g ; W <- W - lr*v
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include "optim.cuh"
#include "tag_internal.h"

namespace tag {
namespace {

__device__ __forceinline__ uint32_t bf16x2_rn(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}

// Segment: n elements; vectorised main body of n/8 groups (8 fp32 in -> 8 bf16 out = 16 B),
// scalar tail. Requires 32-byte aligned src and 16-byte aligned dst for the vector body (the
// host checks and otherwise takes the scalar kernel).
__device__ __forceinline__ void cast_segment(const float* __restrict__ src,
                                             __nv_bfloat16* __restrict__ dst, int64_t n,
                                             int64_t tid, int64_t nthreads) {
    const int64_t groups = n / 8;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    uint4* d4 = reinterpret_cast<uint4*>(dst);
    for (int64_t g = tid; g < groups; g += nthreads) {
        const float4 a = __ldcs(s4 + 2 * g);       // streamed: read once
        const float4 b = __ldcs(s4 + 2 * g + 1);
        uint4 o;
        o.x = bf16x2_rn(a.x, a.y);
        o.y = bf16x2_rn(a.z, a.w);
        o.z = bf16x2_rn(b.x, b.y);
        o.w = bf16x2_rn(b.z, b.w);
        d4[g] = o;                                 // stays in L2 for the all-gather / GEMM
    }
    for (int64_t i = groups * 8 + tid; i < n; i += nthreads) dst[i] = __float2bfloat16_rn(src[i]);
}

__global__ void __launch_bounds__(256)
pack_cast_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ xd, int64_t nx,
                 const float* __restrict__ dy, __nv_bfloat16* __restrict__ dyd, int64_t ny)
{
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    cast_segment(x, xd, nx, tid, nthreads);
    cast_segment(dy, dyd, ny, tid, nthreads);
}

__global__ void __launch_bounds__(256)
pack_cast_scalar_kernel(const float* __restrict__ x, __nv_bfloat16* __restrict__ xd, int64_t nx,
                        const float* __restrict__ dy, __nv_bfloat16* __restrict__ dyd, int64_t ny)
{
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = tid; i < nx; i += nthreads) xd[i] = __float2bfloat16_rn(x[i]);
    for (int64_t i = tid; i < ny; i += nthreads) dyd[i] = __float2bfloat16_rn(dy[i]);
}

// Same-dtype pack: a 16-byte vector copy of both segments (bytes).
__global__ void __launch_bounds__(256)
pack_copy_kernel(const uint8_t* __restrict__ x, uint8_t* __restrict__ xd, int64_t bx,
                 const uint8_t* __restrict__ dy, uint8_t* __restrict__ dyd, int64_t by)
{
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = tid; i < bx / 16; i += nthreads)
        reinterpret_cast<uint4*>(xd)[i] = reinterpret_cast<const uint4*>(x)[i];
    for (int64_t i = (bx / 16) * 16 + tid; i < bx; i += nthreads) xd[i] = x[i];
    for (int64_t i = tid; i < by / 16; i += nthreads)
        reinterpret_cast<uint4*>(dyd)[i] = reinterpret_cast<const uint4*>(dy)[i];
    for (int64_t i = (by / 16) * 16 + tid; i < by; i += nthreads) dyd[i] = dy[i];
}

__global__ void __launch_bounds__(256)
sgd_kernel(const float* __restrict__ dW, float* __restrict__ W, float* __restrict__ V,
           int64_t len, float lr, float mu, float wd)
{
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t n4 = len / 4;
    for (int64_t i = tid; i < n4; i += nthreads) {
        const float4 d = __ldcs(reinterpret_cast<const float4*>(dW) + i);
        float4 w = reinterpret_cast<float4*>(W)[i];
        float4 v = reinterpret_cast<float4*>(V)[i];
        float* df = const_cast<float*>(reinterpret_cast<const float*>(&d));
        float* wf = reinterpret_cast<float*>(&w);
        float* vf = reinterpret_cast<float*>(&v);
#pragma unroll
        for (int e = 0; e < 4; ++e) {
            const float g = __fadd_rn(df[e], __fmul_rn(wd, wf[e]));
            vf[e] = __fadd_rn(__fmul_rn(mu, vf[e]), g);
            wf[e] = __fsub_rn(wf[e], __fmul_rn(lr, vf[e]));
        }
        reinterpret_cast<float4*>(W)[i] = w;
        reinterpret_cast<float4*>(V)[i] = v;
    }
    for (int64_t i = n4 * 4 + tid; i < len; i += nthreads) {
        const float g = __fadd_rn(dW[i], __fmul_rn(wd, W[i]));
        const float vn = __fadd_rn(__fmul_rn(mu, V[i]), g);
        V[i] = vn;
        W[i] = __fsub_rn(W[i], __fmul_rn(lr, vn));
    }
}

int grid_for(int64_t work_items) {
    // a multiple of the SM count (up to 8 resident 256-thread CTAs per SM), no more than needed
    const int64_t per_wave = static_cast<int64_t>(num_sms()) * 8;
    int64_t blocks = (work_items + 255) / 256;
    if (blocks > per_wave) blocks = per_wave;
    if (blocks < 1) blocks = 1;
    return static_cast<int>(blocks);
}

}  // namespace

tag_status_t launch_pack(const void* x, void* x_dst, int64_t nx, const void* dy, void* dy_dst,
                         int64_t ny, tag_dtype_t in, tag_dtype_t wire, cudaStream_t s) {
    if (nx + ny == 0) return TAG_OK;
    if (in == wire) {
        const int64_t es = static_cast<int64_t>(dtype_size(in));
        pack_copy_kernel<<<grid_for((nx + ny) * es / 16 + 1), 256, 0, s>>>(
            static_cast<const uint8_t*>(x), static_cast<uint8_t*>(x_dst), nx * es,
            static_cast<const uint8_t*>(dy), static_cast<uint8_t*>(dy_dst), ny * es);
    } else if (in == TAG_F32 && wire == TAG_BF16) {
        const bool vec = (reinterpret_cast<uintptr_t>(x) % 32 == 0) &&
                         (reinterpret_cast<uintptr_t>(dy) % 32 == 0) &&
                         (reinterpret_cast<uintptr_t>(x_dst) % 16 == 0) &&
                         (reinterpret_cast<uintptr_t>(dy_dst) % 16 == 0);
        if (vec)
            pack_cast_kernel<<<grid_for((nx + ny) / 8 + 1), 256, 0, s>>>(
                static_cast<const float*>(x), static_cast<__nv_bfloat16*>(x_dst), nx,
                static_cast<const float*>(dy), static_cast<__nv_bfloat16*>(dy_dst), ny);
        else
            pack_cast_scalar_kernel<<<grid_for(nx + ny), 256, 0, s>>>(
                static_cast<const float*>(x), static_cast<__nv_bfloat16*>(x_dst), nx,
                static_cast<const float*>(dy), static_cast<__nv_bfloat16*>(dy_dst), ny);
    } else {
        return fail(TAG_ERR_UNSUPPORTED, "pack: unsupported in/wire dtype pair");
    }
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "launch pack kernel");
    count_launch();
    return TAG_OK;
}

namespace {
// 3xTF32 split (recon_tc.cu X3): one element per thread-iteration, grid-stride; non-finite
// values keep hi = value (truncated) and lo = 0 (no inf - inf).
__global__ void __launch_bounds__(256)
tf32_split_kernel(const float* __restrict__ src0, const float* __restrict__ src1,
                  const uint32_t* ctr, float* __restrict__ dst, int64_t K, int64_t cols,
                  int64_t kpad) {
    // a window source: the buffer of the latest gather (device state, see tag_internal.h)
    const float* src = ((load_calls(ctr) - 1u) & 1u) ? src1 : src0;
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    const int64_t total = kpad * cols;
    float* hi = dst;
    float* lo = dst + total;
    for (int64_t i = tid; i < total; i += nthreads) {
        const int64_t row = i / cols;
        float h = 0.f, l = 0.f;
        if (row < K) {
            const float v = src[i];
            // hi = v rounded to the nearest tf32 (10 mantissa bits, ties to even): |lo| <= 2^-11 |v|,
            // so the dropped lo*lo term is <= 2^-22 relative and the lo errors are unbiased
            const uint32_t u = __float_as_uint(v);
            const uint32_t r = (u + 0xfffu + ((u >> 13) & 1u)) & 0xffffe000u;
            h = __uint_as_float(r);
            if (!isfinite(v) || !isfinite(h)) h = __uint_as_float(u & 0xffffe000u);   // no overflow to inf
            l = isfinite(v) ? __fsub_rn(v, h) : 0.f;
            // lo rounded to tf32 too: the tensor core truncates its fp32 inputs, which would
            // bias every lo term toward zero (measured 1.1e-6 -> see tests)
            const uint32_t ul = __float_as_uint(l);
            l = __uint_as_float((ul + 0xfffu + ((ul >> 13) & 1u)) & 0xffffe000u);
        }
        hi[i] = h;
        lo[i] = l;
    }
}
}  // namespace

tag_status_t launch_tf32_split(const float* src, const float* src1, const uint32_t* ctr, float* dst,
                               int64_t K, int64_t cols, int64_t kpad, cudaStream_t s) {
    if (kpad * cols == 0) return TAG_OK;
    tf32_split_kernel<<<grid_for(kpad * cols), 256, 0, s>>>(src, src1, ctr, dst, K, cols, kpad);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "launch tf32_split_kernel");
    count_launch();
    return TAG_OK;
}

namespace {
__global__ void __launch_bounds__(256)
adam_kernel(const float* __restrict__ dW, float* __restrict__ W, float* __restrict__ Mm,
            float* __restrict__ V, int64_t len, AdamConsts c) {
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = tid; i < len; i += nthreads) {
        float w = W[i], m = Mm[i], v = V[i];
        adam_update(dW[i], w, m, v, c);
        W[i] = w;
        Mm[i] = m;
        V[i] = v;
    }
}
}  // namespace

tag_status_t launch_adam(const float* dW, float* W, float* Mm, float* V, int64_t len, float b1,
                         float omb1, float b2, float omb2, float eps, float lr_t, float isbc2,
                         float wd, cudaStream_t s) {
    if (len == 0) return TAG_OK;
    const AdamConsts c{b1, omb1, b2, omb2, eps, lr_t, isbc2, wd};
    adam_kernel<<<grid_for(len), 256, 0, s>>>(dW, W, Mm, V, len, c);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "launch adam_kernel");
    count_launch();
    return TAG_OK;
}

tag_status_t launch_sgd(const float* dW, float* W, float* V, int64_t len, float lr, float mu,
                        float wd, cudaStream_t s) {
    if (len == 0) return TAG_OK;
    sgd_kernel<<<grid_for(len / 4 + 1), 256, 0, s>>>(dW, W, V, len, lr, mu, wd);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "launch sgd_kernel");
    count_launch();
    return TAG_OK;
}

}  // namespace tag
