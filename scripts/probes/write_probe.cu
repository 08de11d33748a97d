// write_probe.cu — HBM write-pattern ceilings on B200 for the reconstruction epilogue's stores.
// Variants write the fc6 dW size (25088 x 4096 fp32 = 411 MB):
//   contig     : grid-stride 16-B stores, consecutive lanes consecutive addresses
//   tile_rows4 : 128x128 fp32 tiles, one warp instruction = 4 rows x 128 B (the epilogue's pattern)
//   tile_rows4_cs : same with st.global.cs (streaming)
//   tile_rows1 : 128x128 tiles, one warp instruction = 1 row x 512 B
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o write_probe write_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void spin(long long cycles) {
    long long t0 = clock64();
    while (clock64() - t0 < cycles) {}
}

__global__ void contig_const(uint4* p, size_t n16) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(0x3fc00000u, 0x3fc00000u, 0x3fc00000u, 0x3fc00000u);   // 1.5f
}

__global__ void contig_rand(uint4* p, size_t n16) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x) {
        uint32_t h = (uint32_t)i * 2654435761u;
        p[i] = make_uint4(h, h ^ 0x9e3779b9u, h * 7u + 1u, h >> 3);
    }
}

__global__ void onestore(uint4* p, size_t n16) {      // torch-like: one 16-B store per thread
    size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
    if (i < n16) p[i] = make_uint4(1, 2, 3, (unsigned)i);
}

__global__ void unroll4(uint4* p, size_t n16) {       // 4 independent stores per thread, block-strided
    size_t base = (size_t)blockIdx.x * blockDim.x * 4 + threadIdx.x;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
        size_t i = base + (size_t)u * blockDim.x;
        if (i < n16) p[i] = make_uint4(1, 2, 3, (unsigned)i);
    }
}

template <int U>
__global__ void persist_unroll(uint4* p, size_t n16) {  // persistent CTAs, U stores in flight
    const size_t chunk = (size_t)blockDim.x * U;        // one CTA-iteration = contiguous chunk
    for (size_t c = blockIdx.x; c * chunk < n16; c += gridDim.x) {
        const size_t base = c * chunk + threadIdx.x;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = base + (size_t)u * blockDim.x;
            if (i < n16) p[i] = make_uint4(1, 2, 3, (unsigned)i);
        }
    }
}

__global__ void tiles_oneshot(float* C, int M, int N) {   // one 128x128 tile per CTA, rows4 pattern
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntn = N / 128;
    const int m0 = (blockIdx.x / ntn) * 128, n0 = (blockIdx.x % ntn) * 128;
    for (int rb = warp * 4; rb < 128; rb += 8 * 4)
        for (int cb = 0; cb < 128; cb += 32) {
            const int r = rb + (lane >> 3), c = cb + (lane & 7) * 4;
            *reinterpret_cast<float4*>(C + (size_t)(m0 + r) * N + n0 + c) = make_float4(1.f, 2.f, 3.f, 4.f);
        }
}

template <int U>
__global__ void persist_dynamic(uint4* p, size_t n16, unsigned* counter) {  // atomic tile queue
    const size_t chunk = (size_t)blockDim.x * U;
    __shared__ unsigned s_c;
    while (true) {
        if (threadIdx.x == 0) s_c = atomicAdd(counter, 1u);
        __syncthreads();
        const size_t c = s_c;
        __syncthreads();
        if (c * chunk >= n16) break;
        const size_t base = c * chunk + threadIdx.x;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const size_t i = base + (size_t)u * blockDim.x;
            if (i < n16) p[i] = make_uint4(1, 2, 3, (unsigned)i);
        }
    }
}

__global__ void tiles_dynamic(float* C, int M, int N, unsigned* counter) {   // 128x128 tiles, queue
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int ntn = N / 128, ntiles = (M / 128) * ntn;
    __shared__ int s_t;
    while (true) {
        if (threadIdx.x == 0) s_t = (int)atomicAdd(counter, 1u);
        __syncthreads();
        const int t = s_t;
        __syncthreads();
        if (t >= ntiles) break;
        const int m0 = (t / ntn) * 128, n0 = (t % ntn) * 128;
        for (int rb = warp * 4; rb < 128; rb += 8 * 4)
            for (int cb = 0; cb < 128; cb += 32) {
                const int r = rb + (lane >> 3), c = cb + (lane & 7) * 4;
                *reinterpret_cast<float4*>(C + (size_t)(m0 + r) * N + n0 + c) = make_float4(1.f, 2.f, 3.f, 4.f);
            }
    }
}

__global__ void contig(uint4* p, size_t n16) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n16; i += (size_t)gridDim.x * blockDim.x)
        p[i] = make_uint4(1, 2, 3, (unsigned)i);
}

template <int MODE>
__global__ void tiles(float* C, int M, int N) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int nwarps = blockDim.x >> 5;
    const int ntn = N / 128, ntiles = (M / 128) * ntn;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int m0 = (t / ntn) * 128, n0 = (t % ntn) * 128;
        // each warp owns 128/nwarps rows... split rows across warps
        for (int rb = warp * 4; rb < 128; rb += nwarps * 4) {
            for (int cb = 0; cb < 128; cb += 32) {     // 32 fp32 = 128 B per row chunk
                if (MODE == 1) {                        // 4 rows x 128 B
                    const int r = rb + (lane >> 3), c = cb + (lane & 7) * 4;
                    float4* dst = reinterpret_cast<float4*>(C + (size_t)(m0 + r) * N + n0 + c);
                    *dst = make_float4(1.f, 2.f, 3.f, 4.f);
                } else if (MODE == 2) {
                    const int r = rb + (lane >> 3), c = cb + (lane & 7) * 4;
                    float4* dst = reinterpret_cast<float4*>(C + (size_t)(m0 + r) * N + n0 + c);
                    __stcs(dst, make_float4(1.f, 2.f, 3.f, 4.f));
                }
            }
            if (MODE == 3) {                            // 1 row x 512 B per instruction, 4 rows
                for (int rr = 0; rr < 4; ++rr) {
                    float4* dst = reinterpret_cast<float4*>(C + (size_t)(m0 + rb + rr) * N + n0 + lane * 4);
                    *dst = make_float4(1.f, 2.f, 3.f, 4.f);
                }
            }
        }
    }
}

int main() {
    const int M = 25088, N = 4096;
    const size_t bytes = (size_t)M * N * 4;
    float* C;
    cudaMalloc(&C, bytes);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    auto run = [&](const char* name, auto fn) {
        for (int i = 0; i < 3; ++i) fn();
        float best = 1e9;
        for (int i = 0; i < 10; ++i) {
            spin<<<1, 1>>>(100000);
            cudaEventRecord(a);
            fn();
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            best = ms < best ? ms : best;
        }
        printf("{\"variant\": \"%s\", \"us\": %.2f, \"GBps\": %.1f}\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9);
    };
    unsigned* ctr;
    cudaMalloc(&ctr, 4);
    run("persist_dynamic_u8_148x1x256", [&] { cudaMemsetAsync(ctr, 0, 4); persist_dynamic<8><<<sms, 256>>>((uint4*)C, bytes / 16, ctr); });
    run("persist_dynamic_u4_148x4x256", [&] { cudaMemsetAsync(ctr, 0, 4); persist_dynamic<4><<<sms * 4, 256>>>((uint4*)C, bytes / 16, ctr); });
    run("tiles_dynamic_148x1x256", [&] { cudaMemsetAsync(ctr, 0, 4); tiles_dynamic<<<sms, 256>>>(C, M, N, ctr); });
    run("tiles_dynamic_148x2x256", [&] { cudaMemsetAsync(ctr, 0, 4); tiles_dynamic<<<sms * 2, 256>>>(C, M, N, ctr); });
    run("persist_u4_148x8x128", [&] { persist_unroll<4><<<sms * 8, 128>>>((uint4*)C, bytes / 16); });
    run("persist_u8_148x4x256", [&] { persist_unroll<8><<<sms * 4, 256>>>((uint4*)C, bytes / 16); });
    run("persist_u16_148x1x256", [&] { persist_unroll<16><<<sms, 256>>>((uint4*)C, bytes / 16); });
    run("persist_u8_148x1x256", [&] { persist_unroll<8><<<sms, 256>>>((uint4*)C, bytes / 16); });
    run("tiles_oneshot_256thr", [&] { tiles_oneshot<<<(M / 128) * (N / 128), 256>>>(C, M, N); });
    run("onestore_128thr", [&] { onestore<<<(unsigned)((bytes / 16 + 127) / 128), 128>>>((uint4*)C, bytes / 16); });
    run("unroll4_128thr", [&] { unroll4<<<(unsigned)((bytes / 16 + 511) / 512), 128>>>((uint4*)C, bytes / 16); });
    run("contig_const_148x8x256", [&] { contig_const<<<sms * 8, 256>>>((uint4*)C, bytes / 16); });
    run("contig_rand_148x8x256", [&] { contig_rand<<<sms * 8, 256>>>((uint4*)C, bytes / 16); });
    run("contig_148x8x256", [&] { contig<<<sms * 8, 256>>>((uint4*)C, bytes / 16); });
    run("contig_148x1x256", [&] { contig<<<sms, 256>>>((uint4*)C, bytes / 16); });
    run("tile_rows4_148x256thr", [&] { tiles<1><<<sms, 256>>>(C, M, N); });
    run("tile_rows4_cs_148x256thr", [&] { tiles<2><<<sms, 256>>>(C, M, N); });
    run("tile_rows1_148x256thr", [&] { tiles<3><<<sms, 256>>>(C, M, N); });
    run("tile_rows4_148x512thr", [&] { tiles<1><<<sms, 512>>>(C, M, N); });
    run("tile_rows4_296x256thr", [&] { tiles<1><<<sms * 2, 256>>>(C, M, N); });
    run("tile_rows4_592x256thr", [&] { tiles<1><<<sms * 4, 256>>>(C, M, N); });
    run("tile_rows4_1184x256thr", [&] { tiles<1><<<sms * 8, 256>>>(C, M, N); });
    return 0;
}
