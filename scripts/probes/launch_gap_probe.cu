// Diagnostic probe (not part of libtag): how long after the previous kernel in the stream ends does
// a persistent 148-CTA kernel start, as a function of its dynamic shared memory, the programmatic
// dependent launch attribute and the previous kernel's own shared-memory use? A one-thread marker
// kernel stamps %globaltimer; the probe kernel stamps its first instruction in every CTA.
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a launch_gap_probe.cu -o launch_gap_probe
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <vector>

__device__ unsigned long long g_t[512];

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}
__global__ void marker(int slot) { g_t[slot] = gt(); }
// the "previous" kernel: optionally with big shared memory of its own
__global__ void prev_kernel(int use) {
    extern __shared__ unsigned char sm[];
    if (use && threadIdx.x == 0) sm[0] = 1;
    __syncthreads();
    if (threadIdx.x == 0) g_t[256 + blockIdx.x] = gt();   // this CTA's end
}
__global__ void __launch_bounds__(320, 1) probe(int slot0) {
    extern __shared__ unsigned char sm[];
    if (threadIdx.x == 0) g_t[slot0 + blockIdx.x] = gt();
    if (threadIdx.x == 0) sm[0] = 1;
}

int main() {
    cudaStream_t s;
    cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    const int G = 148;
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    cudaFuncSetAttribute(prev_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 232448);
    struct V { const char* name; int smem; int pdl; int prev_smem; };
    V vs[] = {{"smem 227KB, pdl, prev 0 smem", 232448, 1, 0},
              {"smem 227KB, no pdl, prev 0 smem", 232448, 0, 0},
              {"smem 100KB, pdl, prev 0 smem", 100 * 1024, 1, 0},
              {"smem 0, pdl, prev 0 smem", 0, 1, 0},
              {"smem 227KB, pdl, prev 227KB smem", 232448, 1, 232448},
              {"smem 0, no pdl, prev 0 smem", 0, 0, 0}};
    std::printf("{\"results\": [");
    bool first = true;
    for (const V& v : vs) {
        std::vector<double> gap, spread;
        for (int rep = 0; rep < 30; ++rep) {
            prev_kernel<<<G, 320, v.prev_smem, s>>>(v.prev_smem > 0);
            cudaLaunchConfig_t cfg{};
            cfg.gridDim = dim3(G);
            cfg.blockDim = dim3(320);
            cfg.dynamicSmemBytes = v.smem;
            cfg.stream = s;
            cudaLaunchAttribute attr[1];
            attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
            attr[0].val.programmaticStreamSerializationAllowed = 1;
            cfg.attrs = attr;
            cfg.numAttrs = v.pdl ? 1 : 0;
            cudaLaunchKernelEx(&cfg, probe, 8);
            cudaStreamSynchronize(s);
            unsigned long long h[512];
            cudaMemcpyFromSymbol(h, g_t, sizeof h);
            unsigned long long mn = ~0ull, mx = 0, pend = 0;
            for (int b = 0; b < G; ++b) pend = std::max(pend, h[256 + b]);
            h[0] = pend;
            for (int b = 0; b < G; ++b) {
                mn = std::min(mn, h[8 + b]);
                mx = std::max(mx, h[8 + b]);
            }
            if (rep >= 5) {
                gap.push_back((mn - h[0]) / 1e3);
                spread.push_back((mx - mn) / 1e3);
            }
        }
        std::sort(gap.begin(), gap.end());
        std::sort(spread.begin(), spread.end());
        std::printf("%s{\"variant\": \"%s\", \"prev_last_cta_end_to_first_cta_us_median\": %.2f, \"cta_start_spread_us\": %.2f}",
                    first ? "" : ", ", v.name, gap[gap.size() / 2], spread[spread.size() / 2]);
        first = false;
    }
    std::printf("]}\n");
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) std::printf("error %s\n", cudaGetErrorString(e));
    return 0;
}
