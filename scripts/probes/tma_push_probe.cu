// Diagnostic probe (not part of libtag): does the factor push land faster over NVLink as TMA bulk
// copies (global -> smem with cp.async.bulk, then smem -> every peer's window with
// cp.async.bulk.global.shared::cta) than as the product's 16-byte SM stores? One process per GPU
// (tma_push_probe.sh), an NCCL symmetric window of n slots per rank; each of 148 CTAs pushes its
// slice of this rank's S-byte slot to slot `me` of every rank (the own included, as the fused
// kernel does), then waits for completion and issues one system-scope fence. Per CTA
// %globaltimer stamps: span = last CTA's fence - first CTA's start; rank 0 prints the max over
// ranks of the median span (NCCL all-reduce), per size and variant.
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I$NCCL/include \
//        tma_push_probe.cu -o tma_push_probe -L$NCCL/lib -l:libnccl.so.2
//   ./tma_push_probe <rank> <nranks> <idfile>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <string>
#include <thread>
#include <vector>

#define CK(x)                                                                                   \
    do {                                                                                        \
        cudaError_t e_ = (x);                                                                   \
        if (e_ != cudaSuccess) {                                                                \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_));    \
            std::exit(1);                                                                       \
        }                                                                                       \
    } while (0)
#define NK(x)                                                                                   \
    do {                                                                                        \
        ncclResult_t r_ = (x);                                                                  \
        if (r_ != ncclSuccess) {                                                                \
            std::fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, ncclGetErrorString(r_));    \
            std::exit(1);                                                                       \
        }                                                                                       \
    } while (0)

constexpr int G = 148;
constexpr int THREADS = 512;
constexpr int CH = 32768;      // TMA chunk bytes
constexpr int NB = 4;          // smem chunk buffers

__device__ __forceinline__ unsigned long long gt() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// the product's way: 16-byte loads, 16-byte stores to every rank's slot (peer order rotated)
__global__ void __launch_bounds__(THREADS, 1)
push_sm(ncclWindow_t win, int n, int me, const uint4* src, long long vecs, size_t slot_bytes,
        unsigned long long* st) {
    if (threadIdx.x == 0) st[2 * blockIdx.x] = gt();
    const long long beg = vecs * blockIdx.x / G, end = vecs * (blockIdx.x + 1) / G;
    for (long long v0 = beg + threadIdx.x; v0 < end; v0 += 4 * THREADS) {
        uint4 val[4];
#pragma unroll
        for (int u = 0; u < 4; ++u)
            if (v0 + u * THREADS < end) val[u] = __ldcs(src + v0 + u * THREADS);
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            if (v0 + u * THREADS >= end) break;
            const size_t off = me * slot_bytes + (v0 + u * THREADS) * 16;
            for (int k = 0; k < n; ++k) {
                const int p = (me + k) % n;
                *reinterpret_cast<uint4*>(ncclGetLsaPointer(win, off, p)) = val[u];
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        st[2 * blockIdx.x + 1] = gt();
    }
}

// TMA bulk copies: one thread per CTA streams its slice through NB smem chunks, each chunk
// stored to every rank with one bulk store per rank
__global__ void __launch_bounds__(THREADS, 1)
push_tma(ncclWindow_t win, int n, int me, const char* src, long long vecs, size_t slot_bytes,
         unsigned long long* st) {
    extern __shared__ __align__(1024) unsigned char sm[];
    __shared__ __align__(8) unsigned long long bars[NB];
    if (threadIdx.x != 0) return;
    st[2 * blockIdx.x] = gt();
    const uint32_t sbase = static_cast<uint32_t>(__cvta_generic_to_shared(sm));
    const uint32_t bbase = static_cast<uint32_t>(__cvta_generic_to_shared(bars));
    for (int b = 0; b < NB; ++b)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(bbase + 8 * b) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    const long long beg = vecs * blockIdx.x / G * 16, end = vecs * (blockIdx.x + 1) / G * 16;
    int c = 0;
    for (long long o = beg; o < end; o += CH, ++c) {
        const int b = c % NB;
        const uint32_t bytes = static_cast<uint32_t>(end - o < CH ? end - o : CH);
        if (c >= NB) asm volatile("cp.async.bulk.wait_group.read %0;" :: "n"(NB - 1) : "memory");
        const uint32_t sb = sbase + b * CH, bar = bbase + 8 * b;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" :: "r"(bar), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     :: "r"(sb), "l"(src + o), "r"(bytes), "r"(bar) : "memory");
        const uint32_t par = (c / NB) & 1;
        asm volatile("{\n\t.reg .pred P;\n\tW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t@!P bra W_%=;\n\t}"
                     :: "r"(bar), "r"(par) : "memory");
        for (int k = 0; k < n; ++k) {
            const int p = (me + k) % n;
            char* dst = static_cast<char*>(ncclGetLsaPointer(win, me * slot_bytes + o, p));
            asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                         :: "l"(dst), "r"(sb), "r"(bytes) : "memory");
        }
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    asm volatile("fence.proxy.async.global;" ::: "memory");
    asm volatile("fence.acq_rel.sys;" ::: "memory");
    st[2 * blockIdx.x + 1] = gt();
}

int main(int argc, char** argv) {
    const int me = std::atoi(argv[1]), n = std::atoi(argv[2]);
    const char* idfile = argv[3];
    CK(cudaSetDevice(me));
    ncclUniqueId id;
    if (me == 0) {
        NK(ncclGetUniqueId(&id));
        std::string tmp = std::string(idfile) + ".tmp";
        std::ofstream(tmp, std::ios::binary).write(reinterpret_cast<char*>(&id), sizeof id);
        std::rename(tmp.c_str(), idfile);
    } else {
        for (;;) {
            std::ifstream f(idfile, std::ios::binary);
            if (f && f.read(reinterpret_cast<char*>(&id), sizeof id)) break;
            std::this_thread::sleep_for(std::chrono::milliseconds(20));
        }
    }
    ncclComm_t comm;
    NK(ncclCommInitRank(&comm, n, id, me));
    const size_t max_slot = 16ull << 20;
    const size_t win_bytes = static_cast<size_t>(n) * max_slot;
    void* base = nullptr;
    NK(ncclMemAlloc(&base, win_bytes));
    CK(cudaMemset(base, 0, win_bytes));
    ncclWindow_t win;
    NK(ncclCommWindowRegister(comm, base, win_bytes, &win, NCCL_WIN_COLL_SYMMETRIC));
    char* src;
    CK(cudaMalloc(&src, max_slot));
    CK(cudaMemset(src, me + 1, max_slot));
    unsigned long long* st;
    CK(cudaMalloc(&st, 2 * G * sizeof(unsigned long long)));
    float* red;
    CK(cudaMalloc(&red, 4 * sizeof(float)));
    cudaStream_t s;
    CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CK(cudaFuncSetAttribute(push_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, NB * CH));
    CK(cudaFuncSetAttribute(push_sm, cudaFuncAttributeMaxDynamicSharedMemorySize, NB * CH));
    const size_t sizes[] = {256u << 10, 1u << 20, 2785280, 8u << 20, 16u << 20};
    if (me == 0) std::printf("{\"n\": %d, \"results\": [", n);
    bool first = true;
    for (int variant = 0; variant < 2; ++variant) {
        for (size_t S : sizes) {
            const long long vecs = static_cast<long long>(S / 16);
            std::vector<float> spans;
            for (int rep = 0; rep < 23; ++rep) {
                NK(ncclAllReduce(red, red, 1, ncclFloat, ncclSum, comm, s));
                if (variant == 0)
                    push_sm<<<G, THREADS, NB * CH, s>>>(win, n, me, reinterpret_cast<const uint4*>(src), vecs, max_slot, st);
                else
                    push_tma<<<G, THREADS, NB * CH, s>>>(win, n, me, src, vecs, max_slot, st);
                CK(cudaGetLastError());
                CK(cudaStreamSynchronize(s));
                std::vector<unsigned long long> h(2 * G);
                CK(cudaMemcpy(h.data(), st, h.size() * 8, cudaMemcpyDeviceToHost));
                unsigned long long a = ~0ull, b = 0;
                for (int i = 0; i < G; ++i) {
                    a = std::min(a, h[2 * i]);
                    b = std::max(b, h[2 * i + 1]);
                }
                if (rep >= 3) spans.push_back((b - a) / 1e3f);
            }
            std::sort(spans.begin(), spans.end());
            float med = spans[spans.size() / 2];
            CK(cudaMemcpy(red + 1, &med, sizeof(float), cudaMemcpyHostToDevice));
            NK(ncclAllReduce(red + 1, red + 2, 1, ncclFloat, ncclMax, comm, s));
            CK(cudaStreamSynchronize(s));
            float mx = 0;
            CK(cudaMemcpy(&mx, red + 2, sizeof(float), cudaMemcpyDeviceToHost));
            bool ok = true;
            for (int p = 0; p < n; ++p) {
                unsigned char b0 = 0, b1 = 0;
                CK(cudaMemcpy(&b0, static_cast<char*>(base) + p * max_slot, 1, cudaMemcpyDeviceToHost));
                CK(cudaMemcpy(&b1, static_cast<char*>(base) + p * max_slot + S - 1, 1, cudaMemcpyDeviceToHost));
                ok = ok && b0 == p + 1 && b1 == p + 1;
            }
            if (me == 0) {
                const double ingress = static_cast<double>(n - 1) * S;
                std::printf("%s{\"variant\": \"%s\", \"slot_bytes\": %zu, \"span_us_max_over_ranks\": %.2f, "
                            "\"ingress_GBps\": %.1f, \"rank0_ok\": %s}", first ? "" : ", ",
                            variant == 0 ? "sm_stores" : "tma_bulk", S, mx, ingress / mx / 1e3,
                            ok ? "true" : "false");
                first = false;
            }
            CK(cudaMemset(base, 0, win_bytes));
            CK(cudaDeviceSynchronize());
            NK(ncclAllReduce(red, red, 1, ncclFloat, ncclSum, comm, s));
            CK(cudaStreamSynchronize(s));
        }
    }
    if (me == 0) std::printf("]}\n");
    CK(cudaDeviceSynchronize());
    NK(ncclCommWindowDeregister(comm, win));
    NK(ncclMemFree(base));
    NK(ncclCommDestroy(comm));
    return 0;
}
