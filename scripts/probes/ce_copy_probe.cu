// Diagnostic probe (not part of libtag): can the copy engines move the SFB factor exchange faster
// than SM stores? Each of n ranks (one process per GPU, launched by ce_copy_probe.sh) owns an NCCL
// symmetric window of n slots; it copies its own S-byte slot into slot `me` of every peer's
// window with cudaMemcpyAsync through the peer's LSA pointer (a flat device VA in this process),
// one stream per peer (optionally split into `chunks` copies per peer on their own streams), then
// writes an arrival flag into each peer's window with cuStreamWriteValue32 (default flags: a
// system-scope fence orders it after the copy); every rank waits for its n - 1 flags with
// cuStreamWaitValue32. The interval [all ranks released by a device barrier -> last flag seen]
// is timed with CUDA events on every rank; rank 0 prints the max over ranks (gathered through
// NCCL) per size. Bootstrap: rank 0 writes the ncclUniqueId to a file.
//
//   nvcc -O2 -std=c++17 -gencode arch=compute_100a,code=sm_100a -I$NCCL/include \
//        ce_copy_probe.cu -o ce_copy_probe -L$NCCL/lib -l:libnccl.so.2 -lcuda
//   ./ce_copy_probe <rank> <nranks> <idfile> [chunks]
#include <cuda.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
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
#define DK(x)                                                                                   \
    do {                                                                                        \
        CUresult r_ = (x);                                                                      \
        if (r_ != CUDA_SUCCESS) {                                                               \
            std::fprintf(stderr, "%s:%d CUresult %d\n", __FILE__, __LINE__, (int)r_);           \
            std::exit(1);                                                                       \
        }                                                                                       \
    } while (0)

__global__ void lsa_ptrs(ncclWindow_t w, int n, unsigned long long* out) {
    for (int p = 0; p < n; ++p) out[p] = reinterpret_cast<unsigned long long>(ncclGetLsaPointer(w, 0, p));
}

int main(int argc, char** argv) {
    const int me = std::atoi(argv[1]), n = std::atoi(argv[2]);
    const char* idfile = argv[3];
    const int chunks = argc > 4 ? std::atoi(argv[4]) : 1;
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
    const size_t max_slot = 32ull << 20;
    const size_t flag_off = static_cast<size_t>(n) * max_slot;
    const size_t win_bytes = flag_off + 4096;
    void* base = nullptr;
    NK(ncclMemAlloc(&base, win_bytes));
    CK(cudaMemset(base, 0, win_bytes));
    ncclWindow_t win;
    NK(ncclCommWindowRegister(comm, base, win_bytes, &win, NCCL_WIN_COLL_SYMMETRIC));
    unsigned long long* dptr;
    CK(cudaMalloc(&dptr, n * sizeof(unsigned long long)));
    lsa_ptrs<<<1, 1>>>(win, n, dptr);
    std::vector<unsigned long long> peer(n);
    CK(cudaMemcpy(peer.data(), dptr, n * sizeof(unsigned long long), cudaMemcpyDeviceToHost));
    char* src;
    CK(cudaMalloc(&src, max_slot));
    CK(cudaMemset(src, me + 1, max_slot));
    float* red;
    CK(cudaMalloc(&red, 4 * sizeof(float)));
    cudaStream_t s0;
    CK(cudaStreamCreateWithFlags(&s0, cudaStreamNonBlocking));
    std::vector<cudaStream_t> ps((n - 1) * chunks);
    for (auto& st : ps) CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    cudaEvent_t e0, e1, fork;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaEventCreateWithFlags(&fork, cudaEventDisableTiming));
    uint32_t* flags_local = reinterpret_cast<uint32_t*>(static_cast<char*>(base) + flag_off);
    const size_t sizes[] = {256u << 10, 1u << 20, 2785280, 8u << 20, 16u << 20, 32u << 20};
    uint32_t iter = 0;
    if (me == 0) std::printf("{\"n\": %d, \"chunks\": %d, \"results\": [", n, chunks);
    bool first = true;
    for (size_t S : sizes) {
        std::vector<float> ts;
        for (int rep = 0; rep < 23; ++rep) {
            ++iter;
            // device barrier: an all-reduce of one float
            NK(ncclAllReduce(red, red, 1, ncclFloat, ncclSum, comm, s0));
            CK(cudaEventRecord(e0, s0));
            CK(cudaEventRecord(fork, s0));
            int k = 0;
            for (int j = 1; j < n; ++j) {
                const int p = (me + j) % n;
                for (int c = 0; c < chunks; ++c, ++k) {
                    cudaStream_t st = ps[k];
                    CK(cudaStreamWaitEvent(st, fork, 0));
                    const size_t lo = S * c / chunks, hi = S * (c + 1) / chunks;
                    char* dst = reinterpret_cast<char*>(peer[p]) + me * max_slot + lo;
                    CK(cudaMemcpyAsync(dst, src + lo, hi - lo, cudaMemcpyDeviceToDevice, st));
                    // flag word [me * 16 + c] on peer p (one per sender and chunk)
                    CUdeviceptr fl = static_cast<CUdeviceptr>(peer[p] + flag_off + 4 * (me * 16 + c));
                    DK(cuStreamWriteValue32(reinterpret_cast<CUstream>(st), fl, iter, CU_STREAM_WRITE_VALUE_DEFAULT));
                }
            }
            for (int j = 1; j < n; ++j) {
                const int p = (me + j) % n;
                for (int c = 0; c < chunks; ++c) {
                    CUdeviceptr fl = reinterpret_cast<CUdeviceptr>(flags_local + p * 16 + c);
                    DK(cuStreamWaitValue32(reinterpret_cast<CUstream>(s0), fl, iter, CU_STREAM_WAIT_VALUE_GEQ));
                }
            }
            CK(cudaEventRecord(e1, s0));
            for (auto& st : ps) {            // join the copy streams before the next iteration
                CK(cudaEventRecord(fork, st));
                CK(cudaStreamWaitEvent(s0, fork, 0));
            }
            CK(cudaStreamSynchronize(s0));
            float ms = 0;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (rep >= 3) ts.push_back(ms * 1000.f);
        }
        std::sort(ts.begin(), ts.end());
        float med = ts[ts.size() / 2];
        // max over ranks of the median
        CK(cudaMemcpy(red + 1, &med, sizeof(float), cudaMemcpyHostToDevice));
        NK(ncclAllReduce(red + 1, red + 2, 1, ncclFloat, ncclMax, comm, s0));
        CK(cudaStreamSynchronize(s0));
        float mx = 0;
        CK(cudaMemcpy(&mx, red + 2, sizeof(float), cudaMemcpyDeviceToHost));
        // check one byte from every peer's slot
        bool ok = true;
        for (int p = 0; p < n; ++p) {
            if (p == me) continue;
            unsigned char b0 = 0, b1 = 0;
            CK(cudaMemcpy(&b0, static_cast<char*>(base) + p * max_slot, 1, cudaMemcpyDeviceToHost));
            CK(cudaMemcpy(&b1, static_cast<char*>(base) + p * max_slot + S - 1, 1, cudaMemcpyDeviceToHost));
            ok = ok && b0 == p + 1 && b1 == p + 1;
        }
        if (me == 0) {
            const double ingress = static_cast<double>(n - 1) * S;
            std::printf("%s{\"slot_bytes\": %zu, \"us_max_over_ranks\": %.2f, \"ingress_GBps\": %.1f, "
                        "\"busbw_frac_of_900\": %.3f, \"rank0_ok\": %s}",
                        first ? "" : ", ", S, mx, ingress / mx / 1e3, ingress / mx / 1e3 / 900.0,
                        ok ? "true" : "false");
            first = false;
        }
    }
    if (me == 0) std::printf("]}\n");
    CK(cudaDeviceSynchronize());
    NK(ncclCommWindowDeregister(comm, win));
    NK(ncclMemFree(base));
    NK(ncclCommDestroy(comm));
    return 0;
}
