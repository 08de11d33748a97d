// push_overlap_probe.cu — diagnostic (not part of libtag): can a few dedicated SMs push this
// rank's factors over NVLink at link speed while the other SMs stream an HBM write (the
// reconstruction's epilogue)? One kernel, one CTA per SM (dynamic smem forces it): CTAs [0, P)
// store `bytes` into slot `rank` of every peer's symmetric window (16-B unicast stores, peer order
// rotated), then one system-scope fence; CTAs [P, grid) write `wbytes` of local HBM. Per-CTA
// %globaltimer stamps give the push span and the write span.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -shared -Xcompiler -fPIC -I$NCCL/include \
//        push_overlap_probe.cu -L$NCCL/lib -l:libnccl.so.2 -o libpushprobe.so
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <cstdint>
#include <cstring>

namespace {

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

__global__ void __launch_bounds__(1024, 1)
probe_kernel(const ncclDevComm comm, ncclWindow_t win, const uint4* src, int64_t vecs, int P,
             float4* hbm, int64_t wvecs, unsigned long long* stamps) {
    const int npeers = comm.lsaSize, me = comm.lsaRank;
    __syncthreads();
    const uint64_t t0 = gtimer();
    if (static_cast<int>(blockIdx.x) < P) {
        if (vecs > 0) {
            const int64_t beg = vecs * blockIdx.x / P, end = vecs * (blockIdx.x + 1) / P;
            for (int64_t v0 = beg + threadIdx.x; v0 < end; v0 += 4 * 1024) {
                uint4 val[4];
#pragma unroll
                for (int u = 0; u < 4; ++u)
                    if (v0 + u * 1024 < end) val[u] = __ldcs(src + v0 + u * 1024);
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    if (v0 + u * 1024 >= end) break;
                    const size_t off = (static_cast<size_t>(me) * vecs + v0 + u * 1024) * 16;
                    for (int k = 0; k < npeers; ++k) {
                        const int p = (me + k) % npeers;
                        *reinterpret_cast<uint4*>(ncclGetLsaPointer(win, off, p)) = val[u];
                    }
                }
            }
        }
        __syncthreads();
        if (threadIdx.x == 0) asm volatile("fence.acq_rel.sys;" ::: "memory");
    } else if (wvecs > 0) {
        const int nw = gridDim.x - P, w = blockIdx.x - P;
        const int64_t beg = wvecs * w / nw, end = wvecs * (w + 1) / nw;
        for (int64_t i = beg + threadIdx.x; i < end; i += 1024) {
            const float f = static_cast<float>(i);
            __stcs(hbm + i, make_float4(f, f + 1.f, f + 2.f, f + 3.f));
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        stamps[2 * blockIdx.x] = t0;
        stamps[2 * blockIdx.x + 1] = gtimer();
    }
}

ncclComm_t g_comm;
ncclDevComm g_dc;
ncclWindow_t g_win;
void* g_winbase;
void* g_src;
void* g_hbm;
unsigned long long* g_stamps;
size_t g_winbytes;

}  // namespace

extern "C" {

int probe_uid(unsigned char* id) {
    ncclUniqueId u;
    if (ncclGetUniqueId(&u) != ncclSuccess) return 1;
    std::memcpy(id, &u, 128);
    return 0;
}

// slot_bytes: bytes this rank pushes (its slot); hbm_bytes: the concurrent write buffer
int probe_init(const unsigned char* id, int nranks, int rank, int dev, size_t slot_bytes,
               size_t hbm_bytes) {
    cudaSetDevice(dev);
    ncclUniqueId u;
    std::memcpy(&u, id, 128);
    if (ncclCommInitRank(&g_comm, nranks, u, rank) != ncclSuccess) return 1;
    ncclDevCommRequirements reqs;
    std::memset(&reqs, 0, sizeof reqs);
    reqs.lsaBarrierCount = 1;
    if (ncclDevCommCreate(g_comm, &reqs, &g_dc) != ncclSuccess) return 2;
    g_winbytes = (slot_bytes * nranks + 4095) & ~size_t(4095);
    if (ncclMemAlloc(&g_winbase, g_winbytes) != ncclSuccess) return 3;
    if (ncclCommWindowRegister(g_comm, g_winbase, g_winbytes, &g_win, NCCL_WIN_COLL_SYMMETRIC) !=
        ncclSuccess)
        return 4;
    if (cudaMalloc(&g_src, slot_bytes) != cudaSuccess) return 5;
    cudaMemset(g_src, 1, slot_bytes);
    if (cudaMalloc(&g_hbm, hbm_bytes) != cudaSuccess) return 6;
    if (cudaMalloc(&g_stamps, 2 * 1024 * sizeof(unsigned long long)) != cudaSuccess) return 7;
    cudaFuncSetAttribute(probe_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 150 * 1024);
    return cudaDeviceSynchronize() == cudaSuccess ? 0 : 8;
}

// one launch; stamps (2 per CTA: start, end, ns) copied to `out` (2 * grid entries)
int probe_run(size_t push_bytes, int P, size_t write_bytes, int grid, unsigned long long* out,
              cudaStream_t s) {
    probe_kernel<<<grid, 1024, 150 * 1024, s>>>(g_dc, g_win, static_cast<const uint4*>(g_src),
                                                 static_cast<int64_t>(push_bytes / 16), P,
                                                 static_cast<float4*>(g_hbm),
                                                 static_cast<int64_t>(write_bytes / 16), g_stamps);
    if (cudaGetLastError() != cudaSuccess) return 1;
    if (cudaStreamSynchronize(s) != cudaSuccess) return 2;
    cudaMemcpy(out, g_stamps, 2 * grid * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    return 0;
}

}  // extern "C"
