// push_gather.cu — steps a1 + a2 fused: every replica PUSHES its (cast) sufficient factors
// straight into the gather buffer of every peer over NVLink 5 / NVSwitch, instead of a pack
// kernel followed by an NCCL all-gather ("the sufficient factors ... are broadcast to all
// devices"; D(D-1) transfers of each cut tensor).
//
// Mechanism: the gather buffers live in an NCCL symmetric window (ncclMemAlloc +
// ncclCommWindowRegister(NCCL_WIN_COLL_SYMMETRIC)); the NCCL 2.28 device API gives every GPU
// load/store-accessible (LSA) pointers into its peers' windows. One kernel per layer, or per
// bucket of layers (tag_sfb_group_*):
//   1. each thread loads 16 output bytes of X_r / dY_r (fp32 -> bf16 RNE cast fused when the
//      wire dtype differs), and stores them into slot r of every peer's window (peer order
//      rotated by rank so the n senders spread over the n receivers);
//   2. an LSA barrier (CTA b of every rank meets CTA b of every peer; release/acquire at system
//      scope) — when the kernel completes on a rank, every peer's slot has landed there.
// The window is double-buffered per plan, so the barrier that ends call t also proves every
// peer has finished reading buffer t-1 (its reconstruction of call t-1 precedes its push of
// call t in stream order): one barrier per call, none before the stores.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>
#include <nccl_device.h>

#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "tag_internal.h"

namespace tag {
namespace {

constexpr int PUSH_THREADS = 512;

__device__ __forceinline__ uint32_t bf16x2_rn(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
    return *reinterpret_cast<uint32_t*>(&h);
}

// One push kernel serves a whole bucket of layers: segment i covers layer i's X slot then its
// dY slot (16-byte output vectors); one LSA barrier per CTA at the end covers all of them.
struct PushLayer {
    const void* X;
    const void* dY;
    ncclWindow_t win;
    size_t off_x, off_dy;   // byte offsets of buffer 0's X_all / dY_all in `win`
    size_t xbuf, ybuf;      // buffer 1's X_all / dY_all are xbuf / ybuf bytes further
    size_t off_flag;        // the window flag area (WIN_* offsets)
    uint32_t* flags;        // the same area, this rank's address
    int64_t vx, vy;         // 16-byte output vectors of this rank's X_r / dY_r
    int64_t vbegin;         // first global vector index of this layer
};

struct PushGroup {
    PushLayer L[MAX_GROUP];
    int count;
    int64_t total;
    int slot;               // this rank's slot (world rank)
    uint32_t* local_ctr;    // self-resetting "last CTA" counter (plan 0's WIN_LOCAL_PUSH)
};

// DBG (diagnostics builds only: scripts/build_variant.sh -DEXP_PUSH_DBG=k, never the product):
// 1 = skip the data stores, 2 = skip the barrier, 3 = full kernel + printf of %globaltimer phase
// stamps from a few CTAs.
#ifndef EXP_PUSH_DBG
#define EXP_PUSH_DBG 0
#endif
__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

template <bool CAST, int DBG = 0>
__global__ void __launch_bounds__(PUSH_THREADS)
push_gather_kernel(const ncclDevComm comm, const __grid_constant__ PushGroup g)
{
    const uint64_t t_start = DBG == 3 ? gtimer() : 0;
    const int npeers = comm.lsaSize;
    const int me = comm.lsaRank;
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nthreads = static_cast<int64_t>(gridDim.x) * blockDim.x;
    // this gather's buffer of every layer: c & 1 (device state, see tag_internal.h)
    __shared__ uint32_t s_calls[MAX_GROUP];
    if (threadIdx.x < g.count) s_calls[threadIdx.x] = load_calls(g.L[threadIdx.x].flags + WIN_CALLS / 4);
    __syncthreads();
    int li = 0;
    for (int64_t v = tid; v < (DBG == 1 ? 0 : g.total); v += nthreads) {
        while (li + 1 < g.count && v >= g.L[li + 1].vbegin) ++li;   // v only grows
        const PushLayer& L = g.L[li];
        const int64_t lv = v - L.vbegin;
        const bool isx = lv < L.vx;
        const int64_t i = isx ? lv : lv - L.vx;
        uint4 val;
        if constexpr (CAST) {
            const float4* src = reinterpret_cast<const float4*>(isx ? L.X : L.dY) + 2 * i;
            const float4 a = __ldcs(src);
            const float4 b = __ldcs(src + 1);
            val = make_uint4(bf16x2_rn(a.x, a.y), bf16x2_rn(a.z, a.w), bf16x2_rn(b.x, b.y),
                             bf16x2_rn(b.z, b.w));
        } else {
            val = __ldcs(reinterpret_cast<const uint4*>(isx ? L.X : L.dY) + i);
        }
        const size_t par = s_calls[li] & 1u;
        const size_t off = isx ? L.off_x + par * L.xbuf + (static_cast<size_t>(g.slot) * L.vx + i) * 16
                               : L.off_dy + par * L.ybuf + (static_cast<size_t>(g.slot) * L.vy + i) * 16;
        for (int k = 0; k < npeers; ++k) {
            const int p = (me + k) % npeers;   // rotate so the senders spread over receivers
            *reinterpret_cast<uint4*>(ncclGetLsaPointer(L.win, off, p)) = val;
        }
    }
    // all of this CTA's stores are released to every peer; CTA b waits for CTA b everywhere
    uint64_t t_data = 0;
    if constexpr (DBG == 3) {
        __syncthreads();
        t_data = gtimer();
    }
    if constexpr (DBG != 2) {
        ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamTagLsa(), blockIdx.x);
        bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
    }
    // The last CTA of this rank (self-resetting counter: every CTA has read c by then) keeps the
    // window's device state in step with the fused path: one arrival per layer on every peer
    // (fused calls wait for n arrivals per call and buffer) and c advanced by one.
    __syncthreads();
    if (threadIdx.x == 0) {
        uint32_t old;
        asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;"
                     : "=r"(old) : "l"(g.local_ctr), "r"(gridDim.x - 1) : "memory");
        if (old == gridDim.x - 1) {
            for (int l = 0; l < g.count; ++l) {
                const size_t fo = g.L[l].off_flag + WIN_ARRIVAL + 4 * (s_calls[l] & 1u);
                for (int k = 0; k < npeers; ++k) {
                    const int p = (me + k) % npeers;
                    uint32_t* ctr = static_cast<uint32_t*>(ncclGetLsaPointer(g.L[l].win, fo, p));
                    asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" :: "l"(ctr) : "memory");
                }
                atomicAdd(g.L[l].flags + WIN_CALLS / 4, 1u);
            }
        }
    }
    if constexpr (DBG == 3) {
        if (threadIdx.x == 0 && (blockIdx.x == 0 || blockIdx.x == gridDim.x - 1 || blockIdx.x == gridDim.x / 2))
            printf("push rank %d cta %d start %llu data +%llu barrier +%llu\n", me, blockIdx.x,
                   (unsigned long long)t_start, (unsigned long long)(t_data - t_start),
                   (unsigned long long)(gtimer() - t_data));
    }
}

// Device-side barrier of the whole comm on a stream (one CTA, LSA barrier index `index`).
__global__ void comm_barrier_kernel(const ncclDevComm comm, int index) {
    ncclLsaBarrierSession<ncclCoopCta> bar(ncclCoopCta(), comm, ncclTeamTagLsa(), index);
    bar.sync(ncclCoopCta(), cuda::memory_order_acq_rel);
}

}  // namespace

tag_status_t launch_comm_barrier(const void* dc, int index, cudaStream_t s) {
    comm_barrier_kernel<<<1, 32, 0, s>>>(*static_cast<const ncclDevComm*>(dc), index);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "launch comm_barrier_kernel");
    count_launch();
    return TAG_OK;
}

tag_status_t push_devcomm_create(ncclComm_t comm, int max_ctas, bool multimem, void** out) {
    ncclDevCommRequirements reqs;
    std::memset(&reqs, 0, sizeof reqs);
    reqs.lsaBarrierCount = max_ctas;
    // NVLink SHARP multicast (one multimem store reaches every GPU): opt-in with the comm flag
    // TAG_COMM_NVLS_MULTICAST. Measured at n = 2 and 4 on B200 it is not faster than one unicast
    // store per peer (the push is latency-bound: 8-11 us unicast vs 13-14 us multicast per CTA
    // slice at n = 2). Collective: every rank must pass the same requirements.
    reqs.lsaMultimem = multimem;
    ncclDevComm* dc = new ncclDevComm;
    ncclResult_t r = ncclDevCommCreate(comm, &reqs, dc);
    if (r != ncclSuccess) {
        delete dc;
        return fail(TAG_ERR_NCCL, std::string("ncclDevCommCreate: ") + ncclGetErrorString(r));
    }
    *out = dc;
    return TAG_OK;
}

void push_devcomm_destroy(ncclComm_t comm, void* dc) {
    if (!dc) return;
    ncclDevCommDestroy(comm, static_cast<ncclDevComm*>(dc));
    delete static_cast<ncclDevComm*>(dc);
}

void* push_devcomm_mc_base(const void* dc) {
    const ncclDevComm* d = static_cast<const ncclDevComm*>(dc);
    return d ? d->lsaMultimem.mcBasePtr : nullptr;
}

bool push_devcomm_all_lsa(const void* dc, int nranks) {
    const ncclDevComm* d = static_cast<const ncclDevComm*>(dc);
    return d && d->lsaSize == nranks && d->nRanks == nranks;
}

int push_grid(int64_t vectors, int max_ctas) {
    int64_t g = (vectors + PUSH_THREADS - 1) / PUSH_THREADS;
    if (g > max_ctas) g = max_ctas;
    if (g > num_sms()) g = num_sms();
    return g < 1 ? 1 : static_cast<int>(g);
}

tag_status_t launch_push_gather_group(const void* dc, const PushSegment* seg, int count, int slot,
                                      tag_dtype_t in, tag_dtype_t wire, int max_ctas,
                                      uint32_t* local_ctr, cudaStream_t s) {
    if (count < 1 || count > MAX_GROUP) return fail(TAG_ERR_INVALID_ARG, "push group size");
    const ncclDevComm& comm = *static_cast<const ncclDevComm*>(dc);
    const int64_t ew = static_cast<int64_t>(dtype_size(wire));
    PushGroup g;
    std::memset(&g, 0, sizeof g);
    int64_t total = 0;
    for (int i = 0; i < count; ++i) {
        PushLayer& L = g.L[i];
        L.X = seg[i].X;
        L.dY = seg[i].dY;
        L.win = static_cast<ncclWindow_t>(seg[i].win);
        L.off_x = seg[i].off_x;
        L.off_dy = seg[i].off_dy;
        L.xbuf = seg[i].xbuf;
        L.ybuf = seg[i].ybuf;
        L.off_flag = seg[i].off_flag;
        L.flags = seg[i].flags;
        L.vx = seg[i].cx * ew / 16;
        L.vy = seg[i].cy * ew / 16;
        L.vbegin = total;
        total += L.vx + L.vy;
    }
    g.count = count;
    g.total = total;
    g.slot = slot;
    g.local_ctr = local_ctr;
    const int grid = push_grid(total, max_ctas);
    if (in == wire)
        push_gather_kernel<false, EXP_PUSH_DBG><<<grid, PUSH_THREADS, 0, s>>>(comm, g);
    else
        push_gather_kernel<true, EXP_PUSH_DBG><<<grid, PUSH_THREADS, 0, s>>>(comm, g);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return cuda_fail(e, "launch push_gather_kernel");
    count_launch();
    return TAG_OK;
}

}  // namespace tag
