// api.cu — the libtag C ABI (include/tag.h): communicator bootstrap, SFB plans, the SFB sync
// path (pack -> NCCL all-gather -> tensor-core reconstruction) and the dense-AllReduce baseline.
// Host-side orchestration only; every arithmetic step runs in the kernels of this library or in
// NCCL. There is no CPU fallback.
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "tag_internal.h"

namespace tag {
// push_gather.cu
tag_status_t push_devcomm_create(ncclComm_t comm, int max_ctas, bool multimem, void** out);
void push_devcomm_destroy(ncclComm_t comm, void* dc);
bool push_devcomm_all_lsa(const void* dc, int nranks);
void* push_devcomm_mc_base(const void* dc);
tag_status_t launch_comm_barrier(const void* dc, int index, cudaStream_t s);
constexpr int PUSH_MAX_CTAS = 148;
#ifndef EXP_PUSH_GRID
#define EXP_PUSH_GRID PUSH_MAX_CTAS   // diagnostics builds: cap on the push kernel's grid
#endif
constexpr int COMM_BARRIER_INDEX = PUSH_MAX_CTAS;   // LSA barrier slot of tag_comm_barrier

std::atomic<uint64_t> g_launches{0};
static thread_local std::string t_last_error;

void set_error(const std::string& msg) { t_last_error = msg; }
tag_status_t fail(tag_status_t st, const std::string& msg) {
    t_last_error = msg;
    return st;
}
tag_status_t cuda_fail(cudaError_t e, const char* what) {
    t_last_error = std::string(what) + ": " + cudaGetErrorString(e);
    return e == cudaErrorMemoryAllocation ? TAG_ERR_OOM : TAG_ERR_CUDA;
}
static tag_status_t nccl_fail(ncclResult_t r, const char* what) {
    t_last_error = std::string(what) + ": " + ncclGetErrorString(r);
    return TAG_ERR_NCCL;
}

int num_sms() {
    static std::atomic<int> cached[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) dev = 0;
    int v = cached[dev].load(std::memory_order_relaxed);
    if (v == 0) {
        if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
            v = 148;
        cached[dev].store(v, std::memory_order_relaxed);
    }
    return v;
}

// ------------------------------------------------------------------------------------------
// scale kernel for the n = 1 "dense all-reduce" (dW <- dW / B) — no collective exists then
// ------------------------------------------------------------------------------------------
namespace {
__global__ void scale_f32_kernel(float* p, int64_t len, float alpha) {
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nt = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = tid; i < len; i += nt) p[i] = __fmul_rn(p[i], alpha);
}
__global__ void scale_bf16_kernel(__nv_bfloat16* p, int64_t len, float alpha) {
    const int64_t tid = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
    const int64_t nt = static_cast<int64_t>(gridDim.x) * blockDim.x;
    for (int64_t i = tid; i < len; i += nt)
        p[i] = __float2bfloat16_rn(__fmul_rn(__bfloat162float(p[i]), alpha));
}
}  // namespace

}  // namespace tag

using namespace tag;

struct tag_comm_s {
    ncclComm_t nccl = nullptr;   // nullptr for a plain one-rank comm (no collective at all)
    int nranks = 1, rank = 0, device = 0;
    void* devcomm = nullptr;     // ncclDevComm (device API: LSA pointers + barriers), or nullptr
    bool lsa_all = false;        // every rank is load/store reachable (one NVLink domain)
    void* mc_base = nullptr;     // NVLS multicast base of the LSA team (multimem stores), or null
};

struct tag_plan_s {
    tag_comm_s* comm = nullptr;
    tag_sfb_desc_t d{};
    int64_t K = 0;
    float alpha = 0.f;             // fl32(1/(nB))
    bool use_tc = false;           // tensor-core reconstruction (else SIMT FFMA)
    void* gx = nullptr;            // gathered X_all  (K x M, wire dtype)   [NCCL gather mode]
    void* gdy = nullptr;           // gathered dY_all (K x N, wire dtype)
    int gather_mode = TAG_GATHER_NONE;
    // NVLink push mode: double-buffered [X_all | dY_all] in an NCCL symmetric window
    void* win_base = nullptr;
    ncclWindow_t win = nullptr;
    // window layout [X buf 0 | X buf 1 | dY buf 0 | dY buf 1 | flags]: each buffer win_kbuf rows
    // (K rounded up to 128, the rows beyond K stay zero: the TMA boxes of the last K block read
    // zeros, and one tensor map covers both buffers)
    int64_t win_kbuf = 0;
    size_t win_xbuf = 0;           // bytes of one X buffer = win_kbuf * M * e_w
    size_t win_ybuf = 0;           // bytes of one dY buffer = win_kbuf * N * e_w
    size_t win_flag_off = 0;       // the window flag area (WIN_* offsets, tag_internal.h)
    uint32_t* flags = nullptr;     // the same area, this rank's device address
    void* lx = nullptr;            // local cast scratch for tag_local_grad (B x M, B x N wire)
    void* ldy = nullptr;
    const void* src_x = nullptr;   // operands of the next reconstruct (set by gather); for the
    const void* src_dy = nullptr;  // window: buffer 0, with buffer 1 and the call counter below
    const void* src_x1 = nullptr;  // (the buffer of the latest gather is read on the device)
    const void* src_dy1 = nullptr;
    const uint32_t* src_ctr = nullptr;
    ncclRedOp_t premul{};
    bool has_premul = false;
    // device staging of tag_sfb_sync_host (allocated on first use)
    void* st_x = nullptr;
    void* st_dy = nullptr;
    void* st_dw = nullptr;
    // fp32 wire on the tensor cores (3xTF32): split [hi ; lo] operands, kpad rows per half
    void* split = nullptr;
    int64_t kpad = 0;
    // Adam on a path without the fused epilogue: dW staged here, then the unfused Adam kernel
    float* adam_dw = nullptr;
    // the reconstruction kernel's dynamic tile-schedule counters (recon_tc.cu), zeroed once
    uint32_t* sched = nullptr;
};

struct tag_group_s {
    std::vector<tag_plan_s*> plans;
    bool push_all = false;     // every plan gathers by NVLink push -> one grouped push kernel
    bool tc_all = false;       // every plan reconstructs on the tensor cores -> one launch
};

namespace {

ncclDataType_t nccl_type(tag_dtype_t t) { return t == TAG_F32 ? ncclFloat32 : ncclBfloat16; }

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

tag_status_t set_device(tag_comm_s* c) {
    cudaError_t e = cudaSetDevice(c->device);
    return e == cudaSuccess ? TAG_OK : cuda_fail(e, "cudaSetDevice");
}

tag_status_t check_async(tag_comm_s* c) {
    if (!c->nccl) return TAG_OK;
    ncclResult_t ar = ncclSuccess;
    ncclResult_t r = ncclCommGetAsyncError(c->nccl, &ar);
    if (r != ncclSuccess) return nccl_fail(r, "ncclCommGetAsyncError");
    if (ar != ncclSuccess && ar != ncclInProgress)
        return fail(TAG_ERR_ASYNC, std::string("asynchronous NCCL error: ") + ncclGetErrorString(ar));
    return TAG_OK;
}

#define TAG_TRY(expr)                         \
    do {                                      \
        tag_status_t _st = (expr);            \
        if (_st != TAG_OK) return _st;        \
    } while (0)

tag_status_t validate_desc(const tag_comm_s* c, const tag_sfb_desc_t* d) {
    if (d->M < 1 || d->N < 1 || d->B < 1)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_plan: M, N, B must be >= 1");
    if (d->n != c->nranks)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_plan: desc.n must equal the comm size");
    if (d->M > INT32_MAX || d->N > INT32_MAX || static_cast<int64_t>(d->n) * d->B > INT32_MAX)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_plan: M, N and n*B must fit in int32");
    auto okdt = [](tag_dtype_t t) { return t == TAG_F32 || t == TAG_BF16; };
    if (!okdt(d->in_dtype) || !okdt(d->wire_dtype) || !okdt(d->out_dtype))
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_plan: unknown dtype");
    if (d->in_dtype == TAG_BF16 && d->wire_dtype == TAG_F32)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_plan: bf16 -> fp32 wire is not a supported pair");
    if (d->fuse_sgd != 0 && d->fuse_sgd != 1)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_plan: fuse_sgd must be 0 or 1");
    if (d->fuse_adam != 0 && d->fuse_adam != 1)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_plan: fuse_adam must be 0 or 1");
    if (d->fuse_adam && d->fuse_sgd)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_plan: fuse_sgd and fuse_adam are exclusive");
    if (d->fuse_adam && !(std::isfinite(d->lr) && std::isfinite(d->weight_decay) &&
                          d->beta1 >= 0.f && d->beta1 < 1.f && d->beta2 >= 0.f && d->beta2 < 1.f &&
                          d->eps > 0.f && std::isfinite(d->eps)))
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_plan: Adam needs finite lr / wd, betas in [0, 1), eps > 0");
    if (d->fuse_adam && d->out_dtype != TAG_F32)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_plan: fuse_adam needs out_dtype = F32");
    if (d->fuse_sgd && !(std::isfinite(d->lr) && std::isfinite(d->momentum) &&
                         std::isfinite(d->weight_decay)))
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_plan: non-finite SGD hyper-parameter");
    if (d->gather != TAG_GATHER_REQ_AUTO && d->gather != TAG_GATHER_REQ_NCCL &&
        d->gather != TAG_GATHER_REQ_PUSH)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_plan: unknown gather request");
    return TAG_OK;
}

tag_status_t check_ptrs(const char* fn, std::initializer_list<const void*> ps) {
    for (const void* p : ps) {
        if (!p) return fail(TAG_ERR_INVALID_ARG, std::string(fn) + ": NULL pointer");
        if (!aligned16(p)) return fail(TAG_ERR_INVALID_ARG, std::string(fn) + ": pointer not 16-byte aligned");
    }
    return TAG_OK;
}

// a plan on a communicator with NCCL (n > 1, or a one-rank loopback comm) exchanges its factors
bool has_collective(const tag_comm_s* c) { return c->nccl != nullptr; }

bool needs_gather_buffers(const tag_comm_s* c, const tag_sfb_desc_t& d) {
    return has_collective(c) || d.in_dtype != d.wire_dtype;
}

// The reconstruction operands of a plan: a plain buffer pair, or the symmetric window's two
// buffers with its call counter (which buffer the latest gather filled is device state).
void set_src_plain(tag_plan_s* p, const void* x, const void* dy) {
    p->src_x = x;
    p->src_dy = dy;
    p->src_x1 = p->src_dy1 = nullptr;
    p->src_ctr = nullptr;
}

size_t win_off_dy(const tag_plan_s* p) { return 2 * p->win_xbuf; }

void set_src_window(tag_plan_s* p) {
    char* w = static_cast<char*>(p->win_base);
    p->src_x = w;
    p->src_x1 = w + p->win_xbuf;
    p->src_dy = w + win_off_dy(p);
    p->src_dy1 = w + win_off_dy(p) + p->win_ybuf;
    p->src_ctr = p->flags + WIN_CALLS / 4;
}

// a's operands from the plan's latest gather; columns col0.. of X_all (sharded rows of dW)
void fill_src(const tag_plan_s* p, ReconArgs& a, int64_t col0 = 0) {
    const size_t xo = static_cast<size_t>(col0) * dtype_size(p->d.wire_dtype);
    a.sched = p->sched;
    a.A = static_cast<const char*>(p->src_x) + xo;
    a.Bm = p->src_dy;
    if (p->src_ctr) {
        a.A1 = static_cast<const char*>(p->src_x1) + xo;
        a.Bm1 = p->src_dy1;
        a.kbuf = p->win_kbuf;
        a.ctr = p->src_ctr;
        a.ctr_mode = 1;
    }
}

PushSegment push_segment(const tag_plan_s* p, const void* X, const void* dY) {
    return PushSegment{X, dY, p->win, 0, win_off_dy(p), p->win_xbuf, p->win_ybuf, p->win_flag_off,
                       p->flags, p->d.B * p->d.M, p->d.B * p->d.N};
}

// Every rank's device work up to here is complete and every rank has reached this point: the
// window of a new plan is zeroed everywhere before any peer can push into it (a late memset
// would wipe a peer's factors and arrival counters), and on destroy no peer still writes into
// a window that is about to be freed.
tag_status_t quiesce_all_ranks(tag_comm_s* c, const char* where) {
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) return cuda_fail(e, where);
    if (c->devcomm && c->lsa_all) {
        TAG_TRY(launch_comm_barrier(c->devcomm, COMM_BARRIER_INDEX, nullptr));
        e = cudaDeviceSynchronize();
        if (e != cudaSuccess) return cuda_fail(e, where);
    }
    return TAG_OK;
}

// a1 + a2: leaves the operands of the reconstruction in plan->src_x / src_dy
tag_status_t do_gather(tag_plan_s* p, const void* X, const void* dY, cudaStream_t s) {
    const tag_sfb_desc_t& d = p->d;
    const int64_t cx = d.B * d.M, cy = d.B * d.N;          // elements per replica
    const size_t ew = dtype_size(d.wire_dtype);
    if (!has_collective(p->comm)) {
        if (d.in_dtype == d.wire_dtype) {
            set_src_plain(p, X, dY);
            return TAG_OK;
        }
        TAG_TRY(launch_pack(X, p->gx, cx, dY, p->gdy, cy, d.in_dtype, d.wire_dtype, s));
        set_src_plain(p, p->gx, p->gdy);
        return TAG_OK;
    }
    const int r = p->comm->rank;
    if (p->gather_mode == TAG_GATHER_NVLINK_PUSH) {
        // a1 + a2 fused: cast and store straight into every peer's window (push_gather.cu); the
        // kernel picks the buffer from the window's call counter and advances it
        PushSegment seg = push_segment(p, X, dY);
        TAG_TRY(launch_push_gather_group(p->comm->devcomm, &seg, 1, r, d.in_dtype, d.wire_dtype,
                                         EXP_PUSH_GRID, p->flags + WIN_LOCAL_PUSH / 4, s));
        set_src_window(p);
        return TAG_OK;
    }
    char* gx = static_cast<char*>(p->gx);
    char* gdy = static_cast<char*>(p->gdy);
    const void* sx = X;
    const void* sdy = dY;
    if (d.in_dtype != d.wire_dtype) {
        // a1: cast into this rank's slot, then gather in place
        sx = gx + r * cx * ew;
        sdy = gdy + r * cy * ew;
        TAG_TRY(launch_pack(X, const_cast<void*>(sx), cx, dY, const_cast<void*>(sdy), cy,
                            d.in_dtype, d.wire_dtype, s));
    }
    // a2: "broadcast to all devices" = all-gather of both factors, rank-major (R12).
    // Same dtype: NCCL reads the caller's buffers directly (no pack pass over HBM).
    const ncclDataType_t t = nccl_type(d.wire_dtype);
    ncclResult_t nr = ncclGroupStart();
    if (nr == ncclSuccess) nr = ncclAllGather(sx, gx, static_cast<size_t>(cx), t, p->comm->nccl, s);
    if (nr == ncclSuccess) nr = ncclAllGather(sdy, gdy, static_cast<size_t>(cy), t, p->comm->nccl, s);
    ncclResult_t ne = ncclGroupEnd();
    if (nr != ncclSuccess) return nccl_fail(nr, "ncclAllGather");
    if (ne != ncclSuccess) return nccl_fail(ne, "ncclGroupEnd");
    set_src_plain(p, p->gx, p->gdy);
    return TAG_OK;
}

// Per-call Adam constants (R22), computed in double and rounded once, shared by the fused
// epilogue and the unfused kernel.
struct AdamCall {
    float b1, omb1, b2, omb2, eps, lr_t, isbc2;
};

AdamCall adam_call(const tag_sfb_desc_t& d, int64_t step) {
    const double b1 = d.beta1, b2 = d.beta2;
    const double bc1 = 1.0 - std::pow(b1, static_cast<double>(step));
    const double bc2 = 1.0 - std::pow(b2, static_cast<double>(step));
    return AdamCall{d.beta1, static_cast<float>(1.0 - b1), d.beta2, static_cast<float>(1.0 - b2),
                    d.eps, static_cast<float>(static_cast<double>(d.lr) / bc1),
                    static_cast<float>(1.0 / std::sqrt(bc2))};
}

void set_adam(ReconArgs& a, float* Mm, const AdamCall* ad) {
    a.opt = ad ? 2 : 1;
    a.Mm = Mm;
    if (ad) {
        a.b1 = ad->b1;
        a.omb1 = ad->omb1;
        a.b2 = ad->b2;
        a.omb2 = ad->omb2;
        a.eps = ad->eps;
        a.lr_t = ad->lr_t;
        a.isbc2 = ad->isbc2;
    }
}

tag_status_t do_recon(tag_plan_s* p, void* dW, bool sgd, float* W, float* V, int64_t K,
                      float alpha, cudaStream_t s, float* Mm = nullptr,
                      const AdamCall* adam = nullptr) {
    if (!p->src_x) return fail(TAG_ERR_INVALID_ARG, "reconstruct: no factors gathered on this plan yet");
    ReconArgs a{};
    fill_src(p, a);
    a.C = dW;
    a.M = p->d.M;
    a.N = p->d.N;
    a.K = K;
    a.wire = p->d.wire_dtype;
    a.out = p->d.out_dtype;
    a.alpha = alpha;
    a.sgd = sgd;
    a.W = W;
    a.V = V;
    a.lr = p->d.lr;
    a.mu = p->d.momentum;
    a.wd = p->d.weight_decay;
    if (sgd) set_adam(a, Mm, adam);
    if (p->use_tc && p->d.wire_dtype == TAG_F32) {
        // 3xTF32: split both operands into [hi ; lo] halves of kp rows (pack_sgd.cu), then the
        // kind::tf32 variant of the tensor-core kernel
        const int64_t kp = (K + TF32_KALIGN - 1) / TF32_KALIGN * TF32_KALIGN;
        float* sx = static_cast<float*>(p->split);
        float* sdy = sx + 2 * kp * p->d.M;
        TAG_TRY(launch_tf32_split(static_cast<const float*>(a.A), static_cast<const float*>(a.A1),
                                  a.ctr, sx, K, p->d.M, kp, s));
        TAG_TRY(launch_tf32_split(static_cast<const float*>(a.Bm), static_cast<const float*>(a.Bm1),
                                  a.ctr, sdy, K, p->d.N, kp, s));
        a.A = sx;
        a.Bm = sdy;
        a.A1 = a.Bm1 = nullptr;
        a.ctr = nullptr;
        a.ctr_mode = 0;
        a.kpad = kp;
    }
    if (p->use_tc && recon_tc_ok(a)) return launch_recon_tc(a, s);
    if (adam) {
        // the SIMT kernel has no Adam epilogue: reconstruct dW (into the caller's buffer or the
        // plan's staging), then the unfused Adam kernel — the same arithmetic (optim.cuh)
        float* dw = static_cast<float*>(dW);
        if (!dw) {
            if (!p->adam_dw) {       // first use, stream-ordered
                cudaError_t e = cudaMallocAsync(&p->adam_dw, static_cast<size_t>(p->d.M * p->d.N) * 4, s);
                if (e != cudaSuccess) {
                    p->adam_dw = nullptr;
                    return cuda_fail(e, "reconstruct: cudaMallocAsync(Adam staging)");
                }
            }
            dw = p->adam_dw;
        }
        a.C = dw;
        a.sgd = false;
        TAG_TRY(launch_recon_simt(a, s));
        return launch_adam(dw, W, Mm, V, p->d.M * p->d.N, adam->b1, adam->omb1, adam->b2,
                           adam->omb2, adam->eps, adam->lr_t, adam->isbc2, p->d.weight_decay, s);
    }
    return launch_recon_simt(a, s);
}

// Fused path (a1 + a2 + a3 + a4 in ONE kernel): every plan gathers by NVLink push without a cast
// and reconstructs on the tensor cores. The reconstruction kernel pushes this rank's factors
// into every peer's window and waits, per layer, on arrival counters before loading its tiles.
// The decision depends only on the plan's descriptor and the epilogue kind (every pointer has
// been validated 16-byte aligned before), so it is the same on every rank: a rank taking the
// fused kernel while a peer took the staged push would wait on a barrier nobody joins.
// opt: 0 = E1 (scale + store), 1 = fused SGD-momentum, 2 = fused Adam.
bool fusable(const tag_plan_s* p, void* dW, int opt = 0) {
    if (p->gather_mode != TAG_GATHER_NVLINK_PUSH || !p->use_tc) return false;
    if (p->d.wire_dtype != TAG_BF16) return false;           // 3xTF32 needs the split pass
    const bool same = p->d.in_dtype == p->d.wire_dtype;
    const bool cast = p->d.in_dtype == TAG_F32 && p->d.wire_dtype == TAG_BF16;
    if (!same && !cast) return false;
    if (EXP_NO_FUSE) return false;                           // diagnostics builds
    ReconArgs a{};
    a.A = p->win_base;
    a.Bm = p->win_base;
    a.C = dW;
    a.M = p->d.M;
    a.N = p->d.N;
    a.K = p->K;
    a.wire = p->d.wire_dtype;
    a.out = p->d.out_dtype;
    if (opt) {
        // the optimizer epilogues store fp32 dW only; a bf16-dW plan takes the staged path
        // whether or not this call passes dW_out (keeps the decision rank-independent)
        if (p->d.out_dtype != TAG_F32) return false;
        // W, v, m are caller pointers checked for alignment already; the window base stands in
        a.sgd = true;
        a.opt = opt;
        a.W = a.V = a.Mm = static_cast<float*>(p->win_base);
    }
    return recon_tc_ok(a);
}

void shard_range(const tag_plan_s* p, int rank, int64_t* begin, int64_t* cnt) {
    const int64_t n = p->d.n, M = p->d.M;
    const int64_t tiles = (M + 127) / 128;
    const int64_t per = (tiles + n - 1) / n;                 // 128-row tiles per rank
    const int64_t b = std::min(M, rank * per * 128);
    const int64_t e = std::min(M, (rank + 1) * per * 128);
    *begin = b;
    *cnt = e - b;
}

tag_status_t fused_sync(tag_plan_s* const* plans, int count, const void* const* X,
                        const void* const* dY, void* const* dW, bool sgd, float* const* W,
                        float* const* V, cudaStream_t s, bool sharded = false,
                        float* const* Mm = nullptr, const AdamCall* adam = nullptr) {
    tag_comm_s* c = plans[0]->comm;
    ReconArgs a[MAX_GROUP];
    for (int i = 0; i < count; ++i) {
        tag_plan_s* p = plans[i];
        const size_t ew = dtype_size(p->d.wire_dtype);
        // both buffers of the window: the kernel pushes into, waits on and reads buffer c & 1 of
        // the window's call counter c, and advances c (no per-call host state)
        char* w = static_cast<char*>(p->win_base);
        a[i] = ReconArgs{};
        a[i].A = w;
        a[i].Bm = w + win_off_dy(p);
        a[i].A1 = w + p->win_xbuf;
        a[i].Bm1 = w + win_off_dy(p) + p->win_ybuf;
        a[i].kbuf = p->win_kbuf;
        a[i].ctr = p->flags + WIN_CALLS / 4;
        a[i].ctr_mode = 2;
        // the dynamic tail schedule (recon_tc.cu): with only the tail's tiles passing through the
        // smem ring, n = 2 / 4 fused steps 100.4 / 115.7-116.2 vs 100.5-100.8 / 117.8 us static
        // (scripts/ab_fused_variants.sh)
        a[i].sched = p->sched;
        a[i].C = dW[i];
        a[i].M = p->d.M;
        a[i].N = p->d.N;
        a[i].K = p->K;
        a[i].wire = p->d.wire_dtype;
        a[i].out = p->d.out_dtype;
        a[i].alpha = p->alpha;
        a[i].sgd = sgd;
        a[i].W = sgd ? W[i] : nullptr;
        a[i].V = sgd ? V[i] : nullptr;
        a[i].lr = p->d.lr;
        a[i].mu = p->d.momentum;
        a[i].wd = p->d.weight_decay;
        if (sgd) set_adam(a[i], Mm ? Mm[i] : nullptr, adam);
        a[i].srcX = X[i];
        a[i].srcY = dY[i];
        a[i].win = p->win;
        a[i].off_x = 0;
        a[i].off_dy = win_off_dy(p);
        a[i].xbuf = p->win_xbuf;
        a[i].ybuf = p->win_ybuf;
        a[i].off_flag = p->win_flag_off;
        a[i].flags = p->flags;
        a[i].cx = p->d.B * p->d.M;
        a[i].cy = p->d.B * p->d.N;
        if (sharded) {
            int64_t rb, rc;
            shard_range(p, c->rank, &rb, &rc);
            a[i].A = static_cast<const char*>(a[i].A) + rb * ew;     // columns rb.. of X_all
            a[i].A1 = static_cast<const char*>(a[i].A1) + rb * ew;
            a[i].lda = p->d.M;
            a[i].M = rc;
        }
    }
    // hierarchical publish: the last CTA of every rank (plan 0's self-resetting local counter)
    // adds 1 per layer on every peer, so each arrival counter grows by exactly n per call
    // whatever grid each rank launched
    FusedGather fg{c->nranks, c->rank, c->mc_base,
                   plans[0]->d.in_dtype == TAG_F32 && plans[0]->d.wire_dtype == TAG_BF16,
                   plans[0]->flags + WIN_LOCAL_FUSED / 4};
    TAG_TRY(launch_recon_tc_group(a, count, s, &fg));
    for (int i = 0; i < count; ++i) set_src_window(plans[i]);
    return TAG_OK;
}

}  // namespace

extern "C" {

const char* tag_version(void) { return "libtag 0.1.0 (sm_100a)"; }

const char* tag_status_string(tag_status_t s) {
    switch (s) {
        case TAG_OK: return "TAG_OK";
        case TAG_ERR_INVALID_ARG: return "TAG_ERR_INVALID_ARG";
        case TAG_ERR_UNSUPPORTED: return "TAG_ERR_UNSUPPORTED";
        case TAG_ERR_CUDA: return "TAG_ERR_CUDA";
        case TAG_ERR_NCCL: return "TAG_ERR_NCCL";
        case TAG_ERR_OOM: return "TAG_ERR_OOM";
        case TAG_ERR_NOT_INITIALIZED: return "TAG_ERR_NOT_INITIALIZED";
        case TAG_ERR_ASYNC: return "TAG_ERR_ASYNC";
    }
    return "TAG_ERR_UNKNOWN";
}

const char* tag_last_error(void) { return t_last_error.c_str(); }

uint64_t tag_kernel_launches(void) { return g_launches.load(std::memory_order_relaxed); }

tag_status_t tag_get_unique_id(unsigned char id[128]) {
    if (!id) return fail(TAG_ERR_INVALID_ARG, "tag_get_unique_id: NULL id");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId u;
    ncclResult_t r = ncclGetUniqueId(&u);
    if (r != ncclSuccess) return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id, &u, 128);
    return TAG_OK;
}

tag_status_t tag_comm_create(const unsigned char id[128], int nranks, int rank, int cuda_device,
                             tag_comm_t* out) {
    return tag_comm_create_ex(id, nranks, rank, cuda_device, TAG_COMM_DEFAULT, out);
}

tag_status_t tag_comm_create_ex(const unsigned char id[128], int nranks, int rank, int cuda_device,
                                unsigned flags, tag_comm_t* out) {
    if (!out) return fail(TAG_ERR_INVALID_ARG, "tag_comm_create: NULL out");
    if (nranks < 1 || rank < 0 || rank >= nranks || cuda_device < 0)
        return fail(TAG_ERR_INVALID_ARG, "tag_comm_create: bad nranks/rank/device");
    if (flags & ~static_cast<unsigned>(TAG_COMM_NVLS_MULTICAST | TAG_COMM_LOOPBACK))
        return fail(TAG_ERR_INVALID_ARG, "tag_comm_create_ex: unknown flag");
    if (nranks > 1 && !id) return fail(TAG_ERR_INVALID_ARG, "tag_comm_create: NULL id");
    const bool loopback = nranks == 1 && (flags & TAG_COMM_LOOPBACK);
    int ndev = 0;
    cudaError_t e = cudaGetDeviceCount(&ndev);
    if (e != cudaSuccess) return cuda_fail(e, "cudaGetDeviceCount");
    if (cuda_device >= ndev) return fail(TAG_ERR_INVALID_ARG, "tag_comm_create: no such CUDA device");
    e = cudaSetDevice(cuda_device);
    if (e != cudaSuccess) return cuda_fail(e, "cudaSetDevice");
    tag_comm_s* c = new tag_comm_s;
    c->nranks = nranks;
    c->rank = rank;
    c->device = cuda_device;
    if (nranks > 1 || loopback) {
        ncclUniqueId u;
        ncclResult_t r = ncclSuccess;
        if (id) std::memcpy(&u, id, 128);
        else r = ncclGetUniqueId(&u);                       // loopback without an id
        if (r == ncclSuccess) r = ncclCommInitRank(&c->nccl, nranks, u, rank);
        if (r != ncclSuccess) {
            delete c;
            return nccl_fail(r, "ncclCommInitRank");
        }
        // device API for the NVLink push gather; without it plans use ncclAllGather
        if (push_devcomm_create(c->nccl, PUSH_MAX_CTAS + 1, (flags & TAG_COMM_NVLS_MULTICAST) != 0,
                                &c->devcomm) == TAG_OK) {
            c->lsa_all = push_devcomm_all_lsa(c->devcomm, nranks);
            c->mc_base = push_devcomm_mc_base(c->devcomm);
        } else {
            c->devcomm = nullptr;
        }
        set_error("");
    }
    *out = c;
    return TAG_OK;
}

tag_status_t tag_comm_destroy(tag_comm_t c) {
    if (!c) return TAG_OK;
    tag_status_t st = TAG_OK;
    if (c->nccl) {
        push_devcomm_destroy(c->nccl, c->devcomm);
        ncclResult_t r = ncclCommDestroy(c->nccl);
        if (r != ncclSuccess) st = nccl_fail(r, "ncclCommDestroy");
    }
    delete c;
    return st;
}

tag_status_t tag_comm_barrier(tag_comm_t c, tag_stream_t stream) {
    if (!c) return fail(TAG_ERR_INVALID_ARG, "tag_comm_barrier: NULL comm");
    if (!has_collective(c)) return TAG_OK;
    TAG_TRY(set_device(c));
    TAG_TRY(check_async(c));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (c->devcomm && c->lsa_all) return launch_comm_barrier(c->devcomm, COMM_BARRIER_INDEX, s);
    return fail(TAG_ERR_UNSUPPORTED, "tag_comm_barrier: needs every rank in one NVLink domain");
}

tag_status_t tag_comm_info(tag_comm_t c, int* nranks, int* rank, int* cuda_device) {
    if (!c) return fail(TAG_ERR_INVALID_ARG, "tag_comm_info: NULL comm");
    if (nranks) *nranks = c->nranks;
    if (rank) *rank = c->rank;
    if (cuda_device) *cuda_device = c->device;
    return TAG_OK;
}

tag_status_t tag_sfb_plan(tag_comm_t c, const tag_sfb_desc_t* d, tag_sfb_plan_t* out) {
    if (!c || !d || !out) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_plan: NULL argument");
    TAG_TRY(validate_desc(c, d));
    TAG_TRY(set_device(c));
    tag_plan_s* p = new tag_plan_s;
    p->comm = c;
    p->d = *d;
    p->K = static_cast<int64_t>(d->n) * d->B;
    p->alpha = static_cast<float>(1.0 / static_cast<double>(p->K));   // fl32(1/(nB)), R1
    // tensor cores need 16-byte factor rows: bf16 operands (kind::f16) or fp32 operands split
    // for 3xTF32 (kind::tf32, R10); other shapes take the SIMT FFMA kernel
    // (3xTF32 only up to K = 4096: the tensor core's accumulation error grows linearly with K —
    // 4.8e-6 relative at K = 2048, 1.9e-5 at 8192 — and the fp32 bar is 1e-5, DESIGN R10)
    p->use_tc = d->M % 8 == 0 && d->N % 8 == 0 &&
                (d->wire_dtype == TAG_BF16 ||
                 (!EXP_F32_SIMT && static_cast<int64_t>(d->n) * d->B <= 4096));
    auto cleanup = [p]() {
        cudaFree(p->split);
        cudaFree(p->sched);
        cudaFree(p->gx);
        cudaFree(p->gdy);
        cudaFree(p->lx);
        cudaFree(p->ldy);
        if (p->win) ncclCommWindowDeregister(p->comm->nccl, p->win);
        if (p->win_base) ncclMemFree(p->win_base);
        delete p;
    };
    const size_t ew = dtype_size(d->wire_dtype);
    if (has_collective(c)) {
        const bool rows16 = (d->B * d->M * static_cast<int64_t>(ew)) % 16 == 0 &&
                            (d->B * d->N * static_cast<int64_t>(ew)) % 16 == 0;
        const bool push_ok = c->devcomm && c->lsa_all && rows16;
        if (d->gather == TAG_GATHER_REQ_PUSH && !push_ok) {
            delete p;
            return fail(TAG_ERR_UNSUPPORTED, "tag_sfb_plan: NVLink push gather requested but not "
                                             "available (ranks not all NVLink load/store reachable, "
                                             "or factor rows not 16-byte multiples)");
        }
        p->gather_mode = (d->gather != TAG_GATHER_REQ_NCCL && push_ok) ? TAG_GATHER_NVLINK_PUSH
                                                                       : TAG_GATHER_NCCL;
    }
    if (p->gather_mode == TAG_GATHER_NVLINK_PUSH) {
        p->win_kbuf = (p->K + 127) / 128 * 128;
        p->win_xbuf = static_cast<size_t>(p->win_kbuf * d->M) * ew;
        p->win_ybuf = static_cast<size_t>(p->win_kbuf * d->N) * ew;
        p->win_flag_off = (2 * (p->win_xbuf + p->win_ybuf) + 255) & ~static_cast<size_t>(255);
        size_t bytes = p->win_flag_off + 256;
        bytes = (bytes + 4095) & ~static_cast<size_t>(4095);      // NCCL_WIN_REQUIRED_ALIGNMENT
        ncclResult_t r = ncclMemAlloc(&p->win_base, bytes);
        if (r == ncclSuccess)
            r = ncclCommWindowRegister(c->nccl, p->win_base, bytes, &p->win, NCCL_WIN_COLL_SYMMETRIC);
        if (r != ncclSuccess) {
            cleanup();
            return nccl_fail(r, "tag_sfb_plan: symmetric gather window");
        }
        p->flags = reinterpret_cast<uint32_t*>(static_cast<char*>(p->win_base) + p->win_flag_off);
        // deterministic initial contents (every slot is overwritten by its owner before use); the
        // call counter and the arrival / local counters start at 0
        cudaError_t e = cudaMemset(p->win_base, 0, bytes);
        if (e != cudaSuccess) {
            cleanup();
            return cuda_fail(e, "tag_sfb_plan: cudaMemset(window)");
        }
        // the zeroed window and arrival counters must exist on EVERY rank before any rank pushes
        tag_status_t qs = quiesce_all_ranks(c, "tag_sfb_plan: window initialisation");
        if (qs != TAG_OK) {
            cleanup();
            return qs;
        }
        if (d->in_dtype != d->wire_dtype) {
            e = cudaMalloc(&p->lx, static_cast<size_t>(d->B * d->M) * ew);
            if (e == cudaSuccess) e = cudaMalloc(&p->ldy, static_cast<size_t>(d->B * d->N) * ew);
            if (e != cudaSuccess) {
                cleanup();
                return cuda_fail(e, "tag_sfb_plan: cudaMalloc(local scratch)");
            }
        }
    } else if (needs_gather_buffers(c, *d)) {
        cudaError_t e = cudaMalloc(&p->gx, static_cast<size_t>(p->K * d->M) * ew);
        if (e == cudaSuccess) e = cudaMalloc(&p->gdy, static_cast<size_t>(p->K * d->N) * ew);
        if (e != cudaSuccess) {
            cleanup();
            return cuda_fail(e, "tag_sfb_plan: cudaMalloc(gather buffers)");
        }
    }
    if (p->use_tc) {
        cudaError_t e = cudaMalloc(&p->sched, 64);
        if (e == cudaSuccess) e = cudaMemset(p->sched, 0, 64);
        if (e != cudaSuccess) {
            cleanup();
            return cuda_fail(e, "tag_sfb_plan: cudaMalloc(tile schedule counters)");
        }
    }
    if (p->use_tc && d->wire_dtype == TAG_F32) {
        p->kpad = (p->K + TF32_KALIGN - 1) / TF32_KALIGN * TF32_KALIGN;
        cudaError_t e = cudaMalloc(&p->split, static_cast<size_t>(2 * p->kpad * (d->M + d->N)) * 4);
        if (e != cudaSuccess) {
            cleanup();
            return cuda_fail(e, "tag_sfb_plan: cudaMalloc(3xTF32 split operands)");
        }
    }
    if (c->nccl) {
        // dense baseline: the 1/(nB) scale rides inside the AllReduce (PreMulSum)
        ncclResult_t r;
        if (d->out_dtype == TAG_F32) {
            float a = p->alpha;
            r = ncclRedOpCreatePreMulSum(&p->premul, &a, ncclFloat32, ncclScalarHostImmediate, c->nccl);
        } else {
            __nv_bfloat16 a = __float2bfloat16_rn(p->alpha);
            r = ncclRedOpCreatePreMulSum(&p->premul, &a, ncclBfloat16, ncclScalarHostImmediate, c->nccl);
        }
        if (r != ncclSuccess) {
            cleanup();
            return nccl_fail(r, "ncclRedOpCreatePreMulSum");
        }
        p->has_premul = true;
    }
    *out = p;
    return TAG_OK;
}

tag_status_t tag_sfb_plan_info(tag_sfb_plan_t p, tag_plan_info_t* out) {
    if (!p || !out) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_plan_info: NULL argument");
    out->tensor_cores = p->use_tc ? 1 : 0;
    out->gather_mode = p->gather_mode;
    out->K = p->K;
    out->alpha = p->alpha;
    out->multicast = (p->gather_mode == TAG_GATHER_NVLINK_PUSH && p->comm->mc_base) ? 1 : 0;
    out->recon_bn = out->recon_ctas = out->recon_box3d = 0;
    if (p->use_tc) {
        ReconArgs a{};
        a.M = p->d.M;
        a.N = p->d.N;
        a.K = p->K;
        a.wire = p->d.wire_dtype;
        a.out = p->d.out_dtype;
        a.sgd = p->d.fuse_sgd || p->d.fuse_adam;   // the optimizer epilogue's tile rule
        recon_tc_describe(&a, 1, &out->recon_bn, &out->recon_ctas, &out->recon_box3d);
    }
    return TAG_OK;
}

tag_status_t tag_sfb_plan_destroy(tag_sfb_plan_t p) {
    if (!p) return TAG_OK;
    set_device(p->comm);
    if (p->win) quiesce_all_ranks(p->comm, "tag_sfb_plan_destroy");   // no peer writes in flight
    cudaFree(p->adam_dw);
    if (p->has_premul) ncclRedOpDestroy(p->premul, p->comm->nccl);
    if (p->win) ncclCommWindowDeregister(p->comm->nccl, p->win);
    if (p->win_base) ncclMemFree(p->win_base);
    cudaFree(p->lx);
    cudaFree(p->ldy);
    cudaFree(p->gx);
    cudaFree(p->gdy);
    cudaFree(p->st_x);
    cudaFree(p->st_dy);
    cudaFree(p->st_dw);
    cudaFree(p->split);
    cudaFree(p->sched);
    delete p;
    return TAG_OK;
}

tag_status_t tag_sfb_gather(tag_sfb_plan_t p, const void* X, const void* dY, tag_stream_t stream) {
    if (!p) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_gather: NULL plan");
    TAG_TRY(check_ptrs("tag_sfb_gather", {X, dY}));
    TAG_TRY(set_device(p->comm));
    TAG_TRY(check_async(p->comm));
    return do_gather(p, X, dY, reinterpret_cast<cudaStream_t>(stream));
}

tag_status_t tag_sfb_reconstruct(tag_sfb_plan_t p, void* dW_out, tag_stream_t stream) {
    if (!p) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_reconstruct: NULL plan");
    TAG_TRY(check_ptrs("tag_sfb_reconstruct", {dW_out}));
    TAG_TRY(set_device(p->comm));
    return do_recon(p, dW_out, false, nullptr, nullptr, p->K, p->alpha,
                    reinterpret_cast<cudaStream_t>(stream));
}

tag_status_t tag_sfb_sync(tag_sfb_plan_t p, const void* X, const void* dY, void* dW_out,
                          tag_stream_t stream) {
    if (!p) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_sync: NULL plan");
    TAG_TRY(check_ptrs("tag_sfb_sync", {X, dY, dW_out}));
    TAG_TRY(set_device(p->comm));
    TAG_TRY(check_async(p->comm));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (fusable(p, dW_out)) return fused_sync(&p, 1, &X, &dY, &dW_out, false, nullptr, nullptr, s);
    TAG_TRY(do_gather(p, X, dY, s));
    return do_recon(p, dW_out, false, nullptr, nullptr, p->K, p->alpha, s);
}

tag_status_t tag_sfb_sync_sgd(tag_sfb_plan_t p, const void* X, const void* dY, float* W, float* v,
                              void* dW_out, tag_stream_t stream) {
    if (!p) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_sync_sgd: NULL plan");
    if (!p->d.fuse_sgd) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_sync_sgd: plan has fuse_sgd = 0");
    TAG_TRY(check_ptrs("tag_sfb_sync_sgd", {X, dY, W, v}));
    if (dW_out) TAG_TRY(check_ptrs("tag_sfb_sync_sgd", {dW_out}));
    TAG_TRY(set_device(p->comm));
    TAG_TRY(check_async(p->comm));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (fusable(p, dW_out, 1)) return fused_sync(&p, 1, &X, &dY, &dW_out, true, &W, &v, s);
    TAG_TRY(do_gather(p, X, dY, s));
    return do_recon(p, dW_out, true, W, v, p->K, p->alpha, s);
}

tag_status_t tag_sfb_sync_adam(tag_sfb_plan_t p, const void* X, const void* dY, float* W, float* m,
                               float* v, int64_t step, void* dW_out, tag_stream_t stream) {
    if (!p) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_sync_adam: NULL plan");
    if (!p->d.fuse_adam) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_sync_adam: plan has fuse_adam = 0");
    if (step < 1) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_sync_adam: step must be >= 1");
    TAG_TRY(check_ptrs("tag_sfb_sync_adam", {X, dY, W, m, v}));
    if (dW_out) TAG_TRY(check_ptrs("tag_sfb_sync_adam", {dW_out}));
    TAG_TRY(set_device(p->comm));
    TAG_TRY(check_async(p->comm));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const AdamCall ad = adam_call(p->d, step);
    if (fusable(p, dW_out, 2)) return fused_sync(&p, 1, &X, &dY, &dW_out, true, &W, &v, s, false, &m, &ad);
    TAG_TRY(do_gather(p, X, dY, s));
    return do_recon(p, dW_out, true, W, v, p->K, p->alpha, s, m, &ad);
}

tag_status_t tag_adam_step(tag_sfb_plan_t p, const float* dW, float* W, float* m, float* v,
                           int64_t step, tag_stream_t stream) {
    if (!p) return fail(TAG_ERR_INVALID_ARG, "tag_adam_step: NULL plan");
    if (step < 1) return fail(TAG_ERR_INVALID_ARG, "tag_adam_step: step must be >= 1");
    if (!(p->d.beta1 >= 0.f && p->d.beta1 < 1.f && p->d.beta2 >= 0.f && p->d.beta2 < 1.f &&
          p->d.eps > 0.f))
        return fail(TAG_ERR_INVALID_ARG, "tag_adam_step: the plan's Adam hyper-parameters are unset");
    TAG_TRY(check_ptrs("tag_adam_step", {dW, W, m, v}));
    TAG_TRY(set_device(p->comm));
    const AdamCall ad = adam_call(p->d, step);
    return launch_adam(dW, W, m, v, p->d.M * p->d.N, ad.b1, ad.omb1, ad.b2, ad.omb2, ad.eps,
                       ad.lr_t, ad.isbc2, p->d.weight_decay, reinterpret_cast<cudaStream_t>(stream));
}

tag_status_t tag_sfb_bias_grad(tag_sfb_plan_t p, void* db_out, tag_stream_t stream) {
    if (!p || !db_out) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_bias_grad: NULL argument");
    if (!p->src_dy) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_bias_grad: no factors gathered on this plan yet");
    TAG_TRY(set_device(p->comm));
    BiasArgs a{p->src_dy, p->src_dy1, p->src_ctr, db_out, p->K, p->d.N, p->d.wire_dtype,
               p->d.out_dtype, p->alpha};
    return launch_bias_grad(&a, 1, reinterpret_cast<cudaStream_t>(stream));
}

tag_status_t tag_sfb_shard_rows(tag_sfb_plan_t p, int rank, int64_t* row_begin, int64_t* row_count) {
    if (!p || !row_begin || !row_count) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_shard_rows: NULL argument");
    if (rank < 0 || rank >= p->d.n) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_shard_rows: bad rank");
    shard_range(p, rank, row_begin, row_count);
    return TAG_OK;
}

tag_status_t tag_sfb_sync_sharded(tag_sfb_plan_t p, const void* X, const void* dY, void* dW_shard,
                                  tag_stream_t stream) {
    if (!p) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_sync_sharded: NULL plan");
    int64_t rb, rc;
    shard_range(p, p->comm->rank, &rb, &rc);
    TAG_TRY(check_ptrs("tag_sfb_sync_sharded", {X, dY}));
    if (rc > 0) TAG_TRY(check_ptrs("tag_sfb_sync_sharded", {dW_shard}));
    TAG_TRY(set_device(p->comm));
    TAG_TRY(check_async(p->comm));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    // the same route on every rank: a rank with an empty shard still launches the fused kernel
    // (one push-only CTA), since its peers wait for its factors
    if (fusable(p, rc > 0 ? dW_shard : nullptr))
        return fused_sync(&p, 1, &X, &dY, &dW_shard, false, nullptr, nullptr, s, true);
    TAG_TRY(do_gather(p, X, dY, s));
    if (rc == 0) return TAG_OK;
    ReconArgs a{};
    fill_src(p, a, rb);
    a.C = dW_shard;
    a.M = rc;
    a.N = p->d.N;
    a.K = p->K;
    a.lda = p->d.M;
    a.wire = p->d.wire_dtype;
    a.out = p->d.out_dtype;
    a.alpha = p->alpha;
    return (p->use_tc && recon_tc_ok(a)) ? launch_recon_tc(a, s) : launch_recon_simt(a, s);
}

// Parameter all-gather of the sharded optimizer step: rank r's rows [rb_r, rb_r + rc_r) of W
// reach every rank. Equal shards: one in-place ncclAllGather; otherwise one ncclBroadcast per
// non-empty shard in a group. n = 1 / no collective: nothing to do.
tag_status_t allgather_rows(tag_plan_s* p, float* W, cudaStream_t s) {
    tag_comm_s* c = p->comm;
    if (!has_collective(c) || c->nranks == 1) return TAG_OK;
    const int64_t N = p->d.N;
    int64_t rb0, rc0;
    shard_range(p, 0, &rb0, &rc0);
    bool equal = true;
    for (int r = 0; r < c->nranks; ++r) {
        int64_t rb, rc;
        shard_range(p, r, &rb, &rc);
        equal = equal && rc == rc0 && rb == r * rc0;
    }
    ncclResult_t r = ncclSuccess;
    if (equal) {
        r = ncclAllGather(W + static_cast<size_t>(c->rank) * rc0 * N, W, static_cast<size_t>(rc0 * N),
                          ncclFloat32, c->nccl, s);
        return r == ncclSuccess ? TAG_OK : nccl_fail(r, "ncclAllGather(W shards)");
    }
    r = ncclGroupStart();
    for (int q = 0; q < c->nranks && r == ncclSuccess; ++q) {
        int64_t rb, rc;
        shard_range(p, q, &rb, &rc);
        if (rc == 0) continue;
        r = ncclBroadcast(W + rb * N, W + rb * N, static_cast<size_t>(rc * N), ncclFloat32, q,
                          c->nccl, s);
    }
    ncclResult_t e = ncclGroupEnd();
    if (r != ncclSuccess) return nccl_fail(r, "ncclBroadcast(W shard)");
    return e == ncclSuccess ? TAG_OK : nccl_fail(e, "ncclGroupEnd");
}

// The sharded optimizer step (f-2, R24) for SGD-momentum (adam == nullptr) or Adam: this rank's
// rows of W with its optimizer-state rows, then the W all-gather.
static tag_status_t sharded_opt(tag_sfb_plan_t p, const void* X, const void* dY, float* W,
                                float* m_shard, float* v_shard, const AdamCall* adam,
                                tag_stream_t stream, const char* fn) {
    if (p->d.out_dtype != TAG_F32) return fail(TAG_ERR_INVALID_ARG, std::string(fn) + ": needs out_dtype = F32");
    int64_t rb, rc;
    shard_range(p, p->comm->rank, &rb, &rc);
    TAG_TRY(check_ptrs(fn, {X, dY, W}));
    if (rc > 0) TAG_TRY(check_ptrs(fn, {v_shard}));
    if (rc > 0 && adam) TAG_TRY(check_ptrs(fn, {m_shard}));
    TAG_TRY(set_device(p->comm));
    TAG_TRY(check_async(p->comm));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    float* Ws = W + rb * p->d.N;               // this rank's rows of W (rb is a multiple of 128)
    void* none = nullptr;
    if (fusable(p, nullptr, adam ? 2 : 1)) {
        // one fused launch: push, reconstruct this rank's rows, the optimizer on them
        TAG_TRY(fused_sync(&p, 1, &X, &dY, &none, true, &Ws, &v_shard, s, true, &m_shard, adam));
    } else {
        TAG_TRY(do_gather(p, X, dY, s));
        if (rc > 0) {
            ReconArgs a{};
            fill_src(p, a, rb);
            a.C = nullptr;
            a.M = rc;
            a.N = p->d.N;
            a.K = p->K;
            a.lda = p->d.M;
            a.wire = p->d.wire_dtype;
            a.out = p->d.out_dtype;
            a.alpha = p->alpha;
            a.sgd = true;
            a.W = Ws;
            a.V = v_shard;
            a.lr = p->d.lr;
            a.mu = p->d.momentum;
            a.wd = p->d.weight_decay;
            set_adam(a, m_shard, adam);
            if (p->use_tc && recon_tc_ok(a)) {
                TAG_TRY(launch_recon_tc(a, s));
            } else if (!adam) {
                TAG_TRY(launch_recon_simt(a, s));
            } else {
                // the SIMT kernel has no Adam epilogue: the shard's dW into the plan's staging,
                // then the unfused Adam kernel on the shard (the same arithmetic, optim.cuh)
                if (!p->adam_dw) {
                    cudaError_t e = cudaMallocAsync(&p->adam_dw, static_cast<size_t>(p->d.M * p->d.N) * 4, s);
                    if (e != cudaSuccess) {
                        p->adam_dw = nullptr;
                        return cuda_fail(e, "cudaMallocAsync(Adam staging)");
                    }
                }
                a.C = p->adam_dw;
                a.sgd = false;
                TAG_TRY(launch_recon_simt(a, s));
                TAG_TRY(launch_adam(p->adam_dw, Ws, m_shard, v_shard, rc * p->d.N, adam->b1, adam->omb1,
                                    adam->b2, adam->omb2, adam->eps, adam->lr_t, adam->isbc2,
                                    p->d.weight_decay, s));
            }
        }
    }
    // parameter all-gather: every rank ends with the whole updated W (ZeRO-style)
    return allgather_rows(p, W, s);
}

tag_status_t tag_sfb_sync_sharded_sgd(tag_sfb_plan_t p, const void* X, const void* dY, float* W,
                                      float* v_shard, tag_stream_t stream) {
    if (!p) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_sync_sharded_sgd: NULL plan");
    if (!p->d.fuse_sgd) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_sync_sharded_sgd: plan has fuse_sgd = 0");
    return sharded_opt(p, X, dY, W, nullptr, v_shard, nullptr, stream, "tag_sfb_sync_sharded_sgd");
}

tag_status_t tag_sfb_sync_sharded_adam(tag_sfb_plan_t p, const void* X, const void* dY, float* W,
                                       float* m_shard, float* v_shard, int64_t step,
                                       tag_stream_t stream) {
    if (!p) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_sync_sharded_adam: NULL plan");
    if (!p->d.fuse_adam) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_sync_sharded_adam: plan has fuse_adam = 0");
    if (step < 1) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_sync_sharded_adam: step must be >= 1");
    const AdamCall ad = adam_call(p->d, step);
    return sharded_opt(p, X, dY, W, m_shard, v_shard, &ad, stream, "tag_sfb_sync_sharded_adam");
}

tag_status_t tag_sfb_sync_host(tag_sfb_plan_t p, const void* X_host, const void* dY_host,
                               void* dW_host, tag_stream_t stream) {
    if (!p) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_sync_host: NULL plan");
    if (!X_host || !dY_host || !dW_host) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_sync_host: NULL pointer");
    TAG_TRY(set_device(p->comm));
    TAG_TRY(check_async(p->comm));
    const tag_sfb_desc_t& d = p->d;
    const size_t bx = static_cast<size_t>(d.B * d.M) * dtype_size(d.in_dtype);
    const size_t bdy = static_cast<size_t>(d.B * d.N) * dtype_size(d.in_dtype);
    const size_t bdw = static_cast<size_t>(d.M * d.N) * dtype_size(d.out_dtype);
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (!p->st_x) {
        // device staging on first use, stream-ordered (no device-wide synchronisation)
        cudaError_t e = cudaMallocAsync(&p->st_x, bx, s);
        if (e == cudaSuccess) e = cudaMallocAsync(&p->st_dy, bdy, s);
        if (e == cudaSuccess) e = cudaMallocAsync(&p->st_dw, bdw, s);
        if (e != cudaSuccess) {
            if (p->st_x) cudaFreeAsync(p->st_x, s);
            if (p->st_dy) cudaFreeAsync(p->st_dy, s);
            if (p->st_dw) cudaFreeAsync(p->st_dw, s);
            p->st_x = p->st_dy = p->st_dw = nullptr;
            return cuda_fail(e, "tag_sfb_sync_host: cudaMallocAsync(staging)");
        }
    }
    cudaError_t e = cudaMemcpyAsync(p->st_x, X_host, bx, cudaMemcpyHostToDevice, s);
    if (e == cudaSuccess) e = cudaMemcpyAsync(p->st_dy, dY_host, bdy, cudaMemcpyHostToDevice, s);
    if (e != cudaSuccess) return cuda_fail(e, "tag_sfb_sync_host: H2D copy");
    TAG_TRY(do_gather(p, p->st_x, p->st_dy, s));
    TAG_TRY(do_recon(p, p->st_dw, false, nullptr, nullptr, p->K, p->alpha, s));
    e = cudaMemcpyAsync(dW_host, p->st_dw, bdw, cudaMemcpyDeviceToHost, s);
    if (e != cudaSuccess) return cuda_fail(e, "tag_sfb_sync_host: D2H copy");
    return TAG_OK;
}

tag_status_t tag_local_grad(tag_sfb_plan_t p, const void* X, const void* dY, void* dW_local,
                            tag_stream_t stream) {
    if (!p) return fail(TAG_ERR_INVALID_ARG, "tag_local_grad: NULL plan");
    TAG_TRY(check_ptrs("tag_local_grad", {X, dY, dW_local}));
    TAG_TRY(set_device(p->comm));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const tag_sfb_desc_t& d = p->d;
    if (d.in_dtype != d.wire_dtype) {
        // same operand precision as the SFB path: cast into this rank's gather slot first
        const size_t ew = dtype_size(d.wire_dtype);
        const int r = p->comm->rank;
        void* lx = p->lx ? p->lx : static_cast<char*>(p->gx) + r * d.B * d.M * ew;
        void* ldy = p->ldy ? p->ldy : static_cast<char*>(p->gdy) + r * d.B * d.N * ew;
        TAG_TRY(launch_pack(X, lx, d.B * d.M, dY, ldy, d.B * d.N, d.in_dtype, d.wire_dtype, s));
        set_src_plain(p, lx, ldy);
    } else {
        set_src_plain(p, X, dY);
    }
    tag_status_t st = do_recon(p, dW_local, false, nullptr, nullptr, d.B, 1.0f, s);
    set_src_plain(p, nullptr, nullptr);   // a later reconstruct needs a fresh gather
    return st;
}

tag_status_t tag_dense_allreduce(tag_sfb_plan_t p, void* dW, tag_stream_t stream) {
    if (!p) return fail(TAG_ERR_INVALID_ARG, "tag_dense_allreduce: NULL plan");
    TAG_TRY(check_ptrs("tag_dense_allreduce", {dW}));
    TAG_TRY(set_device(p->comm));
    TAG_TRY(check_async(p->comm));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const int64_t len = p->d.M * p->d.N;
    if (!p->comm->nccl) {
        const int grid = num_sms() * 4;
        if (p->d.out_dtype == TAG_F32)
            scale_f32_kernel<<<grid, 256, 0, s>>>(static_cast<float*>(dW), len, p->alpha);
        else
            scale_bf16_kernel<<<grid, 256, 0, s>>>(static_cast<__nv_bfloat16*>(dW), len, p->alpha);
        cudaError_t e = cudaGetLastError();
        if (e != cudaSuccess) return cuda_fail(e, "launch scale kernel");
        count_launch();
        return TAG_OK;
    }
    ncclResult_t r = ncclAllReduce(dW, dW, static_cast<size_t>(len), nccl_type(p->d.out_dtype),
                                   p->premul, p->comm->nccl, s);
    if (r != ncclSuccess) return nccl_fail(r, "ncclAllReduce");
    return TAG_OK;
}

tag_status_t tag_ps_sync(tag_sfb_plan_t p, void* dW, int root, tag_stream_t stream) {
    if (!p) return fail(TAG_ERR_INVALID_ARG, "tag_ps_sync: NULL plan");
    TAG_TRY(check_ptrs("tag_ps_sync", {dW}));
    if (root < 0 || root >= p->comm->nranks)
        return fail(TAG_ERR_INVALID_ARG, "tag_ps_sync: root must be a rank of the comm");
    if (!p->comm->nccl) return tag_dense_allreduce(p, dW, stream);     // n = 1: dW / B
    TAG_TRY(set_device(p->comm));
    TAG_TRY(check_async(p->comm));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const size_t len = static_cast<size_t>(p->d.M * p->d.N);
    const ncclDataType_t t = nccl_type(p->d.out_dtype);
    // AddN on the PS (PreMulSum applies 1/(nB) inside the reduction), then the PS sends it back
    ncclResult_t r = ncclReduce(dW, dW, len, t, p->premul, root, p->comm->nccl, s);
    if (r != ncclSuccess) return nccl_fail(r, "ncclReduce");
    r = ncclBroadcast(dW, dW, len, t, root, p->comm->nccl, s);
    if (r != ncclSuccess) return nccl_fail(r, "ncclBroadcast");
    return TAG_OK;
}

tag_status_t tag_sgd_step(tag_sfb_plan_t p, const float* dW, float* W, float* v,
                          tag_stream_t stream) {
    if (!p) return fail(TAG_ERR_INVALID_ARG, "tag_sgd_step: NULL plan");
    TAG_TRY(check_ptrs("tag_sgd_step", {dW, W, v}));
    TAG_TRY(set_device(p->comm));
    return launch_sgd(dW, W, v, p->d.M * p->d.N, p->d.lr, p->d.momentum, p->d.weight_decay,
                      reinterpret_cast<cudaStream_t>(stream));
}

tag_status_t tag_sfb_group_create(const tag_sfb_plan_t* plans, int count, tag_sfb_group_t* out) {
    if (!plans || !out) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_create: NULL argument");
    if (count < 1 || count > MAX_GROUP)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_create: count must be in [1, 32]");
    for (int i = 0; i < count; ++i) {
        const tag_plan_s* p = plans[i];
        if (!p) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_create: NULL plan");
        if (p->comm != plans[0]->comm || p->d.in_dtype != plans[0]->d.in_dtype ||
            p->d.wire_dtype != plans[0]->d.wire_dtype || p->d.out_dtype != plans[0]->d.out_dtype)
            return fail(TAG_ERR_INVALID_ARG,
                        "tag_sfb_group_create: plans must share the comm and the dtypes");
        if (p->d.fuse_sgd != plans[0]->d.fuse_sgd ||
            (p->d.fuse_sgd && (p->d.lr != plans[0]->d.lr || p->d.momentum != plans[0]->d.momentum ||
                               p->d.weight_decay != plans[0]->d.weight_decay)))
            return fail(TAG_ERR_INVALID_ARG,
                        "tag_sfb_group_create: plans must share fuse_sgd and its hyper-parameters");
        if (p->d.fuse_adam != plans[0]->d.fuse_adam ||
            (p->d.fuse_adam && (p->d.lr != plans[0]->d.lr || p->d.beta1 != plans[0]->d.beta1 ||
                                p->d.beta2 != plans[0]->d.beta2 || p->d.eps != plans[0]->d.eps ||
                                p->d.weight_decay != plans[0]->d.weight_decay)))
            return fail(TAG_ERR_INVALID_ARG,
                        "tag_sfb_group_create: plans must share fuse_adam and its hyper-parameters");
        for (int j = 0; j < i; ++j)
            if (plans[j] == p) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_create: duplicate plan");
    }
    tag_group_s* g = new tag_group_s;
    g->plans.assign(plans, plans + count);
    g->push_all = true;
    g->tc_all = true;
    for (tag_plan_s* p : g->plans) {
        g->push_all = g->push_all && p->gather_mode == TAG_GATHER_NVLINK_PUSH;
        g->tc_all = g->tc_all && p->use_tc;
    }
    *out = g;
    return TAG_OK;
}

tag_status_t tag_sfb_group_destroy(tag_sfb_group_t g) {
    delete g;
    return TAG_OK;
}

tag_status_t tag_sfb_group_gather(tag_sfb_group_t g, const void* const* X, const void* const* dY,
                                  tag_stream_t stream) {
    if (!g || !X || !dY) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_gather: NULL argument");
    const int count = static_cast<int>(g->plans.size());
    for (int i = 0; i < count; ++i) TAG_TRY(check_ptrs("tag_sfb_group_gather", {X[i], dY[i]}));
    tag_comm_s* c = g->plans[0]->comm;
    TAG_TRY(set_device(c));
    TAG_TRY(check_async(c));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (g->push_all) {
        PushSegment seg[MAX_GROUP];
        for (int i = 0; i < count; ++i) seg[i] = push_segment(g->plans[i], X[i], dY[i]);
        tag_plan_s* p0 = g->plans[0];
        TAG_TRY(launch_push_gather_group(c->devcomm, seg, count, c->rank, p0->d.in_dtype,
                                         p0->d.wire_dtype, EXP_PUSH_GRID, p0->flags + WIN_LOCAL_PUSH / 4, s));
        for (int i = 0; i < count; ++i) set_src_window(g->plans[i]);
        return TAG_OK;
    }
    // mixed / NCCL mode: one NCCL group around every plan's gather (nested groups are legal)
    const bool nccl = c->nccl != nullptr;
    if (nccl) {
        ncclResult_t r = ncclGroupStart();
        if (r != ncclSuccess) return nccl_fail(r, "ncclGroupStart");
    }
    tag_status_t st = TAG_OK;
    for (int i = 0; i < count && st == TAG_OK; ++i) st = do_gather(g->plans[i], X[i], dY[i], s);
    if (nccl) {
        ncclResult_t r = ncclGroupEnd();
        if (st == TAG_OK && r != ncclSuccess) return nccl_fail(r, "ncclGroupEnd");
    }
    return st;
}

static tag_status_t group_reconstruct(tag_sfb_group_t g, void* const* dW, bool sgd,
                                      float* const* W, float* const* V, tag_stream_t stream,
                                      float* const* Mm = nullptr, const AdamCall* adam = nullptr) {
    const int count = static_cast<int>(g->plans.size());
    for (int i = 0; i < count; ++i) {
        if (!sgd || dW[i]) TAG_TRY(check_ptrs("tag_sfb_group_reconstruct", {dW[i]}));
        if (sgd) TAG_TRY(check_ptrs("tag_sfb_group_sync_sgd", {W[i], V[i]}));
        if (!g->plans[i]->src_x)
            return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_reconstruct: no factors gathered yet");
    }
    TAG_TRY(set_device(g->plans[0]->comm));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    ReconArgs a[MAX_GROUP];
    bool tc = g->tc_all;
    for (int i = 0; i < count; ++i) {
        tag_plan_s* p = g->plans[i];
        a[i] = ReconArgs{};
        fill_src(p, a[i]);
        a[i].C = dW[i];
        a[i].M = p->d.M;
        a[i].N = p->d.N;
        a[i].K = p->K;
        a[i].wire = p->d.wire_dtype;
        a[i].out = p->d.out_dtype;
        a[i].alpha = p->alpha;
        a[i].sgd = sgd;
        a[i].W = sgd ? W[i] : nullptr;
        a[i].V = sgd ? V[i] : nullptr;
        a[i].lr = p->d.lr;
        a[i].mu = p->d.momentum;
        a[i].wd = p->d.weight_decay;
        if (sgd) set_adam(a[i], Mm ? Mm[i] : nullptr, adam);
        tc = tc && recon_tc_ok(a[i]);
    }
    if (tc) return launch_recon_tc_group(a, count, s);
    for (int i = 0; i < count; ++i)
        TAG_TRY(do_recon(g->plans[i], dW[i], sgd, sgd ? W[i] : nullptr, sgd ? V[i] : nullptr,
                         g->plans[i]->K, g->plans[i]->alpha, s, Mm ? Mm[i] : nullptr, adam));
    return TAG_OK;
}

tag_status_t tag_sfb_group_reconstruct(tag_sfb_group_t g, void* const* dW, tag_stream_t stream) {
    if (!g || !dW) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_reconstruct: NULL argument");
    if (g->plans[0]->d.fuse_sgd || g->plans[0]->d.fuse_adam)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_reconstruct: fused-optimizer group, use sync_sgd / sync_adam");
    return group_reconstruct(g, dW, false, nullptr, nullptr, stream);
}

tag_status_t tag_sfb_group_bias_grad(tag_sfb_group_t g, void* const* db, tag_stream_t stream) {
    if (!g || !db) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_bias_grad: NULL argument");
    BiasArgs a[MAX_GROUP];
    const int count = static_cast<int>(g->plans.size());
    for (int i = 0; i < count; ++i) {
        tag_plan_s* p = g->plans[i];
        if (!db[i]) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_bias_grad: NULL db entry");
        if (!p->src_dy)
            return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_bias_grad: no factors gathered yet");
        a[i] = BiasArgs{p->src_dy, p->src_dy1, p->src_ctr, db[i], p->K, p->d.N, p->d.wire_dtype,
                        p->d.out_dtype, p->alpha};
    }
    TAG_TRY(set_device(g->plans[0]->comm));
    return launch_bias_grad(a, count, reinterpret_cast<cudaStream_t>(stream));
}

tag_status_t tag_sfb_group_sync_sgd(tag_sfb_group_t g, const void* const* X, const void* const* dY,
                                    float* const* W, float* const* v, void* const* dW,
                                    tag_stream_t stream) {
    if (!g || !X || !dY || !W || !v)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_sync_sgd: NULL argument");
    if (!g->plans[0]->d.fuse_sgd)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_sync_sgd: plans have fuse_sgd = 0");
    const int count = static_cast<int>(g->plans.size());
    void* none[MAX_GROUP] = {nullptr};
    void* const* dWs = dW ? dW : none;
    bool fuse = true;
    for (int i = 0; i < count; ++i) {
        TAG_TRY(check_ptrs("tag_sfb_group_sync_sgd", {X[i], dY[i], W[i], v[i]}));
        if (dWs[i]) TAG_TRY(check_ptrs("tag_sfb_group_sync_sgd", {dWs[i]}));
        fuse = fuse && fusable(g->plans[i], dWs[i], 1);
    }
    TAG_TRY(set_device(g->plans[0]->comm));
    TAG_TRY(check_async(g->plans[0]->comm));
    if (fuse)
        return fused_sync(g->plans.data(), count, X, dY, dWs, true, W, v,
                          reinterpret_cast<cudaStream_t>(stream));
    TAG_TRY(tag_sfb_group_gather(g, X, dY, stream));
    return group_reconstruct(g, dWs, true, W, v, stream);
}

tag_status_t tag_sfb_group_sync_adam(tag_sfb_group_t g, const void* const* X, const void* const* dY,
                                     float* const* W, float* const* m, float* const* v,
                                     int64_t step, void* const* dW, tag_stream_t stream) {
    if (!g || !X || !dY || !W || !m || !v)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_sync_adam: NULL argument");
    if (!g->plans[0]->d.fuse_adam)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_sync_adam: plans have fuse_adam = 0");
    if (step < 1) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_sync_adam: step must be >= 1");
    const int count = static_cast<int>(g->plans.size());
    void* none[MAX_GROUP] = {nullptr};
    void* const* dWs = dW ? dW : none;
    bool fuse = true;
    for (int i = 0; i < count; ++i) {
        TAG_TRY(check_ptrs("tag_sfb_group_sync_adam", {X[i], dY[i], W[i], m[i], v[i]}));
        if (dWs[i]) TAG_TRY(check_ptrs("tag_sfb_group_sync_adam", {dWs[i]}));
        fuse = fuse && fusable(g->plans[i], dWs[i], 2);
    }
    TAG_TRY(set_device(g->plans[0]->comm));
    TAG_TRY(check_async(g->plans[0]->comm));
    const AdamCall ad = adam_call(g->plans[0]->d, step);
    if (fuse)
        return fused_sync(g->plans.data(), count, X, dY, dWs, true, W, v,
                          reinterpret_cast<cudaStream_t>(stream), false, m, &ad);
    TAG_TRY(tag_sfb_group_gather(g, X, dY, stream));
    return group_reconstruct(g, dWs, true, W, v, stream, m, &ad);
}

tag_status_t tag_sfb_group_sync_sharded(tag_sfb_group_t g, const void* const* X,
                                        const void* const* dY, void* const* dW,
                                        tag_stream_t stream) {
    if (!g || !X || !dY || !dW)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_sync_sharded: NULL argument");
    if (g->plans[0]->d.fuse_sgd || g->plans[0]->d.fuse_adam)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_sync_sharded: fused-optimizer group");
    const int count = static_cast<int>(g->plans.size());
    bool fuse = true;
    for (int i = 0; i < count; ++i) {
        int64_t rb, rc;
        shard_range(g->plans[i], g->plans[i]->comm->rank, &rb, &rc);
        TAG_TRY(check_ptrs("tag_sfb_group_sync_sharded", {X[i], dY[i]}));
        if (rc > 0) TAG_TRY(check_ptrs("tag_sfb_group_sync_sharded", {dW[i]}));
        fuse = fuse && fusable(g->plans[i], rc > 0 ? dW[i] : nullptr);   // rank-independent
    }
    TAG_TRY(set_device(g->plans[0]->comm));
    TAG_TRY(check_async(g->plans[0]->comm));
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (fuse) return fused_sync(g->plans.data(), count, X, dY, dW, false, nullptr, nullptr, s, true);
    TAG_TRY(tag_sfb_group_gather(g, X, dY, stream));
    for (int i = 0; i < count; ++i) {
        tag_plan_s* p = g->plans[i];
        int64_t rb, rc;
        shard_range(p, p->comm->rank, &rb, &rc);
        if (rc == 0) continue;
        ReconArgs r{};
        fill_src(p, r, rb);
        r.C = dW[i];
        r.M = rc;
        r.N = p->d.N;
        r.K = p->K;
        r.lda = p->d.M;
        r.wire = p->d.wire_dtype;
        r.out = p->d.out_dtype;
        r.alpha = p->alpha;
        TAG_TRY((p->use_tc && recon_tc_ok(r)) ? launch_recon_tc(r, s) : launch_recon_simt(r, s));
    }
    return TAG_OK;
}

tag_status_t tag_sfb_group_sync(tag_sfb_group_t g, const void* const* X, const void* const* dY,
                                void* const* dW, tag_stream_t stream) {
    if (!g || !X || !dY || !dW) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_sync: NULL argument");
    if (g->plans[0]->d.fuse_sgd || g->plans[0]->d.fuse_adam)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_group_sync: fused-optimizer group, use sync_sgd / sync_adam");
    const int count = static_cast<int>(g->plans.size());
    bool fuse = true;
    for (int i = 0; i < count; ++i) {
        TAG_TRY(check_ptrs("tag_sfb_group_sync", {X[i], dY[i], dW[i]}));
        fuse = fuse && fusable(g->plans[i], dW[i]);
    }
    if (fuse) {
        TAG_TRY(set_device(g->plans[0]->comm));
        TAG_TRY(check_async(g->plans[0]->comm));
        return fused_sync(g->plans.data(), count, X, dY, dW, false, nullptr, nullptr,
                          reinterpret_cast<cudaStream_t>(stream));
    }
    TAG_TRY(tag_sfb_group_gather(g, X, dY, stream));
    return tag_sfb_group_reconstruct(g, dW, stream);
}

}  // extern "C"
