// tag_internal.h — declarations shared by the libtag translation units (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <atomic>
#include <cstdint>
#include <string>

#include "../../include/tag.h"

// Diagnostics builds only (scripts/build_variant.sh -D...; the product build never sets these):
// EXP_F32_SIMT = fp32 factors on the SIMT FFMA kernel instead of 3xTF32; EXP_NO_FUSE = staged
// push kernel + reconstruction instead of the fused exchange kernel.
#ifndef EXP_F32_SIMT
#define EXP_F32_SIMT 0
#endif
#ifndef EXP_NO_FUSE
#define EXP_NO_FUSE 0
#endif

namespace tag {

// Thread-local error detail behind tag_last_error().
void set_error(const std::string& msg);
tag_status_t fail(tag_status_t st, const std::string& msg);
tag_status_t cuda_fail(cudaError_t e, const char* what);

// Kernel-launch counter behind tag_kernel_launches().
extern std::atomic<uint64_t> g_launches;
inline void count_launch(uint64_t k = 1) { g_launches.fetch_add(k, std::memory_order_relaxed); }

int num_sms();

inline size_t dtype_size(tag_dtype_t t) { return t == TAG_F32 ? 4 : 2; }

// ------------------------------------------------------------------ reconstruction kernels
// dW[m][j] = alpha * sum_{k<K} A[k][m] * Bm[k][j] (A: K x M, Bm: K x N, row-major, wire dtype),
// written as out dtype (epilogue E1), or with the fused SGD-momentum update (epilogue E2).
// The factors a plan gathered into its double-buffered symmetric window live in one of two
// buffers; which one is device state: the window's call counter c (u32, WIN_CALLS below) counts
// every kernel that gathered into the window, so the latest gather used buffer (c - 1) & 1 and a
// gather in flight uses c & 1. Kernels read c on the device instead of taking the buffer from the
// host, which keeps the sync calls free of per-call host state (CUDA-graph capturable).
// Layout of each plan's window flag area (byte offsets from win_flag_off, all u32):
constexpr int WIN_ARRIVAL = 0;      // [2] arrival counters, one per buffer (peers add to them)
constexpr int WIN_LOCAL_FUSED = 8;  // self-resetting "last CTA" counter of the fused kernel
constexpr int WIN_LOCAL_PUSH = 12;  // the same for the push-gather kernel
constexpr int WIN_CALLS = 16;       // c

// Read the call counter of a window (nullptr: a plain single buffer, parity 0). L1 is bypassed:
// the value was written by an earlier kernel of the stream.
__device__ __forceinline__ uint32_t load_calls(const uint32_t* ctr) {
    if (ctr == nullptr) return 1u;   // (1 - 1) & 1 = buffer 0
    uint32_t v;
    asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(ctr) : "memory");
    return v;
}

struct ReconArgs {
    const void* A;       // K x M
    const void* Bm;      // K x N
    // window operands: A / Bm are buffer 0 and buffer 1 starts kbuf rows further (the window
    // holds [X buf 0 | X buf 1 | dY buf 0 | dY buf 1], each buffer kbuf rows, zero beyond K), A1 /
    // Bm1 point at it; ctr is the window's call counter; ctr_mode 1: read the latest gather's
    // buffer ((c - 1) & 1), 2: the fused kernel's own (c & 1)
    const void* A1;
    const void* Bm1;
    int64_t kbuf;
    const uint32_t* ctr;
    int ctr_mode;
    void* C;             // M x N, out dtype; may be nullptr when sgd (no dW write)
    int64_t M, N, K;
    int64_t lda;         // elements between consecutive rows of A (0: M) — row shards of X_all
    int64_t kpad;        // fp32 wire (3xTF32): A, Bm are split [hi ; lo] buffers of kpad rows each
    tag_dtype_t wire;    // operand dtype
    tag_dtype_t out;     // C dtype
    float alpha;
    // E2
    bool sgd;
    float* W;
    float* V;
    float lr, mu, wd;
    // optimizer kind when sgd (= an optimizer epilogue) is set: 1 SGD-momentum, 2 Adam (R22);
    // Adam keeps its first moment in Mm and its second in V
    int opt;
    float* Mm;
    float b1, omb1, b2, omb2, eps, lr_t, isbc2;
    // fused NVLink all-gather (push of this rank's factors inside the reconstruction kernel)
    const void* srcX;      // X_r, dY_r (in dtype: wire dtype, or fp32 with FusedGather::cast)
    const void* srcY;
    void* win;             // ncclWindow_t of the layer's symmetric window
    uint64_t off_x, off_dy;  // buffer 0's X_all / dY_all in the window
    uint64_t xbuf, ybuf;     // buffer 1's X_all / dY_all are xbuf / ybuf bytes further
    uint64_t off_flag;     // the window flag area (WIN_* offsets)
    uint32_t* flags;       // the same area, this rank's device address
    int64_t cx, cy;        // elements of X_r / dY_r
    // dynamic tile schedule counters (2 x u32, zero between launches; owned by the plan whose
    // args are a[0]), or nullptr for the static schedule
    uint32_t* sched;
};

struct FusedGather {
    int npeers;            // LSA team size (== comm size)
    int me;                // LSA rank (== comm rank)
    void* mc_base;         // NVLS multicast base (multimem.st to every GPU at once), or nullptr
    bool cast;             // sources are fp32, the wire is bf16 (RNE cast inside the push)
    // hierarchical publish: CTAs count themselves on a self-resetting local counter (plan 0's
    // WIN_LOCAL_FUSED); the last one of this rank adds 1 to every layer's arrival counter on
    // every peer (n remote atomics per layer, not n * grid) and advances every layer's c
    uint32_t* local_ctr;
};

// Tensor-core path (tcgen05 + TMEM + TMA). Requires 16-byte aligned rows (see recon_tc_ok).
bool recon_tc_ok(const ReconArgs& a);
tag_status_t launch_recon_tc(const ReconArgs& a, cudaStream_t s);
// Grouped form: one persistent launch over all layers' tiles (1 <= count <= MAX_GROUP).
constexpr int MAX_GROUP = 32;   // layers per bucket (kernel parameter space: ~15 KB at 32)
// fused != nullptr: the kernel also pushes this rank's factors to every peer and waits per layer
// on the arrival counters (see recon_tc.cu).
tag_status_t launch_recon_tc_group(const ReconArgs* a, int count, cudaStream_t s,
                                   const FusedGather* fused = nullptr);
// the tile configuration launch_recon_tc_group picks for these layers
void recon_tc_describe(const ReconArgs* a, int count, int* bn, int* ctas, int* box3d);
// SIMT FFMA path: any shape, fp32 or bf16 operands (exact fp32 accumulation in k order).
tag_status_t launch_recon_simt(const ReconArgs& a, cudaStream_t s);

// ------------------------------------------------------------------ pack (a1)
// Casts src (fp32) into dst (bf16, RNE) for two segments in one launch; or copies when the
// dtypes match. Counts are elements.
tag_status_t launch_pack(const void* x, void* x_dst, int64_t nx, const void* dy, void* dy_dst,
                         int64_t ny, tag_dtype_t in, tag_dtype_t wire, cudaStream_t s);

// ------------------------------------------------------------------ NVLink push gather (a1+a2)
struct PushSegment {
    const void* X;
    const void* dY;
    void* win;              // ncclWindow_t
    size_t off_x, off_dy;   // byte offsets of buffer 0's X_all / dY_all in the window
    size_t xbuf, ybuf;      // buffer 1's X_all / dY_all are xbuf / ybuf bytes further
    size_t off_flag;        // the window flag area (WIN_* offsets)
    uint32_t* flags;        // the same area, this rank's device address
    int64_t cx, cy;         // elements of this rank's X_r / dY_r
};
// local_ctr: plan 0's WIN_LOCAL_PUSH (the last CTA after the barrier publishes and advances c)
tag_status_t launch_push_gather_group(const void* dc, const PushSegment* seg, int count, int slot,
                                      tag_dtype_t in, tag_dtype_t wire, int max_ctas,
                                      uint32_t* local_ctr, cudaStream_t s);

// ------------------------------------------------------------------ bias gradient (R17)
struct BiasArgs {
    const void* dy;        // dY_all (K x N, wire dtype); a window: buffer 0
    const void* dy1;       // window buffer 1, or nullptr
    const uint32_t* ctr;   // the window's call counter (latest gather), or nullptr
    void* db;              // N, out dtype
    int64_t K, N;
    tag_dtype_t wire, out;
    float alpha;
};
// db = alpha * column sums of dY_all for 1..MAX_GROUP layers in one launch (bias.cu)
tag_status_t launch_bias_grad(const BiasArgs* a, int count, cudaStream_t s);

// ------------------------------------------------------------------ 3xTF32 operand split
// dst = [hi ; lo] (2*kpad x cols fp32): hi = src rounded to the nearest tf32 (a value kind::tf32
// reads exactly), lo = src - hi (exact in fp32); rows [K, kpad) of both halves are zero.
tag_status_t launch_tf32_split(const float* src, const float* src1, const uint32_t* ctr, float* dst,
                               int64_t K, int64_t cols, int64_t kpad, cudaStream_t s);
constexpr int TF32_KALIGN = 16;   // kpad = K rounded up to the 3xTF32 stage depth

// ------------------------------------------------------------------ unfused Adam (R22)
// W, m, v updated in place from dW (all fp32, len elements); constants as in optim.cuh
tag_status_t launch_adam(const float* dW, float* W, float* Mm, float* V, int64_t len, float b1,
                         float omb1, float b2, float omb2, float eps, float lr_t, float isbc2,
                         float wd, cudaStream_t s);

// ------------------------------------------------------------------ unfused SGD
tag_status_t launch_sgd(const float* dW, float* W, float* V, int64_t len, float lr, float mu,
                        float wd, cudaStream_t s);

}  // namespace tag
