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
struct ReconArgs {
    const void* A;       // K x M
    const void* Bm;      // K x N
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
    uint64_t off_x, off_dy, off_flag;
    int64_t cx, cy;        // elements of X_r / dY_r
    uint32_t flag_target;  // arrival-counter value meaning "all ranks' factors landed"
};

struct FusedGather {
    int npeers;            // LSA team size (== comm size)
    int me;                // LSA rank (== comm rank)
    void* mc_base;         // NVLS multicast base (multimem.st to every GPU at once), or nullptr
    bool cast;             // sources are fp32, the wire is bf16 (RNE cast inside the push)
    // hierarchical publish: CTAs count themselves on a local counter; the last one of this rank
    // adds 1 to every layer's counter on every peer (n remote atomics per layer, not n * grid)
    uint32_t* local_ctr;   // device address (this rank's window)
    uint32_t local_target; // local counter value after this launch's CTAs have all arrived
};

// Tensor-core path (tcgen05 + TMEM + TMA). Requires 16-byte aligned rows (see recon_tc_ok).
bool recon_tc_ok(const ReconArgs& a);
tag_status_t launch_recon_tc(const ReconArgs& a, cudaStream_t s);
// Grouped form: one persistent launch over all layers' tiles (1 <= count <= MAX_GROUP).
constexpr int MAX_GROUP = 32;   // layers per bucket (kernel parameter space: ~15 KB at 32)
// fused != nullptr: the kernel also pushes this rank's factors to every peer and waits per layer
// on the arrival counters (see recon_tc.cu). recon_tc_grid: the CTA count such a launch uses.
tag_status_t launch_recon_tc_group(const ReconArgs* a, int count, cudaStream_t s,
                                   const FusedGather* fused = nullptr);
int recon_tc_grid(const ReconArgs* a, int count);
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
    size_t off_x, off_dy;   // byte offsets of this buffer's X_all / dY_all in the window
    int64_t cx, cy;         // elements of this rank's X_r / dY_r
};
tag_status_t launch_push_gather_group(const void* dc, const PushSegment* seg, int count, int slot,
                                      tag_dtype_t in, tag_dtype_t wire, int max_ctas,
                                      cudaStream_t s);

// ------------------------------------------------------------------ bias gradient (R17)
struct BiasArgs {
    const void* dy;        // dY_all (K x N, wire dtype)
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
tag_status_t launch_tf32_split(const float* src, float* dst, int64_t K, int64_t cols, int64_t kpad,
                               cudaStream_t s);
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
