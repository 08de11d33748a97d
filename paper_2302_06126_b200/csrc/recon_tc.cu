// recon_tc.cu — step a3+a4 of the SFB path on the 5th-generation tensor cores.
//
// dW = alpha * X_all^T dY_all ("MatMul ops on each device can reconstruct identical
// gradients"), K = n*B gathered factor rows, alpha = 1/(nB) (DESIGN R1), fused epilogue
// (E1: scale + fp32/bf16 store; E2: scale + SGD-momentum on W, v, P:543-545 / R14).
//
// Operand layout: both factors are MN-major in their natural row-major form — A_mma[m][k] =
// X_all[k][m] with m contiguous, B_mma[j][k] = dY_all[k][j] with j contiguous — so no transpose
// pass exists anywhere on the path. TMA loads 64-element (128-byte) MN chunks x BK rows with the
// 128-byte swizzle; the UMMA descriptors describe the canonical MN-major SW128 layout
// (LBO = stride between MN chunks, SBO = 1024 B between 8-row K groups). When M and N are
// multiples of 64, each operand's chunks of a stage arrive in ONE 3-D request instead of one per
// chunk (a {64, K, M/64} view with a 128-byte chunk stride; fewer TMA instructions, measured
// 1-2 us faster per bucket at K = 128, neutral elsewhere).
//
// Kernel structure (persistent, warp-specialised, one CTA per SM):
//   warp 0      TMA producer: STAGES-deep smem ring of {A: 128 x BK, B: BN x BK} tiles
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer; accumulators double-buffered
//               in TMEM (2 x BN fp32 columns) so tile t+1's MMAs overlap tile t's epilogue
//   warps 2..9  epilogue: tcgen05.ld 32 rows x 32 cols -> scale -> swizzled smem -> TMA store
//               (E1), or the fused SGD update on W, v (E2). Each TMEM lane quadrant is drained by
//               two warps, each owning half of the tile's columns.
// At the paper's small-batch shapes (K = 32..2048) the epilogue's HBM write of the M x N
// gradient is the binding roof (DESIGN "Roofline"), so the kernel keeps 8 warps of stores in
// flight while the tensor core works one tile ahead.
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <atomic>
#include <climits>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include <nccl.h>
#include <nccl_device.h>

#include "optim.cuh"
#include "ptx.cuh"
#include "tag_internal.h"

namespace tag {
namespace {

constexpr int BM = 128;                  // UMMA M (TMEM lanes)
#ifndef EXP_EPI_WARPS
#define EXP_EPI_WARPS 8
#endif
constexpr int NUM_EPI_WARPS = EXP_EPI_WARPS;
constexpr int EPI_GROUPS = NUM_EPI_WARPS / 4;   // column groups per TMEM lane quadrant
constexpr int NUM_THREADS = 64 + 32 * NUM_EPI_WARPS;   // 320
constexpr int EPI_CHUNK_BYTES = 32 * 128;    // one 32 rows x 128 B transpose buffer
constexpr int SMEM_MAX = 232448;              // 227 KB of dynamic shared memory per CTA
constexpr int TMEM_COLS = 512;
constexpr int SCHED_RING = 16;               // tile ids in flight between the producer and consumers
// Diagnostics only (scripts/build_variant.sh, never the product build): 1 = epilogue skips the
// global stores, 2 = epilogue releases each accumulator without reading it
#ifndef EXP_SGD_EP
#define EXP_SGD_EP 1      // epilogue chunks per round in the optimizer instantiations
#endif
#ifndef EXP_EPI_MODE
#define EXP_EPI_MODE 0
#endif
// Diagnostics builds only: fused-exchange phases (see the kernel), forced tile shapes
// (EXP_RECON_BN = 128 | 256, EXP_RECON_CTAS = 1 | 2; 0 = the measured rule), 2-D instead of
// 3-D TMA boxes (EXP_RECON_NO3D), SIMT FFMA instead of 3xTF32 for fp32 factors (EXP_F32_SIMT).
#ifndef EXP_FUSED_DBG
#define EXP_FUSED_DBG 0
#endif
#ifndef EXP_RECON_BN
#define EXP_RECON_BN 0
#endif
#ifndef EXP_RECON_CTAS
#define EXP_RECON_CTAS 0
#endif
#ifndef EXP_RECON_NO3D
#define EXP_RECON_NO3D 0
#endif

// CTAS = 2: a CTA pair on one TPC runs tcgen05 cta_group::2 — UMMA M = 256 (128 rows of A in
// each CTA's smem), N = BN (BN/2 columns of B in each CTA's smem), each CTA's TMEM holds its
// 128 rows x BN fp32 accumulator. Halves the per-SM smem operand traffic and the L2 re-reads of B.
//
// X3 = true: fp32 factors on the tensor cores with 3xTF32 (kind::tf32). The operand buffers hold
// [hi ; lo] halves (rows [0, Kp) and [Kp, 2Kp), see tf32_split in pack_sgd.cu) and every K step
// issues hi*hi + hi*lo + lo*hi, which recovers ~fp32 accuracy (the dropped lo*lo and the tf32
// truncations are ~2^-21 relative per product) at 3 MMAs per step — free while the epilogue's
// HBM write binds. Stages carry 16 fp32 rows (32-element MN chunks of 128 B) of all four operands.
// EP = epilogue chunks staged per round (2 for the fp32 E1 store, 1 for bf16 / E2 / X3), which
// sizes the per-warp transpose buffers; the operand ring takes the rest of shared memory.
template <int BN, int CTAS, bool X3 = false, int EP = 2, bool LONGK = false>
struct Cfg {
    // X3 keeps two accumulators per tile: hi*hi, and the small hi*lo + lo*hi terms apart, so the
    // big accumulator sees K/8 additions instead of 3K/8 (the tensor core's fp32 accumulation
    // error grows linearly with the number of MMAs; measured, scripts/probes/acc_error.py)
    static constexpr int ACC_COLS = X3 ? 2 * BN : BN;     // TMEM columns per tile
    static constexpr int ACC = TMEM_COLS / ACC_COLS;      // accumulator buffers in TMEM
    static constexpr int ELEMS = X3 ? 32 : 64;            // MN elements per 128-byte chunk
    // factor rows per pipeline stage. CTA pairs (K >= 192) with a one-chunk epilogue (bf16 dW,
    // optimizers) take 128 rows per stage (3 stages of 64 KB; with 3-D boxes one 32 KB TMA
    // request per operand): fc6 at K = 256, bf16 dW, 32 / 64 / 128 rows: 74.6 / 60.1 / 58.1 us
    // (the per-request cost, not bytes, paces the operand stream). With the two-chunk fp32
    // epilogue only 2 such stages fit, which loses at large K (Transformer out-proj K = 2048:
    // 78.8 vs 64.3 us), so those keep 64 rows (5 stages); so do K > 512 layers (LONGK: out-proj
    // K = 2048, bf16 dW: 58.3 us with 64 rows, 60.4 with 128).
    static constexpr int BK = X3 ? 16 : (CTAS == 2 ? (EP == 1 && !LONGK ? 128 : 64) : 32);
    static constexpr int KMMA = X3 ? 8 : 16;              // K per tcgen05.mma
    static constexpr int CHUNK_BYTES = BK * 128;          // one 128-byte-wide MN chunk of BK rows
    static constexpr int A_CHUNKS = BM / ELEMS;
    static constexpr int B_CHUNKS = BN / CTAS / ELEMS;
    static constexpr int HALVES = X3 ? 2 : 1;             // hi and lo operands
    // UMMA smem descriptor: bf16 SWIZZLE_128B (8-row K atoms), tf32 SWIZZLE_128B_BASE32B (4-row)
    static constexpr uint32_t DLAYOUT = X3 ? 1u : 2u;
    static constexpr uint32_t SBO = X3 ? 512u : 1024u;
    static constexpr int A_BYTES = HALVES * A_CHUNKS * CHUNK_BYTES;
    static constexpr int B_BYTES = HALVES * B_CHUNKS * CHUNK_BYTES;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int EPI_BUF_BYTES = EP * EPI_CHUNK_BYTES;   // per epilogue warp
    static constexpr int EPI_BYTES = NUM_EPI_WARPS * EPI_BUF_BYTES;
    // mbarriers + TMEM slot (< 256 B), the tile-schedule ring at +512 (SCHED_RING full / empty
    // barriers and tile ids)
    static constexpr int BAR_BYTES = 1024;
    // as many stages as fit, at most 8 (BN = 128: 8; BN = 256 one CTA: 6; pairs: 3 with a
    // one-chunk epilogue, 2 with the two-chunk fp32 one)
    static constexpr int FIT = (SMEM_MAX - 1024 - EPI_BYTES - BAR_BYTES) / STAGE_BYTES;
    static constexpr int STAGES = X3 ? 4 : (FIT < 8 ? FIT : 8);
    static constexpr int SMEM = 1024 + STAGES * STAGE_BYTES + EPI_BYTES + BAR_BYTES;
    // instruction descriptor: D f32, A/B bf16 (kind::f16) or tf32 (kind::tf32), both MN-major,
    // N = BN, M = 128 * CTAS.
    static constexpr uint32_t FMT = X3 ? 2u : 1u;
    static constexpr uint32_t IDESC = (1u << 4) | (FMT << 7) | (FMT << 10) | (1u << 15) |
                                      (1u << 16) | (uint32_t(BN >> 3) << 17) |
                                      (uint32_t((BM * CTAS) >> 4) << 24);
};

// One launch reconstructs a group of layers (a gradient bucket): their output tiles are
// concatenated in layer order and distributed round-robin over the persistent CTAs, so the
// prologue, pipeline ramp-up and the last partial wave are paid once per bucket, not per layer.
struct LayerParams {
    CUtensorMap tmA;  // X_all (K x M) bf16, box 64 x BK, 128-B swizzle (X3: [hi;lo] fp32, box 32 x BK)
    CUtensorMap tmB;  // dY_all (K x N)
    const uint32_t* ctr;      // window operands: the window's call counter (WIN_CALLS), else null
    int ctr_mode;             // 0: one buffer; 1: buffer (c - 1) & 1 (latest gather); 2: c & 1 (FUSED)
    int kbuf;                 // window operands: rows between the two buffers of tmA / tmB
    void* C;          // dW out (may be nullptr with SGD)
    float* W;
    float* V;         // SGD momentum buffer / Adam second moment
    float* Mm;        // Adam first moment
    int M, N;
    int num_n_blocks, num_k_blocks;
    int k_lo;         // X3: first row of the lo halves (Kp)
    int tile_begin;   // first global tile index of this layer
    int num_m_blocks;
    int m_fast;       // 1: consecutive tiles walk down M (share a B panel), else along N
    int box3;         // 1: tmA / tmB are 3-D maps (64 x BK x chunks): one request per operand
    float alpha;
    // fused all-gather (FUSED = true): this rank's factors are pushed into every peer's window
    const void* srcX;      // X_r (B x M, wire dtype)
    const void* srcY;      // dY_r (B x N)
    ncclWindow_t win;      // the layer's symmetric window
    uint64_t off_x, off_dy;  // buffer 0's X_all / dY_all in the window
    uint64_t xbuf, ybuf;     // buffer 1's are xbuf / ybuf bytes further
    uint64_t off_flag;     // the window flag area (WIN_* offsets)
    uint32_t* flags;       // the same area, this rank's address
    int64_t vx, vy;        // 16-byte vectors of X_r / dY_r
};

// MAXL = 4 (buckets of up to 4 layers) or MAX_GROUP: the kernel parameter block (and every
// launch's copy of it) stays small for the common buckets (measured: 32-layer parameter blocks
// cost ~2 us per launch on the n = 1 bench)
template <int MAXL>
struct GroupParamsT {
    LayerParams L[MAXL];
    int count;
    int num_tiles;
    float lr, mu, wd;
    int opt;               // optimizer epilogue (SGD instantiations): 1 SGD-momentum, 2 Adam
    AdamConsts adam;
    int slot;              // this rank (its slot in X_all / dY_all)
    char* mc_base;         // FUSED: NVLS multicast base of the windows, or nullptr (unicast)
    int cast;              // FUSED: the sources are fp32, cast to bf16 (RNE) on the way out
    uint32_t* local_ctr;   // FUSED: self-resetting hierarchical publish counter
    // dynamic tile schedule (one-CTA tiles): [next-tile counter, finished-CTA counter], zero
    // between launches (the last CTA to finish resets both); nullptr = static round robin
    uint32_t* sched;
};

struct TileRef {
    int li, m0, n0;
};

// m0 is the first row of the (BM * CTAS)-row tile; CTA rank r of a pair owns rows m0 + r * BM.
template <int BN, int CTAS, typename GP>
__device__ __forceinline__ TileRef locate(const GP& gp, int tile) {
    // the last layer whose first tile is <= tile (empty shards share tile_begin with the next
    // layer and are skipped). A linear scan: measured 2.3 us faster per n = 1 bench step than a
    // binary search, whose data-dependent parameter loads sit on every warp's per-tile path
    int li = 0;
    while (li + 1 < gp.count && tile >= gp.L[li + 1].tile_begin) ++li;
    const int t = tile - gp.L[li].tile_begin;
    if (gp.L[li].m_fast) {
        const int nmb = gp.L[li].num_m_blocks;
        return TileRef{li, (t % nmb) * BM * CTAS, (t / nmb) * BN};
    }
    const int nnb = gp.L[li].num_n_blocks;
    return TileRef{li, (t / nnb) * BM * CTAS, (t % nnb) * BN};
}

__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);   // RNE, lo in the low half
    return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ void grid_dep_wait() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
}
__device__ __forceinline__ void grid_dep_launch() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Fused all-gather (a1 + a2 inside the reconstruction kernel). Every CTA pushes an even slice of
// every layer's local factors into slot `rank` of every peer's window (NVLink stores through
// the NCCL LSA mapping; peer order rotated by rank), then — after a CTA barrier — one thread
// issues one system-scope fence and adds 1 to every layer's arrival counter on every peer. The
// TMA producer of each CTA waits for a layer's counter before loading that layer's first tile.
// multicast address of (window, offset): one store there lands in every GPU of the team
__device__ __forceinline__ void* mc_ptr(char* mc_base, ncclWindow_t w, size_t off) {
    return mc_base + static_cast<size_t>(w->mcOffset4K) * 4096 + off;
}

#ifndef EXP_STATIC_SCHED
#define EXP_STATIC_SCHED 0   // diagnostics builds: the static round-robin tile schedule everywhere
#endif
#ifndef EXP_DYN_WAVES
#define EXP_DYN_WAVES 2      // rounds of tiles at the end handed out dynamically
#endif
#ifndef EXP_END_STAMPS
#define EXP_END_STAMPS 0   // diagnostics builds: per-CTA start / end stamps of every launch
#endif
#if EXP_FUSED_DBG == 3 || EXP_END_STAMPS
// diagnostics builds: per-CTA %globaltimer stamps [cta][slot] — 0 start, 1 push stores issued,
// 2 CTA barrier, 3 system-scope fence, 4 local counter add, 5 (last CTA of the rank) second fence +
// remote adds, 6 first arrival wait satisfied, 7 end — printed by the host after each launch
constexpr int DBG_SLOTS = 8;
__device__ unsigned long long g_dbg_stamps[160 * DBG_SLOTS];
#define DBG_STAMP(slot) (g_dbg_stamps[blockIdx.x * DBG_SLOTS + (slot)] = gtimer())
// a one-thread kernel launched right before / after the reconstruction (slot 1 / 2 of row 159)
__global__ void dbg_marker_kernel(int slot) { g_dbg_stamps[159 * DBG_SLOTS + slot] = gtimer(); }
#else
#define DBG_STAMP(slot) ((void)0)
#endif

template <typename GP>
__device__ __forceinline__ void fused_push(const GP& gp, int npeers, int me, uint32_t* calls) {
    if (threadIdx.x == 0) DBG_STAMP(0);
    const int64_t G = gridDim.x;
#ifndef EXP_PUSH_U
#define EXP_PUSH_U 4
#endif
    constexpr int U = EXP_PUSH_U;         // 16-byte loads in flight per thread before the stores
    char* const mc = gp.mc_base;
    for (int li = 0; li < gp.count; ++li) {
        const LayerParams& L = gp.L[li];
        const int64_t V = L.vx + L.vy;
        // this call's buffer: c & 1 of the window's call counter (device state); each thread
        // loads c itself (before this CTA arrives on the local counter, hence before the last CTA
        // advances c) so the load overlaps its first factor loads (no CTA barrier); the
        // producer thread keeps the values for its arrival targets and buffer choice
        calls[li] = load_calls(L.ctr);
        const size_t par = calls[li] & 1u;
        const int64_t beg = V * blockIdx.x / G, end = V * (blockIdx.x + 1) / G;
        for (int64_t v0 = beg + threadIdx.x; v0 < end; v0 += U * static_cast<int64_t>(blockDim.x)) {
            uint4 val[U];
            size_t off[U];
#pragma unroll
            for (int u = 0; u < U; ++u) {
                const int64_t v = v0 + u * static_cast<int64_t>(blockDim.x);
                if (v >= end) break;
                const bool isx = v < L.vx;
                const int64_t i = isx ? v : v - L.vx;
                if (gp.cast) {   // a1: fp32 -> bf16 round-to-nearest-even (DESIGN R11)
                    const float4* src = reinterpret_cast<const float4*>(isx ? L.srcX : L.srcY) + 2 * i;
                    const float4 lo = __ldcs(src), hi = __ldcs(src + 1);
                    val[u] = make_uint4(pack_bf16x2(lo.x, lo.y), pack_bf16x2(lo.z, lo.w),
                                        pack_bf16x2(hi.x, hi.y), pack_bf16x2(hi.z, hi.w));
                } else {
                    val[u] = __ldcs(reinterpret_cast<const uint4*>(isx ? L.srcX : L.srcY) + i);
                }
                off[u] = isx ? L.off_x + par * L.xbuf + (static_cast<size_t>(gp.slot) * L.vx + i) * 16
                             : L.off_dy + par * L.ybuf + (static_cast<size_t>(gp.slot) * L.vy + i) * 16;
            }
#pragma unroll
            for (int u = 0; u < U; ++u) {
                if (v0 + u * static_cast<int64_t>(blockDim.x) >= end) break;
                if (mc != nullptr) {
                    // NVLS: the switch replicates one store to every GPU (this one included)
                    asm volatile("multimem.st.global.v4.f32 [%0], {%1, %2, %3, %4};"
                                 :: "l"(mc_ptr(mc, L.win, off[u])), "r"(val[u].x), "r"(val[u].y),
                                    "r"(val[u].z), "r"(val[u].w) : "memory");
                } else {
                    for (int k = 0; k < npeers; ++k) {
                        const int p = (me + k) % npeers;
                        *reinterpret_cast<uint4*>(ncclGetLsaPointer(L.win, off[u], p)) = val[u];
                    }
                }
            }
        }
    }
    // One system-scope release for the whole slice (a fence per layer costs a NVLink round trip
    // each), then a hierarchical publish: every CTA adds 1 to a local counter and only the last
    // CTA of this rank to arrive adds 1 to every layer's arrival counter on every peer, so each
    // counter sees n remote atomics per call (not n * grid) and its target does not depend on
    // the grid size (ranks may launch different grids, e.g. sharded with uneven shards).
    if (threadIdx.x == 0) DBG_STAMP(1);
    __syncthreads();
    if (threadIdx.x == 0) {
        DBG_STAMP(2);
        asm volatile("fence.acq_rel.sys;" ::: "memory");
        DBG_STAMP(3);
        {
            // self-resetting: the last of the gridDim.x CTAs reads gridDim.x - 1 and leaves 0
            uint32_t old;
            asm volatile("atom.acq_rel.gpu.global.inc.u32 %0, [%1], %2;"
                         : "=r"(old) : "l"(gp.local_ctr), "r"(gridDim.x - 1) : "memory");
            DBG_STAMP(4);
            if (old != gridDim.x - 1) return;              // not the last CTA of this rank
            // every other CTA's slice was released at system scope before its local add,
            // which this acquire observed; make that cumulative for the peers
            asm volatile("fence.acq_rel.sys;" ::: "memory");
        }
        for (int li = 0; li < gp.count; ++li) {
            const size_t fo = gp.L[li].off_flag + WIN_ARRIVAL + 4 * (calls[li] & 1u);
            if (mc != nullptr) {
                asm volatile("multimem.red.relaxed.sys.global.add.u32 [%0], 1;"
                             :: "l"(mc_ptr(mc, gp.L[li].win, fo)) : "memory");
            } else {
                for (int k = 0; k < npeers; ++k) {
                    const int p = (me + k) % npeers;
                    uint32_t* ctr = static_cast<uint32_t*>(ncclGetLsaPointer(gp.L[li].win, fo, p));
                    asm volatile("red.relaxed.sys.global.add.u32 [%0], 1;" :: "l"(ctr) : "memory");
                }
            }
            // every CTA of this rank has read c (it arrived on the local counter after its push)
            atomicAdd(gp.L[li].flags + WIN_CALLS / 4, 1u);
        }
        DBG_STAMP(5);
    }
}

// Producer side: wait until every rank's every CTA has published layer li (acquire, system
// scope), then order those generic-proxy writes before the async-proxy (TMA) reads.
__device__ __forceinline__ void fused_wait(const LayerParams& L, int me, int npeers, uint32_t calls) {
    // every rank adds 1 per call to the counter of the call's buffer, and c is the same on every
    // rank, so call c is complete everywhere when the counter of buffer c & 1 reaches
    // n * (floor(c / 2) + 1)
    const uint32_t target = static_cast<uint32_t>(npeers) * (calls / 2u + 1u);
    const uint32_t* ctr = static_cast<const uint32_t*>(
        ncclGetLsaPointer(L.win, L.off_flag + WIN_ARRIVAL + 4 * (calls & 1u), me));
    const uint64_t t0 = gtimer();
    while (true) {
        uint32_t got;
        asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(got) : "l"(ctr) : "memory");
        if (static_cast<int32_t>(got - target) >= 0) break;
        if (gtimer() - t0 > 10ull * 1000 * 1000 * 1000) __trap();   // a peer never arrived (10 s)
    }
    asm volatile("fence.proxy.async.global;" ::: "memory");
}

template <int BN, int CTAS, bool OUT_BF16, bool SGD, bool FUSED, bool X3, bool LONGK, int MAXL>
__global__ void __launch_bounds__(NUM_THREADS, 1)
recon_tc_kernel(const __grid_constant__ GroupParamsT<MAXL> gp, const int npeers, const int me)
{
    constexpr int EP = OUT_BF16 || X3 ? 1 : (SGD ? EXP_SGD_EP : 2);   // epilogue chunks per round
    using C = Cfg<BN, CTAS, X3, EP, LONGK>;
    static_assert(!X3 || (CTAS == 1 && !FUSED), "3xTF32: single-CTA tiles, staged gather");
    static_assert(C::SMEM <= SMEM_MAX, "shared memory budget");
    extern __shared__ uint8_t smem_raw[];
    // 1024-byte alignment for the SWIZZLE_128B atoms
    const uint32_t base = (ptx::smem_addr(smem_raw) + 1023u) & ~1023u;
    const uint32_t s_stages = base;
    const uint32_t s_epi = s_stages + C::STAGES * C::STAGE_BYTES;
    const uint32_t s_bar = s_epi + C::EPI_BYTES;
    const uint32_t bar_full = s_bar;                       // [STAGES]
    const uint32_t bar_empty = s_bar + 8 * C::STAGES;      // [STAGES]
    const uint32_t bar_tfull = s_bar + 16 * C::STAGES;     // [ACC]
    const uint32_t bar_tempty = bar_tfull + 8 * C::ACC;    // [ACC]
    const uint32_t s_tmem_slot = bar_tempty + 8 * C::ACC;
    // dynamic tile schedule (one-CTA tiles, gp.sched set): the producer takes each CTA's next
    // tile from a global counter and hands it to the MMA issuer and the epilogue warps through a
    // SCHED_RING-deep smem ring (full: 1 arrival, empty: the MMA thread + every epilogue warp)
    const bool dyn = CTAS == 1 && gp.sched != nullptr;
    const uint32_t sch_full = s_bar + 512;                 // [SCHED_RING]
    const uint32_t sch_empty = sch_full + 8 * SCHED_RING;  // [SCHED_RING]
    const uint32_t s_sch = sch_empty + 8 * SCHED_RING;     // int [SCHED_RING]
    uint8_t* gen_base = smem_raw + (base - ptx::smem_addr(smem_raw));
    volatile uint32_t* tmem_slot_ptr =
        reinterpret_cast<volatile uint32_t*>(gen_base + (s_tmem_slot - base));
    const int unit = blockIdx.x / CTAS;      // this CTA's (pair's) index in the tile schedule
    const int nunits = gridDim.x / CTAS;
    volatile int* sch = reinterpret_cast<volatile int*>(gen_base + (s_sch - base));
    // the j-th tile of this CTA (-1: none left) for the MMA issuer (one thread) or an epilogue
    // warp (whole warp: every lane reads the slot before lane 0 frees it)
    // dyn: the first W - EXP_DYN_WAVES rounds (W = full rounds of tiles) are static round robin
    // and every role computes them itself; only the tail's tiles pass through the ring (index
    // j - jst). Only with many short tiles (W >= 8; see the producer).
    const int waves = gp.num_tiles / nunits;
    const int jst = dyn && waves >= 8 ? waves - EXP_DYN_WAVES : INT_MAX;   // static tiles per CTA
    auto next_tile = [&](int j, bool whole_warp) -> int {
        if (j < jst) {
            const int t = unit + j * nunits;
            return t < gp.num_tiles ? t : -1;
        }
        const int jr = j - jst;
        const int r = jr % SCHED_RING;
        ptx::mbar_wait(sch_full + 8 * r, (jr / SCHED_RING) & 1);
        const int t = sch[r];
        if (whole_warp) __syncwarp();
        if (!whole_warp || ptx::lane_id() == 0) ptx::mbar_arrive(sch_empty + 8 * r);
        return t;
    };

    if (EXP_END_STAMPS && threadIdx.x == 0) DBG_STAMP(1);   // first instruction
    const uint32_t warp = threadIdx.x >> 5;
    const uint32_t lane = threadIdx.x & 31;
    const uint32_t crank = CTAS == 2 ? ptx::cluster_ctarank() : 0;   // 0 = leader of the pair

    // ---- prologue (overlaps the previous kernel's tail under programmatic dependent launch)
    if (warp == 0 && lane == 0) {
        for (int i = 0; i < gp.count; ++i) {
            if (gp.L[i].M == 0) continue;             // empty shard: no tensor maps
            ptx::tma_prefetch_desc(&gp.L[i].tmA);
            ptx::tma_prefetch_desc(&gp.L[i].tmB);
        }
        for (int s = 0; s < C::STAGES; ++s) {
            ptx::mbar_init(bar_full + 8 * s, CTAS);      // pair: the leader's, armed by both
            ptx::mbar_init(bar_empty + 8 * s, 1);
        }
        for (int a = 0; a < C::ACC; ++a) {
            ptx::mbar_init(bar_tfull + 8 * a, 1);
            ptx::mbar_init(bar_tempty + 8 * a, NUM_EPI_WARPS * CTAS);   // pair: both CTAs drain
        }
        if (dyn)
            for (int r = 0; r < SCHED_RING; ++r) {
                ptx::mbar_init(sch_full + 8 * r, 1);
                ptx::mbar_init(sch_empty + 8 * r, 1 + NUM_EPI_WARPS);
            }
        ptx::fence_mbar_init();
    }
    if (warp == 1) {
        if constexpr (CTAS == 2) ptx::tmem_alloc_cg2<TMEM_COLS>(s_tmem_slot);
        else ptx::tmem_alloc<TMEM_COLS>(s_tmem_slot);
    }
    ptx::tc_fence_before();
    if constexpr (CTAS == 2) ptx::cluster_sync();
    else __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = *tmem_slot_ptr;
    // no global memory is touched before the previous grid in the stream has completed
    grid_dep_wait();
    if (EXP_END_STAMPS && threadIdx.x == 0) DBG_STAMP(0);
    // Diagnostics builds only (scripts/build_variant.sh -DEXP_FUSED_DBG=k, never the product):
    // 1 = no push and no wait, 2 = push without the arrival wait, 3 = phase stamps.
    uint32_t calls[MAXL];                     // window operands: each layer's call counter c
    if constexpr (FUSED) {
        if (EXP_FUSED_DBG != 1) fused_push(gp, npeers, me, calls);
        else for (int i = 0; i < gp.count; ++i) calls[i] = load_calls(gp.L[i].ctr);
    }

    if (warp == 0) {
        // ===================================================== TMA producer
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            uint32_t ready = 0;               // layers whose call counter (and, FUSED, factors) are known
            // dyn: the first W - 2 rounds (W = full rounds of tiles) are static round robin, the
            // last tiles are handed out by the counter, each fetched one tile ahead, so CTAs that
            // ran fast take the tail (VGG bucket n = 1: 84.7 -> 83.9 us; measured, all-dynamic
            // schedules lose 13 %: the counter's latency under full HBM write traffic is exposed
            // on every tile). Only with many short tiles (W >= 8): the BERT-L optimizer bucket
            // (W = 3, ~5 us tiles) is 0.8 us slower with a dynamic tail.
            const int slim = jst == INT_MAX ? 0 : jst * nunits;       // first dynamic tile
            int next = -1;
            for (int j = 0;; ++j) {
                int tile;
                if (j < jst) {
                    tile = unit + j * nunits;
                    if (tile >= gp.num_tiles) tile = -1;
                } else {
                    tile = next < gp.num_tiles ? next : -1;
                }
                if (j >= jst) {
                    const int jr = j - jst;
                    const int r = jr % SCHED_RING;
                    if (jr >= SCHED_RING) ptx::mbar_wait(sch_empty + 8 * r, ((jr / SCHED_RING) - 1) & 1);
                    sch[r] = tile;
                    ptx::mbar_arrive(sch_full + 8 * r);
                }
                if (tile < 0) break;
                // the following dynamic tile, fetched now: its latency overlaps this tile's loads
                if (j + 1 >= jst) next = slim + static_cast<int>(atomicAdd(gp.sched, 1u));
                const TileRef tr = locate<BN, CTAS>(gp, tile);
                const LayerParams& Lp = gp.L[tr.li];
                if (!(ready & (1u << tr.li))) {
                    // FUSED: c was read before this CTA's push (the kernel advances it later);
                    // a reconstruction of an earlier gather reads it here
                    if (!FUSED) calls[tr.li] = Lp.ctr_mode ? load_calls(Lp.ctr) : 1u;
                    if constexpr (FUSED) {
                        if (EXP_FUSED_DBG == 0 || EXP_FUSED_DBG == 3)
                            fused_wait(Lp, me, npeers, calls[tr.li]);
                        if (ready == 0) DBG_STAMP(6);
                    }
                    ready |= 1u << tr.li;
                }
                // window operands: the FUSED kernel reads its own gather's buffer (c & 1), a
                // later reconstruction the latest gather's ((c - 1) & 1)
                const uint32_t cc = calls[tr.li];
                const bool buf1 = Lp.ctr_mode == 2 ? (cc & 1u) : Lp.ctr_mode == 1 ? ((cc - 1u) & 1u) : false;
                const CUtensorMap* tmA = &Lp.tmA;
                const CUtensorMap* tmB = &Lp.tmB;
                const int krow = buf1 ? Lp.kbuf : 0;     // the buffer's first row in the maps
                const int nkb = gp.L[tr.li].num_k_blocks;
                for (int kb = 0; kb < nkb; ++kb) {
                    ptx::mbar_wait(bar_empty + 8 * stage, phase ^ 1);
                    const uint32_t fb = bar_full + 8 * stage;
                    const uint32_t sa = s_stages + stage * C::STAGE_BYTES;
                    const uint32_t sb = sa + C::A_BYTES;
                    const int am0 = tr.m0 + static_cast<int>(crank) * BM;          // my A rows
                    const int bn0 = tr.n0 + static_cast<int>(crank) * (BN / CTAS); // my B cols
                    if constexpr (CTAS == 2) {
                        // both halves land on the leader's barrier, which the leader arms for
                        // the pair's bytes; the peer adds its arrival (count 2)
                        const uint32_t fbl = ptx::mapa(fb, 0);
                        if (crank == 0) ptx::mbar_arrive_expect_tx(fb, CTAS * C::STAGE_BYTES);
                        else ptx::mbar_arrive_cluster(fbl);
                        if (gp.L[tr.li].box3) {
                            // all MN chunks of an operand in one 3-D request (16 KB each)
                            ptx::tma_load_3d_cg2(sa, tmA, fbl, 0, kb * C::BK + krow, am0 / C::ELEMS);
                            ptx::tma_load_3d_cg2(sb, tmB, fbl, 0, kb * C::BK + krow, bn0 / C::ELEMS);
                            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
                            continue;
                        }
#pragma unroll
                        for (int c = 0; c < C::A_CHUNKS; ++c)
                            ptx::tma_load_2d_cg2(sa + c * C::CHUNK_BYTES, tmA, fbl, am0 + C::ELEMS * c, kb * C::BK + krow);
#pragma unroll
                        for (int c = 0; c < C::B_CHUNKS; ++c)
                            ptx::tma_load_2d_cg2(sb + c * C::CHUNK_BYTES, tmB, fbl, bn0 + C::ELEMS * c, kb * C::BK + krow);
                    } else {
                        ptx::mbar_arrive_expect_tx(fb, C::STAGE_BYTES);
                        if (!X3 && gp.L[tr.li].box3) {
                            ptx::tma_load_3d(sa, tmA, fb, 0, kb * C::BK + krow, am0 / C::ELEMS);
                            ptx::tma_load_3d(sb, tmB, fb, 0, kb * C::BK + krow, bn0 / C::ELEMS);
                            if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
                            continue;
                        }
#pragma unroll
                        for (int h = 0; h < C::HALVES; ++h) {     // X3: h = 1 loads the lo rows
                            const int kr = kb * C::BK + h * gp.L[tr.li].k_lo + krow;
#pragma unroll
                            for (int c = 0; c < C::A_CHUNKS; ++c)
                                ptx::tma_load_2d(sa + (h * C::A_CHUNKS + c) * C::CHUNK_BYTES, tmA, fb,
                                                 am0 + C::ELEMS * c, kr);
#pragma unroll
                            for (int c = 0; c < C::B_CHUNKS; ++c)
                                ptx::tma_load_2d(sb + (h * C::B_CHUNKS + c) * C::CHUNK_BYTES, tmB, fb,
                                                 bn0 + C::ELEMS * c, kr);
                        }
                    }
                    if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
                }
            }
            if (jst != INT_MAX) {
                // this CTA's last fetch has returned: the last CTA to get here re-arms the
                // counters for the next launch (stream order / griddepcontrol.wait keep launches apart)
                __threadfence();
                if (atomicAdd(gp.sched + 1, 1u) == gridDim.x - 1) {
                    atomicExch(gp.sched, 0u);
                    atomicExch(gp.sched + 1, 0u);
                }
            }
        }
    } else if (warp == 1) {
        // ===================================================== MMA issuer (one thread; the
        // leader CTA's only, for a pair)
        if (lane == 0 && crank == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int acc = 0;
            uint32_t acc_phase = 0;
            for (int j = 0;; ++j) {
                const int tile = next_tile(j, false);
                if (tile < 0) break;
                const int nkb = gp.L[locate<BN, CTAS>(gp, tile).li].num_k_blocks;
                ptx::mbar_wait(bar_tempty + 8 * acc, acc_phase ^ 1);   // epilogue drained it
                ptx::tc_fence_after();
                const uint32_t d_tmem = tmem_base + acc * C::ACC_COLS;
                for (int kb = 0; kb < nkb; ++kb) {
                    ptx::mbar_wait(bar_full + 8 * stage, phase);        // TMA landed
                    ptx::tc_fence_after();
                    const uint32_t sa = s_stages + stage * C::STAGE_BYTES;
                    const uint32_t sb = sa + C::A_BYTES;
#pragma unroll
                    for (int kk = 0; kk < C::BK / C::KMMA; ++kk) {
                        // KMMA rows of 128 B per UMMA_K step (bf16: two 8-row swizzle atoms)
                        const uint32_t ko = kk * C::KMMA * 128;
                        const uint64_t ad = ptx::sw128_desc(sa + ko, C::CHUNK_BYTES, C::SBO, C::DLAYOUT);
                        const uint64_t bd = ptx::sw128_desc(sb + ko, C::CHUNK_BYTES, C::SBO, C::DLAYOUT);
                        if constexpr (X3) {
                            const uint64_t adl = ptx::sw128_desc(sa + C::A_CHUNKS * C::CHUNK_BYTES + ko,
                                                                 C::CHUNK_BYTES, C::SBO, C::DLAYOUT);
                            const uint64_t bdl = ptx::sw128_desc(sb + C::B_CHUNKS * C::CHUNK_BYTES + ko,
                                                                 C::CHUNK_BYTES, C::SBO, C::DLAYOUT);
                            ptx::mma_tf32(d_tmem + BN, adl, bd, C::IDESC, (kb | kk) != 0);  // lo * hi
                            ptx::mma_tf32(d_tmem + BN, ad, bdl, C::IDESC, 1);               // hi * lo
                            ptx::mma_tf32(d_tmem, ad, bd, C::IDESC, (kb | kk) != 0);        // hi * hi
                        } else if constexpr (CTAS == 2) {
                            ptx::mma_f16_cg2(d_tmem, ad, bd, C::IDESC, (kb | kk) != 0);
                        } else {
                            ptx::mma_f16(d_tmem, ad, bd, C::IDESC, (kb | kk) != 0);
                        }
                    }
                    // frees the smem slot (both CTAs' slots for a pair)
                    if constexpr (CTAS == 2) ptx::mma_commit_cg2_mc(bar_empty + 8 * stage, 0x3);
                    else ptx::mma_commit(bar_empty + 8 * stage);
                    if (++stage == C::STAGES) { stage = 0; phase ^= 1; }
                }
                // accumulator ready (both CTAs' epilogues for a pair)
                if constexpr (CTAS == 2) ptx::mma_commit_cg2_mc(bar_tfull + 8 * acc, 0x3);
                else ptx::mma_commit(bar_tfull + 8 * acc);
                if (++acc == C::ACC) { acc = 0; acc_phase ^= 1; }
            }
            // all MMAs of this CTA are issued: let the next kernel in the stream start launching
            grid_dep_launch();
        }
    } else {
        // ===================================================== epilogue warps
        // TMEM -> registers (one output row per lane) -> x alpha (-> RNE bf16) -> 128B-swizzled
        // smem transpose -> coalesced 16-byte streaming stores, four FULL 128-byte lines per warp
        // instruction. (Measured: direct 8-byte stores from the 16x256b TMEM layout — whole
        // 32-B sectors but 8 lines per instruction — write HBM ~15 % slower at K = 32.)
        const int ew = warp - 2;                 // 0..7
        const int quad = warp & 3;               // TMEM lane quadrant this warp may access
        const int half = ew >> 2;                // which column group of the tile
        constexpr int GC = BN / EPI_GROUPS;      // columns per group
        const uint32_t sbuf = s_epi + ew * C::EPI_BUF_BYTES;
        constexpr int ESZ = OUT_BF16 ? 2 : 4;
        constexpr int COLS_PER_CHUNK = 128 / ESZ;               // 128 bytes of output per row
        constexpr int CHUNKS = GC / COLS_PER_CHUNK;
        static_assert(CHUNKS >= 1, "epilogue column group narrower than one 128-byte chunk");
        constexpr int VEC = 16 / ESZ;                           // output elements per 16 B
        constexpr int PAIR = EP;                                // chunks staged per round
        const int sub = lane >> 3;               // row within a 4-row group (write-out phase)
        const int cj = lane & 7;                 // 16-byte column slot (write-out phase)
        int acc = 0;
        uint32_t acc_phase = 0;
        const float lr = gp.lr, mu = gp.mu, wd = gp.wd;
        const uint32_t tempty_leader = CTAS == 2 ? ptx::mapa(bar_tempty, 0) : bar_tempty;
        for (int j = 0;; ++j) {
            const int tile = next_tile(j, true);
            if (tile < 0) break;
            const TileRef tr = locate<BN, CTAS>(gp, tile);
            // this tile's layer parameters, read once into registers
            const LayerParams& lp = gp.L[tr.li];
            uint8_t* const Cp = static_cast<uint8_t*>(lp.C);
            float* const Wp = lp.W;
            float* const Vp = lp.V;
            const int M = lp.M, N = lp.N;
            const float alpha = lp.alpha;
            const int n0 = tr.n0;
            const int row0 = tr.m0 + static_cast<int>(crank) * BM + 32 * quad;  // first row
#ifndef EXP_OPT_PREFETCH
#define EXP_OPT_PREFETCH 0
#endif
            if constexpr (SGD && EXP_OPT_PREFETCH) {
                // Diagnostics builds (the round-1 product, before the hoisted loads below): pull
                // this warp's rows of the optimizer state into L2 while the accumulator is still
                // being computed. With the loads hoisted it costs 1-2 us on the BERT-L bucket.
                auto prefetch_tile = [&](int t) {
                    const TileRef pr = locate<BN, CTAS>(gp, t);
                    const LayerParams& pl = gp.L[pr.li];
                    const int r = pr.m0 + static_cast<int>(crank) * BM + 32 * quad + static_cast<int>(lane);
                    const int c0 = pr.n0 + half * GC;
                    if (r < pl.M && c0 < pl.N) {
                        const int64_t base = static_cast<int64_t>(r) * pl.N + c0;
                        const int lines = ((pl.N - c0 < GC ? pl.N - c0 : GC) * 4 + 127) / 128;
                        for (int j = 0; j < lines; ++j) {
                            ptx::prefetch_l2(pl.W + base + 32 * j);
                            ptx::prefetch_l2(pl.V + base + 32 * j);
                            if (gp.opt == 2) ptx::prefetch_l2(pl.Mm + base + 32 * j);
                        }
                    }
                };
                if (EXP_OPT_PREFETCH == 1 || tile == unit) prefetch_tile(tile);
                if (EXP_OPT_PREFETCH == 2 && tile + nunits < gp.num_tiles) prefetch_tile(tile + nunits);
            }
#ifndef EXP_OPT_HOIST
#define EXP_OPT_HOIST 1
#endif
            // HOIST: the optimizer state of a full chunk does not depend on the accumulator —
            // all 8 rows' loads (per lane) are issued before the accumulator wait / TMEM read /
            // transpose, so their latency overlaps those and the Adam math of the previous chunk
            // (measured, scripts/opt_epilogue_ab.py: Adam 59.5 -> 48.0 us on the BERT-L bucket)
            constexpr bool HOIST = SGD && EXP_OPT_HOIST;
            if (!HOIST) {
                ptx::mbar_wait(bar_tfull + 8 * acc, acc_phase);
                ptx::tc_fence_after();
            }
            const uint32_t t_row = tmem_base + (static_cast<uint32_t>(32 * quad) << 16) + acc * C::ACC_COLS;
            // chunks of this warp's column half that hold any output column (warp-uniform)
            int nch = (N - (n0 + half * GC) + COLS_PER_CHUNK - 1) / COLS_PER_CHUNK;
            nch = nch < 0 ? 0 : (nch > CHUNKS ? CHUNKS : nch);
            if (EXP_EPI_MODE == 2) nch = 0;
            if (nch == 0) {                       // nothing to read: release the accumulator
                if (HOIST) {
                    ptx::mbar_wait(bar_tfull + 8 * acc, acc_phase);
                    ptx::tc_fence_after();
                }
                ptx::tc_fence_before();
                __syncwarp();
                if (lane == 0) {
                    if constexpr (CTAS == 2) ptx::mbar_arrive_cluster(tempty_leader + 8 * acc);
                    else ptx::mbar_arrive(bar_tempty + 8 * acc);
                }
            }
#pragma unroll 1
            for (int ch = 0; ch < nch; ch += PAIR) {
                const int np = (nch - ch) < PAIR ? (nch - ch) : PAIR;    // chunks this round
                [[maybe_unused]] float4 hw[8], hv[8], hm[8];
                [[maybe_unused]] const bool hfull =
                    row0 + 32 <= M && n0 + half * GC + (ch + 1) * COLS_PER_CHUNK <= N;
                if constexpr (HOIST) {
                    if (hfull) {
                        const int64_t o = static_cast<int64_t>(row0 + sub) * N + n0 + half * GC +
                                          ch * COLS_PER_CHUNK + cj * VEC;
                        const float4* wp4 = reinterpret_cast<const float4*>(Wp + o);
                        const float4* vp4 = reinterpret_cast<const float4*>(Vp + o);
                        const int64_t gs = static_cast<int64_t>(N);          // 4 rows, in float4
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            hw[i] = __ldcs(wp4 + i * gs);
                            hv[i] = __ldcs(vp4 + i * gs);
                        }
                        if (gp.opt == 2) {
                            const float4* mp4 = reinterpret_cast<const float4*>(lp.Mm + o);
#pragma unroll
                            for (int i = 0; i < 8; ++i) hm[i] = __ldcs(mp4 + i * gs);
                        }
                    }
#ifndef EXP_OPT_PF_NEXT
#define EXP_OPT_PF_NEXT 1
#endif
                    if (EXP_OPT_PF_NEXT && CHUNKS >= 4 && ch + 1 < nch &&
                        row0 + static_cast<int>(lane) < M) {
                        // wide tiles (4 chunks per warp): the next chunk's rows (one 128-B line per
                        // lane and array) into L2 as well, so its hoisted loads hit L2 (measured,
                        // scripts/opt_epilogue_ab.py: BERT-L bucket at K = 8B SGD 42.0 -> 37.9 us,
                        // Adam 62.5 -> 52.3; with 2 chunks per warp (K = B) no gain, Adam +2 us)
                        const int64_t o = static_cast<int64_t>(row0 + lane) * N + n0 + half * GC +
                                          (ch + 1) * COLS_PER_CHUNK;
                        ptx::prefetch_l2(Wp + o);
                        ptx::prefetch_l2(Vp + o);
                        if (gp.opt == 2) ptx::prefetch_l2(lp.Mm + o);
                    }
#ifndef EXP_OPT_PF_TILE
#define EXP_OPT_PF_TILE 1
#endif
                    if (EXP_OPT_PF_TILE && (CHUNKS >= 4 || gp.opt == 1) && ch + 1 == nch &&
                        tile + nunits < gp.num_tiles) {
                        // at a tile's last chunk: the first chunk rows of this unit's next tile in
                        // the static order (with a dynamic tail the guess may miss; only a hint)
                        // into L2. Measured (scripts/opt_epilogue_ab.py): BERT-L SGD at K = B
                        // 30.9-31.7 -> 29.7 us, Adam at K = 8B 52.3 -> 50.2, Transformer SGD / Adam
                        // at K = 8B 89 -> 87 / 120 -> 117; Adam on 2-chunk tiles +1-2 us (skipped)
                        const TileRef nt = locate<BN, CTAS>(gp, tile + nunits);
                        const LayerParams& nl = gp.L[nt.li];
                        const int r = nt.m0 + static_cast<int>(crank) * BM + 32 * quad + static_cast<int>(lane);
                        const int c0 = nt.n0 + half * GC;
                        if (r < nl.M && c0 < nl.N) {
                            const int64_t o = static_cast<int64_t>(r) * nl.N + c0;
                            ptx::prefetch_l2(nl.W + o);
                            ptx::prefetch_l2(nl.V + o);
                            if (gp.opt == 2) ptx::prefetch_l2(nl.Mm + o);
                        }
                    }
                    if (ch == 0) {
                        ptx::mbar_wait(bar_tfull + 8 * acc, acc_phase);
                        ptx::tc_fence_after();
                    }
                }
                uint32_t w[PAIR][32];                                    // 128 B of row per chunk
                // ---- TMEM -> registers: every load of the round issued before one wait
#pragma unroll
                for (int q = 0; q < PAIR; ++q) {
                    if (q >= np) break;
                    const uint32_t tc = t_row + half * GC + (ch + q) * COLS_PER_CHUNK;
                    if constexpr (OUT_BF16) {
                        uint32_t r0[32], r1[32];
                        ptx::tmem_ld_32x32b_x32(tc, r0);
                        ptx::tmem_ld_32x32b_x32(tc + 32, r1);
                        ptx::tmem_wait_ld();
                        if constexpr (X3) {       // + the lo accumulator, one fp32 add (RN)
                            uint32_t l[32];
                            ptx::tmem_ld_32x32b_x32(tc + BN, l);
                            ptx::tmem_wait_ld();
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                r0[i] = __float_as_uint(__fadd_rn(__uint_as_float(r0[i]), __uint_as_float(l[i])));
                            ptx::tmem_ld_32x32b_x32(tc + BN + 32, l);
                            ptx::tmem_wait_ld();
#pragma unroll
                            for (int i = 0; i < 32; ++i)
                                r1[i] = __float_as_uint(__fadd_rn(__uint_as_float(r1[i]), __uint_as_float(l[i])));
                        }
#pragma unroll
                        for (int i = 0; i < 16; ++i) {
                            w[q][i] = pack_bf16x2(__fmul_rn(__uint_as_float(r0[2 * i]), alpha),
                                                  __fmul_rn(__uint_as_float(r0[2 * i + 1]), alpha));
                            w[q][16 + i] = pack_bf16x2(__fmul_rn(__uint_as_float(r1[2 * i]), alpha),
                                                       __fmul_rn(__uint_as_float(r1[2 * i + 1]), alpha));
                        }
                    } else {
                        ptx::tmem_ld_32x32b_x32(tc, w[q]);
                    }
                }
                if constexpr (!OUT_BF16) {
                    ptx::tmem_wait_ld();
                    if constexpr (X3) {           // + the lo accumulator (PAIR = 1), one fp32 add
                        uint32_t l[32];
                        ptx::tmem_ld_32x32b_x32(t_row + half * GC + ch * COLS_PER_CHUNK + BN, l);
                        ptx::tmem_wait_ld();
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            w[0][i] = __float_as_uint(__fadd_rn(__uint_as_float(w[0][i]), __uint_as_float(l[i])));
                    }
#pragma unroll
                    for (int q = 0; q < PAIR; ++q)
#pragma unroll
                        for (int i = 0; i < 32; ++i)
                            w[q][i] = __float_as_uint(__fmul_rn(__uint_as_float(w[q][i]), alpha));
                }
                if (ch + np >= nch) {
                    // last TMEM read of this accumulator by this warp: hand it back to the MMA
                    ptx::tc_fence_before();
                    __syncwarp();
                    if (lane == 0) {
                    if constexpr (CTAS == 2) ptx::mbar_arrive_cluster(tempty_leader + 8 * acc);
                    else ptx::mbar_arrive(bar_tempty + 8 * acc);
                }
                }
                if constexpr (EXP_EPI_MODE == 3 || EXP_EPI_MODE == 4) {
                    // diagnostics: 3 = direct 16-B stores of each lane's row segment (no smem),
                    // 4 = TMEM read only
#pragma unroll
                    for (int q = 0; q < PAIR; ++q) {
                        if (q >= np) break;
                        const int gc = n0 + half * GC + (ch + q) * COLS_PER_CHUNK;
                        const int r = row0 + static_cast<int>(lane);
                        if (EXP_EPI_MODE == 4) {
                            uint32_t x = 0;
                            for (int i = 0; i < 32; ++i) x ^= w[q][i];
                            if (x == 0x7f7f7f7fu && r < 0) Cp[0] = 1;
                            continue;
                        }
                        if (r >= M || gc + COLS_PER_CHUNK > N) continue;
                        uint4* g = reinterpret_cast<uint4*>(Cp + (static_cast<int64_t>(r) * N + gc) * ESZ);
#pragma unroll
                        for (int j = 0; j < 8; ++j)
                            __stcs(g + j, make_uint4(w[q][4 * j], w[q][4 * j + 1], w[q][4 * j + 2], w[q][4 * j + 3]));
                    }
                    continue;
                }
                // ---- registers -> 128B-swizzled smem (row `lane`), conflict-free
                __syncwarp();                     // previous round's smem reads are done
#pragma unroll
                for (int q = 0; q < PAIR; ++q) {
                    if (q >= np) break;
                    const uint32_t rowaddr = sbuf + q * 4096 + lane * 128;
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        ptx::st_shared_v4(rowaddr + ((j ^ (lane & 7)) << 4), w[q][4 * j],
                                          w[q][4 * j + 1], w[q][4 * j + 2], w[q][4 * j + 3]);
                }
                __syncwarp();
                // ---- smem -> global: lane reads 16 B of row 4i+sub; 4 full lines per store
#pragma unroll
                for (int q = 0; q < PAIR; ++q) {
                    if (q >= np) break;
                    const int gcol = n0 + half * GC + (ch + q) * COLS_PER_CHUNK + cj * VEC;
                    const bool col_ok = gcol < N;   // N % 8 == 0: a 16-B slot is all in or out
                    const int64_t off0 = static_cast<int64_t>(row0 + sub) * N + gcol;
                    const int64_t step = 4 * static_cast<int64_t>(N);
                    // warp-uniform: every row and column of this 32 x 128-B chunk is in range
                    const bool full = row0 + 32 <= M &&
                                      n0 + half * GC + (ch + q + 1) * COLS_PER_CHUNK <= N;
                    const uint32_t sq = sbuf + q * 4096 + sub * 128;
                    const uint32_t sw0 = (cj ^ sub) << 4, sw1 = (cj ^ (sub + 4)) << 4;
                    if (EXP_EPI_MODE == 1 && full && !SGD) {
                        uint32_t a, b, c, d, x = 0;
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            ptx::ld_shared_v4(sq + i * 512 + ((i & 1) ? sw1 : sw0), a, b, c, d);
                            x ^= a ^ b ^ c ^ d;
                        }
                        if (x == 0x7f7f7f7fu && row0 < 0) Cp[0] = 1;   // keep the loads
                        continue;
                    }
                    if (full && !SGD) {
                        // fast path (all but the edge tiles): no per-store predicates, the global
                        // address advances by 4 rows per store
                        uint4* gp4 = reinterpret_cast<uint4*>(Cp + off0 * ESZ);
                        const int64_t gstep = step * ESZ / 16;
#pragma unroll
                        for (int i = 0; i < 8; ++i) {
                            uint32_t a, b, c, d;
                            ptx::ld_shared_v4(sq + i * 512 + ((i & 1) ? sw1 : sw0), a, b, c, d);
                            __stcs(gp4 + i * gstep, make_uint4(a, b, c, d));
                        }
                        continue;
                    }
                    if constexpr (SGD) {
                        if (full && gp.opt == 2) {
                            // E3 Adam fast path: W, m, v of four rows in flight at a time
                            float4* wp4 = reinterpret_cast<float4*>(Wp + off0);
                            float4* mp4 = reinterpret_cast<float4*>(lp.Mm + off0);
                            float4* vp4 = reinterpret_cast<float4*>(Vp + off0);
                            const int64_t gstep = step / 4;
#pragma unroll
                            for (int hh = 0; hh < 2; ++hh) {
                                float4 wv[4], mv[4], vv[4];
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    const int r = 4 * hh + i;
                                    if constexpr (HOIST) {
                                        wv[i] = hw[r];
                                        mv[i] = hm[r];
                                        vv[i] = hv[r];
                                    } else {
                                        wv[i] = __ldcs(wp4 + r * gstep);
                                        mv[i] = __ldcs(mp4 + r * gstep);
                                        vv[i] = __ldcs(vp4 + r * gstep);
                                    }
                                }
#pragma unroll
                                for (int i = 0; i < 4; ++i) {
                                    const int r = 4 * hh + i;
                                    uint32_t dw[4];
                                    ptx::ld_shared_v4(sq + r * 512 + ((r & 1) ? sw1 : sw0), dw[0],
                                                      dw[1], dw[2], dw[3]);
                                    float* wf = reinterpret_cast<float*>(&wv[i]);
                                    float* mf = reinterpret_cast<float*>(&mv[i]);
                                    float* vf = reinterpret_cast<float*>(&vv[i]);
#pragma unroll
                                    for (int e = 0; e < 4; ++e)
                                        adam_update(__uint_as_float(dw[e]), wf[e], mf[e], vf[e], gp.adam);
                                    __stcs(wp4 + r * gstep, wv[i]);
                                    __stcs(mp4 + r * gstep, mv[i]);
                                    __stcs(vp4 + r * gstep, vv[i]);
                                    if (Cp != nullptr)
                                        __stcs(reinterpret_cast<uint4*>(Cp + (off0 + r * step) * ESZ),
                                               make_uint4(dw[0], dw[1], dw[2], dw[3]));
                                }
                            }
                            continue;
                        }
                        if (full) {
                            // E2 fast path: all 16 loads of W and v in flight before any math
                            // (the per-row load -> update -> store chain would serialise on the
                            // HBM latency 8 times per chunk)
                            float4* wp4 = reinterpret_cast<float4*>(Wp + off0);
                            float4* vp4 = reinterpret_cast<float4*>(Vp + off0);
                            const int64_t gstep = step / 4;
#ifndef EXP_SGD_ROWS
#define EXP_SGD_ROWS 4
#endif
                            constexpr int RW = EXP_SGD_ROWS;     // rows of W, v in flight
#pragma unroll
                            for (int h0 = 0; h0 < 8; h0 += RW) {
                            float4 wv[RW], vv[RW];
#pragma unroll
                            for (int i = 0; i < RW; ++i) {
                                if constexpr (HOIST) {
                                    wv[i] = hw[h0 + i];
                                    vv[i] = hv[h0 + i];
                                } else {
                                    wv[i] = __ldcs(wp4 + (h0 + i) * gstep);
                                    vv[i] = __ldcs(vp4 + (h0 + i) * gstep);
                                }
                            }
#pragma unroll
                            for (int ii = 0; ii < RW; ++ii) {
                                const int i = h0 + ii;
                                uint32_t dw[4];
                                ptx::ld_shared_v4(sq + i * 512 + ((i & 1) ? sw1 : sw0), dw[0],
                                                  dw[1], dw[2], dw[3]);
                                float* wf = reinterpret_cast<float*>(&wv[ii]);
                                float* vf = reinterpret_cast<float*>(&vv[ii]);
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    // E2 (R14): g = dW + wd*W ; v = mu*v + g ; W -= lr*v
                                    const float g = __fadd_rn(__uint_as_float(dw[e]), __fmul_rn(wd, wf[e]));
                                    vf[e] = __fadd_rn(__fmul_rn(mu, vf[e]), g);
                                    wf[e] = __fsub_rn(wf[e], __fmul_rn(lr, vf[e]));
                                }
                                __stcs(wp4 + i * gstep, wv[ii]);
                                __stcs(vp4 + i * gstep, vv[ii]);
                                if (Cp != nullptr)
                                    __stcs(reinterpret_cast<uint4*>(Cp + (off0 + i * step) * ESZ),
                                           make_uint4(dw[0], dw[1], dw[2], dw[3]));
                            }
                            }
                            continue;
                        }
                    }
#pragma unroll
                    for (int i = 0; i < 8; ++i) {
                        const int r = 4 * i + sub;
                        uint32_t a, b, c, d;
                        ptx::ld_shared_v4(sq + i * 512 + ((i & 1) ? sw1 : sw0), a, b, c, d);
                        if (!col_ok || row0 + r >= M) continue;
                        const int64_t off = off0 + i * step;
                        if constexpr (SGD) {
                            float4* wp = reinterpret_cast<float4*>(Wp + off);
                            float4* vp = reinterpret_cast<float4*>(Vp + off);
                            float4 wv = __ldcs(wp);
                            float4 vv = __ldcs(vp);
                            const float dv[4] = {__uint_as_float(a), __uint_as_float(b),
                                                 __uint_as_float(c), __uint_as_float(d)};
                            float* wf = reinterpret_cast<float*>(&wv);
                            float* vf = reinterpret_cast<float*>(&vv);
                            if (gp.opt == 2) {
                                // E3 Adam (R22)
                                float4* mp = reinterpret_cast<float4*>(lp.Mm + off);
                                float4 mv = __ldcs(mp);
                                float* mf = reinterpret_cast<float*>(&mv);
#pragma unroll
                                for (int e = 0; e < 4; ++e) adam_update(dv[e], wf[e], mf[e], vf[e], gp.adam);
                                __stcs(mp, mv);
                            } else {
                                // E2 (R14): g = dW + wd*W ; v = mu*v + g ; W -= lr*v   (fp32)
#pragma unroll
                                for (int e = 0; e < 4; ++e) {
                                    const float g = __fadd_rn(dv[e], __fmul_rn(wd, wf[e]));
                                    vf[e] = __fadd_rn(__fmul_rn(mu, vf[e]), g);
                                    wf[e] = __fsub_rn(wf[e], __fmul_rn(lr, vf[e]));
                                }
                            }
                            __stcs(wp, wv);
                            __stcs(vp, vv);
                            if (Cp == nullptr) continue;
                        }
                        __stcs(reinterpret_cast<uint4*>(Cp + off * ESZ), make_uint4(a, b, c, d));
                    }
                }
            }
            if (++acc == C::ACC) { acc = 0; acc_phase ^= 1; }
        }
    }

    ptx::tc_fence_before();
    if constexpr (CTAS == 2) ptx::cluster_sync();   // the leader's MMAs into the peer are done
    else __syncthreads();
    ptx::tc_fence_after();
    if ((FUSED || EXP_END_STAMPS) && threadIdx.x == 0) DBG_STAMP(7);
    if (warp == 1) {
        if constexpr (CTAS == 2) ptx::tmem_dealloc_cg2<TMEM_COLS>(tmem_base);
        else ptx::tmem_dealloc<TMEM_COLS>(tmem_base);
    }
}

// ------------------------------------------------------------------ host side
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* f = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

// Row-major rows x cols matrix; box = box_cols x box_rows; 128-byte swizzle.
bool encode_2d(CUtensorMap* m, const void* ptr, CUtensorMapDataType dt, int esize, int64_t rows,
               int64_t cols, int box_cols, int box_rows, int64_t ld = 0,
               CUtensorMapSwizzle swz = CU_TENSOR_MAP_SWIZZLE_128B) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(cols), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>((ld ? ld : cols) * esize)};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(box_cols), static_cast<cuuint32_t>(box_rows)};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(m, dt, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, swz,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// The same operand as a 3-D map {64 elements, rows, cols / 64 chunks} with a 128-byte chunk
// stride: one box of `chunks` chunks x box_rows rows lands as consecutive 128-B-swizzled chunks,
// exactly the 2-D layout, in one request. Needs cols % 64 == 0 (no chunk straddles a row end).
bool encode_3d(CUtensorMap* m, const void* ptr, int64_t rows, int64_t cols, int box_rows,
               int chunks, int64_t ld = 0) {
    auto enc = get_encode();
    if (!enc) return false;
    cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows), static_cast<cuuint64_t>(cols / 64)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>((ld ? ld : cols) * 2), 128};
    cuuint32_t box[3] = {64, static_cast<cuuint32_t>(box_rows), static_cast<cuuint32_t>(chunks)};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(ptr), dims, strides,
                     box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                     CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// one CTA (pair) per SM (TPC), at most one per tile; a FUSED launch keeps at least one unit even
// with no tiles (every rank must push its factors)
#ifndef EXP_RECON_SMS
#define EXP_RECON_SMS 0   // diagnostics builds: SMs the persistent grid may use (0 = all)
#endif
int grid_for(int tiles, int ctas, bool fused) {
    const int units = (EXP_RECON_SMS ? EXP_RECON_SMS : num_sms()) / ctas;
    int g = tiles < units ? tiles : units;
    if (fused && g < 1) g = 1;
    return ctas * g;
}

int tiles_for(const ReconArgs* a, int count, int bn, int ctas) {
    int64_t tiles = 0;
    for (int i = 0; i < count; ++i)
        tiles += ((a[i].M + BM * ctas - 1) / (BM * ctas)) * ((a[i].N + bn - 1) / bn);
    return static_cast<int>(tiles);
}

bool use_wide(const ReconArgs* a, int count) {
    int64_t kmax = 0;
    for (int i = 0; i < count; ++i) kmax = a[i].K > kmax ? a[i].K : kmax;
    // Small K (the HBM-write-bound regime of the paper's small-batch layers): BN = 128 tiles,
    // 4 TMEM accumulators, finer tail. K >= 96: BN = 256 (and a CTA pair, cta_group::2, from
    // K = 192): the operand re-reads from L2 bind first there (fc6 at K = 256, one CTA: 102 us
    // at BN = 128, 88 us at BN = 256 with L2 throughput saturated); the pair halves B's again.
    bool wide = kmax >= 96;
    // Optimizer epilogues (16-24 B of HBM traffic per dW element) stay on 128 x 128 tiles up to
    // K = 512: BERT-L E2 bucket (scripts/sgd_bucket_time.py) 31.7 / 33.8 / 35.9 us at K = 128 /
    // 256 / 512 vs 35.7 / 37.9 / 40.0 with wide tiles; at K = 1024 wide pairs win (42.0 vs 46.0)
    if (a[0].sgd) wide = kmax > 512;
    if (EXP_RECON_BN) wide = EXP_RECON_BN == 256;   // diagnostics builds
    return wide;
}

int use_ctas(const ReconArgs* a, int count) {
    if (!use_wide(a, count)) return 1;
    if (EXP_RECON_CTAS) return EXP_RECON_CTAS == 1 ? 1 : 2;   // diagnostics builds
    int64_t kmax = 0;
    for (int i = 0; i < count; ++i) kmax = a[i].K > kmax ? a[i].K : kmax;
    // measured on the VGG-19 bucket (scripts/tile_sweep.py): K = 128 one CTA x 256 columns 96 us
    // (pairs 101, 128-col tiles 99); K = 256 pairs 107 us (one CTA 112)
    return kmax >= 192 ? 2 : 1;
}

// Big (256 x 256 pair) tiles only when they fill at least half the TPCs; a small-output bucket
// (e.g. Transformer FFN at K = 256: 16 pair tiles) runs faster on 4x as many 128 x 128 tiles.
// Measured (scripts/recon_time.py): fc8 4096 x 1000 at K = 256 (64 pair tiles) 13.3 vs 15.3 us,
// AlexNet / VGG-16 fc8 at K = 512 15.3 vs 19.4 us with big tiles from half a round (was: a full
// round); fc7, FFN, out-proj unchanged.
bool big_tiles(const ReconArgs* a, int count) {
    if (!use_wide(a, count)) return false;
    if (EXP_RECON_BN) return true;   // diagnostics builds force it
    const int ctas = use_ctas(a, count);
#ifndef EXP_BIG_FRAC
#define EXP_BIG_FRAC 2   // big tiles from 1 / EXP_BIG_FRAC of a full round of units
#endif
    return tiles_for(a, count, 256, ctas) * EXP_BIG_FRAC >= num_sms() / ctas;
}

template <int BN, int CTAS, bool OUT_BF16, bool SGD, bool FUSED, bool X3, bool LONGK, int MAXL>
tag_status_t launch_m(const ReconArgs* a, int count, cudaStream_t s, const FusedGather* fg) {
    using C = Cfg<BN, CTAS, X3, (OUT_BF16 || X3 ? 1 : (SGD ? EXP_SGD_EP : 2)), LONGK>;
    GroupParamsT<MAXL> gp;
    std::memset(&gp, 0, sizeof gp);
    int tiles = 0;
    for (int i = 0; i < count; ++i) {
        LayerParams& L = gp.L[i];
        const CUtensorMapDataType odt = X3 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
        const int oes = X3 ? 4 : 2;
        const int64_t orows = X3 ? 2 * a[i].kpad : a[i].K;      // X3: [hi ; lo], Kp rows each
        const CUtensorMapSwizzle oswz = X3 ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_128B;
        L.box3 = !X3 && !EXP_RECON_NO3D && a[i].M % 64 == 0 && a[i].N % 64 == 0 && a[i].lda % 64 == 0 ? 1 : 0;
        if (a[i].M == 0) {
            // an empty row shard (sharded sync, more ranks than 128-row tiles): no tiles and no
            // tensor maps; in a FUSED launch the layer's factors are still pushed to the peers
        } else {
            // window operands: one map over both buffers (2 * kbuf rows; rows K..kbuf of each
            // buffer stay zero, so the last K block of buffer 0 never reads buffer 1)
            const int64_t rows = a[i].ctr_mode && a[i].ctr ? 2 * a[i].kbuf : orows;
            if (L.box3) {
                if (!encode_3d(&L.tmA, a[i].A, rows, a[i].M, C::BK, C::A_CHUNKS, a[i].lda) ||
                    !encode_3d(&L.tmB, a[i].Bm, rows, a[i].N, C::BK, C::B_CHUNKS))
                    return fail(TAG_ERR_CUDA, "cuTensorMapEncodeTiled (3-D) failed for the factor operands");
            } else if (!encode_2d(&L.tmA, a[i].A, odt, oes, rows, a[i].M, C::ELEMS, C::BK, a[i].lda, oswz) ||
                       !encode_2d(&L.tmB, a[i].Bm, odt, oes, rows, a[i].N, C::ELEMS, C::BK, 0, oswz)) {
                return fail(TAG_ERR_CUDA, "cuTensorMapEncodeTiled failed for the factor operands");
            }
        }
        L.ctr = a[i].ctr;
        L.ctr_mode = a[i].ctr ? a[i].ctr_mode : 0;
        L.kbuf = static_cast<int>(a[i].kbuf);
        L.k_lo = X3 ? static_cast<int>(a[i].kpad) : 0;
        L.C = a[i].C;
        L.W = a[i].W;
        L.V = a[i].V;
        L.Mm = a[i].Mm;
        L.M = static_cast<int>(a[i].M);
        L.N = static_cast<int>(a[i].N);
        L.num_n_blocks = static_cast<int>((a[i].N + BN - 1) / BN);
        L.num_k_blocks = static_cast<int>((a[i].K + C::BK - 1) / C::BK);
        L.tile_begin = tiles;
        L.alpha = a[i].alpha;
        L.num_m_blocks = static_cast<int>((a[i].M + BM * CTAS - 1) / (BM * CTAS));
        // Raster: when dY_all (K x N) no longer fits comfortably in L2, walk M first so the
        // concurrently running tiles share each B panel (read once from HBM); otherwise walk N
        // (whole output rows written together, better DRAM page locality for the epilogue).
        L.m_fast = (a[i].K * a[i].N * 2 > (32ll << 20)) ? 1 : 0;
        tiles += L.num_m_blocks * L.num_n_blocks;
        if constexpr (FUSED) {
            L.srcX = a[i].srcX;
            L.srcY = a[i].srcY;
            L.win = static_cast<ncclWindow_t>(a[i].win);
            L.off_x = a[i].off_x;
            L.off_dy = a[i].off_dy;
            L.xbuf = a[i].xbuf;
            L.ybuf = a[i].ybuf;
            L.off_flag = a[i].off_flag;
            L.flags = a[i].flags;
            L.vx = a[i].cx * 2 / 16;
            L.vy = a[i].cy * 2 / 16;
        }
    }
    gp.count = count;
    gp.num_tiles = tiles;
    gp.lr = a[0].lr;
    gp.mu = a[0].mu;
    gp.wd = a[0].wd;
    gp.opt = a[0].opt;
    gp.adam = AdamConsts{a[0].b1, a[0].omb1, a[0].b2, a[0].omb2, a[0].eps, a[0].lr_t, a[0].isbc2,
                         a[0].wd};
    gp.slot = FUSED ? fg->me : 0;
    gp.mc_base = FUSED ? static_cast<char*>(fg->mc_base) : nullptr;
    gp.cast = FUSED && fg->cast ? 1 : 0;
    gp.local_ctr = FUSED ? fg->local_ctr : nullptr;
    gp.sched = CTAS == 1 && !EXP_STATIC_SCHED ? a[0].sched : nullptr;
    auto kern = recon_tc_kernel<BN, CTAS, OUT_BF16, SGD, FUSED, X3, LONGK, MAXL>;
    // the shared-memory opt-in, once per instantiation and device (thread-safe)
    static std::atomic<uint64_t> attr_set{0};
    int dev = 0;
    cudaGetDevice(&dev);
    const uint64_t bit = 1ull << (dev & 63);
    if (!(attr_set.load(std::memory_order_acquire) & bit)) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             C::SMEM);
        if (e != cudaSuccess) return cuda_fail(e, "cudaFuncSetAttribute(recon_tc)");
        attr_set.fetch_or(bit, std::memory_order_release);
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(grid_for(tiles, CTAS, FUSED)));
    cfg.blockDim = dim3(NUM_THREADS);
    cfg.dynamicSmemBytes = C::SMEM;
    cfg.stream = s;
    cudaLaunchAttribute attr[2];
    int na = 0;
#ifndef EXP_NO_PDL
#define EXP_NO_PDL 0
#endif
    if (!EXP_NO_PDL) {
        attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;   // PDL (see kernel)
        attr[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    if (CTAS == 2) {
        attr[na].id = cudaLaunchAttributeClusterDimension;                  // CTA pair on one TPC
        attr[na].val.clusterDim.x = CTAS;
        attr[na].val.clusterDim.y = 1;
        attr[na++].val.clusterDim.z = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = na;
    const int npeers = FUSED ? fg->npeers : 1, me = FUSED ? fg->me : 0;
#if EXP_FUSED_DBG == 3
    if (FUSED) {
        static unsigned long long zero[160 * DBG_SLOTS];
        cudaMemcpyToSymbolAsync(g_dbg_stamps, zero, sizeof zero, 0, cudaMemcpyHostToDevice, s);
    }
#endif
#if EXP_END_STAMPS
    {
        static unsigned long long zero[160 * DBG_SLOTS];
        cudaMemcpyToSymbolAsync(g_dbg_stamps, zero, sizeof zero, 0, cudaMemcpyHostToDevice, s);
        dbg_marker_kernel<<<1, 1, 0, s>>>(1);
    }
#endif
    cudaError_t e = cudaLaunchKernelEx(&cfg, kern, gp, npeers, me);
    if (e != cudaSuccess) return cuda_fail(e, "launch recon_tc_kernel");
#if EXP_END_STAMPS
    {
        // diagnostics builds: how unevenly the persistent CTAs finish (us from the earliest start)
        static unsigned long long st[160 * DBG_SLOTS];
        dbg_marker_kernel<<<1, 1, 0, s>>>(2);
        cudaStreamSynchronize(s);
        cudaMemcpyFromSymbol(st, g_dbg_stamps, sizeof st);
        const int G = static_cast<int>(cfg.gridDim.x);
        unsigned long long t0 = ~0ull, f0 = ~0ull, f1 = 0, e1 = 0;
        for (int b = 0; b < G; ++b) {
            t0 = st[b * DBG_SLOTS] < t0 ? st[b * DBG_SLOTS] : t0;
            f0 = st[b * DBG_SLOTS + 1] < f0 ? st[b * DBG_SLOTS + 1] : f0;
            f1 = st[b * DBG_SLOTS + 1] > f1 ? st[b * DBG_SLOTS + 1] : f1;
            e1 = st[b * DBG_SLOTS + 7] > e1 ? st[b * DBG_SLOTS + 7] : e1;
        }
        const unsigned long long m1 = st[159 * DBG_SLOTS + 1], m2 = st[159 * DBG_SLOTS + 2];
        std::fprintf(stderr, "[launch stamps] marker -> first CTA %.2f, CTA first instr spread %.2f, "
                     "first instr -> body %.2f, body -> last end %.2f, last end -> marker %.2f, "
                     "marker -> marker %.2f us\n", (f0 - m1) / 1e3, (f1 - f0) / 1e3, (t0 - f0) / 1e3,
                     (e1 - t0) / 1e3, (m2 - e1) / 1e3, (m2 - m1) / 1e3);
        std::vector<double> s0, s7;
        for (int b = 0; b < G; ++b) {
            s0.push_back((st[b * DBG_SLOTS] - t0) / 1000.0);
            s7.push_back((st[b * DBG_SLOTS + 7] - t0) / 1000.0);
        }
        std::sort(s0.begin(), s0.end());
        std::sort(s7.begin(), s7.end());
        std::fprintf(stderr, "[end stamps] grid %d tiles %d start max %.2f end min %.2f p10 %.2f "
                     "p50 %.2f p90 %.2f max %.2f us\n", G, tiles, s0.back(), s7[0],
                     s7[G / 10], s7[G / 2], s7[G * 9 / 10], s7.back());
    }
#endif
#if EXP_FUSED_DBG == 3
    if (FUSED) {
        // diagnostics builds: phase stamps (max over CTAs, us from the earliest CTA start)
        static unsigned long long st[160 * DBG_SLOTS];
        cudaStreamSynchronize(s);
        cudaMemcpyFromSymbol(st, g_dbg_stamps, sizeof st);
        const int G = static_cast<int>(cfg.gridDim.x);
        unsigned long long t0 = ~0ull;
        for (int b = 0; b < G; ++b)
            if (st[b * DBG_SLOTS] && st[b * DBG_SLOTS] < t0) t0 = st[b * DBG_SLOTS];
        double mx[DBG_SLOTS] = {0}, mn[DBG_SLOTS];
        for (int k = 0; k < DBG_SLOTS; ++k) mn[k] = 1e30;
        for (int b = 0; b < G; ++b)
            for (int k = 0; k < DBG_SLOTS; ++k)
                if (st[b * DBG_SLOTS + k]) {
                    const double v = (st[b * DBG_SLOTS + k] - t0) / 1000.0;
                    mx[k] = v > mx[k] ? v : mx[k];
                    mn[k] = v < mn[k] ? v : mn[k];
                }
        std::fprintf(stderr, "[fused dbg] rank %d grid %d us (min..max over CTAs): start %.1f..%.1f "
                     "stores_issued %.1f..%.1f cta_barrier %.1f..%.1f sys_fence %.1f..%.1f "
                     "local_add %.1f..%.1f publish(last CTA) %.1f wait_done %.1f..%.1f end %.1f..%.1f\n",
                     fg->me, G, mn[0], mx[0], mn[1], mx[1], mn[2], mx[2], mn[3], mx[3], mn[4], mx[4],
                     mx[5], mn[6], mx[6], mn[7], mx[7]);
    }
#endif
    count_launch();
    return TAG_OK;
}

template <int BN, int CTAS, bool OUT_BF16, bool SGD, bool FUSED, bool X3 = false,
          bool LONGK = false>
tag_status_t launch_t(const ReconArgs* a, int count, cudaStream_t s, const FusedGather* fg) {
    if (count <= 4) return launch_m<BN, CTAS, OUT_BF16, SGD, FUSED, X3, LONGK, 4>(a, count, s, fg);
    return launch_m<BN, CTAS, OUT_BF16, SGD, FUSED, X3, LONGK, MAX_GROUP>(a, count, s, fg);
}

template <bool FUSED>
tag_status_t dispatch(const ReconArgs* a, int count, cudaStream_t s, const FusedGather* fg) {
    if (a[0].wire == TAG_F32) {                 // 3xTF32: 128 x 128 tiles, staged gather only
        if constexpr (FUSED) return fail(TAG_ERR_UNSUPPORTED, "recon: fp32 wire is not fused");
        if (a[0].sgd) return launch_t<128, 1, false, true, false, true>(a, count, s, fg);
        if (a[0].out == TAG_BF16) return launch_t<128, 1, true, false, false, true>(a, count, s, fg);
        return launch_t<128, 1, false, false, false, true>(a, count, s, fg);
    }
    const bool wide = big_tiles(a, count);
    const bool pair = wide && use_ctas(a, count) == 2;
    int64_t kmax = 0;
    for (int i = 0; i < count; ++i) kmax = a[i].K > kmax ? a[i].K : kmax;
    const bool longk = kmax > 512;        // CTA-pair stages of 64 instead of 128 rows (see Cfg)
    if (a[0].sgd) {
        if (!wide) return launch_t<128, 1, false, true, FUSED>(a, count, s, fg);
        if (pair && longk) return launch_t<256, 2, false, true, FUSED, false, true>(a, count, s, fg);
        return pair ? launch_t<256, 2, false, true, FUSED>(a, count, s, fg)
                    : launch_t<256, 1, false, true, FUSED>(a, count, s, fg);
    }
    if (a[0].out == TAG_BF16) {
        if (!wide) return launch_t<128, 1, true, false, FUSED>(a, count, s, fg);
        if (pair && longk) return launch_t<256, 2, true, false, FUSED, false, true>(a, count, s, fg);
        return pair ? launch_t<256, 2, true, false, FUSED>(a, count, s, fg)
                    : launch_t<256, 1, true, false, FUSED>(a, count, s, fg);
    }
    if (!wide) return launch_t<128, 1, false, false, FUSED>(a, count, s, fg);
    return pair ? launch_t<256, 2, false, false, FUSED>(a, count, s, fg)
                : launch_t<256, 1, false, false, FUSED>(a, count, s, fg);
}

}  // namespace

bool recon_tc_ok(const ReconArgs& a) {
    if (a.wire == TAG_F32 && a.kpad < a.K) return false;  // 3xTF32 needs the split [hi ; lo] operands
    if (a.wire == TAG_F32 && (EXP_F32_SIMT || a.lda)) return false;
    if (a.M % 8 || a.N % 8 || a.lda % 8) return false;   // 16-byte rows for TMA (bf16)
    if (a.M > INT32_MAX || a.N > INT32_MAX || a.K > INT32_MAX) return false;
    if (a.sgd && a.out == TAG_BF16 && a.C) return false;  // E2 writes fp32 dW only
    if (reinterpret_cast<uintptr_t>(a.A) % 16 || reinterpret_cast<uintptr_t>(a.Bm) % 16)
        return false;
    if (a.C && reinterpret_cast<uintptr_t>(a.C) % 16) return false;
    if (a.sgd && (reinterpret_cast<uintptr_t>(a.W) % 16 || reinterpret_cast<uintptr_t>(a.V) % 16))
        return false;
    if (a.sgd && a.opt == 2 && (a.Mm == nullptr || reinterpret_cast<uintptr_t>(a.Mm) % 16)) return false;
    return true;
}

void recon_tc_describe(const ReconArgs* a, int count, int* bn, int* ctas, int* box3d) {
    if (a[0].wire == TAG_F32) {                  // 3xTF32: 128 x 128 single-CTA tiles
        *bn = 128, *ctas = 1, *box3d = 0;
        return;
    }
    const bool wide = big_tiles(a, count);
    *bn = wide ? 256 : 128;
    *ctas = wide ? use_ctas(a, count) : 1;
    *box3d = !EXP_RECON_NO3D && a[0].M % 64 == 0 && a[0].N % 64 == 0 && a[0].lda % 64 == 0 ? 1 : 0;
}

tag_status_t launch_recon_tc_group(const ReconArgs* a, int count, cudaStream_t s,
                                   const FusedGather* fused) {
    if (count < 1 || count > MAX_GROUP) return fail(TAG_ERR_INVALID_ARG, "recon group size");
    for (int i = 0; i < count; ++i)
        if (a[i].sgd != a[0].sgd || a[i].out != a[0].out || a[i].wire != a[0].wire ||
            (a[i].sgd && a[i].opt != a[0].opt))
            return fail(TAG_ERR_INVALID_ARG, "recon group: mixed epilogues or operand dtypes");
    return fused ? dispatch<true>(a, count, s, fused) : dispatch<false>(a, count, s, nullptr);
}

tag_status_t launch_recon_tc(const ReconArgs& a, cudaStream_t s) {
    return launch_recon_tc_group(&a, 1, s);
}

}  // namespace tag
