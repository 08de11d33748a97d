/*
 * tag.h — C ABI of libtag: B200-native sufficient-factor-broadcasting (SFB) gradient
 * synchronisation for replicated fully-connected / MatMul layers, the data-parallel hot path of
 * TAG (Zhang et al., "Expediting Distributed DNN Training with Device Topology-Aware Graph
 * Deployment", arXiv 2302.06126).
 *
 * Citations: P:n = line n of the paper's LaTeX source; S:n = line n of SPEC.md.
 * DESIGN.md lists every reading taken where the paper is silent (R1..R20).
 *
 * The method (Fig. "fig:sfb_impl"): n data-parallel replicas of a Dense
 * layer with weight W (M x N; M = input features = the paper's H1, N = output features = H2) each
 * hold a batch shard of B rows. Replica r owns its sufficient factors
 *     X_r  (B x M)  — the layer input x
 *     dY_r (B x N)  — the gradient w.r.t. the output ∇
 * Instead of all-reducing the M x N gradient, the factors are broadcast (all-gathered) to every
 * replica and every replica reconstructs the identical gradient
 *     dW = alpha * sum_{r<n} X_r^T dY_r = alpha * X_all^T dY_all,   K = n*B,  alpha = 1/(n*B)
 * ("MatMul ops on each device can reconstruct identical gradients"; alpha: DESIGN R1).
 *
 * Conventions for every call below
 *   - All matrices are dense, row-major, contiguous. Device pointers must be 16-byte aligned.
 *   - dtype of X / dY = desc.in_dtype; of dW_out = desc.out_dtype. W and v are always fp32.
 *   - Every call that takes a cudaStream_t is stream-ordered and asynchronous: it only enqueues
 *     work; inputs must stay unmodified and all buffers alive until the stream passes the call.
 *   - One plan (or a group containing it) is used by one stream at a time: its gather buffers,
 *     window call counter and the reconstruction's tile-schedule counters are per plan, so calls
 *     on the same plan from two streams must be ordered (events) — different plans are
 *     independent.
 *   - CUDA graphs: the calls keep no per-call state on the host. Which half of a plan's
 *     double-buffered symmetric window a gather fills, and the arrival-counter targets of the fused
 *     exchange, derive on the device from a call counter in the window, so tag_sfb_sync*, the group
 *     calls, tag_sfb_gather / tag_sfb_reconstruct and the bias calls can be captured in a CUDA
 *     graph and replayed (collectively: every rank replays the same sequence). Calls that go
 *     through NCCL collectives (desc.gather = NCCL, tag_dense_allreduce, tag_ps_sync, the sharded
 *     W all-gather) follow NCCL's own capture rules.
 *   - Ownership: the caller owns X, dY, dW_out, W, v and all host buffers. The plan owns its
 *     gather buffers, staging buffers, TMA descriptors and NCCL reduction op; the comm owns the
 *     NCCL communicator. Destroy plans before their comm.
 *   - Collective calls (marked COLLECTIVE) must be made by every rank of the comm, in the same
 *     order, with identical descriptors — the NCCL rule.
 *   - Errors: argument validation happens on the host before anything is enqueued; an invalid
 *     argument returns TAG_ERR_INVALID_ARG with no side effects. CUDA / NCCL failures return
 *     TAG_ERR_CUDA / TAG_ERR_NCCL; an asynchronous NCCL error detected on entry returns
 *     TAG_ERR_ASYNC. tag_last_error() gives a thread-local human-readable detail. Nothing throws
 *     across the ABI. There is no CPU fallback: without a usable CUDA device every compute call
 *     fails with TAG_ERR_CUDA.
 */
#ifndef TAG_H_
#define TAG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the library builds with -fvisibility=hidden */
#endif

typedef struct CUstream_st* tag_stream_t; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
    TAG_OK = 0,
    TAG_ERR_INVALID_ARG = 1,
    TAG_ERR_UNSUPPORTED = 2,
    TAG_ERR_CUDA = 3,
    TAG_ERR_NCCL = 4,
    TAG_ERR_OOM = 5,
    TAG_ERR_NOT_INITIALIZED = 6,
    TAG_ERR_ASYNC = 7
} tag_status_t;

typedef enum { TAG_F32 = 0, TAG_BF16 = 1 } tag_dtype_t;

/* Per-layer synchronisation choice: Replicate-with-AllReduce, SFB
 * ("Duplicate" of the gradient op, P:363-365 / P:523-524), Replicate-with-PS (only
 * from the profiled selector when a PS curve is given); NONE when n = 1. */
typedef enum {
    TAG_SYNC_ALLREDUCE = 0,
    TAG_SYNC_SFB = 1,
    TAG_SYNC_NONE = 2,
    TAG_SYNC_PS = 3
} tag_choice_t;

/* Readings of the SFB communication term (DESIGN R2): north_star's gathered bytes n*S (default),
 * the paper ILP's D(D-1)*S broadcast term, or the physical all-gather wire (n-1)*S. */
typedef enum { TAG_RULE_NORTHSTAR = 0, TAG_RULE_PAPER_ILP = 1, TAG_RULE_WIRE = 2 } tag_rule_t;

typedef struct tag_comm_s* tag_comm_t;
typedef struct tag_plan_s* tag_sfb_plan_t;

/* ------------------------------------------------------------------------------------------ */
/* Library info                                                                               */
/* ------------------------------------------------------------------------------------------ */
const char* tag_version(void);
const char* tag_status_string(tag_status_t s);
/* Detail of the last error raised on the calling thread ("" if none). Valid until the next call. */
const char* tag_last_error(void);
/* Number of libtag kernels launched by this process so far (all plans, all streams). */
uint64_t tag_kernel_launches(void);

/* ------------------------------------------------------------------------------------------ */
/* Communicator bootstrap (one process per GPU, P:716-718 NCCL; DESIGN "Multi-GPU")           */
/* ------------------------------------------------------------------------------------------ */
/* Rank 0 creates a 128-byte id (ncclGetUniqueId); the caller broadcasts it to every rank with
 * its own transport (torch.distributed in the Python binding). */
tag_status_t tag_get_unique_id(unsigned char id[128]);
/* COLLECTIVE. Sets the CUDA device to `cuda_device` for the calling thread and creates the NCCL
 * communicator of `nranks` ranks. nranks == 1 is valid and creates no NCCL communicator (`id` may
 * be NULL then): plans on it skip the exchange entirely. *out is set only on success.
 * Equivalent to tag_comm_create_ex(..., TAG_COMM_DEFAULT, out). */
tag_status_t tag_comm_create(const unsigned char id[128], int nranks, int rank, int cuda_device,
                             tag_comm_t* out);
typedef enum {
    TAG_COMM_DEFAULT = 0,
    /* NVLink SHARP: the fused push stores once to the multicast address of the LSA team instead
     * of once per peer (needs NVLS; ignored when unavailable). Same results, bit for bit. */
    TAG_COMM_NVLS_MULTICAST = 1,
    /* nranks == 1 only: create a real one-rank NCCL communicator (device communicator, symmetric
     * windows, PreMulSum op) so that every collective code path of the library runs with n = 1:
     * the fused push into the (own) window with its arrival counters, the push-gather kernel and
     * its LSA barrier, ncclAllGather, the PreMulSum ncclAllReduce, the PS reduce + broadcast and
     * the sharded calls. Results equal those of the plain one-rank comm (the same values, since
     * the exchange of one rank is a copy). `id` may be NULL (the library makes one). */
    TAG_COMM_LOOPBACK = 2
} tag_comm_flags_t;
/* COLLECTIVE. tag_comm_create with flags (a bitwise OR of tag_comm_flags_t; every rank must pass
 * the same flags). Errors: TAG_ERR_INVALID_ARG (unknown flag, bad rank/device, NULL id with
 * nranks > 1), TAG_ERR_NCCL. */
tag_status_t tag_comm_create_ex(const unsigned char id[128], int nranks, int rank, int cuda_device,
                                unsigned flags, tag_comm_t* out);
/* COLLECTIVE. Destroys the communicator. NULL is a no-op. */
tag_status_t tag_comm_destroy(tag_comm_t comm);
tag_status_t tag_comm_info(tag_comm_t comm, int* nranks, int* rank, int* cuda_device);
/* COLLECTIVE. Stream-ordered device-side barrier of all ranks (one-CTA kernel on the NCCL LSA
 * barrier): work enqueued on `stream` after it starts only once every rank's stream reached it.
 * No-op for nranks == 1; TAG_ERR_UNSUPPORTED if the ranks are not all NVLink load/store
 * reachable. Used to align ranks before a timed region. */
tag_status_t tag_comm_barrier(tag_comm_t comm, tag_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* SFB plan: one replicated Dense layer                                                       */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
    int64_t M;               /* input features (H1); rows of dW                      */
    int64_t N;               /* output features (H2); columns of dW                  */
    int64_t B;               /* rows (samples / tokens) per replica                         */
    int n;                   /* replicas; must equal the comm size                          */
    tag_dtype_t in_dtype;    /* dtype of X and dY as the caller holds them                  */
    tag_dtype_t wire_dtype;  /* dtype of the broadcast factors: F32->F32, BF16->BF16 or     */
                             /* F32->BF16 (RNE cast in the pack kernel, DESIGN R11)         */
    tag_dtype_t out_dtype;   /* dtype of dW_out (F32 default; BF16 = RNE of the fp32 value) */
    int fuse_sgd;            /* 1: tag_sfb_sync_sgd applies SGD-momentum in the epilogue    */
    float lr, momentum, weight_decay; /* optimizer hyper-parameters, frozen in the plan (R14) */
    int fuse_adam;           /* 1: tag_sfb_sync_adam applies Adam in the epilogue (R22);     */
                             /* exclusive with fuse_sgd; uses lr and weight_decay too        */
    float beta1, beta2, eps; /* Adam hyper-parameters (also read by tag_adam_step)           */
    int gather;              /* tag_gather_request_t: how step a2 moves the factors (0 = auto)*/
} tag_sfb_desc_t;

/* tag_sfb_desc_t.gather (must be identical on every rank):
 *   AUTO: NVLink push into the peers' symmetric windows when every rank is NVLink load/store
 *         reachable and the factor rows are 16-byte multiples, else ncclAllGather;
 *   NCCL: always ncclAllGather (pack first when casting) — the library-collective baseline;
 *   PUSH: the NVLink push or TAG_ERR_UNSUPPORTED from tag_sfb_plan.
 * Ignored on a one-rank comm without NCCL (TAG_GATHER_NONE: nothing is exchanged). */
typedef enum {
    TAG_GATHER_REQ_AUTO = 0,
    TAG_GATHER_REQ_NCCL = 1,
    TAG_GATHER_REQ_PUSH = 2
} tag_gather_request_t;

/* COLLECTIVE. Validates `desc`, allocates the gather buffers (n*B*M and n*B*N elements of the
 * wire dtype) and staging, and creates the PreMulSum(1/(nB)) NCCL op used by the dense path.
 * Errors: TAG_ERR_INVALID_ARG (bad dims/dtypes, n != comm size, unknown gather request),
 * TAG_ERR_UNSUPPORTED (gather = PUSH where the push is unavailable), TAG_ERR_OOM, TAG_ERR_NCCL. */
tag_status_t tag_sfb_plan(tag_comm_t comm, const tag_sfb_desc_t* desc, tag_sfb_plan_t* out);
/* COLLECTIVE. NULL is a no-op. The caller must ensure no work using the plan is still pending. */
tag_status_t tag_sfb_plan_destroy(tag_sfb_plan_t plan);

/* Which implementation a plan selected (host query, no device work). */
typedef enum {
    TAG_GATHER_NONE = 0,        /* one-rank comm without NCCL: nothing to exchange             */
    TAG_GATHER_NCCL = 1,        /* pack (if casting) + ncclAllGather                           */
    TAG_GATHER_NVLINK_PUSH = 2  /* fused pack+push into peers' symmetric windows + LSA barrier */
} tag_gather_mode_t;
typedef struct {
    int tensor_cores;           /* 1: tcgen05 reconstruction; 0: SIMT FFMA (fp32 wire, odd rows) */
    int gather_mode;            /* tag_gather_mode_t                                            */
    int64_t K;                  /* n * B                                                        */
    float alpha;                /* fl32(1/(nB)), the fused epilogue scale                       */
    int multicast;              /* 1: the fused push uses NVLS multimem stores (one store reaches */
                                /*    every GPU); 0: one unicast store per peer                   */
    /* the tensor-core launch this plan's reconstruction uses alone — its fused optimizer      */
    /* epilogue's launch when fuse_sgd / fuse_adam is set (0 when tensor_cores == 0):          */
    int recon_bn;               /* output tile columns: 128 or 256                               */
    int recon_ctas;             /* 1: one CTA per 128-row tile; 2: CTA pair (tcgen05 cta_group::2,*/
                                /*    256-row tiles)                                             */
    int recon_box3d;            /* 1: each operand stage is one 3-D TMA box (bf16 factors, M and */
                                /*    N multiples of 64); 0: one 2-D box per 64-column chunk     */
} tag_plan_info_t;
tag_status_t tag_sfb_plan_info(tag_sfb_plan_t plan, tag_plan_info_t* out);

/* COLLECTIVE (n > 1). The SFB synchronisation of one layer, steps a1-a4:
 *   a1 pack   : if in_dtype != wire_dtype, RNE-cast X_r and dY_r into this rank's slot of the
 *               gather buffers (16-byte vectorised kernel);
 *   a2 gather : X_r and dY_r reach every replica over NVLink ("broadcast to all devices"):
 *               fused with a1 as a push into the peers' symmetric windows (NCCL device API,
 *               TAG_GATHER_NVLINK_PUSH), or an ncclAllGather (TAG_GATHER_NCCL) when the rows are
 *               not 16-byte multiples, the ranks are not all NVLink-reachable, or the descriptor
 *               asks for it (desc.gather = TAG_GATHER_REQ_NCCL);
 *   a3 recon  : dW = alpha * X_all^T dY_all on the tensor cores (K = n*B), alpha = 1/(nB);
 *   a4 store  : dW_out <- dW in out_dtype (fused epilogue).
 * X: B x M, dY: B x N (in_dtype, device). dW_out: M x N (out_dtype, device), overwritten.
 * dW_out is bitwise identical on every rank. n = 1: a3-a4 only, alpha = 1/B. */
tag_status_t tag_sfb_sync(tag_sfb_plan_t plan, const void* X, const void* dY, void* dW_out,
                          tag_stream_t stream);

/* Stage split of tag_sfb_sync for staged timing: gather = a1 + a2 into the plan's gather
 * buffers (COLLECTIVE for n > 1); reconstruct = a3 + a4 from the most recent gather on the same
 * stream. tag_sfb_gather followed by tag_sfb_reconstruct == tag_sfb_sync. */
tag_status_t tag_sfb_gather(tag_sfb_plan_t plan, const void* X, const void* dY,
                            tag_stream_t stream);
tag_status_t tag_sfb_reconstruct(tag_sfb_plan_t plan, void* dW_out, tag_stream_t stream);

/* COLLECTIVE (n > 1). tag_sfb_sync with the optimizer op fused into the reconstruction epilogue
 * (the ApplyGradient op l that consumes the gradient; SGD-momentum per R14):
 *   g = dW + wd*W ; v <- momentum*v + g ; W <- W - lr*v        (W, v: M x N fp32, in place)
 * dW_out may be NULL (then dW is never written to HBM). Requires desc.fuse_sgd = 1. */
tag_status_t tag_sfb_sync_sgd(tag_sfb_plan_t plan, const void* X, const void* dY, float* W,
                              float* v, void* dW_out, tag_stream_t stream);

/* COLLECTIVE (n > 1). tag_sfb_sync with Adam fused into the epilogue (the optimizer the paper
 * trains with; torch.optim.Adam semantics, DESIGN R22), step t >= 1 (bias corrections):
 *   g = dW + wd*W ; m <- b1*m + (1-b1)*g ; v <- b2*v + (1-b2)*g*g ;
 *   W <- W - (lr/(1-b1^t)) * m / (sqrt(v)/sqrt(1-b2^t) + eps)       (W, m, v: M x N fp32)
 * dW_out may be NULL. Requires desc.fuse_adam = 1 (and out_dtype F32). Bitwise equal to
 * tag_sfb_sync followed by tag_adam_step. */
tag_status_t tag_sfb_sync_adam(tag_sfb_plan_t plan, const void* X, const void* dY, float* W,
                               float* m, float* v, int64_t step, void* dW_out, tag_stream_t stream);

/* COLLECTIVE (n > 1). End-to-end form with HOST buffers: copies X and dY (pinned or pageable
 * host memory, in_dtype) to plan-owned device staging, runs tag_sfb_sync into plan-owned device
 * memory and copies dW (out_dtype) back to dW_host. Stream-ordered like the others: the host
 * buffers are read / written when the stream reaches the copies. */
tag_status_t tag_sfb_sync_host(tag_sfb_plan_t plan, const void* X_host, const void* dY_host,
                               void* dW_host, tag_stream_t stream);

/* Sharded reconstruction: rank r reconstructs only rows
 * [row_begin, row_begin + row_count) of dW — a contiguous run of 128-row tiles — so each GPU
 * writes M*N/n gradient elements instead of M*N (the HBM write is the reconstruction's binding
 * roof). Every rank still receives all factors; the shards of ranks 0..n-1 tile dW exactly, in
 * rank order, and each shard is bitwise equal to the same rows of tag_sfb_sync's dW. This is a
 * variant, not the paper's semantics (the paper's Duplicate leaves the full gradient on every
 * replica): it fits a sharded (ZeRO-style) optimizer. tag_sfb_shard_rows is a host
 * query; row_count may be 0 (more ranks than 128-row tiles). */
tag_status_t tag_sfb_shard_rows(tag_sfb_plan_t plan, int rank, int64_t* row_begin,
                                int64_t* row_count);
/* COLLECTIVE (n > 1). dW_shard: row_count x N in out_dtype (may be NULL when row_count == 0). */
tag_status_t tag_sfb_sync_sharded(tag_sfb_plan_t plan, const void* X, const void* dY,
                                  void* dW_shard, tag_stream_t stream);

/* COLLECTIVE (n > 1). Sharded optimizer step + parameter all-gather (ZeRO-style; SURVEY §8(f)
 * rank 2; the Duplicate replicates the gradient op, and here the optimizer op l is
 * sharded instead of replicated): every rank receives all factors (a1 + a2, fused push), rank r
 * reconstructs only its rows [row_begin, row_begin + row_count) of dW (tag_sfb_shard_rows) and
 * applies SGD-momentum to those rows of W and to its momentum shard in the same epilogue (dW is
 * never stored), then the updated rows of W are all-gathered (one in-place ncclAllGather when
 * the shards are equal, else one ncclBroadcast per shard) so every rank ends with the whole W.
 * W: M x N fp32, the full parameter (read and written only in this rank's rows before the
 * all-gather; every row is overwritten by its owner's result). v_shard: row_count x N fp32, this
 * rank's momentum rows (may be NULL when row_count == 0). Requires desc.fuse_sgd = 1 and
 * out_dtype F32. W after the call is bitwise equal to tag_sfb_sync_sgd's on every rank (the same
 * per-row arithmetic), and v_shard to the same rows of its v. n = 1: one shard, no all-gather.
 * Errors: TAG_ERR_INVALID_ARG (plan without fuse_sgd, NULL / misaligned pointers). */
tag_status_t tag_sfb_sync_sharded_sgd(tag_sfb_plan_t plan, const void* X, const void* dY, float* W,
                                      float* v_shard, tag_stream_t stream);
/* COLLECTIVE (n > 1). The same with Adam (desc.fuse_adam = 1, step t >= 1, R22): m_shard and
 * v_shard are this rank's row_count x N moment rows; W after the call is bitwise equal to
 * tag_sfb_sync_adam's on every rank. */
tag_status_t tag_sfb_sync_sharded_adam(tag_sfb_plan_t plan, const void* X, const void* dY, float* W,
                                       float* m_shard, float* v_shard, int64_t step,
                                       tag_stream_t stream);

/* Bias gradient of the layer (y = x W + b; DESIGN R17): db = alpha * sum_k dY_all[k][:], the
 * column sums of the gathered output gradients — the bias is the weight of a constant input, so
 * its gradient is the outer product of the ones vector with the factor dY that SFB already
 * broadcasts; no communication. Reads the dY_all of this plan's most
 * recent synchronisation on `stream` (tag_sfb_sync, _sgd, _sharded, _gather, or a group call
 * containing the plan); at n = 1 without a cast that is the caller's dY, which must still be
 * valid. db_out: N elements of out_dtype (device), overwritten; bitwise identical on every rank
 * (fixed summation order, no atomics). Not collective. Errors: TAG_ERR_INVALID_ARG (NULL, or no
 * factors gathered yet). */
tag_status_t tag_sfb_bias_grad(tag_sfb_plan_t plan, void* db_out, tag_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* Buckets: several layers synchronised together                                             */
/* ------------------------------------------------------------------------------------------ */
/* A group (bucket) of 1..32 plans of the same comm, the same in/wire/out dtypes and the same
 * fuse_sgd setting (and SGD hyper-parameters). tag_sfb_group_sync runs steps a1-a4 of every layer with ONE push kernel (one LSA
 * barrier; or one grouped NCCL call) and ONE persistent tensor-core launch over all layers' output
 * tiles, so launch latency, pipeline ramp-up, the last partial wave and the barrier latency are
 * paid once per bucket instead of once per layer. Results are bitwise identical to calling
 * tag_sfb_sync on each plan. The group borrows the plans (destroy the group first). Creating a
 * group is host-only; using it is COLLECTIVE: every rank must build the same groups in the same
 * plan order. X[i], dY[i], dW[i] are the arguments tag_sfb_sync would take for plans[i]. */
typedef struct tag_group_s* tag_sfb_group_t;
tag_status_t tag_sfb_group_create(const tag_sfb_plan_t* plans, int count, tag_sfb_group_t* out);
tag_status_t tag_sfb_group_destroy(tag_sfb_group_t group);
tag_status_t tag_sfb_group_sync(tag_sfb_group_t group, const void* const* X,
                                const void* const* dY, void* const* dW, tag_stream_t stream);
/* Same with the SGD-momentum epilogue of every layer fused (all plans need fuse_sgd = 1 and the
 * same lr / momentum / weight_decay): W[i], v[i] fp32 M x N in place; dW may be NULL (no dW
 * written) or an array whose entries may be NULL. */
tag_status_t tag_sfb_group_sync_sgd(tag_sfb_group_t group, const void* const* X,
                                    const void* const* dY, float* const* W, float* const* v,
                                    void* const* dW, tag_stream_t stream);
/* Same with Adam (all plans fuse_adam = 1 with identical hyper-parameters); m[i], v[i] fp32. */
tag_status_t tag_sfb_group_sync_adam(tag_sfb_group_t group, const void* const* X,
                                     const void* const* dY, float* const* W, float* const* m,
                                     float* const* v, int64_t step, void* const* dW,
                                     tag_stream_t stream);
/* Sharded form of tag_sfb_group_sync: dW_shard[i] is plans[i]'s row shard for this rank
 * (tag_sfb_shard_rows). One fused launch when every plan takes the fused path and every shard is
 * non-empty; otherwise one gather + per-plan reconstructions. */
tag_status_t tag_sfb_group_sync_sharded(tag_sfb_group_t group, const void* const* X,
                                        const void* const* dY, void* const* dW_shard,
                                        tag_stream_t stream);
/* Stage split, as for single plans: gather = a1 + a2 of every layer, reconstruct = a3 + a4. */
tag_status_t tag_sfb_group_gather(tag_sfb_group_t group, const void* const* X,
                                  const void* const* dY, tag_stream_t stream);
tag_status_t tag_sfb_group_reconstruct(tag_sfb_group_t group, void* const* dW,
                                       tag_stream_t stream);
/* tag_sfb_bias_grad of every plan of the group in ONE launch: db[i] (N_i elements, out_dtype). */
tag_status_t tag_sfb_group_bias_grad(tag_sfb_group_t group, void* const* db,
                                     tag_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* Dense-gradient baseline ("Replicate with AllReduce")                 */
/* ------------------------------------------------------------------------------------------ */
/* Local, unscaled gradient of this replica: dW_local = X_r^T dY_r (K = B) in out_dtype, operands
 * cast to wire_dtype first (same tensor-core path as the reconstruction). Not collective. */
tag_status_t tag_local_grad(tag_sfb_plan_t plan, const void* X, const void* dY, void* dW_local,
                            tag_stream_t stream);
/* COLLECTIVE. In place: dW <- (1/(nB)) * sum_ranks dW, one ncclAllReduce whose PreMulSum op
 * applies the scale inside the collective (P:566 ring AllReduce). dW: M x N out_dtype.
 * n = 1: dW <- dW / B. */
tag_status_t tag_dense_allreduce(tag_sfb_plan_t plan, void* dW, tag_stream_t stream);
/* COLLECTIVE. "Replicate with PS": the parameter server `root` aggregates the local
 * gradients (AddN, with the 1/(nB) scale as PreMulSum: ncclReduce) and sends the result back to
 * every replica (ncclBroadcast). In place, like tag_dense_allreduce: dW (M x N out_dtype) holds
 * this rank's unscaled local gradient on entry and (1/(nB)) * sum_ranks dW on exit, bitwise
 * identical on every rank. The paper picks the PS round-robin over the device group
 * (S:367): pass root = layer index mod n. n = 1: dW <- dW / B. Errors:
 * TAG_ERR_INVALID_ARG (root outside [0, n), NULL / misaligned dW). */
tag_status_t tag_ps_sync(tag_sfb_plan_t plan, void* dW, int root, tag_stream_t stream);
/* Unfused optimizer step of the dense path (same arithmetic as the fused epilogue):
 * g = dW + wd*W; v <- momentum*v + g; W <- W - lr*v. dW fp32 (out_dtype must be F32). */
tag_status_t tag_sgd_step(tag_sfb_plan_t plan, const float* dW, float* W, float* v,
                          tag_stream_t stream);
/* Unfused Adam step with the plan's beta1 / beta2 / eps / lr / weight_decay (same arithmetic as
 * the fused epilogue, step t >= 1): W, m, v updated in place from dW (fp32, M x N). */
tag_status_t tag_adam_step(tag_sfb_plan_t plan, const float* dW, float* W, float* m, float* v,
                           int64_t step, tag_stream_t stream);

/* ------------------------------------------------------------------------------------------ */
/* Selector: per-layer SFB vs AllReduce (the paper's SFB ILP, for one MatMul cut)  */
/* ------------------------------------------------------------------------------------------ */
typedef struct {
    int64_t M, N, B;          /* layer dims and rows per replica                              */
    tag_dtype_t factor_dtype; /* e_w: bytes per factor element on the wire                    */
    tag_dtype_t grad_dtype;   /* e_g: bytes per gradient element the dense path all-reduces   */
} tag_layer_t;

typedef struct {
    int n;                     /* replicas D                                           */
    uint64_t link_bytes_per_s; /* tau: bottleneck bandwidth between the D devices     */
    uint64_t tensor_flops;     /* F: T_g = 2*M*N*B / F (linear model P:326-328); 0 = ignore   */
    int rule;                  /* tag_rule_t                                                   */
} tag_topology_t;

/* Host only; no device or communicator work. For each layer i, out[i] is
 *   TAG_SYNC_NONE      if n <= 1;
 *   TAG_SYNC_SFB       iff (n-1)*T_g + c_rule*S/tau < 2(n-1)/n * G/tau  strictly, with
 *                      S = B(M+N)e_w, G = M*N*e_g, c_rule = n | n(n-1) | n-1 (R2, R4);
 *   TAG_SYNC_ALLREDUCE otherwise (ties keep AllReduce).
 * Evaluated exactly in 128-bit integers after clearing denominators (R4c), so the decision is
 * bit-exact and identical on every rank. Errors: TAG_ERR_INVALID_ARG for NULL pointers,
 * num_layers < 0, non-positive dims, tau = 0, or an unknown rule/dtype; TAG_ERR_UNSUPPORTED if
 * an intermediate would overflow 127 bits. */
tag_status_t tag_sfb_select(const tag_layer_t* layers, int num_layers, const tag_topology_t* topo,
                            tag_choice_t* out);

/* Profiled selector (the paper's profiler; SPEC fit_comm / predict S:197-214;
 * SURVEY §8(f) rank 4): the two synchronisation costs are read from curves measured on the
 * machine (e.g. scripts/profile_comm.py) instead of the analytic ring formula, so per-collective
 * latency is part of the decision. Curve: count >= 2 points, bytes strictly increasing; the time
 * at x is the piecewise-linear interpolation between consecutive points, extended by the first /
 * last segment outside them, evaluated in integer ns with floor rounding and clamped
 * at 0. Decision per layer (S = B(M+N)e_w, G = M N e_g):
 *   SFB iff gather((n-1) S) + floor((n-1) 2MNB 1e9 / F) < allreduce(G)   [F = 0: no compute term]
 * ties keep AllReduce; n = 1 -> NONE. With a PS curve (ps.count >= 2; count 0 = no PS option,
 * "Replicate with PS"), PS is chosen iff ps(G) is strictly below both other costs
 * (ties: AllReduce, then SFB). Exact integer arithmetic (bit-identical on every rank and
 * to oracle/selector.py). Limits (TAG_ERR_INVALID_ARG beyond): n <= 65536, M, N, B <= 2^24,
 * curve ns <= 2^40, bytes <= 2^62.
 * Measured op times (the paper profiles every op at the batch size, instead of the
 * linear model P:326-328): when recon_ns and local_ns are both non-NULL, recon_ns[i] is the
 * measured time of layer i's reconstruction at K = nB (tag_sfb_reconstruct) and local_ns[i] that
 * of the dense path's local gradient at K = B (tag_local_grad), e.g. from
 * scripts/profile_compute.py, and the costs become
 *   SFB = gather((n-1) S) + recon_ns[i],  AllReduce = local_ns[i] + allreduce(G),
 *   PS  = local_ns[i] + ps(G)
 * (same tie rule; tensor_flops is then ignored). Each value <= 2^40. */
typedef struct {
    int count;
    const uint64_t* bytes;
    const uint64_t* ns;
} tag_curve_t;
typedef struct {
    int n;
    tag_curve_t gather;      /* x = bytes each rank receives: (n-1) * B(M+N) e_w */
    tag_curve_t allreduce;   /* x = gradient bytes M N e_g */
    uint64_t tensor_flops;   /* F; 0 drops the compute term */
    tag_curve_t ps;          /* x = gradient bytes M N e_g (tag_ps_sync); count 0: no PS option */
    const uint64_t* recon_ns;  /* [num_layers] measured reconstruction ns at K = nB, or NULL */
    const uint64_t* local_ns;  /* [num_layers] measured local-gradient ns at K = B, or NULL  */
} tag_profiled_topology_t;
tag_status_t tag_sfb_select_profiled(const tag_layer_t* layers, int num_layers,
                                     const tag_profiled_topology_t* topo, tag_choice_t* out);

/* General SFB cut ILP: for one gradient tensor (g, l) of a
 * replicated op group V, choose which ops to duplicate (alpha_i) so as to
 *   min (D-1) sum_i alpha_i T_i + D(D-1) sum_{(j,i) in E} b_ji L_ji / tau - 2 alpha_g (D-1)/D L_gl / tau
 *   s.t. alpha_k <= sum_{(k,i) in E} alpha_i (k != l),  b_ji >= alpha_i - alpha_j,  binary.
 * Readings (DESIGN R20): alpha_l = 1 and T_l excluded; edge_src = -1 marks a
 * producer outside the group (alpha 0); edges into l are not cut candidates; b_ji = max(0,
 * alpha_i - alpha_j). Solved exactly in polynomial time as ONE s-t minimum cut ("similar to the
 * min-cut problem"; derivation in csrc/ilp.cpp) with integer costs (T in ns, L in
 * bytes, tau in bytes/s); among optimal assignments the one duplicating the fewest ops is
 * returned (it is unique), so an objective of exactly 0 keeps the all-zero one. The
 * Fig. 5 MatMul instance reduces to tag_sfb_select's TAG_RULE_PAPER_ILP. Host only.
 * Errors: TAG_ERR_INVALID_ARG (bad indices, cycles, D outside [1, 1024], tau 0, num_ops outside
 * [2, 64], > 4096 edges), TAG_ERR_UNSUPPORTED (T > 2^40 ns or bytes > 2^50: 127-bit range). */
typedef struct {
    int num_ops;                 /* |V|, 2..64; ops are 0..num_ops-1                         */
    int l, g;                    /* the optimizer op and the op producing its gradient        */
    const uint64_t* op_ns;       /* T_i: compute time of op i at the per-replica batch, ns    */
    int num_edges;
    const int* edge_src;         /* j: producer op, or -1 for a producer outside the group    */
    const int* edge_dst;         /* i: consumer op (an op of the group)                       */
    const uint64_t* edge_bytes;  /* L_ji                                                      */
    uint64_t grad_bytes;         /* L_gl                                                      */
    int D;                       /* replicas                                                  */
    uint64_t tau;                /* bottleneck bandwidth, bytes/s                             */
} tag_sfb_ilp_t;
/* alpha_out[num_ops]: 1 = duplicate; objective_s: the optimum in seconds (0 for all-zero). */
tag_status_t tag_sfb_ilp_solve(const tag_sfb_ilp_t* inst, uint8_t* alpha_out, double* objective_s);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* TAG_H_ */
