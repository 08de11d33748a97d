/*
 * tag_oracle.c — CPU reference ("oracle") for the SFB gradient-synchronisation hot path of
 * TAG (Zhang et al., arXiv 2302.06126).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference legs may load this library. The product path (paper_2302_06126_b200/, libtag)
 * never links, imports or calls it, and shares no header, helper or constant with it.
 *
 * Plain, slow, obviously correct, fp64. Every function cites the passage it follows
 * (P:n = /root/reference/PAPER.md line n; S:n = SPEC.md line n). No blocking, fusion or
 * reordering of the arithmetic beyond what the cited definition states. Loops over independent
 * output rows are split across OpenMP threads; each output element is still accumulated by one
 * thread, in the order the definition gives, so results are deterministic.
 *
 * Notation: n replicas, B rows per replica, layer W in R^{M x N}
 * (M = input features = the paper's H1, N = output features = H2), K = n*B.
 * X  : n*B*M doubles, replica-major: X[r][b][m]   (replica r's layer input x,   P:520-526)
 * dY : n*B*N doubles, replica-major: dY[r][b][j]  (replica r's output grad ∇,   P:520-526)
 * dW : M*N doubles, row-major dW[m][j]  (the paper's H2 x H1 gradient, transposed; R15)
 */
#include <stdint.h>
#include <string.h>
#include <stdlib.h>

/* ---------------------------------------------------------------------------------------------
 * Dense route: "Replicate with AllReduce" — every replica computes its own gradient of the
 * MatMul, then the gradients are summed across replicas ("AllReduce ...
 * op is inserted when a parameter is replicated"; SplitSum semantics of gradient ops P:300-302).
 *   G_r[m][j] = sum_{b<B} X_r[b][m] * dY_r[b][j]          (per-replica triple loop)
 *   S[m][j]   = sum_{r<n} G_r[m][j]                         (summed in rank order)
 * Returns the unscaled sum S; oracle_dense_dw applies the scale alpha = 1/(nB) (R1).
 * ------------------------------------------------------------------------------------------- */
void oracle_dense_sum(int64_t n, int64_t B, int64_t M, int64_t N,
                      const double* X, const double* dY, double* S)
{
    #pragma omp parallel
    {
        double* G = (double*)malloc((size_t)(N > 0 ? N : 1) * sizeof(double));
        #pragma omp for schedule(static)
        for (int64_t m = 0; m < M; ++m) {
            double* Srow = S + m * N;
            for (int64_t j = 0; j < N; ++j) Srow[j] = 0.0;
            for (int64_t r = 0; r < n; ++r) {
                /* G_r row m: sum over this replica's B rows, in row order */
                for (int64_t j = 0; j < N; ++j) G[j] = 0.0;
                for (int64_t b = 0; b < B; ++b) {
                    const double x = X[(r * B + b) * M + m];
                    const double* dyrow = dY + (r * B + b) * N;
                    for (int64_t j = 0; j < N; ++j) G[j] += x * dyrow[j];
                }
                /* AllReduce-sum: add replica r's gradient */
                for (int64_t j = 0; j < N; ++j) Srow[j] += G[j];
            }
        }
        free(G);
    }
}

/* dW_dense = (1/(nB)) * S  — the global-batch mean gradient (reading R1). */
void oracle_dense_dw(int64_t n, int64_t B, int64_t M, int64_t N,
                     const double* X, const double* dY, double* dW)
{
    oracle_dense_sum(n, B, M, N, X, dY, dW);
    const double nb = (double)(n * B);
    for (int64_t i = 0; i < M * N; ++i) dW[i] = dW[i] / nb;
}

/* ---------------------------------------------------------------------------------------------
 * SFB route ("sufficient factors ... can generate a gradient tensor, usually by an
 * outer product"; "the sufficient factors, ∇ and x, are broadcast to all devices, and
 * MatMul ops on each device can reconstruct identical gradients").
 *   X_all  = vstack_r X_r   (K x M),   dY_all = vstack_r dY_r  (K x N), rank order (broadcast)
 *   S      = sum_{k<K} X_all[k,:]^T (outer) dY_all[k,:]     (rank-1 accumulation, k order)
 * With the replica-major input layout, X and dY already are X_all and dY_all.
 * ------------------------------------------------------------------------------------------- */
void oracle_sfb_sum(int64_t n, int64_t B, int64_t M, int64_t N,
                    const double* X_all, const double* dY_all, double* S)
{
    const int64_t K = n * B;
    #pragma omp parallel for schedule(static)
    for (int64_t m = 0; m < M; ++m) {
        double* Srow = S + m * N;
        for (int64_t j = 0; j < N; ++j) Srow[j] = 0.0;
        /* rank-1 update number k touches row m with weight X_all[k][m] */
        for (int64_t k = 0; k < K; ++k) {
            const double x = X_all[k * M + m];
            const double* dyrow = dY_all + k * N;
            for (int64_t j = 0; j < N; ++j) Srow[j] += x * dyrow[j];
        }
    }
}

void oracle_sfb_dw(int64_t n, int64_t B, int64_t M, int64_t N,
                   const double* X_all, const double* dY_all, double* dW)
{
    oracle_sfb_sum(n, B, M, N, X_all, dY_all, dW);
    const double nb = (double)(n * B);
    for (int64_t i = 0; i < M * N; ++i) dW[i] = dW[i] / nb;
}

/* ---------------------------------------------------------------------------------------------
 * Single entries of the SFB sum, one by one, for full-size sampled parity:
 *   S[m][j] = sum_{k<K} X_all[k][m] * dY_all[k][j],  for each requested flat index m*N + j.
 * ------------------------------------------------------------------------------------------- */
void oracle_sfb_sum_entries(int64_t n, int64_t B, int64_t M, int64_t N,
                            const double* X_all, const double* dY_all,
                            int64_t count, const int64_t* flat_idx, double* out)
{
    const int64_t K = n * B;
    #pragma omp parallel for schedule(static)
    for (int64_t i = 0; i < count; ++i) {
        const int64_t m = flat_idx[i] / N, j = flat_idx[i] % N;
        double s = 0.0;
        for (int64_t k = 0; k < K; ++k) s += X_all[k * M + m] * dY_all[k * N + j];
        out[i] = s;
    }
}

/* ---------------------------------------------------------------------------------------------
 * SGD with momentum applied to the reconstructed gradient (the optimizer op l = ApplyGradient
 * that consumes the gradient; north_star "fused SGD/momentum update on W").
 * PyTorch SGD semantics (R14): dampening 0, no Nesterov, weight decay folded into g.
 *   g  = dW + wd * W
 *   v' = mu * v + g
 *   W' = W - lr * v'
 * ------------------------------------------------------------------------------------------- */
void oracle_sgd_momentum(int64_t len, const double* dW, double* W, double* v,
                         double lr, double mu, double wd)
{
    for (int64_t i = 0; i < len; ++i) {
        const double g = dW[i] + wd * W[i];
        v[i] = mu * v[i] + g;
        W[i] = W[i] - lr * v[i];
    }
}

/* ---------------------------------------------------------------------------------------------
 * Round-to-nearest-even fp32 -> bf16 (R11: the wire cast of the factor pack).
 * bf16 keeps the top 16 bits of the IEEE-754 binary32 pattern. The dropped low half is compared
 * against half an ulp (0x8000): above -> round up, below -> truncate, exactly half -> round to
 * the even result. NaN stays a (quiet) NaN.
 * ------------------------------------------------------------------------------------------- */
static uint16_t rne_bf16(float f)
{
    uint32_t u;
    memcpy(&u, &f, sizeof u);
    if ((u & 0x7f800000u) == 0x7f800000u && (u & 0x007fffffu) != 0u)
        return (uint16_t)((u >> 16) | 0x0040u);               /* quiet NaN */
    uint32_t upper = u >> 16, lower = u & 0xffffu;
    if (lower > 0x8000u || (lower == 0x8000u && (upper & 1u))) upper += 1u;
    return (uint16_t)upper;
}

void oracle_cast_bf16(int64_t len, const float* in, uint16_t* out)
{
    for (int64_t i = 0; i < len; ++i) out[i] = rne_bf16(in[i]);
}

/* ---------------------------------------------------------------------------------------------
 * Bias gradient of the Dense layer y = x W + b (R17). The sufficient factors "can
 * generate a gradient tensor, usually by an outer product": the bias is the weight
 * of a constant input 1, so its gradient is the outer product of the ones vector with dY, i.e.
 * the column sums of dY — it needs only the factor dY that SFB already broadcasts.
 * Dense route (AllReduce of per-replica bias gradients):
 *   db_r[j] = sum_{b<B} dY_r[b][j];   S_b[j] = sum_{r<n} db_r[j]   (rank order)
 * SFB route (from the gathered dY_all):
 *   S_b[j] = sum_{k<K} dY_all[k][j]                                  (k order)
 * Both return the unscaled sum (length N); the scale is alpha = 1/(nB) as for dW (R1).
 * ------------------------------------------------------------------------------------------- */
void oracle_dense_bias_sum(int64_t n, int64_t B, int64_t N, const double* dY, double* S)
{
    for (int64_t j = 0; j < N; ++j) {
        double s = 0.0;
        for (int64_t r = 0; r < n; ++r) {
            double g = 0.0;
            for (int64_t b = 0; b < B; ++b) g += dY[(r * B + b) * N + j];
            s += g;
        }
        S[j] = s;
    }
}

void oracle_sfb_bias_sum(int64_t n, int64_t B, int64_t N, const double* dY_all, double* S)
{
    const int64_t K = n * B;
    for (int64_t j = 0; j < N; ++j) S[j] = 0.0;
    for (int64_t k = 0; k < K; ++k)
        for (int64_t j = 0; j < N; ++j) S[j] += dY_all[k * N + j];
}

/* ---------------------------------------------------------------------------------------------
 * Adam applied to the reconstructed gradient (the optimizer the paper trains with, "Adam
 * optimizer"; R22: torch.optim.Adam semantics, L2 weight decay folded into g,
 * bias-corrected moments, step t >= 1):
 *   g  = dW + wd * W
 *   m' = b1 * m + (1 - b1) * g
 *   v' = b2 * v + (1 - b2) * g * g
 *   W' = W - lr * (m' / (1 - b1^t)) / (sqrt(v' / (1 - b2^t)) + eps)
 * ------------------------------------------------------------------------------------------- */
#include <math.h>
void oracle_adam(int64_t len, const double* dW, double* W, double* m, double* v, double lr,
                 double b1, double b2, double eps, double wd, int64_t t)
{
    const double bc1 = 1.0 - pow(b1, (double)t), bc2 = 1.0 - pow(b2, (double)t);
    for (int64_t i = 0; i < len; ++i) {
        const double g = dW[i] + wd * W[i];
        m[i] = b1 * m[i] + (1.0 - b1) * g;
        v[i] = b2 * v[i] + (1.0 - b2) * g * g;
        W[i] = W[i] - lr * (m[i] / bc1) / (sqrt(v[i] / bc2) + eps);
    }
}
