/*
 * c_abi_example.c — libtag used from plain C11, no Python and no PyTorch: the boundary of the
 * SFB hot path (include/tag.h) as a C program sees it.
 *
 *   gcc -std=c11 -Wall -Wextra -Werror -I include -I /usr/local/cuda/include \
 *       examples/c_abi_example.c -o c_abi_example \
 *       -L paper_2302_06126_b200 -ltag -Wl,-rpath,$PWD/paper_2302_06126_b200 \
 *       -L /usr/local/cuda/lib64 -lcudart
 *   ./c_abi_example            # host calls + one SFB sync on GPU 0 (n = 1), checked exactly
 *   ./c_abi_example --host     # host-only calls (selector, ILP): runs without a GPU
 *
 * The GPU part reconstructs dW = (1/B) X^T dY for one 1024 x 512 layer, B = 64 rows, from
 * small-integer bf16 factors, and compares every element with a double-precision loop: with
 * integer inputs and alpha = 2^-6 the fp32 result is exact, so the check is bit-for-bit
 * (the same pin as tests/test_gpu_recon.py). Exit code 0 iff every check passed.
 */
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <cuda_runtime_api.h>

#include "tag.h"

#define CHECK_TAG(call)                                                                  \
    do {                                                                                 \
        tag_status_t st_ = (call);                                                       \
        if (st_ != TAG_OK) {                                                             \
            fprintf(stderr, "%s failed: %s (%s)\n", #call, tag_status_string(st_),       \
                    tag_last_error());                                                   \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

#define CHECK_CUDA(call)                                                                 \
    do {                                                                                 \
        cudaError_t e_ = (call);                                                         \
        if (e_ != cudaSuccess) {                                                         \
            fprintf(stderr, "%s failed: %s\n", #call, cudaGetErrorString(e_));           \
            return 1;                                                                    \
        }                                                                                \
    } while (0)

/* bf16 bit pattern of a small integer (exact: the top half of its fp32 pattern) */
static uint16_t bf16_of_int(int v) {
    float f = (float)v;
    uint32_t u;
    memcpy(&u, &f, sizeof u);
    return (uint16_t)(u >> 16);
}

static int host_part(void) {
    printf("%s\n", tag_version());
    /* per-layer selector for VGG-19 fc6 / fc8 at n = 8 (north_star rule + compute term) */
    tag_layer_t layers[2] = {{25088, 4096, 32, TAG_BF16, TAG_F32}, {4096, 1000, 32, TAG_BF16, TAG_F32}};
    tag_topology_t topo = {8, 900000000000ull, 1421400000000000ull, TAG_RULE_NORTHSTAR};
    tag_choice_t choice[2];
    CHECK_TAG(tag_sfb_select(layers, 2, &topo, choice));
    printf("select n=8: fc6 -> %s, fc8 -> %s\n", choice[0] == TAG_SYNC_SFB ? "SFB" : "AllReduce",
           choice[1] == TAG_SYNC_SFB ? "SFB" : "AllReduce");
    if (choice[0] != TAG_SYNC_SFB) return 1;
    /* the general SFB cut ILP on SPEC's worked example: objective -9.7e-4 s */
    uint64_t op_ns[2] = {10000, 0};
    int src[3] = {0, -1, -1}, dst[3] = {1, 0, 0};
    uint64_t eb[3] = {1000000, 5000, 5000};
    tag_sfb_ilp_t inst = {2, 1, 0, op_ns, 3, src, dst, eb, 1000000, 2, 1000000000ull};
    uint8_t alpha[2];
    double obj = 0.0;
    CHECK_TAG(tag_sfb_ilp_solve(&inst, alpha, &obj));
    printf("ilp: alpha = [%d, %d], objective = %.3e s\n", alpha[0], alpha[1], obj);
    if (!(alpha[0] == 1 && alpha[1] == 1 && obj < -9.69e-4 && obj > -9.71e-4)) return 1;
    /* invalid arguments fail cleanly, never crash */
    if (tag_sfb_select(NULL, 1, &topo, choice) != TAG_ERR_INVALID_ARG) return 1;
    return 0;
}

static int gpu_part(void) {
    const int64_t M = 1024, N = 512, B = 64;
    const size_t nx = (size_t)(B * M), ny = (size_t)(B * N), nw = (size_t)(M * N);
    uint16_t* hx = malloc(nx * sizeof *hx);
    uint16_t* hy = malloc(ny * sizeof *hy);
    int* ix = malloc(nx * sizeof *ix);
    int* iy = malloc(ny * sizeof *iy);
    float* hw = malloc(nw * sizeof *hw);
    if (!hx || !hy || !ix || !iy || !hw) return 1;
    uint32_t seed = 12345u;
    for (size_t i = 0; i < nx; ++i) {
        seed = seed * 1664525u + 1013904223u;
        ix[i] = (int)((seed >> 16) % 7u) - 3;
        hx[i] = bf16_of_int(ix[i]);
    }
    for (size_t i = 0; i < ny; ++i) {
        seed = seed * 1664525u + 1013904223u;
        iy[i] = (int)((seed >> 16) % 7u) - 3;
        hy[i] = bf16_of_int(iy[i]);
    }
    tag_comm_t comm = NULL;
    CHECK_TAG(tag_comm_create(NULL, 1, 0, 0, &comm));
    tag_sfb_desc_t desc = {.M = M, .N = N, .B = B, .n = 1, .in_dtype = TAG_BF16,
                           .wire_dtype = TAG_BF16, .out_dtype = TAG_F32};
    tag_sfb_plan_t plan = NULL;
    CHECK_TAG(tag_sfb_plan(comm, &desc, &plan));
    void *dx, *dy, *dw;
    CHECK_CUDA(cudaMalloc(&dx, nx * 2));
    CHECK_CUDA(cudaMalloc(&dy, ny * 2));
    CHECK_CUDA(cudaMalloc(&dw, nw * 4));
    CHECK_CUDA(cudaMemcpy(dx, hx, nx * 2, cudaMemcpyHostToDevice));
    CHECK_CUDA(cudaMemcpy(dy, hy, ny * 2, cudaMemcpyHostToDevice));
    CHECK_TAG(tag_sfb_sync(plan, dx, dy, dw, NULL));
    CHECK_CUDA(cudaDeviceSynchronize());
    CHECK_CUDA(cudaMemcpy(hw, dw, nw * 4, cudaMemcpyDeviceToHost));
    int64_t bad = 0;
    for (int64_t m = 0; m < M; ++m)
        for (int64_t j = 0; j < N; ++j) {
            double s = 0.0;
            for (int64_t b = 0; b < B; ++b) s += (double)ix[b * M + m] * (double)iy[b * N + j];
            if ((double)hw[m * N + j] != s / (double)B) ++bad;
        }
    printf("tag_sfb_sync %lld x %lld, B = %lld: %lld mismatches\n", (long long)M, (long long)N,
           (long long)B, (long long)bad);
    CHECK_TAG(tag_sfb_plan_destroy(plan));
    CHECK_TAG(tag_comm_destroy(comm));
    cudaFree(dx);
    cudaFree(dy);
    cudaFree(dw);
    free(hx); free(hy); free(ix); free(iy); free(hw);
    return bad == 0 ? 0 : 1;
}

int main(int argc, char** argv) {
    const int host_only = argc > 1 && strcmp(argv[1], "--host") == 0;
    if (host_part() != 0) return 1;
    if (host_only) return 0;
    return gpu_part();
}
