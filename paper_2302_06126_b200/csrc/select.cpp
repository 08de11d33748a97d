// select.cpp — step a6: per-layer SFB vs AllReduce selector (host only).
//
// The paper's per-gradient SFB ILP (P:563-567 objective, P:569-574 constraints, notation
// P:578-600) restricted to one Dense-layer MatMul cut {x, ∇} (DESIGN R4b): duplicating the
// gradient op g (alpha_g = 1) costs
//     (n-1) T_g  +  c_rule * S / tau        (extra compute; factor broadcast)
// and saves the ring AllReduce  2 (n-1)/n * G / tau, with
//     S = B (M + N) e_w   (per-replica cut bytes L_x + L_∇, R3),   G = M N e_g,
//     T_g = 2 M N B / F   (linear compute model; F = 0 drops the term, R4),
//     c_rule = n (north_star, default) | n(n-1) (paper ILP) | n-1 (all-gather wire) (R2).
// SFB iff strictly cheaper; ties keep AllReduce; n = 1 -> NONE.
//
// Evaluated exactly: multiply by n * tau * F > 0 and compare 128-bit integers (R4c):
//     F > 0 : n(n-1) 2MNB tau + n c S F  <  2 (n-1) G F
//     F = 0 : n c S                      <  2 (n-1) G
// Overflow of any intermediate is detected and reported, never wrapped.
#include <cstdint>

#include "tag_internal.h"

namespace tag {
namespace {

using i128 = __int128;
using u128 = unsigned __int128;

// a * b with overflow detection on non-negative 127-bit values.
bool mul(i128 a, i128 b, i128* out) {
    if (a < 0 || b < 0) return false;
    if (a == 0 || b == 0) { *out = 0; return true; }
    const u128 lim = (static_cast<u128>(1) << 127) - 1;
    if (static_cast<u128>(a) > lim / static_cast<u128>(b)) return false;
    *out = a * b;
    return true;
}

bool add(i128 a, i128 b, i128* out) {
    const i128 lim = static_cast<i128>((static_cast<u128>(1) << 127) - 1);
    if (a < 0 || b < 0 || a > lim - b) return false;
    *out = a + b;
    return true;
}

bool mul_all(std::initializer_list<i128> xs, i128* out) {
    i128 acc = 1;
    for (i128 x : xs)
        if (!mul(acc, x, &acc)) return false;
    *out = acc;
    return true;
}

}  // namespace
}  // namespace tag

extern "C" tag_status_t tag_sfb_select(const tag_layer_t* layers, int num_layers,
                                       const tag_topology_t* topo, tag_choice_t* out) {
    using namespace tag;
    if (num_layers < 0) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_select: num_layers < 0");
    if (num_layers > 0 && (!layers || !out))
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_select: NULL layers/out");
    if (!topo) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_select: NULL topology");
    if (topo->n < 1) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_select: n < 1");
    if (topo->link_bytes_per_s == 0) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_select: tau = 0");
    if (topo->rule < TAG_RULE_NORTHSTAR || topo->rule > TAG_RULE_WIRE)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_select: unknown rule");
    for (int i = 0; i < num_layers; ++i) {
        const tag_layer_t& L = layers[i];
        if (L.M < 1 || L.N < 1 || L.B < 1)
            return fail(TAG_ERR_INVALID_ARG, "tag_sfb_select: layer dims must be >= 1");
        if ((L.factor_dtype != TAG_F32 && L.factor_dtype != TAG_BF16) ||
            (L.grad_dtype != TAG_F32 && L.grad_dtype != TAG_BF16))
            return fail(TAG_ERR_INVALID_ARG, "tag_sfb_select: unknown dtype");
    }
    // decide everything first, write `out` only if every layer succeeds (no partial output)
    const i128 n = topo->n;
    const i128 tau = static_cast<i128>(topo->link_bytes_per_s);
    const i128 F = static_cast<i128>(topo->tensor_flops);
    const i128 c = topo->rule == TAG_RULE_NORTHSTAR ? n : topo->rule == TAG_RULE_PAPER_ILP ? n * (n - 1) : n - 1;
    for (int pass = 0; pass < 2; ++pass) {
        for (int i = 0; i < num_layers; ++i) {
            const tag_layer_t& L = layers[i];
            tag_choice_t choice;
            if (n <= 1) {
                choice = TAG_SYNC_NONE;
            } else {
                const i128 M = L.M, N = L.N, B = L.B;
                const i128 ew = static_cast<i128>(dtype_size(L.factor_dtype));
                const i128 eg = static_cast<i128>(dtype_size(L.grad_dtype));
                i128 S, G, lhs, rhs, t1, t2;
                bool ok = mul_all({B, M + N, ew}, &S) && mul_all({M, N, eg}, &G);
                if (F > 0) {
                    ok = ok && mul_all({n, n - 1, 2, M, N, B, tau}, &t1) &&
                         mul_all({n, c, S, F}, &t2) && add(t1, t2, &lhs) &&
                         mul_all({2, n - 1, G, F}, &rhs);
                } else {
                    ok = ok && mul_all({n, c, S}, &lhs) && mul_all({2, n - 1, G}, &rhs);
                }
                if (!ok) return fail(TAG_ERR_UNSUPPORTED, "tag_sfb_select: 127-bit overflow");
                choice = lhs < rhs ? TAG_SYNC_SFB : TAG_SYNC_ALLREDUCE;
            }
            if (pass == 1) out[i] = choice;
        }
    }
    return TAG_OK;
}
