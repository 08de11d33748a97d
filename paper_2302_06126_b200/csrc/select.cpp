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

namespace tag {
namespace {

// floor(a / b) for b > 0 (C++ division truncates toward zero)
i128 floor_div(i128 a, i128 b) {
    i128 q = a / b;
    if ((a % b != 0) && (a < 0)) --q;
    return q;
}

bool curve_ok(const tag_curve_t& c) {
    if (c.count < 2 || !c.bytes || !c.ns) return false;
    for (int i = 1; i < c.count; ++i)
        if (c.bytes[i] <= c.bytes[i - 1]) return false;
    for (int i = 0; i < c.count; ++i)      // bounds that keep every product below 2^127
        if (c.bytes[i] > (1ull << 62) || c.ns[i] > (1ull << 40)) return false;
    return true;
}

// piecewise-linear time in ns at x bytes, floor-rounded, clamped at 0
i128 curve_ns(const tag_curve_t& c, i128 x) {
    int i = 0;                                   // segment [i, i+1]
    while (i + 2 < c.count && x > static_cast<i128>(c.bytes[i + 1])) ++i;
    const i128 b0 = c.bytes[i], b1 = c.bytes[i + 1];
    const i128 t0 = c.ns[i], t1 = c.ns[i + 1];
    i128 t = t0 + floor_div((x - b0) * (t1 - t0), b1 - b0);
    return t < 0 ? 0 : t;
}

}  // namespace
}  // namespace tag

extern "C" tag_status_t tag_sfb_select_profiled(const tag_layer_t* layers, int num_layers,
                                                const tag_profiled_topology_t* topo,
                                                tag_choice_t* out) {
    using namespace tag;
    if (num_layers < 0 || !topo || (num_layers > 0 && (!layers || !out)))
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_select_profiled: bad arguments");
    if (topo->n < 1 || topo->n > 65536)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_select_profiled: n must be in [1, 65536]");
    if (!curve_ok(topo->gather) || !curve_ok(topo->allreduce))
        return fail(TAG_ERR_INVALID_ARG,
                    "tag_sfb_select_profiled: curves need >= 2 points with increasing bytes");
    const bool has_ps = topo->ps.count != 0;
    if (has_ps && !curve_ok(topo->ps))
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_select_profiled: bad PS curve");
    for (int i = 0; i < num_layers; ++i) {
        const tag_layer_t& L = layers[i];
        if (L.M < 1 || L.N < 1 || L.B < 1 || L.M > (1ll << 24) || L.N > (1ll << 24) ||
            L.B > (1ll << 24))
            return fail(TAG_ERR_INVALID_ARG, "tag_sfb_select_profiled: layer dims out of range");
        if ((L.factor_dtype != TAG_F32 && L.factor_dtype != TAG_BF16) ||
            (L.grad_dtype != TAG_F32 && L.grad_dtype != TAG_BF16))
            return fail(TAG_ERR_INVALID_ARG, "tag_sfb_select_profiled: unknown dtype");
    }
    const bool measured = topo->recon_ns != nullptr && topo->local_ns != nullptr;
    if ((topo->recon_ns != nullptr) != (topo->local_ns != nullptr))
        return fail(TAG_ERR_INVALID_ARG,
                    "tag_sfb_select_profiled: recon_ns and local_ns go together");
    if (measured)
        for (int i = 0; i < num_layers; ++i)
            if (topo->recon_ns[i] > (1ull << 40) || topo->local_ns[i] > (1ull << 40))
                return fail(TAG_ERR_INVALID_ARG, "tag_sfb_select_profiled: op time above 2^40 ns");
    const i128 n = topo->n;
    const i128 F = static_cast<i128>(topo->tensor_flops);
    for (int i = 0; i < num_layers; ++i) {
        const tag_layer_t& L = layers[i];
        if (n <= 1) {
            out[i] = TAG_SYNC_NONE;
            continue;
        }
        const i128 M = L.M, N = L.N, B = L.B;
        const i128 S = B * (M + N) * static_cast<i128>(dtype_size(L.factor_dtype));
        const i128 G = M * N * static_cast<i128>(dtype_size(L.grad_dtype));
        i128 t_sfb = curve_ns(topo->gather, (n - 1) * S);
        i128 t_ar = curve_ns(topo->allreduce, G);
        i128 t_local = 0;
        if (measured) {
            // the measured ops: SFB reconstructs at K = nB, the dense paths compute
            // the local gradient at K = B before their collective
            t_sfb += static_cast<i128>(topo->recon_ns[i]);
            t_local = static_cast<i128>(topo->local_ns[i]);
            t_ar += t_local;
        } else if (F > 0) {
            t_sfb += floor_div((n - 1) * 2 * M * N * B * 1000000000, F);
        }
        // AllReduce unless strictly beaten; then SFB; then PS if strictly below the best so far
        tag_choice_t c = TAG_SYNC_ALLREDUCE;
        i128 best = t_ar;
        if (t_sfb < best) { c = TAG_SYNC_SFB; best = t_sfb; }
        if (has_ps && t_local + curve_ns(topo->ps, G) < best) c = TAG_SYNC_PS;
        out[i] = c;
    }
    return TAG_OK;
}
