// ilp.cpp — the general SFB cut ILP of TAG, host only.
//
// For one gradient tensor (g, l) of a replicated op group V the paper decides which ops to
// "Duplicate" (alpha_i = 1) by
//   min (D-1) sum_i alpha_i T_i + D(D-1) sum_{(j,i) in E} b_ji L_ji / tau - 2 alpha_g (D-1)/D L_gl/tau
//   s.t. alpha_k <= sum_{(k,i) in E} alpha_i  (k in V \ {l}),  b_ji >= alpha_i - alpha_j
// (objective P:563-567, constraints P:569-574, notation P:585-594; the paper runs Cbc, P:615-616,
// and calls it "an integer linear program similar to the min-cut problem, but with additional node
// weights on one side of the cut").
//
// Readings (DESIGN R20): alpha_l = 1 with T_l excluded; a producer outside
// the group (src = -1) has alpha = 0; edges into l are not cut candidates (l runs on every replica
// in both options; the gradient's own synchronisation is the third term); b_ji is the smallest
// feasible value max(0, alpha_i - alpha_j) because it only adds cost.
//
// Exact polynomial solution. Every cost term except the gradient saving is non-negative, so the
// optimum is either alpha = 0 (objective 0) or alpha_g = 1 with the set S of duplicated ops
// minimising  sum_{k in S} c_k + sum_{(j,i): i in S, j not in S} w_ji  over S containing g. Without
// constraint 1 that is a submodular pseudo-boolean minimisation, i.e. ONE s-t minimum cut: node k
// on the source side <=> k in S; unary c_k = edge k->t; pairwise w_ji [i in S, j not] = edge i->j;
// an outside producer = edge i->t; g forced by s->g of infinite capacity. Constraint 1 is then
// automatic for the inclusion-minimal minimum cut (the source side reachable in the residual
// graph): an op of S without a consumer in S u {l} could be dropped at no extra cost, contradicting
// minimality. That minimal set is also the unique optimum with the fewest ops (min cuts form a
// lattice), which is the tie-break the oracle's brute force applies. SFB iff its cost minus the
// saving is < 0 (ties keep AllReduce).
//
// Integer units: every term multiplied by D * tau * 1e9 — compute (D-1) T_i[ns] D tau, broadcast
// D^2 (D-1) 1e9 L_ji, saving 2 (D-1) 1e9 L_gl — in 128-bit integers (input bounds keep every sum
// below 2^122), so decisions equal the oracle's exact rationals.
#include <cstdint>
#include <cstring>
#include <vector>

#include "tag_internal.h"

namespace tag {
namespace {

using i128 = __int128;

// Dinic's max flow on a tiny graph (<= 66 nodes, <= 4096 + 130 arcs), 128-bit capacities.
struct MaxFlow {
    struct Arc { int to; i128 cap; };
    std::vector<Arc> arcs;
    std::vector<std::vector<int>> adj;
    std::vector<int> level, it;
    explicit MaxFlow(int n) : adj(n), level(n), it(n) {}
    void add(int u, int v, i128 c) {
        adj[u].push_back(static_cast<int>(arcs.size()));
        arcs.push_back({v, c});
        adj[v].push_back(static_cast<int>(arcs.size()));
        arcs.push_back({u, 0});
    }
    bool bfs(int s, int t) {
        std::fill(level.begin(), level.end(), -1);
        std::vector<int> q{s};
        level[s] = 0;
        for (size_t h = 0; h < q.size(); ++h)
            for (int a : adj[q[h]])
                if (arcs[a].cap > 0 && level[arcs[a].to] < 0) {
                    level[arcs[a].to] = level[q[h]] + 1;
                    q.push_back(arcs[a].to);
                }
        return level[t] >= 0;
    }
    i128 dfs(int u, int t, i128 f) {
        if (u == t) return f;
        for (int& i = it[u]; i < static_cast<int>(adj[u].size()); ++i) {
            Arc& e = arcs[adj[u][i]];
            if (e.cap > 0 && level[e.to] == level[u] + 1) {
                const i128 d = dfs(e.to, t, f < e.cap ? f : e.cap);
                if (d > 0) {
                    e.cap -= d;
                    arcs[adj[u][i] ^ 1].cap += d;
                    return d;
                }
            }
        }
        return 0;
    }
    i128 run(int s, int t) {
        i128 flow = 0;
        while (bfs(s, t)) {
            std::fill(it.begin(), it.end(), 0);
            while (i128 f = dfs(s, t, (static_cast<i128>(1) << 125))) flow += f;
        }
        return flow;
    }
    // nodes reachable from s in the residual graph = the minimal source side
    std::vector<char> source_side(int s) {
        std::vector<char> seen(adj.size(), 0);
        std::vector<int> q{s};
        seen[s] = 1;
        for (size_t h = 0; h < q.size(); ++h)
            for (int a : adj[q[h]])
                if (arcs[a].cap > 0 && !seen[arcs[a].to]) {
                    seen[arcs[a].to] = 1;
                    q.push_back(arcs[a].to);
                }
        return seen;
    }
};

bool has_cycle(int V, const std::vector<int>& src, const std::vector<int>& dst) {
    std::vector<int> indeg(V, 0);
    std::vector<std::vector<int>> out(V);
    for (size_t e = 0; e < src.size(); ++e)
        if (src[e] >= 0) {
            out[src[e]].push_back(dst[e]);
            ++indeg[dst[e]];
        }
    std::vector<int> q;
    for (int i = 0; i < V; ++i)
        if (!indeg[i]) q.push_back(i);
    size_t seen = 0;
    while (!q.empty()) {
        const int k = q.back();
        q.pop_back();
        ++seen;
        for (int i : out[k])
            if (--indeg[i] == 0) q.push_back(i);
    }
    return seen != static_cast<size_t>(V);
}

}  // namespace
}  // namespace tag

extern "C" tag_status_t tag_sfb_ilp_solve(const tag_sfb_ilp_t* in, uint8_t* alpha_out,
                                          double* objective_s) {
    using namespace tag;
    if (!in || !alpha_out) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_ilp_solve: NULL argument");
    const int V = in->num_ops;
    if (V < 2 || V > 64) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_ilp_solve: num_ops must be in [2, 64]");
    if (in->l < 0 || in->l >= V || in->g < 0 || in->g >= V || in->l == in->g)
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_ilp_solve: bad l / g");
    if (in->D < 1 || in->D > 1024 || in->tau == 0 || in->tau > (1ull << 44))
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_ilp_solve: D in [1, 1024], tau in [1, 2^44]");
    if (in->num_edges < 0 || in->num_edges > 4096 || !in->op_ns ||
        (in->num_edges > 0 && (!in->edge_src || !in->edge_dst || !in->edge_bytes)))
        return fail(TAG_ERR_INVALID_ARG, "tag_sfb_ilp_solve: bad edge arrays");
    if (in->grad_bytes > (1ull << 50))
        return fail(TAG_ERR_UNSUPPORTED, "tag_sfb_ilp_solve: grad_bytes > 2^50");
    std::vector<int> src(in->edge_src, in->edge_src + in->num_edges);
    std::vector<int> dst(in->edge_dst, in->edge_dst + in->num_edges);
    for (int e = 0; e < in->num_edges; ++e) {
        if (dst[e] < 0 || dst[e] >= V || src[e] < -1 || src[e] >= V || src[e] == dst[e])
            return fail(TAG_ERR_INVALID_ARG, "tag_sfb_ilp_solve: bad edge endpoints");
        if (in->edge_bytes[e] > (1ull << 50))
            return fail(TAG_ERR_UNSUPPORTED, "tag_sfb_ilp_solve: edge bytes > 2^50");
    }
    for (int i = 0; i < V; ++i)
        if (in->op_ns[i] > (1ull << 40)) return fail(TAG_ERR_UNSUPPORTED, "tag_sfb_ilp_solve: T > 2^40 ns");
    if (has_cycle(V, src, dst)) return fail(TAG_ERR_INVALID_ARG, "tag_sfb_ilp_solve: the op group has a cycle");

    const i128 D = in->D, tau = static_cast<i128>(in->tau), G9 = 1000000000;
    const int s = V, t = V + 1;                   // l (index in->l) is left out of the cut graph
    MaxFlow mf(V + 2);
    const i128 inf = static_cast<i128>(1) << 124;
    for (int k = 0; k < V; ++k)
        if (k != in->l) {
            const i128 c = (D - 1) * static_cast<i128>(in->op_ns[k]) * D * tau;   // [k in S]
            if (c > 0) mf.add(k, t, c);
        }
    for (int e = 0; e < in->num_edges; ++e) {
        const int j = src[e], i = dst[e];
        if (i == in->l) continue;                                   // not a cut candidate
        const i128 w = D * D * (D - 1) * G9 * static_cast<i128>(in->edge_bytes[e]);
        if (w == 0) continue;
        if (j < 0 || j == in->l) mf.add(i, t, w);                   // producer never in S
        else mf.add(i, j, w);                                       // [i in S, j not in S]
    }
    mf.add(s, in->g, inf);                                          // alpha_g = 1
    const i128 cost = mf.run(s, t);
    const i128 save = 2 * (D - 1) * G9 * static_cast<i128>(in->grad_bytes);
    const bool sfb = cost - save < 0;
    std::vector<char> side = mf.source_side(s);
    for (int k = 0; k < V; ++k) alpha_out[k] = k == in->l ? 1 : (sfb && side[k] ? 1 : 0);
    if (objective_s)
        *objective_s = sfb ? static_cast<double>(cost - save) /
                                 (static_cast<double>(D) * static_cast<double>(tau) * 1e9)
                           : 0.0;
    return TAG_OK;
}
