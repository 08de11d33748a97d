"""Pins for the CPU oracle (`-m "not gpu"`): the oracle is checked against things other than itself —
values the paper/SPEC print, closed forms, invariants, exact-rational brute force, and textbook
library routines — so that a dropped term, wrong sign/index or transposed operand fails a test.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

from paper_2302_06126_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
SHAPES = [(1, 1, 1, 2), (3, 5, 2, 3), (17, 33, 3, 4), (64, 32, 4, 2), (130, 257, 5, 2)]  # (M,N,B,n)


def _rel_fro(a, r):
    return np.linalg.norm(a - r) / np.linalg.norm(r)


def _inputs(M, N, B, n, dist="normal", cid=900):
    return synth.all_factors(cid, M * 1000 + N, n, M, N, B, dist, dist)


# ---------------------------------------------------------------------------------------------
# Lossless: SFB reconstruction == dense AllReduce result
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("M,N,B,n", SHAPES)
def test_lossless_random(oracle_mod, M, N, B, n):
    X, dY = _inputs(M, N, B, n)
    d, s = oracle_mod.dense_dw(X, dY), oracle_mod.sfb_dw(X, dY)
    assert _rel_fro(s, d) <= 1e-13


@pytest.mark.parametrize("M,N,B,n", SHAPES)
def test_lossless_integers_exact(oracle_mod, M, N, B, n):
    X, dY = _inputs(M, N, B, n, "int3")
    assert np.array_equal(oracle_mod.dense_sum(X, dY), oracle_mod.sfb_sum(X, dY))
    assert np.array_equal(oracle_mod.dense_dw(X, dY), oracle_mod.sfb_dw(X, dY))


# ---------------------------------------------------------------------------------------------
# Brute force with exact rationals (P:520-526 definition written out element by element)
# ---------------------------------------------------------------------------------------------
@pytest.mark.parametrize("M,N,B,n", [(1, 1, 1, 2), (3, 5, 2, 3), (4, 3, 3, 2)])
@pytest.mark.parametrize("dist", ["int3", "normal"])
def test_bruteforce_fractions(oracle_mod, M, N, B, n, dist):
    X, dY = _inputs(M, N, B, n, dist)
    got = oracle_mod.sfb_dw(X, dY)
    got_dense = oracle_mod.dense_dw(X, dY)
    for m in range(M):
        for j in range(N):
            exact = sum(Fraction(float(X[r, b, m])) * Fraction(float(dY[r, b, j]))
                        for r in range(n) for b in range(B)) / (n * B)
            if dist == "int3":
                # K <= 6 products of small integers: the fp64 sum is exact; /nB rounds once
                assert got[m, j] == float(exact) and got_dense[m, j] == float(exact)
            else:
                assert abs(Fraction(got[m, j]) - exact) <= abs(exact) * Fraction(1, 2 ** 48) + \
                    Fraction(1, 2 ** 60)


def test_fixture_shapes_against_fractions_integer_sum(oracle_mod):
    """(130,257,5,2) and (17,33,3,4): non-power-of-two nB and odd tiles; integer sums exact."""
    for (M, N, B, n) in [(17, 33, 3, 4), (130, 257, 5, 2)]:
        X, dY = _inputs(M, N, B, n, "int3")
        S = oracle_mod.sfb_sum(X, dY)
        Xi, dYi = X.astype(np.int64), dY.astype(np.int64)
        exact = np.zeros((M, N), dtype=np.int64)
        for r in range(n):
            exact += Xi[r].T @ dYi[r]          # integer matmul: exact
        assert np.array_equal(S, exact.astype(np.float64))


# ---------------------------------------------------------------------------------------------
# Textbook reductions
# ---------------------------------------------------------------------------------------------
def test_n1_reduces_to_matmul(oracle_mod):
    """n = 1: dW = (1/B) X^T dY — checked against torch.matmul in fp64 (a library routine)."""
    X, dY = _inputs(96, 80, 7, 1)
    ref = (torch.from_numpy(X[0]).double().T @ torch.from_numpy(dY[0]).double()).numpy() / 7
    assert _rel_fro(oracle_mod.sfb_dw(X, dY), ref) <= 1e-14


def test_dense_sum_is_sum_of_replica_products(oracle_mod):
    X, dY = _inputs(40, 24, 6, 3)
    ref = sum(X[r].astype(np.float64).T @ dY[r].astype(np.float64) for r in range(3))
    assert _rel_fro(oracle_mod.dense_sum(X, dY), ref) <= 1e-14
    # orientation pin: dW[m][j] pairs input feature m with output feature j
    m, j = 7, 19
    direct = sum(float(X[r, b, m]) * float(dY[r, b, j]) for r in range(3) for b in range(6))
    assert abs(oracle_mod.dense_sum(X, dY)[m, j] - direct) <= 1e-12 * max(1.0, abs(direct))


def test_scale_ones(oracle_mod):
    """X = 1, dY = 1 -> every entry of the (1/(nB))-scaled gradient is exactly 1."""
    for (M, N, B, n) in [(5, 3, 3, 3), (64, 32, 4, 2), (8, 8, 7, 5)]:
        X = np.ones((n, B, M), np.float32)
        dY = np.ones((n, B, N), np.float32)
        assert np.all(oracle_mod.sfb_dw(X, dY) == 1.0)
        assert np.all(oracle_mod.dense_dw(X, dY) == 1.0)


def test_scale_is_global_batch_mean(oracle_mod):
    """Replicating one replica's factors n times leaves the mean gradient unchanged (alpha=1/(nB))."""
    X, dY = _inputs(12, 10, 4, 1, "int3")
    one = oracle_mod.sfb_dw(X, dY)
    rep = oracle_mod.sfb_dw(np.repeat(X, 4, axis=0), np.repeat(dY, 4, axis=0))
    assert np.array_equal(one, rep)


def test_rank_bound(oracle_mod):
    """rank(dW) <= nB (the gradient is the product of two smaller matrices); Gaussian
    factors with nB < min(M, N) give rank exactly nB."""
    X, dY = _inputs(64, 32, 4, 2)
    s = np.linalg.svd(oracle_mod.sfb_dw(X, dY), compute_uv=False)
    assert s[8] / s[0] < 1e-12
    assert s[7] / s[0] > 1e-6


def test_entries_match_full(oracle_mod):
    X, dY = _inputs(130, 257, 5, 2)
    full = oracle_mod.sfb_sum(X, dY)
    idx = np.random.default_rng(0).integers(0, 130 * 257, 300)
    assert np.array_equal(oracle_mod.sfb_sum_entries(X, dY, idx), full.ravel()[idx])


# ---------------------------------------------------------------------------------------------
# SGD-momentum (R14): closed form for a constant gradient
# ---------------------------------------------------------------------------------------------
def test_sgd_closed_form(oracle_mod):
    g = np.random.default_rng(1).standard_normal((6, 5))
    W0 = np.random.default_rng(2).standard_normal((6, 5))
    W, v = W0.copy(), np.zeros_like(W0)
    lr, mu, k = 0.05, 0.9, 7
    for _ in range(k):
        W, v = oracle_mod.sgd_momentum(g, W, v, lr, mu, 0.0)
    vk = g * (1 - mu ** k) / (1 - mu)
    Wk = W0 - lr * g * sum((1 - mu ** j) / (1 - mu) for j in range(1, k + 1))
    assert np.allclose(v, vk, rtol=1e-13, atol=1e-15)
    assert np.allclose(W, Wk, rtol=1e-13, atol=1e-15)


def test_sgd_weight_decay_folds_into_gradient(oracle_mod):
    rs = np.random.default_rng(3)
    g, W0, v0 = rs.standard_normal((4, 4)), rs.standard_normal((4, 4)), rs.standard_normal((4, 4))
    a = oracle_mod.sgd_momentum(g, W0, v0, 0.1, 0.5, 0.01)
    b = oracle_mod.sgd_momentum(g + 0.01 * W0, W0, v0, 0.1, 0.5, 0.0)
    assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    # mu = 0, wd = 0 is plain gradient descent W - lr*g (P:283 GradientDescent)
    c = oracle_mod.sgd_momentum(g, W0, v0, 0.1, 0.0, 0.0)
    assert np.allclose(c[0], W0 - 0.1 * g, rtol=0, atol=1e-15)


# ---------------------------------------------------------------------------------------------
# RNE fp32 -> bf16 cast (R11), pinned to torch's CPU conversion (a library routine)
# ---------------------------------------------------------------------------------------------
def test_bf16_rne_matches_torch(oracle_mod):
    rs = np.random.default_rng(4)
    x = np.concatenate([
        rs.standard_normal(100000).astype(np.float32),
        (rs.standard_normal(1000) * 1e-38).astype(np.float32),            # subnormals
        np.array([0.0, -0.0, np.inf, -np.inf, 3.4e38, -3.4e38, 1.0, 1 + 2 ** -8, 1 + 3 * 2 ** -8,
                  1 + 2 ** -9, 1 + 3 * 2 ** -9], np.float32),               # exact ties, both ways
    ])
    ours = oracle_mod.cast_bf16_bits(x)
    ref = torch.from_numpy(x).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(ours, ref)
    nan = oracle_mod.cast_bf16_bits(np.array([np.nan], np.float32))
    assert np.isnan(oracle_mod.bf16_bits_to_f64(nan)[0])


def test_bf16_tie_rounds_to_even(oracle_mod):
    # 1 + 2^-8 is exactly half-way between bf16 1.0 and 1 + 2^-7: even mantissa (1.0) wins
    assert oracle_mod.bf16_bits_to_f64(oracle_mod.cast_bf16_bits(
        np.array([1 + 2 ** -8], np.float32)))[0] == 1.0
    assert oracle_mod.bf16_bits_to_f64(oracle_mod.cast_bf16_bits(
        np.array([1 + 3 * 2 ** -8], np.float32)))[0] == 1 + 2 ** -6


# ---------------------------------------------------------------------------------------------
# Byte counts, ring AllReduce, ILP objective (golden values printed by the paper / SPEC)
# ---------------------------------------------------------------------------------------------
def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def test_spec_volume_fixture(oracle_mod):
    g = _golden("spec_volume.json")
    S = oracle_mod.selector
    assert S.sfb_elements_fig5(g["H1"], g["H2"], g["B"]) == g["sfb_elements"]
    assert S.gradient_elements(g["H1"], g["H2"]) == g["gradient_elements"]
    assert g["gradient_elements"] // g["sfb_elements"] == g["reduction"]
    # north_star's gathered-bytes count coincides with Fig. 5 at D = 2 (R2), in elements
    assert S.sfb_gathered_bytes(g["D"], g["B"], g["H1"], g["H2"], 1) == g["sfb_elements"]
    # and the all-gather wire per rank is half of it at D = 2
    assert S.allgather_ingress_bytes(2, 4, 256, 256, 1) == 2048


def test_spec_ring_allreduce(oracle_mod):
    for c in _golden("spec_ring_allreduce.json")["cases"]:
        t = oracle_mod.selector.ring_allreduce_time(c["D"], c["size_bytes"], c["tau"])
        assert t == Fraction(c["seconds"])


def _simulate_ring_allreduce(n, chunks):
    """Independent brute force: a ring AllReduce of n ranks' vectors, each split into n chunks —
    reduce-scatter (n-1 steps: rank r sends its running sum of chunk (r - s) mod n to r+1), then
    all-gather (n-1 steps: the owner of a finished chunk passes it on). Returns (per-rank result,
    elements each rank sent)."""
    data = [[list(c) for c in chunks_r] for chunks_r in chunks]      # data[rank][chunk] = list
    sent = [0] * n
    for s in range(n - 1):                                           # reduce-scatter
        msgs = []
        for r in range(n):
            c = (r - s) % n
            msgs.append(((r + 1) % n, c, list(data[r][c])))
            sent[r] += len(data[r][c])
        for dst, c, vals in msgs:
            data[dst][c] = [a + b for a, b in zip(data[dst][c], vals)]
    for s in range(n - 1):                                           # all-gather
        msgs = []
        for r in range(n):
            c = (r + 1 - s) % n
            msgs.append(((r + 1) % n, c, list(data[r][c])))
            sent[r] += len(data[r][c])
        for dst, c, vals in msgs:
            data[dst][c] = vals
    return data, sent


def test_ring_allreduce_bytes_brute_force(oracle_mod):
    """ring_allreduce_bytes (P:566 / P:611-612: 2(D-1)/D * L per rank) against a simulated ring
    that also checks the reduction itself; and its time equals ring_allreduce_time."""
    S = oracle_mod.selector
    rng = np.random.default_rng(7)
    for n in (2, 3, 4, 8):
        for M, N in ((4, 6), (8, 3), (5, 8)):
            L = M * N * n                            # elements; divisible into n equal chunks
            vecs = [rng.integers(-5, 5, L).tolist() for _ in range(n)]
            chunks = [[v[c * (L // n):(c + 1) * (L // n)] for c in range(n)] for v in vecs]
            data, sent = _simulate_ring_allreduce(n, chunks)
            want = [sum(col) for col in zip(*vecs)]
            for r in range(n):
                assert sum(data[r], []) == want
            for e_g in (2, 4):
                assert all(Fraction(x * e_g) == S.ring_allreduce_bytes(n, M * n, N, e_g) for x in sent)
                assert S.ring_allreduce_bytes(n, M * n, N, e_g) / Fraction(10 ** 9) == \
                    S.ring_allreduce_time(n, M * n * N * e_g, 10 ** 9)


def test_spec_ilp_objective(oracle_mod):
    S = oracle_mod.selector
    c1, c2 = _golden("spec_sfb_ilp.json")["cases"]
    obj = S.ilp_objective(c1["D"], Fraction(c1["T_g"]), c1["cut_bytes"], c1["L_gl"], c1["tau"])
    assert obj == Fraction(c1["objective"])
    L = c1["as_layer"]
    layer = dict(M=L["M"], N=L["N"], B=L["B"], e_w=L["e_w"], e_g=L["e_g"])
    topo = dict(n=2, tau=c1["tau"], F=L["F"], rule=S.RULE_PAPER_ILP)
    sfb, ar = S.sfb_cost_terms(layer, topo)
    assert sfb - ar == Fraction(c1["objective"])
    for rule in (S.RULE_PAPER_ILP, S.RULE_NORTHSTAR, S.RULE_WIRE):
        assert S.select(layer, dict(topo, rule=rule)) == S.CHOICE_SFB
    # WIRE reading at D = 2: (n-1) S / tau instead of n(n-1) S / tau -> -9.8e-4
    sfb, ar = S.sfb_cost_terms(layer, dict(topo, rule=S.RULE_WIRE))
    assert sfb - ar == Fraction("-9.8e-4")
    # second SPEC case: cut == gradient size, zero compute, D = 2 -> keep AllReduce (alpha = 0)
    assert S.ilp_objective(2, 0, c2["cut_bytes"], c2["L_gl"], c2["tau"]) > 0
    layer2 = dict(M=1000, N=1000, B=1, e_w=500, e_g=1)      # S = 1e6 B = G, T_g dropped (F = 0)
    assert S.select(layer2, dict(n=2, tau=c2["tau"], F=0, rule=S.RULE_PAPER_ILP)) == \
        S.CHOICE_ALLREDUCE


def test_selector_n1_and_tie(oracle_mod):
    S = oracle_mod.selector
    lay = dict(M=16, N=16, B=4, e_w=2, e_g=2)
    assert S.select(lay, dict(n=1, tau=1, F=0)) == S.CHOICE_NONE
    # exact tie: n^2 S = 4*256 = 1024 = 2 (n-1) G -> AllReduce
    sfb, ar = S.sfb_cost_terms(lay, dict(n=2, tau=10 ** 9, F=0))
    assert sfb == ar
    assert S.select(lay, dict(n=2, tau=10 ** 9, F=0)) == S.CHOICE_ALLREDUCE
    assert S.select(dict(lay, B=3), dict(n=2, tau=10 ** 9, F=0)) == S.CHOICE_SFB


def test_selector_integer_form_equals_fraction_form(oracle_mod):
    S = oracle_mod.selector
    rs = np.random.default_rng(5)
    for _ in range(3000):
        lay = dict(M=int(rs.integers(1, 40000)), N=int(rs.integers(1, 40000)),
                   B=int(rs.integers(1, 600)), e_w=int(rs.choice([2, 4])),
                   e_g=int(rs.choice([2, 4])))
        topo = dict(n=int(rs.integers(1, 17)), tau=int(rs.integers(1, 10 ** 12)),
                    F=int(rs.choice([0, int(rs.integers(1, 3 * 10 ** 15))])),
                    rule=int(rs.integers(0, 3)))
        assert S.select(lay, topo) == S.select_integer_form(lay, topo)


def test_appendix_a_decision_table(oracle_mod):
    S = oracle_mod.selector
    name = {S.CHOICE_ALLREDUCE: "AR", S.CHOICE_SFB: "SFB", S.CHOICE_NONE: "NONE"}
    cases = _golden("appendix_a_decisions.json")["cases"]
    assert len(cases) == 200
    for c in cases:
        lay = dict(M=c["M"], N=c["N"], B=c["B"], e_w=c["e_w"], e_g=c["e_g"])
        topo = dict(n=c["n"], tau=c["tau"], F=c["F"], rule=c["rule"])
        assert name[S.select(lay, topo)] == c["expect"], c


# ---------------------------------------------------------------------------------------------
# Profiled selector (paper's profiler P:323-334; SPEC fit_comm S:197-205)
# ---------------------------------------------------------------------------------------------
def test_spec_fit_comm_interpolation(oracle_mod):
    g = _golden("spec_fit_comm.json")
    for x, want in g["queries"]:
        assert oracle_mod.selector.curve_ns(g["points"], x) == want


def test_curve_first_segment_and_clamp(oracle_mod):
    S = oracle_mod.selector
    pts = [(1000, 5000), (2000, 9000), (4000, 10000)]
    assert S.curve_ns(pts, 500) == 3000          # extended below the first point
    assert S.curve_ns(pts, 0) == 1000
    assert S.curve_ns([(1000, 100), (2000, 5000)], 0) == 0      # clamped at 0
    assert S.curve_ns(pts, 3000) == 9500         # second segment
    assert S.curve_ns(pts, 8000) == 12000        # last segment's slope


def test_profiled_reduces_to_ring_model(oracle_mod):
    """Linear curves t = bytes / tau (gather) and t = 2(n-1)/n G / tau (ring AR), no latency: the
    profiled rule decides like the analytic WIRE rule (F = 0) wherever it is not a tie."""
    S = oracle_mod.selector
    rs = np.random.default_rng(21)
    tau = 10 ** 9                                 # 1 byte per ns
    checked = 0
    for _ in range(2000):
        n = int(rs.integers(2, 17))
        lay = dict(M=int(rs.integers(8, 5000)), N=int(rs.integers(8, 5000)),
                   B=int(rs.integers(1, 300)), e_w=2, e_g=4)
        gather = [(0, 0), (10 ** 12, 10 ** 12)]
        ar = [(0, 0), (n * 10 ** 12, 2 * (n - 1) * 10 ** 12)]     # slope 2(n-1)/n
        sfb_ns = (n - 1) * lay["B"] * (lay["M"] + lay["N"]) * 2
        ar_exact = Fraction(2 * (n - 1) * lay["M"] * lay["N"] * 4, n)
        if abs(sfb_ns - ar_exact) <= 1:
            continue                              # floor rounding may flip exact ties
        want = S.select(lay, dict(n=n, tau=tau, F=0, rule=S.RULE_WIRE))
        assert S.select_profiled(lay, n, gather, ar) == want
        checked += 1
    assert checked > 1900


def test_profiled_latency_flips_small_layers(oracle_mod):
    """A fixed per-call latency on the gather (the measured NVLink push floor) turns tiny layers
    to AllReduce that the bandwidth-only model sends to SFB — the reason for profiling."""
    S = oracle_mod.selector
    lay = dict(M=1024, N=1024, B=2, e_w=2, e_g=4)        # BERT-L pooler, n = 8
    gather = [(0, 20000), (10 ** 9, 20000 + 10 ** 9 // 700)]      # 20 us + 700 GB/s
    ar = [(0, 8000), (10 ** 9, 8000 + 10 ** 9 // 700)]            # 8 us + 700 GB/s
    assert S.select(lay, dict(n=8, tau=900 * 10 ** 9, F=0)) == S.CHOICE_SFB
    assert S.select_profiled(lay, 8, gather, ar) == S.CHOICE_ALLREDUCE
    big = dict(M=25088, N=4096, B=32, e_w=2, e_g=4)        # VGG-19 fc6 stays SFB
    assert S.select_profiled(big, 8, gather, ar) == S.CHOICE_SFB


# ------------------------------------------------------------------ bias gradient (R17)
def test_bias_dense_equals_sfb_and_numpy(oracle_mod):
    """Lossless for the bias too: the AllReduce route (per-replica column sums, rank order) and
    the SFB route (column sums of dY_all) agree, exactly on integers; numpy's sum pins both."""
    rs = np.random.default_rng(51)
    for n, B, N in ((1, 1, 1), (2, 4, 32), (3, 5, 17), (8, 32, 1000)):
        dYi = rs.integers(-3, 4, (n, B, N)).astype(np.float64)
        assert np.array_equal(oracle_mod.dense_bias_sum(dYi), oracle_mod.sfb_bias_sum(dYi))
        assert np.array_equal(oracle_mod.sfb_bias_sum(dYi), dYi.sum(axis=(0, 1)))
        dYr = rs.standard_normal((n, B, N))
        np.testing.assert_allclose(oracle_mod.dense_bias_sum(dYr), oracle_mod.sfb_bias_sum(dYr),
                                   rtol=1e-13, atol=1e-13)
        np.testing.assert_allclose(oracle_mod.sfb_bias(dYr), dYr.reshape(n * B, N).mean(axis=0),
                                   rtol=1e-13, atol=1e-13)


def test_bias_is_weight_gradient_of_a_constant_input(oracle_mod):
    """the gradient is an outer product of the factors. Appending a constant-1 column
    to x makes the bias a row of W, and its gradient row equals the SFB bias sum."""
    rs = np.random.default_rng(52)
    n, B, M, N = 3, 4, 6, 9
    X = rs.integers(-3, 4, (n, B, M)).astype(np.float64)
    dY = rs.integers(-3, 4, (n, B, N)).astype(np.float64)
    Xa = np.concatenate([X, np.ones((n, B, 1))], axis=2)
    S = oracle_mod.sfb_sum(Xa, dY)
    assert np.array_equal(S[M], oracle_mod.sfb_bias_sum(dY))


def test_bias_fractions_and_ones(oracle_mod):
    """Exact rationals on a tiny case; dY = 1 gives db = 1 after the 1/(nB) scale."""
    n, B, N = 2, 3, 4
    vals = [[[Fraction(1, 1 + r + b + j) for j in range(N)] for b in range(B)] for r in range(n)]
    want = [sum(vals[r][b][j] for r in range(n) for b in range(B)) for j in range(N)]
    got = oracle_mod.sfb_bias_sum(np.array(vals, dtype=np.float64))
    for j in range(N):
        assert abs(Fraction(got[j]) - want[j]) <= Fraction(1, 10 ** 14)
    assert np.array_equal(oracle_mod.sfb_bias(np.ones((n, B, N))), np.ones(N))


def test_profiled_ps_option(oracle_mod):
    """Replicate-with-PS in the profiled selector: a PS curve equal to the AllReduce
    curve never wins (tie keeps AllReduce), one strictly below both wins, and one equal to SFB's
    cost keeps SFB; without a PS curve the two-way rule is unchanged."""
    S = oracle_mod.selector
    lay = dict(M=4096, N=4096, B=32, e_w=2, e_g=4)
    G = 4096 * 4096 * 4
    gather = [(1, 10_000), (10 ** 9, 10 ** 9)]          # cheap SFB
    ar = [(1, 10_000), (10 ** 9, 2 * 10 ** 9)]
    assert S.select_profiled(lay, 2, gather, ar) == S.CHOICE_SFB
    assert S.select_profiled(lay, 2, gather, ar, 0, ar) == S.CHOICE_SFB
    t_sfb = S.curve_ns(gather, 1 * 32 * (4096 + 4096) * 2)
    cheap_ps = [(0, 0), (2 * G, 2 * (t_sfb - 1))]        # ps(G) = t_sfb - 1 < t_sfb
    assert S.curve_ns(cheap_ps, G) == t_sfb - 1
    assert S.select_profiled(lay, 2, gather, ar, 0, cheap_ps) == S.CHOICE_PS
    tie_ps = [(0, 0), (2 * G, 2 * t_sfb)]
    assert S.select_profiled(lay, 2, gather, ar, 0, tie_ps) == S.CHOICE_SFB
    expensive_gather = [(1, 10 ** 9), (10 ** 9, 10 ** 10)]
    assert S.select_profiled(lay, 2, expensive_gather, ar, 0, ar) == S.CHOICE_ALLREDUCE
    assert S.select_profiled(lay, 1, gather, ar, 0, cheap_ps) == S.CHOICE_NONE


# ------------------------------------------------------------------ Adam (R22)
def test_adam_first_step_closed_form(oracle_mod):
    """t = 1: the bias corrections undo the (1 - b) factors, so W1 = W0 - lr g / (|g| + eps)."""
    rs = np.random.default_rng(71)
    g = rs.standard_normal(1000)
    W0 = rs.standard_normal(1000)
    W1, m1, v1 = oracle_mod.adam(g, W0, np.zeros(1000), np.zeros(1000), 1e-3, 0.9, 0.999, 1e-8, 0.0, 1)
    np.testing.assert_allclose(m1, 0.1 * g, rtol=1e-15)
    np.testing.assert_allclose(v1, 0.001 * g * g, rtol=1e-14)
    np.testing.assert_allclose(W1, W0 - 1e-3 * g / (np.abs(g) + 1e-8), rtol=1e-12, atol=1e-15)


def test_adam_matches_torch_optim(oracle_mod):
    """Three steps against torch.optim.Adam in float64 (an independent implementation), with
    weight decay; the gradient changes every step."""
    rs = np.random.default_rng(72)
    W = rs.standard_normal((16, 8))
    p = torch.nn.Parameter(torch.from_numpy(W.copy()))
    opt = torch.optim.Adam([p], lr=3e-3, betas=(0.8, 0.95), eps=1e-6, weight_decay=0.01)
    m, v = np.zeros_like(W), np.zeros_like(W)
    for t in range(1, 4):
        g = rs.standard_normal(W.shape)
        p.grad = torch.from_numpy(g.copy())
        opt.step()
        W, m, v = oracle_mod.adam(g, W, m, v, 3e-3, 0.8, 0.95, 1e-6, 0.01, t)
        np.testing.assert_allclose(W, p.detach().numpy(), rtol=1e-12, atol=1e-14)


def test_profiled_measured_op_times_reduce_to_linear_model(oracle_mod):
    """Measured op times that follow the linear model — recon time =
    local time + floor((n-1) 2MNB 1e9 / F) — give the analytic-compute decision exactly, with and
    without the PS option, whatever the local time; a measured reconstruction slower than the
    model by more than the margin flips SFB to AllReduce."""
    S = oracle_mod.selector
    rs = np.random.default_rng(41)
    flips = 0
    for _ in range(2000):
        def curve():
            b = np.cumsum(rs.integers(1, 10 ** 8, int(rs.integers(2, 6)))).tolist()
            return list(zip(b, rs.integers(1000, 10 ** 7, len(b)).tolist()))
        g, a, ps = curve(), curve(), curve()
        n = int(rs.integers(2, 9))
        F = int(rs.integers(10 ** 12, 3 * 10 ** 15))
        L = dict(M=int(rs.integers(1, 30000)), N=int(rs.integers(1, 30000)),
                 B=int(rs.integers(1, 2048)), e_w=int(rs.choice([2, 4])), e_g=int(rs.choice([2, 4])))
        extra = ((n - 1) * 2 * L["M"] * L["N"] * L["B"] * 10 ** 9) // F
        local = int(rs.integers(0, 10 ** 6))
        for p in (None, ps):
            want = S.select_profiled(L, n, g, a, F, p)
            assert S.select_profiled(L, n, g, a, 0, p, recon_ns=local + extra, local_ns=local) == want
        if S.select_profiled(L, n, g, a, F) == S.CHOICE_SFB:
            margin = S.curve_ns(a, L["M"] * L["N"] * L["e_g"]) - (
                S.curve_ns(g, (n - 1) * L["B"] * (L["M"] + L["N"]) * L["e_w"]) + extra)
            assert margin > 0
            assert S.select_profiled(L, n, g, a, 0, None, recon_ns=local + extra + margin,
                                     local_ns=local) == S.CHOICE_ALLREDUCE
            flips += 1
    assert flips > 100
