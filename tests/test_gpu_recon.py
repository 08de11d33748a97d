"""GPU parity of the single-GPU SFB path through the C ABI (`-m gpu`): reconstruction (tcgen05 and
SIMT kernels), pack/cast, epilogues E1/E2, dense local gradient, host-buffer e2e form, edge cases.

Virtual-n: NCCL cannot put two ranks on one GPU, so the n-replica reconstruction
is exercised with a 1-rank plan whose B' = n*B rows are the n replicas' factors stacked
rank-major — the same K = nB contraction and the same alpha = 1/(nB) as after the all-gather.
Tolerances (north_star; DESIGN "Parity"): bit-exact on small-integer inputs; relative Frobenius
<= 1e-5 against the oracle fed the exact operand values; <= 2e-2 against the user's fp32 values
for bf16 wire factors.
"""
import numpy as np
import pytest
import torch

from paper_2302_06126_b200 import synth

pytestmark = pytest.mark.gpu

TORCH = {"f32": torch.float32, "bf16": torch.bfloat16}


def rel_fro(a, r):
    a = np.asarray(a, np.float64)
    r = np.asarray(r, np.float64)
    return float(np.linalg.norm(a - r) / max(np.linalg.norm(r), 1e-300))


@pytest.fixture(scope="module")
def comm1(tag, cuda):
    c = tag.Comm(1, 0, 0)
    yield c
    c.close()


def to_dev(a, dt):
    return torch.from_numpy(np.ascontiguousarray(a)).to(TORCH[dt]).to("cuda")


def exact_values(a, dt):
    """The values the GPU operates on (fp32 -> bf16 is torch RNE), as fp64."""
    return torch.from_numpy(np.ascontiguousarray(a)).to(TORCH[dt]).double().numpy()


def run_sync(tag, comm, Xall, dYall, in_dt="bf16", wire_dt="bf16", out_dt="f32"):
    K, M = Xall.shape
    N = dYall.shape[1]
    plan = tag.SfbPlan(comm, M, N, K, in_dt, wire_dt, out_dt)
    dW = torch.full((M, N), float("nan"), dtype=TORCH[out_dt], device="cuda")
    plan.sync(to_dev(Xall, in_dt), to_dev(dYall, in_dt), dW)
    torch.cuda.synchronize()
    plan.close()
    return dW


def expected_int(oracle_mod, Xall, dYall, n_times_b, out_dt):
    """Bit pattern the epilogue must produce for integer inputs: fl32(S * fl32(1/(nB))) and, for a
    bf16 output, RNE of that fp32 value (DESIGN "Parity")."""
    S = oracle_mod.sfb_sum(Xall[None], dYall[None])
    assert np.all(np.abs(S) < 2 ** 24)           # fp32 accumulation is exact
    e = S.astype(np.float32) * np.float32(1.0 / n_times_b)
    if out_dt == "f32":
        return e
    return oracle_mod.bf16_bits_to_f64(oracle_mod.cast_bf16_bits(e)).astype(np.float32)


# tensor-core shapes (M, N multiples of 8) and SIMT shapes (odd), K = n*B with ragged tails
TC_SHAPES = [(64, 32, 8), (128, 256, 32), (136, 264, 40), (520, 1000, 64), (1024, 4096, 256),
             (256, 512, 5), (8, 8, 1), (384, 768, 2048), (4096, 1000, 256), (200, 264, 300),
             (128, 8, 33), (8, 136, 512), (264, 520, 100), (4096, 1024, 128)]
SIMT_SHAPES = [(1, 1, 2), (3, 5, 6), (17, 33, 12), (130, 257, 10)]


@pytest.mark.parametrize("M,N,K", TC_SHAPES + SIMT_SHAPES)
@pytest.mark.parametrize("out_dt", ["f32", "bf16"])
def test_integer_inputs_bit_exact(tag, comm1, oracle_mod, M, N, K, out_dt):
    X = synth.draw("int3", K, M, synth.rng(50, M, N, 0))
    dY = synth.draw("int3", K, N, synth.rng(50, M, N, 1))
    dW = run_sync(tag, comm1, X, dY, "bf16", "bf16", out_dt).float().cpu().numpy()
    want = expected_int(oracle_mod, X, dY, K, out_dt)
    assert np.array_equal(dW.view(np.uint32), want.view(np.uint32)), \
        f"max |diff| {np.abs(dW - want).max()}"


# CTA-pair shapes (>= 74 pair tiles, K >= 192): 3-D boxes with ragged n-block and K tails, and
# 2-D boxes (M not a multiple of 64) with ragged M, N and K; K > 512 takes 64-row stages
PAIR_SHAPES = [((4352, 2112, 264), True), ((4104, 2008, 200), False), ((4352, 2112, 600), True)]


@pytest.mark.parametrize("shape,box3d", PAIR_SHAPES)
@pytest.mark.parametrize("out_dt", ["f32", "bf16"])
def test_pair_path_integer_bit_exact(tag, comm1, oracle_mod, shape, box3d, out_dt):
    M, N, K = shape
    plan = tag.SfbPlan(comm1, M, N, K, "bf16", "bf16", out_dt)
    info = plan.info()
    plan.close()
    assert (info["recon_bn"], info["recon_ctas"], info["recon_box3d"]) == (256, 2, box3d), info
    X = synth.draw("int3", K, M, synth.rng(51, M, N, 0))
    dY = synth.draw("int3", K, N, synth.rng(51, M, N, 1))
    dW = run_sync(tag, comm1, X, dY, "bf16", "bf16", out_dt).float().cpu().numpy()
    want = expected_int(oracle_mod, X, dY, K, out_dt)
    assert np.array_equal(dW.view(np.uint32), want.view(np.uint32)), \
        f"max |diff| {np.abs(dW - want).max()}"


@pytest.mark.parametrize("M,N,K,want", [(128, 256, 32, (128, 1, True)), (136, 264, 40, (128, 1, False)),
                                         (4096, 4096, 128, (256, 1, True)),
                                         (25088, 4096, 256, (256, 2, True))])
def test_plan_info_tile_config(tag, comm1, M, N, K, want):
    plan = tag.SfbPlan(comm1, M, N, K)
    i = plan.info()
    plan.close()
    assert (i["recon_bn"], i["recon_ctas"], i["recon_box3d"]) == want, i


@pytest.mark.parametrize("n,B", [(1, 32), (2, 32), (4, 32), (8, 32), (8, 64)])
def test_virtual_n_random_vgg_fc7(tag, comm1, oracle_mod, n, B):
    """VGG-19 fc7 shape (4096 x 4096) at K = n*B: post-ReLU X, masked small dY (d-2 recipe)."""
    X, dY = synth.all_factors(2, 7, n, 4096, 4096, B, "relu", "masked_small")
    Xall, dYall = X.reshape(n * B, 4096), dY.reshape(n * B, 4096)
    dW = run_sync(tag, comm1, Xall, dYall).cpu().numpy()
    ref_exact = oracle_mod.sfb_dw(exact_values(X, "bf16"), exact_values(dY, "bf16"))
    ref_user = oracle_mod.sfb_dw(X, dY)
    assert rel_fro(dW, ref_exact) <= 1e-5
    assert rel_fro(dW, ref_user) <= 2e-2


def test_fp32_toy_config(tag, comm1, oracle_mod):
    """Config 1: M=64, N=32, B=4, n=2, fp32 end to end (3xTF32 tensor-core path): <= 1e-5."""
    X, dY = synth.all_factors(1, 0, 2, 64, 32, 4, "normal", "normal")
    dW = run_sync(tag, comm1, X.reshape(8, 64), dY.reshape(8, 32), "f32", "f32", "f32")
    assert rel_fro(dW.cpu().numpy(), oracle_mod.sfb_dw(X, dY)) <= 1e-5


@pytest.mark.parametrize("M,N,K", [(512, 2048, 256), (100, 36, 7), (4096, 1000, 32),
                                   (136, 264, 37), (1024, 4096, 2048), (8, 8, 1)])
def test_fp32_wire_random(tag, comm1, oracle_mod, M, N, K):
    """fp32 factors: 3xTF32 on the tensor cores (M, N multiples of 8) or SIMT FFMA (100 x 36)."""
    X = synth.draw("normal", K, M, synth.rng(51, M, N, 0))
    dY = synth.draw("normal", K, N, synth.rng(51, M, N, 1))
    dW = run_sync(tag, comm1, X, dY, "f32", "f32", "f32")
    assert rel_fro(dW.cpu().numpy(), oracle_mod.sfb_dw(X[None], dY[None])) <= 1e-5


def test_pack_cast_is_rne(tag, comm1, oracle_mod):
    """fp32 inputs, bf16 wire: with dY = identity rows, dW[m][b] = alpha * bf16(X[b][m]) exactly,
    so the pack kernel's cast is compared bit for bit with the oracle's RNE cast."""
    K, M = 16, 4104                                # 4104*16 = 65664 values incl. vector tail
    X = synth.draw("normal", K, M, synth.rng(52, 0, 0, 0))
    X[0, :8] = [1 + 2 ** -8, 1 + 3 * 2 ** -8, -(1 + 2 ** -8), 2 ** -120, 3.0e38, 0.0, -1.5, 1.0]   # all finite in bf16
    dY = np.eye(K, dtype=np.float32)
    dW = run_sync(tag, comm1, X, dY, "f32", "bf16", "f32").cpu().numpy()   # M x K
    cast = oracle_mod.bf16_bits_to_f64(oracle_mod.cast_bf16_bits(X)).astype(np.float32)
    want = (cast.T * np.float32(1.0 / K)).astype(np.float32)
    assert np.array_equal(dW.view(np.uint32), want.view(np.uint32))


@pytest.mark.parametrize("M,N,K,out_dt", [(4096, 1000, 32, "f32"), (25088, 4096, 32, "f32"),
                                          (25088, 4096, 256, "f32"), (25088, 4096, 256, "bf16")])
def test_full_size_sampled(tag, comm1, oracle_mod, M, N, K, out_dt):
    """VGG-19 fc8 / fc6 at n = 1, B = 32 — the bench's launch configuration — and fc6 at K = 256
    (north_star's n = 8 contraction: the CTA-pair kernel the bench's virtual_n8_recon times).
    4000 sampled entries against the oracle computed one by one, plus whole-matrix properties."""
    layer = {1000: 8, 4096: 6}[N]
    X, dY = synth.all_factors(2, layer, 1, M, N, K, "relu",
                              "softmax_onehot" if N == 1000 else "masked_small")
    dW = run_sync(tag, comm1, X[0], dY[0], out_dt=out_dt).float().cpu().numpy()
    idx = np.random.default_rng(7).integers(0, M * N, 4000)
    Xe, dYe = exact_values(X, "bf16"), exact_values(dY, "bf16")
    ref = oracle_mod.sfb_sum_entries(Xe, dYe, idx) / K
    # bf16 dW: one RNE rounding of each entry (relative 2^-9) on top of the fp32 result
    assert rel_fro(dW.ravel()[idx], ref) <= (1e-5 if out_dt == "f32" else 4e-3)
    if out_dt == "bf16":   # every sampled entry within half a bf16 ulp (+ the fp32 error)
        assert np.all(np.abs(dW.ravel()[idx] - ref) <= 2.0 ** -8 * np.abs(ref) + 1e-30)
    assert np.isfinite(dW).all()
    # rank <= K property, checked on a random sketch of the whole matrix (fp32 dW: the bf16
    # rounding of every entry is full-rank noise at the 2^-9 level)
    if out_dt != "f32":
        return
    g = torch.Generator(device="cuda").manual_seed(0)
    sketch = torch.from_numpy(dW).cuda().double() @ torch.randn(N, 2 * K, device="cuda",
                                                                dtype=torch.float64, generator=g)
    s = torch.linalg.svdvals(sketch).cpu().numpy()
    assert s[K] / s[0] < 1e-5


def test_local_grad_and_dense_n1(tag, comm1, oracle_mod):
    M, N, B = 1024, 512, 48
    X = synth.draw("int3", B, M, synth.rng(53, 0, 0, 0))
    dY = synth.draw("int3", B, N, synth.rng(53, 0, 0, 1))
    plan = tag.SfbPlan(comm1, M, N, B, "bf16", "bf16", "f32")
    Xd, dYd = to_dev(X, "bf16"), to_dev(dY, "bf16")
    loc = torch.empty(M, N, device="cuda")
    plan.local_grad(Xd, dYd, loc)
    torch.cuda.synchronize()
    S = oracle_mod.sfb_sum(X[None], dY[None])
    assert np.array_equal(loc.cpu().numpy(), S.astype(np.float32))        # unscaled, exact
    plan.dense_allreduce(loc)                                             # n = 1: dW <- dW / B
    sfb = torch.empty(M, N, device="cuda")
    plan.sync(Xd, dYd, sfb)
    torch.cuda.synchronize()
    assert torch.equal(loc, sfb)
    plan.close()


@pytest.mark.parametrize("M,N,K,want", [(1024, 4096, 512, (128, 1)), (4096, 4096, 1024, (256, 2)),
                                         (4096, 5120, 32, (128, 1))])
def test_fused_sgd_tile_configs_equal_unfused(tag, comm1, M, N, K, want):
    """E2 on both optimizer tile rules (128 x 128 tiles up to K = 512, CTA pairs with 64-row
    stages above; 4096 x 5120: 8 rounds of tiles, dynamic tail): fused == reconstruct +
    tag_sgd_step, bit for bit, over two steps."""
    rs = np.random.default_rng(79)
    X = torch.from_numpy(rs.standard_normal((K, M)).astype(np.float32)).to(torch.bfloat16).cuda()
    dY = torch.from_numpy(rs.standard_normal((K, N)).astype(np.float32)).to(torch.bfloat16).cuda()
    W0 = torch.from_numpy((0.02 * rs.standard_normal((M, N))).astype(np.float32)).cuda()
    hp = dict(lr=1e-3, momentum=0.9, weight_decay=1e-2)
    p = tag.SfbPlan(comm1, M, N, K, fuse_sgd=True, **hp)
    i = p.info()
    assert (i["recon_bn"], i["recon_ctas"]) == want, i
    W1, v1 = W0.clone(), torch.zeros_like(W0)
    W2, v2 = W0.clone(), torch.zeros_like(W0)
    dW = torch.empty_like(W0)
    for _ in range(2):
        p.sync_sgd(X, dY, W1, v1, None)
        p.sync(X, dY, dW)
        p.sgd_step(dW, W2, v2)
    torch.cuda.synchronize()
    p.close()
    assert torch.equal(W1, W2) and torch.equal(v1, v2)
    assert not torch.equal(W1, W0)


def test_fused_sgd_matches_unfused_and_oracle(tag, comm1, oracle_mod):
    """E2: the fused epilogue equals reconstruct + tag_sgd_step bit for bit, and the fp64 oracle
    (BERT-L pooler shape, virtual n = 8, B = 2; lr 1e-3, mu 0.9, wd 1e-2)."""
    n, B, M, N = 8, 2, 1024, 1024
    X, dY = synth.all_factors(5, 3, n, M, N, B, "tanh", "small")
    W0, v0 = synth.sgd_state(5, 3, M, N)
    v0 = (v0 + 1e-4 * synth.draw("normal", M, N, synth.rng(5, 3, 0, 9))).astype(np.float32)
    hp = dict(lr=1e-3, momentum=0.9, weight_decay=1e-2)
    plan = tag.SfbPlan(comm1, M, N, n * B, "bf16", "bf16", "f32", fuse_sgd=True, **hp)
    Xd, dYd = to_dev(X.reshape(n * B, M), "bf16"), to_dev(dY.reshape(n * B, N), "bf16")
    W1, v1 = torch.from_numpy(W0).cuda(), torch.from_numpy(v0).cuda()
    dW1 = torch.empty(M, N, device="cuda")
    plan.sync_sgd(Xd, dYd, W1, v1, dW1)
    W2, v2 = torch.from_numpy(W0).cuda(), torch.from_numpy(v0).cuda()
    dW2 = torch.empty(M, N, device="cuda")
    plan.sync(Xd, dYd, dW2)
    plan.sgd_step(dW2, W2, v2)
    W3, v3 = torch.from_numpy(W0).cuda(), torch.from_numpy(v0).cuda()
    plan.sync_sgd(Xd, dYd, W3, v3, None)                 # no dW write at all
    torch.cuda.synchronize()
    assert torch.equal(dW1, dW2) and torch.equal(W1, W2) and torch.equal(v1, v2)
    assert torch.equal(W1, W3) and torch.equal(v1, v3)
    g = oracle_mod.sfb_dw(exact_values(X, "bf16"), exact_values(dY, "bf16"))
    Wr, vr = oracle_mod.sgd_momentum(g, W0, v0, hp["lr"], hp["momentum"], hp["weight_decay"])
    assert rel_fro(v1.cpu().numpy(), vr) <= 1e-5
    # W' = W - lr*v is rounded to fp32 once per element: at most 1 ulp(W') plus the v error
    W1n = W1.cpu().numpy()
    tol = np.spacing(np.abs(Wr).astype(np.float32)) + hp["lr"] * (1e-5 * np.abs(vr) + 1e-12)
    assert np.all(np.abs(W1n - Wr) <= tol)
    assert rel_fro(W1n, Wr) <= 1e-6
    plan.close()


def test_sync_host_matches_device(tag, comm1):
    M, N, B = 4096, 1000, 32
    X, dY = synth.factors(2, 8, 0, M, N, B, "relu", "softmax_onehot")
    plan = tag.SfbPlan(comm1, M, N, B, "bf16", "bf16", "f32")
    Xh = torch.from_numpy(X).to(torch.bfloat16).pin_memory()
    dYh = torch.from_numpy(dY).to(torch.bfloat16).pin_memory()
    dWh = torch.empty(M, N).pin_memory()
    plan.sync_host(Xh, dYh, dWh)
    dWd = torch.empty(M, N, device="cuda")
    plan.sync(Xh.cuda(), dYh.cuda(), dWd)
    torch.cuda.synchronize()
    assert torch.equal(dWh, dWd.cpu())
    plan.close()


def test_stage_split_equals_sync(tag, comm1):
    M, N, B = 512, 2048, 256
    X, dY = synth.factors(4, 2, 0, M, N, B, "normal", "small")
    plan = tag.SfbPlan(comm1, M, N, B, "f32", "bf16", "bf16")
    Xd, dYd = to_dev(X, "f32"), to_dev(dY, "f32")
    a = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
    b = torch.empty_like(a)
    plan.sync(Xd, dYd, a)
    plan.gather(Xd, dYd)
    plan.reconstruct(b)
    torch.cuda.synchronize()
    assert torch.equal(a, b)
    plan.close()


def test_invalid_arguments_have_no_side_effects(tag, comm1):
    with pytest.raises(tag.TagError) as e:
        tag.SfbPlan(comm1, 0, 4, 4)
    assert e.value.status == tag.ERR_INVALID_ARG
    plan = tag.SfbPlan(comm1, 64, 32, 8)
    X = torch.zeros(8, 64, dtype=torch.bfloat16, device="cuda")
    dY = torch.zeros(8, 32, dtype=torch.bfloat16, device="cuda")
    dW = torch.full((64, 32), 7.0, device="cuda")
    before = tag.kernel_launches()
    st = tag._lib.tag_sfb_sync(plan._h, tag._vp(X.data_ptr() + 2), tag._vp(dY.data_ptr()),
                               tag._vp(dW.data_ptr()), tag._vp(0))
    assert st == tag.ERR_INVALID_ARG
    st = tag._lib.tag_sfb_sync(plan._h, tag._vp(0), tag._vp(dY.data_ptr()),
                               tag._vp(dW.data_ptr()), tag._vp(0))
    assert st == tag.ERR_INVALID_ARG
    torch.cuda.synchronize()
    assert tag.kernel_launches() == before and torch.all(dW == 7.0)
    # reconstruct before any gather on a fresh plan is an error, not garbage
    with pytest.raises(tag.TagError):
        plan.reconstruct(dW)
    with pytest.raises(tag.TagError):
        plan.sync_sgd(X, dY, torch.zeros(64, 32, device="cuda"), torch.zeros(64, 32, device="cuda"))
    plan.close()


def test_launch_counter_counts_kernels(tag, comm1):
    plan = tag.SfbPlan(comm1, 4096, 1000, 32)
    X = torch.ones(32, 4096, dtype=torch.bfloat16, device="cuda")
    dY = torch.ones(32, 1000, dtype=torch.bfloat16, device="cuda")
    dW = torch.empty(4096, 1000, device="cuda")
    before = tag.kernel_launches()
    plan.sync(X, dY, dW)
    torch.cuda.synchronize()
    assert tag.kernel_launches() - before == 1          # n = 1, bf16 in == wire: recon only
    assert torch.all(dW == 1.0)                          # X = dY = 1 -> dW = 1 (scale pin)
    plan.close()


@pytest.mark.parametrize("layers,out_dt", [
    ([(25088, 4096, 32), (4096, 4096, 32), (4096, 1000, 32)], "f32"),      # VGG-19 FC bucket
    ([(512, 32000, 256), (512, 2048, 256), (2048, 512, 256)], "bf16"),     # Transformer bucket
    ([(136, 264, 40), (130, 257, 10), (8, 8, 1)], "f32"),                  # mixed TC + SIMT shapes
])
def test_group_equals_per_plan(tag, comm1, layers, out_dt):
    """One push + one persistent launch for a bucket == tag_sfb_sync per layer, bit for bit."""
    plans, Xs, dYs, ref, got = [], [], [], [], []
    for li, (M, N, K) in enumerate(layers):
        X = synth.draw("normal", K, M, synth.rng(70, li, 0, 0))
        dY = synth.draw("small", K, N, synth.rng(70, li, 0, 1))
        plan = tag.SfbPlan(comm1, M, N, K, "bf16", "bf16", out_dt)
        plans.append(plan)
        Xs.append(to_dev(X, "bf16"))
        dYs.append(to_dev(dY, "bf16"))
        r = torch.empty(M, N, dtype=TORCH[out_dt], device="cuda")
        plan.sync(Xs[-1], dYs[-1], r)
        ref.append(r)
        got.append(torch.full((M, N), float("nan"), dtype=TORCH[out_dt], device="cuda"))
    group = tag.SfbGroup(plans)
    before = tag.kernel_launches()
    group.sync(Xs, dYs, got)
    torch.cuda.synchronize()
    launches = tag.kernel_launches() - before
    if all(p.info()["tensor_cores"] for p in plans):
        assert launches == 1                 # n = 1, no cast: one grouped reconstruction
    for r, g in zip(ref, got):
        assert torch.equal(r, g)
    group.close()
    for p in plans:
        p.close()


def test_group_of_32_layers(tag, comm1):
    """A whole 12-block FFN stack (24 layers, 768 x 3072 / 3072 x 768) plus 8 small layers — the
    32-layer bucket limit — in one launch == per-layer syncs, bit for bit; 33 plans rejected."""
    layers = [(768, 3072, 64) if i % 2 == 0 else (3072, 768, 64) for i in range(24)]
    layers += [(136 + 8 * i, 264, 64) for i in range(8)]
    plans, Xs, dYs, ref, got = [], [], [], [], []
    for li, (M, N, K) in enumerate(layers):
        X = synth.draw("int3", K, M, synth.rng(71, li, 0, 0))
        dY = synth.draw("int3", K, N, synth.rng(71, li, 0, 1))
        plan = tag.SfbPlan(comm1, M, N, K, "bf16", "bf16", "bf16")
        plans.append(plan)
        Xs.append(to_dev(X, "bf16"))
        dYs.append(to_dev(dY, "bf16"))
        r = torch.empty(M, N, dtype=torch.bfloat16, device="cuda")
        plan.sync(Xs[-1], dYs[-1], r)
        ref.append(r)
        got.append(torch.full((M, N), float("nan"), dtype=torch.bfloat16, device="cuda"))
    group = tag.SfbGroup(plans)
    before = tag.kernel_launches()
    group.sync(Xs, dYs, got)
    torch.cuda.synchronize()
    assert tag.kernel_launches() - before == 1
    assert all(torch.equal(r, g) for r, g in zip(ref, got))
    extra = tag.SfbPlan(comm1, 64, 32, 8, "bf16", "bf16", "bf16")
    with pytest.raises(tag.TagError) as e:
        tag.SfbGroup(plans + [extra])
    assert e.value.status == tag.ERR_INVALID_ARG
    extra.close()
    group.close()
    for p in plans:
        p.close()


def test_group_validation(tag, comm1):
    a = tag.SfbPlan(comm1, 64, 32, 8, "bf16", "bf16", "f32")
    b = tag.SfbPlan(comm1, 64, 32, 8, "bf16", "bf16", "bf16")
    with pytest.raises(tag.TagError) as e:
        tag.SfbGroup([a, b])                       # mixed out dtypes
    assert e.value.status == tag.ERR_INVALID_ARG
    with pytest.raises(tag.TagError):
        tag.SfbGroup([a, a])                       # duplicate plan
    with pytest.raises(tag.TagError):
        tag.SfbGroup([])
    a.close()
    b.close()


def test_group_sgd_equals_per_plan(tag, comm1):
    """BERT-large bucket (FFN1, FFN2, pooler; virtual n = 8) with the SGD epilogue fused: one
    grouped launch == tag_sfb_sync_sgd per layer, bit for bit (W, v and dW)."""
    hp = dict(lr=1e-3, momentum=0.9, weight_decay=1e-4)
    specs = [(1024, 4096, 8 * 128, "normal"), (4096, 1024, 8 * 128, "gelu"), (1024, 1024, 8 * 2, "tanh")]
    plans, Xs, dYs, W1, v1, W2, v2, d1, d2 = [], [], [], [], [], [], [], [], []
    for li, (M, N, K, xd) in enumerate(specs):
        X = synth.draw(xd, K, M, synth.rng(80, li, 0, 0))
        dY = synth.draw("small", K, N, synth.rng(80, li, 0, 1))
        W0, _ = synth.sgd_state(80, li, M, N)
        p = tag.SfbPlan(comm1, M, N, K, "bf16", "bf16", "f32", fuse_sgd=True, **hp)
        plans.append(p)
        Xs.append(to_dev(X, "bf16"))
        dYs.append(to_dev(dY, "bf16"))
        for Wl, vl, dl in ((W1, v1, d1), (W2, v2, d2)):
            Wl.append(torch.from_numpy(W0).cuda())
            vl.append(torch.zeros(M, N, device="cuda"))
            dl.append(torch.empty(M, N, device="cuda"))
    for _ in range(2):
        for i, p in enumerate(plans):
            p.sync_sgd(Xs[i], dYs[i], W1[i], v1[i], d1[i])
    g = tag.SfbGroup(plans)
    for _ in range(2):
        g.sync_sgd(Xs, dYs, W2, v2, d2)
    torch.cuda.synchronize()
    for i in range(len(plans)):
        assert torch.equal(W1[i], W2[i]) and torch.equal(v1[i], v2[i]) and torch.equal(d1[i], d2[i])
    with pytest.raises(tag.TagError):
        g.sync(Xs, dYs, d2)                        # fuse_sgd groups only take sync_sgd
    g.close()
    for p in plans:
        p.close()


# ------------------------------------------------------------------ bias gradient (R17)
def expected_bias_int(oracle_mod, dYall, K, out_dt):
    """fl32(S_b * fl32(1/K)) (RNE to bf16 for a bf16 output) for integer dY: S_b is exact."""
    S = oracle_mod.sfb_bias_sum(dYall[None])
    e = S.astype(np.float32) * np.float32(1.0 / K)
    if out_dt == "f32":
        return e
    return oracle_mod.bf16_bits_to_f64(oracle_mod.cast_bf16_bits(e)).astype(np.float32)


@pytest.mark.parametrize("M,N,K", [(64, 32, 8), (136, 264, 40), (4096, 1000, 256), (256, 512, 5),
                                   (3, 5, 6), (130, 257, 10), (64, 32000, 256), (8, 8, 2048)])
@pytest.mark.parametrize("out_dt", ["f32", "bf16"])
def test_bias_grad_bit_exact(tag, comm1, oracle_mod, M, N, K, out_dt):
    X = synth.draw("int3", K, M, synth.rng(60, M, N, 0))
    dY = synth.draw("int3", K, N, synth.rng(60, M, N, 1))
    plan = tag.SfbPlan(comm1, M, N, K, "bf16", "bf16", out_dt)
    dW = torch.empty((M, N), dtype=TORCH[out_dt], device="cuda")
    db = torch.full((N,), float("nan"), dtype=TORCH[out_dt], device="cuda")
    Xd, dYd = to_dev(X, "bf16"), to_dev(dY, "bf16")
    plan.sync(Xd, dYd, dW)
    plan.bias_grad(db)
    torch.cuda.synchronize()
    plan.close()
    got = db.float().cpu().numpy()
    want = expected_bias_int(oracle_mod, dY, K, out_dt)
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))


def test_bias_grad_random_fp32_wire_and_cast(tag, comm1, oracle_mod):
    """fp32 wire (toy) and the fp32 -> bf16 cast path read the right dY_all; <= 1e-5 vs the oracle
    on the operand values the GPU used."""
    rs = np.random.default_rng(61)
    for in_dt, wire_dt, M, N, K in (("f32", "f32", 64, 32, 8), ("f32", "bf16", 520, 1000, 64)):
        X = rs.standard_normal((K, M)).astype(np.float32)
        dY = rs.standard_normal((K, N)).astype(np.float32)
        plan = tag.SfbPlan(comm1, M, N, K, in_dt, wire_dt, "f32")
        dW = torch.empty((M, N), device="cuda")
        db = torch.empty((N,), device="cuda")
        plan.sync(to_dev(X, in_dt), to_dev(dY, in_dt), dW)
        plan.bias_grad(db)
        torch.cuda.synchronize()
        plan.close()
        want = oracle_mod.sfb_bias(exact_values(dY, wire_dt)[None])
        assert rel_fro(db.cpu().numpy(), want) <= 1e-5


def test_group_bias_grad_equals_per_plan(tag, comm1):
    rs = np.random.default_rng(62)
    layers = [(4096, 1000, 32), (1024, 4096, 32), (512, 2048, 32)]
    plans, Xs, dYs, dWs = [], [], [], []
    for M, N, K in layers:
        plans.append(tag.SfbPlan(comm1, M, N, K))
        Xs.append(torch.from_numpy(rs.standard_normal((K, M))).to(torch.bfloat16).cuda())
        dYs.append(torch.from_numpy(rs.standard_normal((K, N))).to(torch.bfloat16).cuda())
        dWs.append(torch.empty((M, N), device="cuda"))
    g = tag.SfbGroup(plans)
    g.sync(Xs, dYs, dWs)
    dbs = [torch.empty((p.N,), device="cuda") for p in plans]
    g.bias_grad(dbs)
    for p, X, dY, dW, db in zip(plans, Xs, dYs, dWs, dbs):
        p.sync(X, dY, dW)
        one = torch.empty_like(db)
        p.bias_grad(one)
        torch.cuda.synchronize()
        assert torch.equal(one, db)
    g.close()
    for p in plans:
        p.close()


def test_bias_grad_before_sync_is_an_error(tag, comm1):
    plan = tag.SfbPlan(comm1, 64, 32, 8)
    with pytest.raises(tag.TagError) as e:
        plan.bias_grad(torch.empty((32,), device="cuda"))
    assert e.value.status == tag.ERR_INVALID_ARG
    plan.close()


@pytest.mark.parametrize("M,N,K", [(64, 32, 8), (136, 264, 40), (4096, 1000, 256), (256, 512, 5),
                                   (1024, 4096, 33)])
@pytest.mark.parametrize("out_dt", ["f32", "bf16"])
def test_fp32_wire_integer_bit_exact(tag, comm1, oracle_mod, M, N, K, out_dt):
    """3xTF32 on integers: hi = x, lo = 0, so the tensor-core sum is exact (same pin as bf16)."""
    X = synth.draw("int3", K, M, synth.rng(63, M, N, 0))
    dY = synth.draw("int3", K, N, synth.rng(63, M, N, 1))
    plan = tag.SfbPlan(comm1, M, N, K, "f32", "f32", out_dt)
    assert plan.info()["tensor_cores"]
    dW = torch.full((M, N), float("nan"), dtype=TORCH[out_dt], device="cuda")
    plan.sync(to_dev(X, "f32"), to_dev(dY, "f32"), dW)
    torch.cuda.synchronize()
    plan.close()
    want = expected_int(oracle_mod, X, dY, K, out_dt)
    assert np.array_equal(dW.float().cpu().numpy().view(np.uint32), want.view(np.uint32))


def test_fp32_wire_lo_halves_matter(tag, comm1, oracle_mod):
    """Values with mantissa bits below tf32's 10: one TF32 pass would be off by ~1e-4; 3xTF32
    must stay within 1e-6 of the fp64 oracle."""
    rs = np.random.default_rng(64)
    K, M, N = 64, 256, 512
    X = (1.0 + rs.random((K, M)) * 2.0 ** -11).astype(np.float32)   # only low mantissa bits vary
    dY = (1.0 + rs.random((K, N)) * 2.0 ** -11).astype(np.float32)
    plan = tag.SfbPlan(comm1, M, N, K, "f32", "f32", "f32")
    dW = torch.empty((M, N), device="cuda")
    plan.sync(to_dev(X, "f32"), to_dev(dY, "f32"), dW)
    torch.cuda.synchronize()
    plan.close()
    want = oracle_mod.sfb_dw(X.astype(np.float64)[None], dY.astype(np.float64)[None])
    err = np.abs(dW.cpu().numpy() - want).max() / np.abs(want).max()
    assert err <= 1e-6, err


def test_fp32_wire_sgd_fused(tag, comm1, oracle_mod):
    """E2 on the 3xTF32 path equals the unfused update bit for bit."""
    rs = np.random.default_rng(65)
    K, M, N = 32, 512, 1024
    X = torch.from_numpy(rs.standard_normal((K, M)).astype(np.float32)).cuda()
    dY = torch.from_numpy(rs.standard_normal((K, N)).astype(np.float32)).cuda()
    W0 = torch.from_numpy(rs.standard_normal((M, N)).astype(np.float32)).cuda()
    v0 = torch.from_numpy(rs.standard_normal((M, N)).astype(np.float32)).cuda()
    p = tag.SfbPlan(comm1, M, N, K, "f32", "f32", "f32", fuse_sgd=True, lr=1e-2, momentum=0.9)
    W1, v1 = W0.clone(), v0.clone()
    p.sync_sgd(X, dY, W1, v1, None)
    dW = torch.empty((M, N), device="cuda")
    p.sync(X, dY, dW)
    W2, v2 = W0.clone(), v0.clone()
    p.sgd_step(dW, W2, v2)
    torch.cuda.synchronize()
    p.close()
    assert torch.equal(W1, W2) and torch.equal(v1, v2)


# ------------------------------------------------------------------ Adam epilogue (R22)
ADAM_HP = dict(lr=1e-3, beta1=0.9, beta2=0.999, eps=1e-8, weight_decay=0.01)


@pytest.mark.parametrize("M,N,K,wire", [(4096, 1000, 32, "bf16"), (1024, 4096, 128, "bf16"),
                                         (4096, 5120, 32, "bf16"),
                                         (4096, 4096, 256, "bf16"), (4096, 4096, 1024, "bf16"),
                                         (512, 1024, 32, "f32"),
                                         (130, 257, 10, "bf16"), (136, 264, 40, "bf16")])
def test_adam_fused_equals_unfused(tag, comm1, M, N, K, wire):  # noqa: E302
    """E3 (tensor-core epilogue; SIMT shapes: reconstruction + unfused kernel) == tag_sfb_sync
    followed by tag_adam_step, bit for bit, over three steps (one CTA, CTA pairs, 3xTF32)."""
    rs = np.random.default_rng(73)
    dt = TORCH[wire]
    X = torch.from_numpy(rs.standard_normal((K, M)).astype(np.float32)).to(dt).cuda()
    dY = torch.from_numpy(rs.standard_normal((K, N)).astype(np.float32)).to(dt).cuda()
    W0 = torch.from_numpy((0.02 * rs.standard_normal((M, N))).astype(np.float32)).cuda()
    p = tag.SfbPlan(comm1, M, N, K, wire, wire, "f32", fuse_adam=True, **ADAM_HP)
    W1, m1, v1 = W0.clone(), torch.zeros_like(W0), torch.zeros_like(W0)
    W2, m2, v2 = W0.clone(), torch.zeros_like(W0), torch.zeros_like(W0)
    dW = torch.empty_like(W0)
    for t in (1, 2, 3):
        p.sync_adam(X, dY, W1, m1, v1, t)
        p.sync(X, dY, dW)
        p.adam_step(dW, W2, m2, v2, t)
    torch.cuda.synchronize()
    p.close()
    assert torch.equal(W1, W2) and torch.equal(m1, m2) and torch.equal(v1, v2)
    assert not torch.equal(W1, W0)


def test_adam_matches_oracle(tag, comm1, oracle_mod):
    """Two fused Adam steps vs the fp64 oracle (reconstruction from the exact bf16 operands, then
    torch.optim.Adam-semantics updates): the weight change agrees to 1e-4 relative."""
    rs = np.random.default_rng(74)
    K, M, N = 64, 520, 1000
    X = rs.standard_normal((K, M)).astype(np.float32)
    dY = rs.standard_normal((K, N)).astype(np.float32)
    W0 = (0.02 * rs.standard_normal((M, N))).astype(np.float32)
    p = tag.SfbPlan(comm1, M, N, K, "bf16", "bf16", "f32", fuse_adam=True, **ADAM_HP)
    W, m, v = torch.from_numpy(W0).cuda(), torch.zeros((M, N), device="cuda"), torch.zeros((M, N), device="cuda")
    for t in (1, 2):
        p.sync_adam(to_dev(X, "bf16"), to_dev(dY, "bf16"), W, m, v, t)
    torch.cuda.synchronize()
    p.close()
    dW = oracle_mod.sfb_dw(exact_values(X, "bf16")[None], exact_values(dY, "bf16")[None])
    Wr, mr, vr = W0.astype(np.float64), np.zeros((M, N)), np.zeros((M, N))
    # the plan holds its hyper-parameters as fp32 (tag_sfb_desc_t): fl32(0.999) makes 1 - beta2
    # differ from 0.001 by 1.3e-5 relative, so the oracle is given the same fp32 values
    hp32 = {k: float(np.float32(v)) for k, v in ADAM_HP.items()}
    for t in (1, 2):
        Wr, mr, vr = oracle_mod.adam(dW, Wr, mr, vr, hp32["lr"], hp32["beta1"], hp32["beta2"],
                                     hp32["eps"], hp32["weight_decay"], t)
    assert rel_fro(W.cpu().numpy() - W0, Wr - W0) <= 1e-4
    assert rel_fro(m.cpu().numpy(), mr) <= 1e-5 and rel_fro(v.cpu().numpy(), vr) <= 1e-5


def test_group_adam_equals_per_plan(tag, comm1):
    rs = np.random.default_rng(75)
    layers = [(4096, 1000, 32), (1024, 4096, 32), (512, 2048, 32)]
    plans, Xs, dYs, Ws, ms, vs, W2, m2, v2 = [], [], [], [], [], [], [], [], []
    for M, N, K in layers:
        plans.append(tag.SfbPlan(comm1, M, N, K, fuse_adam=True, **ADAM_HP))
        Xs.append(torch.from_numpy(rs.standard_normal((K, M))).to(torch.bfloat16).cuda())
        dYs.append(torch.from_numpy(rs.standard_normal((K, N))).to(torch.bfloat16).cuda())
        w = torch.from_numpy((0.02 * rs.standard_normal((M, N))).astype(np.float32)).cuda()
        Ws.append(w.clone()); W2.append(w.clone())
        ms.append(torch.zeros_like(w)); m2.append(torch.zeros_like(w))
        vs.append(torch.zeros_like(w)); v2.append(torch.zeros_like(w))
    g = tag.SfbGroup(plans)
    for t in (1, 2):
        g.sync_adam(Xs, dYs, Ws, ms, vs, t)
        for i, p in enumerate(plans):
            p.sync_adam(Xs[i], dYs[i], W2[i], m2[i], v2[i], t)
    torch.cuda.synchronize()
    assert all(torch.equal(a, b) for a, b in zip(Ws + ms + vs, W2 + m2 + v2))
    g.close()
    for p in plans:
        p.close()


def test_adam_validation(tag, comm1):
    with pytest.raises(tag.TagError):
        tag.SfbPlan(comm1, 64, 32, 8, fuse_adam=True, fuse_sgd=True, lr=1e-3)
    with pytest.raises(tag.TagError):
        tag.SfbPlan(comm1, 64, 32, 8, fuse_adam=True, lr=1e-3, beta1=1.0)
    with pytest.raises(tag.TagError):
        tag.SfbPlan(comm1, 64, 32, 8, "bf16", "bf16", "bf16", fuse_adam=True, lr=1e-3)
    p = tag.SfbPlan(comm1, 64, 32, 8, fuse_adam=True, lr=1e-3)
    X, dY = torch.zeros((8, 64), dtype=torch.bfloat16, device="cuda"), torch.zeros((8, 32), dtype=torch.bfloat16, device="cuda")
    W, m, v = (torch.zeros((64, 32), device="cuda") for _ in range(3))
    with pytest.raises(tag.TagError):
        p.sync_adam(X, dY, W, m, v, 0)                      # step must be >= 1
    with pytest.raises(tag.TagError):
        p.sync_sgd(X, dY, W, v)                             # not an SGD plan
    p.close()


def test_cuda_graph_capture_n1(tag, comm1, oracle_mod):
    """On a one-rank comm without NCCL a bucket sync is one kernel with no per-call host state, so
    it can be captured in a CUDA graph and replayed (new inputs copied into the captured buffers
    between replays); every replay is bit exact."""
    layers = [(520, 264, 24), (4096, 1000, 32)]
    plans = [tag.SfbPlan(comm1, M, N, K, "bf16", "bf16", "f32") for (M, N, K) in layers]
    g = tag.SfbGroup(plans)
    Xs = [torch.empty(K, M, dtype=torch.bfloat16, device="cuda") for (M, N, K) in layers]
    dYs = [torch.empty(K, N, dtype=torch.bfloat16, device="cuda") for (M, N, K) in layers]
    outs = [torch.empty(M, N, device="cuda") for (M, N, K) in layers]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g.sync(Xs, dYs, outs, s)                 # warm-up outside capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        g.sync(Xs, dYs, outs, s)
    for rep in range(3):
        wants = []
        for li, (M, N, K) in enumerate(layers):
            X = synth.draw("int3", K, M, synth.rng(90 + rep, li, 0, 0))
            dY = synth.draw("int3", K, N, synth.rng(90 + rep, li, 0, 1))
            Xs[li].copy_(torch.from_numpy(X).to(torch.bfloat16))
            dYs[li].copy_(torch.from_numpy(dY).to(torch.bfloat16))
            wants.append(expected_int(oracle_mod, X, dY, K, "f32"))
        graph.replay()
        torch.cuda.synchronize()
        for o, w in zip(outs, wants):
            assert np.array_equal(o.cpu().numpy().view(np.uint32), w.view(np.uint32))
    g.close()
    for p in plans:
        p.close()


def test_dynamic_tail_schedule_repeated_and_captured(tag, comm1, oracle_mod):
    """Buckets of >= 8 rounds of one-CTA tiles hand their last two rounds out through a device
    counter that the last CTA re-arms (recon_tc.cu): back-to-back launches, two plans interleaved
    on one stream, and a CUDA graph of three launches replayed twice are all bit exact."""
    M, N, K = 4096, 5120, 32             # 1280 tiles of 128 x 128: 8 rounds on 148 SMs
    rs = np.random.default_rng(77)
    X = rs.integers(-3, 4, (K, M)).astype(np.float32)
    dY = rs.integers(-3, 4, (K, N)).astype(np.float32)
    want = expected_int(oracle_mod, X, dY, K, "f32").view(np.uint32)
    p1 = tag.SfbPlan(comm1, M, N, K, "bf16", "bf16", "f32")
    p2 = tag.SfbPlan(comm1, M, N, K, "bf16", "bf16", "f32")
    Xd, dYd = to_dev(X, "bf16"), to_dev(dY, "bf16")
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    outs = [torch.full((M, N), float("nan"), device="cuda") for _ in range(4)]
    with torch.cuda.stream(s):
        for i in range(8):
            (p1 if i % 2 == 0 else p2).sync(Xd, dYd, outs[i % 4], s)
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(o.cpu().numpy().view(np.uint32), want)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        for i in range(3):
            p1.sync(Xd, dYd, outs[i], s)
    for _ in range(2):
        for o in outs[:3]:
            o.fill_(float("nan"))
        with torch.cuda.stream(s):
            g.replay()
        torch.cuda.synchronize()
        for o in outs[:3]:
            assert np.array_equal(o.cpu().numpy().view(np.uint32), want)
    # two plans (own counters) running concurrently on two streams
    s2 = torch.cuda.Stream()
    s2.wait_stream(torch.cuda.current_stream())
    for o in outs:
        o.fill_(float("nan"))
    torch.cuda.synchronize()
    for i in range(6):
        with torch.cuda.stream(s):
            p1.sync(Xd, dYd, outs[i % 2], s)
        with torch.cuda.stream(s2):
            p2.sync(Xd, dYd, outs[2 + i % 2], s2)
    torch.cuda.synchronize()
    for o in outs:
        assert np.array_equal(o.cpu().numpy().view(np.uint32), want)
    p1.close()
    p2.close()
