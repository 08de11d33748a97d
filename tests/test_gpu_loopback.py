"""Every collective code path of libtag on ONE GPU, through a one-rank NCCL communicator
(TAG_COMM_LOOPBACK, `-m gpu`).

A plain one-rank comm has no NCCL communicator and skips the exchange (n = 1). A loopback comm is
a real one-rank `ncclComm` with the device communicator, symmetric windows and the PreMulSum op,
so the paths that otherwise run only at n > 1 execute here against the oracle:
  * the fused exchange + reconstruction kernel (`recon_tc_kernel<..., FUSED = true>`): the push of
    this rank's factors through the LSA pointer of the symmetric window, the system-scope release,
    the hierarchical publish on the local and arrival counters, the producer's arrival wait, TMA
    loads from the window, the fp32 -> bf16 cast inside the push, both window parities;
  * the staged push kernel `push_gather_kernel` and its LSA barrier (tag_sfb_gather);
  * `ncclAllGather` (desc.gather = NCCL), with and without the pack cast;
  * the dense baseline's `ncclAllReduce` with PreMulSum(1/(nB)), the PS `ncclReduce` + `ncclBroadcast`;
  * the sharded calls and the fused optimizer epilogues on the fused path.
P:522-523 ("MatMul ops on each device can reconstruct identical gradients"), P:356-358 (dense
route). Integer inputs make every result exact, so the checks are bit for bit; random VGG-shaped
inputs are checked at the north_star tolerance (1e-5 relative Frobenius on the exact operands).
The same matrix at n = 2 and 4 is scripts/multi_gpu_check.py (tests/test_gpu_multi.py).
"""
import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_2302_06126_b200 import synth

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
TORCH = {"f32": torch.float32, "bf16": torch.bfloat16}


@pytest.fixture(scope="module")
def loop(tag, cuda):
    c = tag.Comm.loopback_comm(0)
    yield c
    c.close()


def ints(cid, M, N, B):
    X = synth.draw("int3", B, M, synth.rng(cid, M, N, 0))
    dY = synth.draw("int3", B, N, synth.rng(cid, M, N, 1))
    return X, dY


def want_int(oracle_mod, X, dY, out_dt="f32"):
    """fl32(S * fl32(1/B)) (one rank: K = B), RNE to bf16 for a bf16 dW (DESIGN "Parity")."""
    S = oracle_mod.sfb_sum(X[None], dY[None])
    e = S.astype(np.float32) * np.float32(1.0 / X.shape[0])
    if out_dt == "f32":
        return e
    return oracle_mod.bf16_bits_to_f64(oracle_mod.cast_bf16_bits(e)).astype(np.float32)


def same_bits(got, want):
    got = got.float().cpu().numpy()
    return np.array_equal(got.view(np.uint32), want.view(np.uint32))


def dev(a, dt):
    return torch.from_numpy(np.ascontiguousarray(a)).to(TORCH[dt]).cuda()


def test_loopback_plan_modes(tag, loop):
    """The loopback comm selects the collective paths, the plain one-rank comm does not."""
    p = tag.SfbPlan(loop, 256, 512, 32)
    assert p.info()["gather"] == "nvlink_push"
    p.close()
    p = tag.SfbPlan(loop, 256, 512, 32, gather="nccl")
    assert p.info()["gather"] == "nccl_allgather"
    p.close()
    plain = tag.Comm(1, 0, 0)
    p = tag.SfbPlan(plain, 256, 512, 32)
    assert p.info()["gather"] == "none"
    p.close()
    p = tag.SfbPlan(plain, 256, 512, 32, gather="push")   # nothing to exchange: request ignored
    assert p.info()["gather"] == "none"
    p.close()
    plain.close()
    loop.barrier()          # the LSA-barrier kernel on one rank
    torch.cuda.synchronize()


# (M, N, B): one-CTA tiles (K < 192) and CTA pairs (K = 256, the fused cta_group::2 kernel at
# north_star's n = 8 contraction depth), ragged M, N
FUSED_SHAPES = [(520, 264, 24), (4096, 1000, 32), (4096, 4096, 256), (520, 264, 256)]


@pytest.mark.parametrize("M,N,B", FUSED_SHAPES)
@pytest.mark.parametrize("in_dt", ["bf16", "f32"])
@pytest.mark.parametrize("out_dt", ["f32", "bf16"])
def test_fused_push_bit_exact(tag, loop, oracle_mod, M, N, B, in_dt, out_dt):
    """tag_sfb_sync on the fused kernel (in_dt f32: cast to the bf16 wire inside the push); three
    calls cover both window parities and the running arrival-counter targets."""
    X, dY = ints(70, M, N, B)
    plan = tag.SfbPlan(loop, M, N, B, in_dt, "bf16", out_dt)
    assert plan.info()["gather"] == "nvlink_push"
    want = want_int(oracle_mod, X, dY, out_dt)
    Xd, dYd = dev(X, in_dt), dev(dY, in_dt)
    for _ in range(3):
        dW = torch.full((M, N), float("nan"), dtype=TORCH[out_dt], device="cuda")
        plan.sync(Xd, dYd, dW)
        torch.cuda.synchronize()
        assert same_bits(dW, want)
    plan.close()


@pytest.mark.parametrize("in_dt", ["bf16", "f32"])
def test_staged_push_gather(tag, loop, oracle_mod, in_dt):
    """tag_sfb_gather = push_gather_kernel (store into the window + LSA barrier), then
    tag_sfb_reconstruct from the window; also the group form (one push kernel for a bucket)."""
    shapes = [(520, 264, 24), (4096, 1000, 32)]
    plans, Xs, dYs, wants = [], [], [], []
    for M, N, B in shapes:
        X, dY = ints(71, M, N, B)
        plans.append(tag.SfbPlan(loop, M, N, B, in_dt, "bf16", "f32"))
        Xs.append(dev(X, in_dt))
        dYs.append(dev(dY, in_dt))
        wants.append(want_int(oracle_mod, X, dY))
    for _ in range(2):
        for p, x, dy, w in zip(plans, Xs, dYs, wants):
            dW = torch.full((p.M, p.N), float("nan"), device="cuda")
            p.gather(x, dy)
            p.reconstruct(dW)
            torch.cuda.synchronize()
            assert same_bits(dW, w)
    g = tag.SfbGroup(plans)
    for _ in range(2):
        outs = [torch.full((p.M, p.N), float("nan"), device="cuda") for p in plans]
        g.gather(Xs, dYs)
        g.reconstruct(outs)
        torch.cuda.synchronize()
        assert all(same_bits(o, w) for o, w in zip(outs, wants))
    g.close()
    for p in plans:
        p.close()


@pytest.mark.parametrize("in_dt,out_dt", [("bf16", "f32"), ("f32", "f32"), ("bf16", "bf16")])
def test_nccl_allgather_mode(tag, loop, oracle_mod, in_dt, out_dt):
    """desc.gather = NCCL: (pack cast +) ncclAllGather into the plan's buffers, then reconstruct."""
    M, N, B = 4096, 1000, 32
    X, dY = ints(72, M, N, B)
    plan = tag.SfbPlan(loop, M, N, B, in_dt, "bf16", out_dt, gather="nccl")
    assert plan.info()["gather"] == "nccl_allgather"
    dW = torch.full((M, N), float("nan"), dtype=TORCH[out_dt], device="cuda")
    for _ in range(2):
        plan.sync(dev(X, in_dt), dev(dY, in_dt), dW)
    torch.cuda.synchronize()
    assert same_bits(dW, want_int(oracle_mod, X, dY, out_dt))
    plan.close()


def test_fp32_wire_toy_config(tag, loop, oracle_mod):
    """Config 1's dtypes (fp32 in, on the wire, out) at 64 x 32: ncclAllGather (fp32 rows are not
    pushed when not 16-byte multiples) or push, then 3xTF32 / SIMT reconstruction, <= 1e-5."""
    M, N, B = 64, 32, 4
    X, dY = synth.factors(1, 0, 0, M, N, B, "normal", "normal")
    plan = tag.SfbPlan(loop, M, N, B, "f32", "f32", "f32")
    dW = torch.empty(M, N, device="cuda")
    plan.sync(dev(X, "f32"), dev(dY, "f32"), dW)
    torch.cuda.synchronize()
    ref = oracle_mod.sfb_dw(X[None].astype(np.float64), dY[None].astype(np.float64))
    err = np.linalg.norm(dW.cpu().numpy() - ref) / np.linalg.norm(ref)
    assert err <= 1e-5, err
    plan.close()


def test_dense_allreduce_premulsum_and_ps(tag, loop, oracle_mod):
    """Dense baseline: tag_local_grad + ncclAllReduce with PreMulSum(1/(nB)); Replicate-with-PS:
    ncclReduce (PreMulSum) to root 0 + ncclBroadcast. Random VGG fc8-shaped inputs vs the oracle's
    dense route <= 1e-5; integer inputs bit exact (1/B is a power of two)."""
    M, N, B = 4096, 1000, 32
    X, dY = synth.factors(2, 2, 0, M, N, B, "relu", "softmax_onehot")
    Xe = torch.from_numpy(X).to(torch.bfloat16).double().numpy()
    dYe = torch.from_numpy(dY).to(torch.bfloat16).double().numpy()
    ref = oracle_mod.dense_dw(Xe[None], dYe[None])
    plan = tag.SfbPlan(loop, M, N, B)
    for sync in ("allreduce", "ps"):
        dW = torch.empty(M, N, device="cuda")
        plan.local_grad(dev(X, "bf16"), dev(dY, "bf16"), dW)
        if sync == "allreduce":
            plan.dense_allreduce(dW)
        else:
            plan.ps_sync(dW, 0)
        torch.cuda.synchronize()
        err = np.linalg.norm(dW.cpu().numpy() - ref) / np.linalg.norm(ref)
        assert err <= 1e-5, (sync, err)
    with pytest.raises(tag.TagError) as e:
        plan.ps_sync(torch.empty(M, N, device="cuda"), 1)
    assert e.value.status == tag.ERR_INVALID_ARG
    Xi, dYi = ints(73, M, N, B)
    dW = torch.empty(M, N, device="cuda")
    plan.local_grad(dev(Xi, "bf16"), dev(dYi, "bf16"), dW)
    plan.dense_allreduce(dW)
    torch.cuda.synchronize()
    assert same_bits(dW, want_int(oracle_mod, Xi, dYi))
    plan.close()


@pytest.mark.parametrize("M,N,B", [(520, 264, 24), (25088, 4096, 32), (1000, 264, 256)])
def test_sharded_fused(tag, loop, oracle_mod, M, N, B):
    """tag_sfb_sync_sharded on the fused kernel (one rank: the shard is every row) == the oracle."""
    X, dY = ints(74, M, N, B)
    plan = tag.SfbPlan(loop, M, N, B)
    rb, rc = plan.shard_rows()
    assert (rb, rc) == (0, M)
    shard = torch.full((M, N), float("nan"), device="cuda")
    for _ in range(2):
        plan.sync_sharded(dev(X, "bf16"), dev(dY, "bf16"), shard)
    torch.cuda.synchronize()
    if M * N <= 1 << 22:
        assert same_bits(shard, want_int(oracle_mod, X, dY))
    else:       # fc6: sampled entries computed one by one by the oracle
        idx = np.random.default_rng(0).integers(0, M * N, 4000)
        S = oracle_mod.sfb_sum_entries(X[None], dY[None], idx)
        w = S.astype(np.float32) * np.float32(1.0 / B)
        got = shard.cpu().numpy().reshape(-1)[idx]
        assert np.array_equal(got.view(np.uint32), w.view(np.uint32))
    plan.close()


def test_group_fused_bucket_and_sharded(tag, loop, oracle_mod):
    """One fused launch for a bucket (tag_sfb_group_sync, _sync_sharded) == per-layer syncs."""
    shapes = [(4096, 4096, 32), (4096, 1000, 32), (520, 264, 32)]
    plans, Xs, dYs, wants = [], [], [], []
    for M, N, B in shapes:
        X, dY = ints(75, M, N, B)
        plans.append(tag.SfbPlan(loop, M, N, B))
        Xs.append(dev(X, "bf16"))
        dYs.append(dev(dY, "bf16"))
        wants.append(want_int(oracle_mod, X, dY))
    g = tag.SfbGroup(plans)
    for _ in range(3):
        outs = [torch.full((p.M, p.N), float("nan"), device="cuda") for p in plans]
        g.sync(Xs, dYs, outs)
        torch.cuda.synchronize()
        assert all(same_bits(o, w) for o, w in zip(outs, wants))
        shards = [torch.full((p.M, p.N), float("nan"), device="cuda") for p in plans]
        g.sync_sharded(Xs, dYs, shards)
        torch.cuda.synchronize()
        assert all(same_bits(o, w) for o, w in zip(shards, wants))
    g.close()
    for p in plans:
        p.close()


@pytest.mark.parametrize("K", [32, 256])
def test_fused_optimizers(tag, loop, K):
    """The fused exchange with the SGD-momentum (E2) and Adam (E3) epilogues == sync + the unfused
    optimizer kernels, bit for bit, three steps."""
    M, N = 1024, 1024
    X, dY = synth.factors(5, 3, 0, M, N, K, "tanh", "small")
    W0, v0 = synth.sgd_state(5, 3, M, N)
    Xd, dYd = dev(X, "bf16"), dev(dY, "bf16")
    ps = tag.SfbPlan(loop, M, N, K, fuse_sgd=True, lr=1e-3, momentum=0.9, weight_decay=1e-4)
    W1, v1 = torch.from_numpy(W0).cuda(), torch.from_numpy(v0).cuda()
    W2, v2 = W1.clone(), v1.clone()
    dW2 = torch.empty(M, N, device="cuda")
    for _ in range(3):
        ps.sync_sgd(Xd, dYd, W1, v1, None)
        ps.sync(Xd, dYd, dW2)
        ps.sgd_step(dW2, W2, v2)
    torch.cuda.synchronize()
    assert torch.equal(W1, W2) and torch.equal(v1, v2)
    ps.close()
    pa = tag.SfbPlan(loop, M, N, K, fuse_adam=True, lr=1e-3, weight_decay=0.01)
    W1, m1, v1 = torch.from_numpy(W0).cuda(), torch.zeros(M, N, device="cuda"), torch.zeros(M, N, device="cuda")
    W2, m2, v2 = W1.clone(), m1.clone(), v1.clone()
    for t in (1, 2, 3):
        pa.sync_adam(Xd, dYd, W1, m1, v1, t)
        pa.sync(Xd, dYd, dW2)
        pa.adam_step(dW2, W2, m2, v2, t)
    torch.cuda.synchronize()
    assert torch.equal(W1, W2) and torch.equal(m1, m2) and torch.equal(v1, v2)
    pa.close()


def test_fused_sgd_bf16_dw_takes_staged_path(tag, loop, oracle_mod):
    """a fuse_sgd plan with a bf16 dW_out must not run the fused fp32-dW epilogue (it
    would write 4-byte elements into a 2-byte buffer). Integer inputs: W, v equal those of an
    fp32-dW plan bit for bit, and dW_out == RNE(the exact dW); the guard rows after dW stay intact."""
    M, N, B = 520, 264, 24
    X, dY = ints(76, M, N, B)
    W0, v0 = synth.sgd_state(65, 0, M, N)
    pa = tag.SfbPlan(loop, M, N, B, "bf16", "bf16", "bf16", fuse_sgd=True, lr=1e-3, momentum=0.9)
    pb = tag.SfbPlan(loop, M, N, B, "bf16", "bf16", "f32", fuse_sgd=True, lr=1e-3, momentum=0.9)
    Wa, va = torch.from_numpy(W0).cuda(), torch.from_numpy(v0).cuda()
    Wb, vb = Wa.clone(), va.clone()
    buf = torch.full((2 * M, N), 7.0, dtype=torch.bfloat16, device="cuda")
    dWa = buf[:M]
    for _ in range(2):
        pa.sync_sgd(dev(X, "bf16"), dev(dY, "bf16"), Wa, va, dWa)
        pb.sync_sgd(dev(X, "bf16"), dev(dY, "bf16"), Wb, vb, None)
    torch.cuda.synchronize()
    assert torch.equal(Wa, Wb) and torch.equal(va, vb)
    assert same_bits(dWa, want_int(oracle_mod, X, dY, "bf16"))
    assert bool((buf[M:] == 7.0).all())
    pa.close()
    pb.close()


def test_bias_grad_from_window(tag, loop, oracle_mod):
    """db from the dY_all the fused sync left in the window (R17), bit exact on integers."""
    M, N, B = 520, 264, 24
    X, dY = ints(77, M, N, B)
    plan = tag.SfbPlan(loop, M, N, B)
    plan.sync(dev(X, "bf16"), dev(dY, "bf16"), torch.empty(M, N, device="cuda"))
    db = torch.full((N,), float("nan"), device="cuda")
    plan.bias_grad(db)
    torch.cuda.synchronize()
    want = oracle_mod.sfb_bias_sum(dY[None]).astype(np.float32) * np.float32(1.0 / B)
    assert np.array_equal(db.cpu().numpy().view(np.uint32), want.view(np.uint32))
    plan.close()


@pytest.mark.parametrize("gather", ["auto", "nccl"])
def test_multi_gpu_check_loopback(gather):
    """The whole n > 1 parity script (scripts/multi_gpu_check.py) on the loopback comm."""
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "multi_gpu_check.py"),
                        "--loopback", "--gather", gather], capture_output=True, text=True,
                       timeout=900, cwd=ROOT)
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"] and res["n"] == 1, res
    want = "nccl_allgather" if gather == "nccl" else "nvlink_push"
    assert want in res["gather_modes"], res


def test_sharded_sgd_with_parameter_allgather(tag, loop):
    """f-2 on one rank: the sharded SGD step (one shard = every row) through the fused exchange
    equals the replicated fused SGD bit for bit, three steps (n = 2 / 4 with real shards:
    scripts/multi_gpu_check.py, check 13)."""
    M, N, B = 520, 264, 24
    X, dY = synth.factors(66, 1, 0, M, N, B, "normal", "small")
    W0, v0 = synth.sgd_state(66, 1, M, N)
    plan = tag.SfbPlan(loop, M, N, B, fuse_sgd=True, lr=1e-3, momentum=0.9, weight_decay=1e-4)
    Xd, dYd = dev(X, "bf16"), dev(dY, "bf16")
    Wr, vr = torch.from_numpy(W0).cuda(), torch.from_numpy(v0).cuda()
    Ws, vs = Wr.clone(), vr.clone()
    for _ in range(3):
        plan.sync_sgd(Xd, dYd, Wr, vr, None)
        plan.sync_sharded_sgd(Xd, dYd, Ws, vs)
    torch.cuda.synchronize()
    assert torch.equal(Ws, Wr) and torch.equal(vs, vr)
    plan.close()


def test_fused_bucket_of_32_layers(tag, loop, oracle_mod):
    """The fused exchange with the 32-layer bucket limit (32 per-layer arrival counters, one push
    kernel) == the oracle, bit for bit, two calls (both window parities)."""
    layers = [(256 + 64 * (i % 4), 264 + 8 * (i % 3), 24) for i in range(32)]
    plans, Xs, dYs, wants = [], [], [], []
    for li, (M, N, B) in enumerate(layers):
        X, dY = ints(80 + li, M, N, B)
        plans.append(tag.SfbPlan(loop, M, N, B))
        Xs.append(dev(X, "bf16"))
        dYs.append(dev(dY, "bf16"))
        wants.append(want_int(oracle_mod, X, dY))
    g = tag.SfbGroup(plans)
    for _ in range(2):
        outs = [torch.full((p.M, p.N), float("nan"), device="cuda") for p in plans]
        g.sync(Xs, dYs, outs)
        torch.cuda.synchronize()
        assert all(same_bits(o, w) for o, w in zip(outs, wants))
    g.close()
    for p in plans:
        p.close()


def test_cuda_graph_capture_exchange(tag, loop, oracle_mod):
    """The window's buffer choice and arrival targets are device state (the window call counter),
    so the fused exchange (a bucket sync), the staged push + reconstruct and the bias gradient can
    be captured once and replayed, interleaved with ordinary calls; every replay is bit exact."""
    layers = [(520, 264, 24), (4096, 1000, 32)]
    plans = [tag.SfbPlan(loop, M, N, B) for (M, N, B) in layers]
    g = tag.SfbGroup(plans)
    Xs = [torch.empty(B, M, dtype=torch.bfloat16, device="cuda") for (M, N, B) in layers]
    dYs = [torch.empty(B, N, dtype=torch.bfloat16, device="cuda") for (M, N, B) in layers]
    outs = [torch.empty(M, N, device="cuda") for (M, N, B) in layers]
    outs2 = [torch.empty(M, N, device="cuda") for (M, N, B) in layers]
    dbs = [torch.empty(N, device="cuda") for (M, N, B) in layers]
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        g.sync(Xs, dYs, outs, s)                  # warm-up outside capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph, stream=s):
        g.sync(Xs, dYs, outs, s)                  # fused exchange + reconstruction
        plans[1].gather(Xs[1], dYs[1], s)         # staged push + LSA barrier
        plans[1].reconstruct(outs2[1], s)
        for p, db in zip(plans, dbs):
            p.bias_grad(db, s)
    for rep in range(4):
        wants, bwant = [], []
        for li, (M, N, B) in enumerate(layers):
            X, dY = ints(100 + rep * 7 + li, M, N, B)
            Xs[li].copy_(torch.from_numpy(X).to(torch.bfloat16))
            dYs[li].copy_(torch.from_numpy(dY).to(torch.bfloat16))
            wants.append(want_int(oracle_mod, X, dY))
            bwant.append(oracle_mod.sfb_bias_sum(dY[None]).astype(np.float32) * np.float32(1.0 / B))
        graph.replay()
        torch.cuda.synchronize()
        assert all(same_bits(o, w) for o, w in zip(outs, wants))
        assert same_bits(outs2[1], wants[1])
        assert all(np.array_equal(d.cpu().numpy().view(np.uint32), w.view(np.uint32))
                   for d, w in zip(dbs, bwant))
        if rep % 2 == 0:                          # an ordinary call between replays
            o = torch.full((layers[0][0], layers[0][1]), float("nan"), device="cuda")
            plans[0].sync(Xs[0], dYs[0], o)
            torch.cuda.synchronize()
            assert same_bits(o, wants[0])
    g.close()
    for p in plans:
        p.close()


def test_sharded_adam_with_parameter_allgather(tag, loop):
    """f-2 with Adam on one rank (loopback): == the replicated fused Adam bit for bit, 3 steps."""
    M, N, B = 520, 264, 24
    X, dY = synth.factors(69, 1, 0, M, N, B, "normal", "small")
    W0, _ = synth.sgd_state(69, 1, M, N)
    plan = tag.SfbPlan(loop, M, N, B, fuse_adam=True, lr=1e-3, weight_decay=0.01)
    Xd, dYd = dev(X, "bf16"), dev(dY, "bf16")
    Wr = torch.from_numpy(W0).cuda()
    mr, vr = torch.zeros_like(Wr), torch.zeros_like(Wr)
    Ws, ms, vs = Wr.clone(), mr.clone(), vr.clone()
    for t in (1, 2, 3):
        plan.sync_adam(Xd, dYd, Wr, mr, vr, t)
        plan.sync_sharded_adam(Xd, dYd, Ws, ms, vs, t)
    torch.cuda.synchronize()
    assert torch.equal(Ws, Wr) and torch.equal(ms, mr) and torch.equal(vs, vr)
    plan.close()
