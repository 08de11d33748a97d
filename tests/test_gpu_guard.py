"""Out-of-bounds write detection without compute-sanitizer (closed on this GPU pool: runs under it
left GPUs needing a reset). Every caller-owned output of every kernel family is placed inside a
larger allocation whose guard bands hold a sentinel bit pattern; after the calls the bands must be
untouched and the output bit-exact (integer inputs, oracle). Covers ragged tile edges (M, N not
multiples of the tile, K not a multiple of the stage depth), the CTA-pair kernel, the optimizer
epilogues (W, v, m written in place), the fused exchange on a loopback comm, the sharded shard and
the bias vector. `-m gpu`.
"""
import numpy as np
import pytest
import torch

from paper_2302_06126_b200 import synth

pytestmark = pytest.mark.gpu
TDT = {"f32": torch.float32, "bf16": torch.bfloat16}
GUARD = 4096          # guard elements on each side (16-byte multiple for both dtypes)


def guarded(shape, dt, fill=None):
    """(buffer, view): view is a contiguous tensor of `shape` inside buffer, GUARD elements from
    either end; the guard bands hold 0x7F (bytes)."""
    n = int(np.prod(shape))
    buf = torch.empty(n + 2 * GUARD, dtype=TDT[dt], device="cuda")
    buf.view(torch.uint8).fill_(0x7F)
    view = buf[GUARD:GUARD + n].view(*shape)
    if fill is not None:
        view.copy_(fill)
    return buf, view


def bands_intact(buf, n):
    b = buf.view(torch.uint8)
    es = buf.element_size()
    lo, hi = b[:GUARD * es], b[(GUARD + n) * es:]
    return bool((lo == 0x7F).all()) and bool((hi == 0x7F).all())


def ints(cid, M, N, K):
    return (synth.draw("int3", K, M, synth.rng(cid, M, N, 0)),
            synth.draw("int3", K, N, synth.rng(cid, M, N, 1)))


def want(oracle_mod, X, dY, out_dt):
    S = oracle_mod.sfb_sum(X[None], dY[None])
    e = S.astype(np.float32) * np.float32(1.0 / X.shape[0])
    if out_dt == "bf16":
        e = oracle_mod.bf16_bits_to_f64(oracle_mod.cast_bf16_bits(e)).astype(np.float32)
    return e


@pytest.fixture(scope="module")
def comms(tag, cuda):
    plain = tag.Comm(1, 0, 0)
    loop = tag.Comm.loopback_comm(0)
    yield {"plain": plain, "loop": loop}
    loop.close()
    plain.close()


# (M, N, K, in, wire, out): one-CTA tiles, CTA pairs, 3xTF32, SIMT, cast, bf16 dW; ragged edges
CASES = [(264, 520, 40, "bf16", "bf16", "f32"), (136, 1000, 33, "bf16", "bf16", "bf16"),
         (520, 264, 256, "bf16", "bf16", "f32"), (392, 136, 300, "bf16", "bf16", "bf16"),
         (136, 264, 40, "f32", "f32", "f32"), (130, 257, 10, "bf16", "bf16", "f32"),
         (264, 520, 40, "f32", "bf16", "f32")]


@pytest.mark.parametrize("case", CASES)
@pytest.mark.parametrize("cname", ["plain", "loop"])
def test_dw_guard_bands(tag, comms, oracle_mod, case, cname):
    M, N, K, i, w, o = case
    X, dY = ints(95, M, N, K)
    plan = tag.SfbPlan(comms[cname], M, N, K, i, w, o)
    buf, dW = guarded((M, N), o)
    Xd = torch.from_numpy(X).to(TDT[i]).cuda()
    dYd = torch.from_numpy(dY).to(TDT[i]).cuda()
    for _ in range(2):
        plan.sync(Xd, dYd, dW)
    bbuf, db = guarded((N,), o)
    plan.bias_grad(db)
    torch.cuda.synchronize()
    assert bands_intact(buf, M * N) and bands_intact(bbuf, N)
    got = dW.float().cpu().numpy()
    assert np.array_equal(got.view(np.uint32), want(oracle_mod, X, dY, o).view(np.uint32))
    plan.close()


@pytest.mark.parametrize("opt", ["sgd", "adam"])
@pytest.mark.parametrize("M,N,K", [(264, 520, 40), (520, 264, 256), (130, 264, 24)])
@pytest.mark.parametrize("cname", ["plain", "loop"])
def test_optimizer_state_guard_bands(tag, comms, opt, M, N, K, cname):
    X, dY = ints(96, M, N, K)
    W0, v0 = synth.sgd_state(96, 0, M, N)
    kw = dict(fuse_adam=True, lr=1e-3) if opt == "adam" else dict(fuse_sgd=True, lr=1e-3, momentum=0.9)
    plan = tag.SfbPlan(comms[cname], M, N, K, **kw)
    Xd = torch.from_numpy(X).to(torch.bfloat16).cuda()
    dYd = torch.from_numpy(dY).to(torch.bfloat16).cuda()
    bw, W = guarded((M, N), "f32", torch.from_numpy(W0))
    bv, v = guarded((M, N), "f32", torch.from_numpy(v0))
    bm, m = guarded((M, N), "f32", torch.zeros(M, N))
    bd, dW = guarded((M, N), "f32")
    for t in (1, 2):
        if opt == "adam":
            plan.sync_adam(Xd, dYd, W, m, v, t, dW)
        else:
            plan.sync_sgd(Xd, dYd, W, v, dW)
    torch.cuda.synchronize()
    assert all(bands_intact(b, M * N) for b in (bw, bv, bm, bd))
    assert bool(torch.isfinite(W).all())
    plan.close()


@pytest.mark.parametrize("M,N,B", [(520, 264, 24), (25088 // 8, 4096, 32)])
def test_sharded_guard_bands(tag, comms, M, N, B):
    X, dY = ints(97, M, N, B)
    plan = tag.SfbPlan(comms["loop"], M, N, B)
    rb, rc = plan.shard_rows()
    buf, sh = guarded((rc, N), "f32")
    plan.sync_sharded(torch.from_numpy(X).to(torch.bfloat16).cuda(),
                      torch.from_numpy(dY).to(torch.bfloat16).cuda(), sh)
    torch.cuda.synchronize()
    assert bands_intact(buf, rc * N)
    plan.close()
