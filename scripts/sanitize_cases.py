#!/usr/bin/env python3
"""Small cases of every libtag kernel for compute-sanitizer (memcheck / racecheck / synccheck):

    compute-sanitizer --tool memcheck python scripts/sanitize_cases.py

one-CTA tensor-core tiles (bf16 and fp32 dW, ragged edges), CTA pairs (cta_group::2, K = 256),
3xTF32, the SIMT kernel, the fused SGD / Adam epilogues, pack, bias, and — on a one-rank NCCL
loopback comm — the fused exchange kernel (push into the symmetric window, hierarchical publish,
arrival wait), the staged push kernel with its LSA barrier, the PreMulSum AllReduce. Every result
is checked bit for bit against the oracle (integer inputs), so a sanitizer-induced slowdown that
broke an ordering would show as a failure too. Prints one JSON line; exit code 0 iff all pass.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure)
from paper_2302_06126_b200 import synth, tag  # noqa: E402

TDT = {"f32": torch.float32, "bf16": torch.bfloat16}


def ints(cid, M, N, K):
    return (synth.draw("int3", K, M, synth.rng(cid, M, N, 0)),
            synth.draw("int3", K, N, synth.rng(cid, M, N, 1)))


def want(X, dY, out_dt):
    S = oracle.sfb_sum(X[None], dY[None])
    e = S.astype(np.float32) * np.float32(1.0 / X.shape[0])
    if out_dt == "bf16":
        e = oracle.bf16_bits_to_f64(oracle.cast_bf16_bits(e)).astype(np.float32)
    return e


def main():
    torch.cuda.set_device(0)
    res = {}
    plain = tag.Comm(1, 0, 0)
    loop = tag.Comm.loopback_comm(0)
    cases = [("tc1_bf16", plain, 264, 520, 40, "bf16", "bf16", "f32"),
             ("tc1_bf16_out", plain, 264, 520, 40, "bf16", "bf16", "bf16"),
             ("pair_k256", plain, 520, 264, 256, "bf16", "bf16", "f32"),
             ("x3_tf32", plain, 136, 264, 40, "f32", "f32", "f32"),
             ("simt", plain, 130, 257, 10, "bf16", "bf16", "f32"),
             ("pack_cast", plain, 264, 520, 40, "f32", "bf16", "f32"),
             ("fused_loop", loop, 264, 520, 40, "bf16", "bf16", "f32"),
             ("fused_loop_cast", loop, 264, 520, 40, "f32", "bf16", "f32"),
             ("fused_loop_pair", loop, 520, 264, 256, "bf16", "bf16", "bf16"),
             ("nccl_loop", loop, 264, 520, 40, "bf16", "bf16", "f32")]
    for name, comm, M, N, K, i, w, o in cases:
        X, dY = ints(90, M, N, K)
        plan = tag.SfbPlan(comm, M, N, K, i, w, o, gather="nccl" if name == "nccl_loop" else "auto")
        dW = torch.full((M, N), float("nan"), dtype=TDT[o], device="cuda")
        Xd = torch.from_numpy(X).to(TDT[i]).cuda()
        dYd = torch.from_numpy(dY).to(TDT[i]).cuda()
        for _ in range(2):
            plan.sync(Xd, dYd, dW)
        db = torch.empty(N, device="cuda", dtype=TDT[o])
        plan.bias_grad(db)
        torch.cuda.synchronize()
        got = dW.float().cpu().numpy()
        res[name] = bool(np.array_equal(got.view(np.uint32), want(X, dY, o).view(np.uint32)))
        if comm is loop and name == "fused_loop":
            # staged: push kernel + LSA barrier, then reconstruct; dense PreMulSum AllReduce
            plan.gather(Xd, dYd)
            plan.reconstruct(dW)
            dense = torch.empty(M, N, device="cuda")
            plan.local_grad(Xd, dYd, dense)
            plan.dense_allreduce(dense)
            torch.cuda.synchronize()
            w_ = want(X, dY, "f32")
            res["staged_loop"] = bool(np.array_equal(dW.cpu().numpy().view(np.uint32), w_.view(np.uint32)))
            res["dense_loop"] = bool(np.array_equal(dense.cpu().numpy().view(np.uint32), w_.view(np.uint32)))
        plan.close()
    # fused optimizer epilogues (plain comm: E2 / E3 on one-CTA tiles; loopback: fused exchange)
    for name, comm, K in [("sgd_plain", plain, 32), ("sgd_loop", loop, 32), ("adam_loop_pair", loop, 256)]:
        M, N = 256, 264
        X, dY = ints(91, M, N, K)
        W0, v0 = synth.sgd_state(91, 0, M, N)
        adam = name.startswith("adam")
        kw = dict(fuse_adam=True, lr=1e-3) if adam else dict(fuse_sgd=True, lr=1e-3, momentum=0.9)
        plan = tag.SfbPlan(comm, M, N, K, **kw)
        Xd = torch.from_numpy(X).to(torch.bfloat16).cuda()
        dYd = torch.from_numpy(dY).to(torch.bfloat16).cuda()
        W1, v1 = torch.from_numpy(W0).cuda(), torch.from_numpy(v0).cuda()
        W2, v2 = W1.clone(), v1.clone()
        m1, m2 = torch.zeros_like(W1), torch.zeros_like(W1)
        dW = torch.empty(M, N, device="cuda")
        for t in (1, 2):
            if adam:
                plan.sync_adam(Xd, dYd, W1, m1, v1, t)
                plan.sync(Xd, dYd, dW)
                plan.adam_step(dW, W2, m2, v2, t)
            else:
                plan.sync_sgd(Xd, dYd, W1, v1, None)
                plan.sync(Xd, dYd, dW)
                plan.sgd_step(dW, W2, v2)
        torch.cuda.synchronize()
        res[name] = bool(torch.equal(W1, W2) and torch.equal(v1, v2) and torch.equal(m1, m2))
        plan.close()
    loop.close()
    plain.close()
    ok = all(res.values())
    print(json.dumps({"ok": ok, "results": res}), flush=True)
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
