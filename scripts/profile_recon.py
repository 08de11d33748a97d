#!/usr/bin/env python3
"""Small driver for ncu: runs `--iters` SFB syncs of one layer (virtual n replicas stacked on one
GPU, K = n*B) through the C ABI. Used for `ncu --set full -k regex:recon_tc` captures."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_06126_b200 import synth, tag  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--layer", default="fc6")
ap.add_argument("--n", type=int, default=1, help="virtual replicas (K = n*B)")
ap.add_argument("--iters", type=int, default=5)
ap.add_argument("--out", default="f32")
ap.add_argument("--sgd", action="store_true")
ap.add_argument("--group", action="store_true", help="all layers of the config in one bucket")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
if a.group:
    comm = tag.Comm(1, 0, 0)
    plans, Xs, dYs, dWs = [], [], [], []
    for li, L in enumerate(cfg.layers):
        X, dY = synth.all_factors(cfg.cid, li, a.n, L.M, L.N, L.B, L.x_dist, L.dy_dist)
        K = a.n * L.B
        plans.append(tag.SfbPlan(comm, L.M, L.N, K, "bf16", "bf16", a.out, fuse_sgd=a.sgd, lr=1e-3,
                                 momentum=0.9))
        Xs.append(torch.from_numpy(X.reshape(K, L.M)).to(torch.bfloat16).cuda())
        dYs.append(torch.from_numpy(dY.reshape(K, L.N)).to(torch.bfloat16).cuda())
        dWs.append(torch.empty(L.M, L.N, dtype=torch.float32 if a.out == "f32" else torch.bfloat16,
                               device="cuda"))
    g = tag.SfbGroup(plans)
    Ws = [torch.zeros(p.M, p.N, device="cuda") for p in plans] if a.sgd else None
    vs = [torch.zeros(p.M, p.N, device="cuda") for p in plans] if a.sgd else None
    for _ in range(a.iters):
        if a.sgd:       # E2: the bench's --config 5 step (no dW stored)
            g.sync_sgd(Xs, dYs, Ws, vs, None)
        else:
            g.sync(Xs, dYs, dWs)
    torch.cuda.synchronize()
    print(f"ok group config {a.config} n={a.n} iters={a.iters}")
    g.close()
    for p in plans:
        p.close()
    comm.close()
    sys.exit(0)
li, L = next((i, L) for i, L in enumerate(cfg.layers) if L.name == a.layer)
X, dY = synth.all_factors(cfg.cid, li, a.n, L.M, L.N, L.B, L.x_dist, L.dy_dist)
comm = tag.Comm(1, 0, 0)
K = a.n * L.B
plan = tag.SfbPlan(comm, L.M, L.N, K, "bf16", "bf16", a.out, fuse_sgd=a.sgd, lr=1e-3, momentum=0.9)
Xd = torch.from_numpy(X.reshape(K, L.M)).to(torch.bfloat16).cuda()
dYd = torch.from_numpy(dY.reshape(K, L.N)).to(torch.bfloat16).cuda()
dW = torch.empty(L.M, L.N, dtype=torch.float32 if a.out == "f32" else torch.bfloat16, device="cuda")
W = torch.zeros(L.M, L.N, device="cuda") if a.sgd else None
v = torch.zeros(L.M, L.N, device="cuda") if a.sgd else None
for _ in range(a.iters):
    if a.sgd:
        plan.sync_sgd(Xd, dYd, W, v, None)
    else:
        plan.sync(Xd, dYd, dW)
torch.cuda.synchronize()
print(f"ok {a.layer} M={L.M} N={L.N} K={K} iters={a.iters}")
plan.close()
comm.close()
