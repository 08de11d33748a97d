#!/usr/bin/env python3
"""The BERT-L E2 bucket (FFN1, FFN2, pooler; fused SGD-momentum epilogue, one grouped launch) at
virtual n = 1, 2, 4, 8 on one GPU (K = n*B), clean L2, median of 10; tile configs selectable by
environment variables (TAG_RECON_BN=128|256). Diagnostics for the E2 tile choice."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_06126_b200 import synth, tag  # noqa: E402

cfg = synth.CONFIGS[5]
comm = tag.Comm(1, 0, 0)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
out = {}
for nv in (1, 2, 4, 8):
    plans, Xs, dYs, Ws, vs = [], [], [], [], []
    for L in cfg.layers:
        K = nv * L.B
        plans.append(tag.SfbPlan(comm, L.M, L.N, K, fuse_sgd=True, lr=1e-3, momentum=0.9,
                                 weight_decay=0.0))
        Xs.append(torch.randn(K, L.M, device="cuda").to(torch.bfloat16))
        dYs.append(torch.randn(K, L.N, device="cuda").to(torch.bfloat16))
        Ws.append(torch.randn(L.M, L.N, device="cuda") * 0.02)
        vs.append(torch.zeros(L.M, L.N, device="cuda"))
    g = tag.SfbGroup(plans)
    ts = []
    for it in range(13):
        flush.zero_()
        flush.sum()
        torch.cuda._sleep(1_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.sync_sgd(Xs, dYs, Ws, vs)
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
    out[f"K={nv * cfg.layers[0].B}"] = round(statistics.median(ts) * 1e3, 2)
    g.close()
    for p in plans:
        p.close()
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("TAG_")}, "us": out}))
comm.close()
