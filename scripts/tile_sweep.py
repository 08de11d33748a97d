#!/usr/bin/env python3
"""Reconstruction tile-config sweep on one GPU: the VGG-19 FC bucket (one grouped launch) at
virtual n = 1, 2, 4, 8 (K = 32 n), for the tile configs selectable by environment variables.
Run once per config, e.g. TAG_RECON_BN=256 python scripts/tile_sweep.py."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_06126_b200 import synth, tag  # noqa: E402

cfg = synth.CONFIGS[int(os.environ.get("CONFIG", "2"))]
comm = tag.Comm(1, 0, 0)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
out = {}
for nv in (1, 2, 4, 8):
    plans, Xs, dYs, dWs = [], [], [], []
    for li, L in enumerate(cfg.layers):
        K = nv * L.B
        plans.append(tag.SfbPlan(comm, L.M, L.N, K))
        Xs.append(torch.randn(K, L.M, device="cuda").to(torch.bfloat16))
        dYs.append(torch.randn(K, L.N, device="cuda").to(torch.bfloat16))
        dWs.append(torch.empty(L.M, L.N, device="cuda"))
    g = tag.SfbGroup(plans)
    ts = []
    for it in range(13):
        flush.zero_()
        flush.sum()            # leave L2 holding clean lines (no write-back inside the timing)
        torch.cuda._sleep(1_000_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.sync(Xs, dYs, dWs)
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
    out[f"K={nv * cfg.layers[0].B}"] = round(statistics.median(ts) * 1e3, 2)
    g.close()
    for p in plans:
        p.close()
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("TAG_RECON")},
                  "us": out}))
