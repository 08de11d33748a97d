#!/usr/bin/env python3
"""Event-timed reconstruction of one layer (virtual n replicas on one GPU, K = n*B), L2 left
clean between runs; prints us and the tensor-peak fraction. Diagnostics for tile sweeps."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_06126_b200 import synth, tag  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--layer", default="fc6")
ap.add_argument("--n", type=int, default=8)
ap.add_argument("--out", default="bf16")
ap.add_argument("--wire", default="bf16", help="bf16 (kind::f16) or f32 (3xTF32)")
a = ap.parse_args()
cfg = synth.CONFIGS[a.config]
L = next(L for L in cfg.layers if L.name == a.layer)
K = a.n * L.B
comm = tag.Comm(1, 0, 0)
wdt = torch.bfloat16 if a.wire == "bf16" else torch.float32
plan = tag.SfbPlan(comm, L.M, L.N, K, a.wire, a.wire, a.out)
X = torch.randn(K, L.M, device="cuda").to(wdt)
dY = torch.randn(K, L.N, device="cuda").to(wdt)
dW = torch.empty(L.M, L.N, device="cuda", dtype=torch.float32 if a.out == "f32" else torch.bfloat16)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
ts = []
for it in range(13):
    flush.zero_()
    flush.sum()
    torch.cuda._sleep(1_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    plan.sync(X, dY, dW)
    e1.record()
    torch.cuda.synchronize()
    if it >= 3:
        ts.append(e0.elapsed_time(e1))
us = statistics.median(ts) * 1e3
print(json.dumps({"layer": a.layer, "K": K, "wire": a.wire, "out": a.out, "us": round(us, 2),
                  "tensor_frac": round(2 * L.M * L.N * K / (us * 1e-6) / 1687.1e12, 3),
                  "simt": bool(os.environ.get("TAG_F32_SIMT")),
                  "lib": os.path.basename(tag.LIB_PATH)}))
plan.close()
comm.close()
