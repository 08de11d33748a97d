#!/usr/bin/env python3
"""A/B timing of the fused optimizer epilogues (E2 SGD-momentum, E3 Adam) on one GPU: the BERT-L
FFN/pooler bucket (bench --config 5) and the Transformer bucket (config 4) as one grouped
launch, at K = B (n = 1) and K = 8B (north_star's n = 8 contraction, virtual replicas stacked).
Median of CUDA-event-timed runs with L2 flushed in between; HBM fraction of the algorithmic
bytes (16 B per element for SGD, 24 for Adam, + the factors) against MEASURED_PEAKS.json.

    TAG_LIB_PATH=build_exp/libtag_<v>.so python scripts/opt_epilogue_ab.py --label <v>
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_06126_b200 import synth, tag  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--label", default="product")
ap.add_argument("--reps", type=int, default=25)
args = ap.parse_args()
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
peak = None
try:
    pk = json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))
    peak = pk.get("hbm_gbs")
except (OSError, ValueError):
    pass
comm = tag.Comm(1, 0, 0)
flush = torch.empty(64 * 1024 * 1024, device="cuda")


def timed(fn):
    ts = []
    for it in range(args.reps + 3):
        flush.zero_()
        flush.sum()
        torch.cuda._sleep(200_000)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
    return statistics.median(ts) * 1e3


out = {"label": args.label, "lib": os.environ.get("TAG_LIB_PATH", "")}
for cid in (5, 4):
    cfg = synth.CONFIGS[cid]
    for nv in (1, 8):
        for opt in ("sgd", "adam"):
            plans, Xs, dYs, Ws, vs, ms = [], [], [], [], [], []
            nbytes = 0
            for L in cfg.layers:
                K = nv * L.B
                kw = dict(fuse_sgd=True, lr=1e-3, momentum=0.9) if opt == "sgd" else dict(fuse_adam=True, lr=1e-3)
                plans.append(tag.SfbPlan(comm, L.M, L.N, K, "bf16", "bf16", "f32", **kw))
                Xs.append(torch.randn(K, L.M, device="cuda").to(torch.bfloat16))
                dYs.append(torch.randn(K, L.N, device="cuda").to(torch.bfloat16))
                Ws.append(torch.randn(L.M, L.N, device="cuda"))
                vs.append(torch.rand(L.M, L.N, device="cuda"))
                ms.append(torch.randn(L.M, L.N, device="cuda") if opt == "adam" else None)
                nbytes += K * (L.M + L.N) * 2 + L.M * L.N * (16 if opt == "sgd" else 24)
            g = tag.SfbGroup(plans)
            if opt == "sgd":
                us = timed(lambda: g.sync_sgd(Xs, dYs, Ws, vs, None))
            else:
                us = timed(lambda: g.sync_adam(Xs, dYs, Ws, ms, vs, 1, None))
            g.close()
            for p in plans:
                p.close()
            key = f"c{cid}_n{nv}_{opt}"
            out[key] = {"us": round(us, 2), "frac": round(nbytes / us / 1e3 / peak, 3) if peak else None}
comm.close()
print(json.dumps(out), flush=True)
