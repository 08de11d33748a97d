#!/usr/bin/env python3
"""Where does a small layer's reconstruction time go? One GPU, one layer per launch, median
CUDA-event µs (device spin ahead of the start event so the host enqueue is not timed), with and
without an L2 flush before each run: an empty torch kernel (the event floor), then
tag_sfb_reconstruct of growing layers at K = 16 and K = 256, fp32 / bf16 dW.

    python scripts/small_layer_latency.py [--reps 30]
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_06126_b200 import tag  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=30)
ap.add_argument("--label", default="")
args = ap.parse_args()
comm = tag.Comm(1, 0, 0)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
s = torch.cuda.Stream()


def timed(fn, do_flush):
    ts = []
    for it in range(args.reps + 3):
        if do_flush:
            flush.zero_()
            flush.sum()
        torch.cuda.synchronize()
        with torch.cuda.stream(s):
            torch.cuda._sleep(1_000_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
    return round(statistics.median(ts) * 1e3, 2)


x = torch.zeros(1, device="cuda")
out = {"label": args.label,
       "empty_torch_kernel_us": timed(lambda: x.add_(1), False)}
shapes = [(128, 128), (1024, 1024), (4096, 1000), (4096, 4096)]
for K in (16, 256):
    for M, N in shapes:
        for odt in ("f32", "bf16"):
            p = tag.SfbPlan(comm, M, N, K, "bf16", "bf16", odt)
            X = torch.randn(K, M, device="cuda").to(torch.bfloat16)
            dY = torch.randn(K, N, device="cuda").to(torch.bfloat16)
            dW = torch.empty(M, N, device="cuda", dtype=torch.float32 if odt == "f32" else torch.bfloat16)
            p.gather(X, dY, s)
            key = f"K{K}_{M}x{N}_{odt}"
            out[key] = {"flushed": timed(lambda: p.reconstruct(dW, s), True),
                        "warm": timed(lambda: p.reconstruct(dW, s), False)}
            p.close()
comm.close()
print(json.dumps(out), flush=True)
