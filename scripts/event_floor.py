#!/usr/bin/env python3
"""The CUDA-event timing floor on this GPU: two events recorded back to back after a device spin,
then 1 / 10 empty torch kernels between them, then one and ten back-to-back reconstructions of
small layers (per-launch = slope). Median µs over reps. Separates the event/launch floor from a
small kernel's own duration (scripts/small_layer_latency.py times one launch per interval).

    python scripts/event_floor.py [--reps 30]
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
args = ap.parse_args()
s = torch.cuda.Stream()


def timed(fn):
    ts = []
    for it in range(args.reps + 3):
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
    return round(statistics.median(ts) * 1e3, 3)


x = torch.zeros(1, device="cuda")


def kern(k):
    def f():
        for _ in range(k):
            x.add_(1)
    return f


out = {"events_only_us": timed(lambda: None), "empty_kernel_x1_us": timed(kern(1)),
       "empty_kernel_x10_us": timed(kern(10)), "empty_kernel_x50_us": timed(kern(50))}
ge = torch.cuda.CUDAGraph()
with torch.cuda.stream(s):
    kern(10)()
torch.cuda.synchronize()
with torch.cuda.graph(ge, stream=s):
    kern(10)()
out["empty_kernel_graph_x10_us"] = timed(lambda: ge.replay())
comm = tag.Comm(1, 0, 0)
for M, N, K in ((1024, 1024, 16), (4096, 1000, 256), (4096, 4096, 256), (25088, 4096, 256)):
    p = tag.SfbPlan(comm, M, N, K, "bf16", "bf16", "bf16")
    X = torch.randn(K, M, device="cuda").to(torch.bfloat16)
    dY = torch.randn(K, N, device="cuda").to(torch.bfloat16)
    dW = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    p.gather(X, dY, s)
    t1 = timed(lambda: p.reconstruct(dW, s))

    def ten():
        for _ in range(10):
            p.reconstruct(dW, s)
    t10 = timed(ten)
    # the same ten launches captured once into a CUDA graph: no host enqueue inside the interval
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        ten()
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=s):
        ten()
    g1 = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g1, stream=s):
        p.reconstruct(dW, s)
    tg1 = timed(lambda: g1.replay())
    tg10 = timed(lambda: g.replay())
    out[f"recon_{M}x{N}_K{K}_bf16"] = {"x1_us": t1, "x10_us": t10,
                                       "per_launch_us": round((t10 - t1) / 9, 3),
                                       "graph_x1_us": tg1, "graph_x10_us": tg10,
                                       "graph_per_launch_us": round((tg10 - tg1) / 9, 3)}
    p.close()
comm.close()
print(json.dumps(out), flush=True)
