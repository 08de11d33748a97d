#!/usr/bin/env python3
"""Probe: device->host copy throughput of a 411 MB buffer into pinned memory, one copy vs the
same bytes split over several streams (several copy engines); also host->device."""
import json
import torch

N = 411 * 1024 * 1024 // 4
d = torch.randn(N, device="cuda")
h = torch.empty(N, dtype=torch.float32).pin_memory()
res = {}
for nstreams in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    chunk = (N + nstreams - 1) // nstreams
    for direction in ("d2h", "h2d"):
        ts = []
        for it in range(6):
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record()
            for i, s in enumerate(streams):
                s.wait_event(e0)
                with torch.cuda.stream(s):
                    lo, hi = i * chunk, min(N, (i + 1) * chunk)
                    if direction == "d2h":
                        h[lo:hi].copy_(d[lo:hi], non_blocking=True)
                    else:
                        d[lo:hi].copy_(h[lo:hi], non_blocking=True)
            for s in streams:
                torch.cuda.current_stream().wait_stream(s)
            e1.record()
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(e0.elapsed_time(e1))
        res[f"{direction}_{nstreams}"] = round(N * 4 / (min(ts) * 1e-3) / 1e9, 1)
print(json.dumps({"GBps": res}))
