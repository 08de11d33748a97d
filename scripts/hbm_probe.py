#!/usr/bin/env python3
"""Practical HBM ceilings on this B200 for the reconstruction's traffic shape: write-only
(torch fill_) and copy (read+write, the MEASURED_PEAKS definition) of the fc6 dW size."""
import json
import torch

nbytes = 25088 * 4096 * 4
a = torch.empty(nbytes // 4, device="cuda")
b = torch.empty_like(a)
res = {}
for name, fn in [("write_fill", lambda: a.fill_(1.5)), ("copy", lambda: b.copy_(a))]:
    for _ in range(5):
        fn()
    ts = []
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda._sleep(50000)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    t = min(ts)
    moved = nbytes if name == "write_fill" else 2 * nbytes
    res[name] = {"bytes": moved, "best_ms": t, "GBps": moved / (t * 1e-3) / 1e9}
print(json.dumps(res))
