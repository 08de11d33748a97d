#!/usr/bin/env python3
"""Copy-engine peer copies vs the SM push (one process, 2+ GPUs): device-to-device
cudaMemcpyAsync (torch .copy_ across devices uses the copy engines over NVLink when peer access is
on) of S bytes from GPU 0 to GPU 1, event-timed on GPU 0's stream; and the same copy issued while
GPU 1 streams a 411 MB write (does the CE keep its bandwidth under an HBM-bound kernel?)."""
import json
import statistics

import torch

assert torch.cuda.device_count() >= 2
res = {}
for mb in (0.33, 0.85, 2.7, 8.2, 19.0, 128.0):
    n = int(mb * 1e6) // 4
    a = torch.randn(n, device="cuda:0")
    b = torch.empty(n, device="cuda:1")
    s = torch.cuda.Stream(device="cuda:0")
    ts = []
    for it in range(23):
        with torch.cuda.stream(s):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            b.copy_(a, non_blocking=True)
            e1.record(s)
        torch.cuda.synchronize("cuda:0")
        torch.cuda.synchronize("cuda:1")
        if it >= 3:
            ts.append(e0.elapsed_time(e1) * 1e3)
    t = statistics.median(ts)
    res[f"{mb}MB"] = {"us": round(t, 2), "GBps": round(mb * 1e3 / t, 1)}
# under load: GPU 1 writes 411 MB while GPU 0 copies 2.7 MB into it
big = torch.empty(411 * 1024 * 1024 // 4, device="cuda:1")
n = int(2.7e6) // 4
a = torch.randn(n, device="cuda:0")
b = torch.empty(n, device="cuda:1")
ts = []
for it in range(13):
    with torch.cuda.device(1):
        big.fill_(float(it))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    b.copy_(a, non_blocking=True)
    e1.record()
    torch.cuda.synchronize("cuda:0")
    torch.cuda.synchronize("cuda:1")
    if it >= 3:
        ts.append(e0.elapsed_time(e1) * 1e3)
res["2.7MB_under_411MB_write"] = {"us": round(statistics.median(ts), 2)}
print(json.dumps(res))
