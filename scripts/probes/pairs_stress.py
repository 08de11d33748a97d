#!/usr/bin/env python3
"""Stress probe (torchrun): many fused syncs of a 4096 x 4096 layer at K = 256 (the CTA-pair fused
kernel), synchronising every few calls; prints the first failure (or "ok")."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2302_06126_b200 import dist as tdist  # noqa: E402
from paper_2302_06126_b200 import tag  # noqa: E402

rank, local_rank, world = tdist.init_from_env()
torch.cuda.set_device(local_rank)
comm = tdist.bootstrap_comm(tag, local_rank)
M, N = int(os.environ.get("M", 4096)), int(os.environ.get("N", 4096))
B = int(os.environ.get("KTOT", 256)) // world
plan = tag.SfbPlan(comm, M, N, B)
X = torch.randn(B, M, device="cuda").to(torch.bfloat16)
dY = torch.randn(B, N, device="cuda").to(torch.bfloat16)
dW = torch.empty(M, N, device="cuda")
t0 = time.time()
iters = int(os.environ.get("ITERS", 300))
try:
    for i in range(iters):
        plan.sync(X, dY, dW)
        if i % 10 == 9:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    msg = f"ok {iters} syncs in {time.time() - t0:.1f}s"
except Exception as e:  # noqa: BLE001
    msg = f"FAIL at ~{i} after {time.time() - t0:.1f}s: {str(e).splitlines()[0]}"
print(f"rank {rank}: {msg}", flush=True)
os._exit(0)
