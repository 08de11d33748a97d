#!/usr/bin/env python3
"""Driver for an ncu capture of the factor pack (step a1): fp32 X_r, dY_r of VGG-19 fc6 cast to
the bf16 wire (pack_cast_kernel), n = 1, then the reconstruction. `--iters` syncs."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_06126_b200 import tag  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--B", type=int, default=256)
a = ap.parse_args()
M, N = 25088, 4096
comm = tag.Comm(1, 0, 0)
plan = tag.SfbPlan(comm, M, N, a.B, "f32", "bf16", "f32")
X = torch.randn(a.B, M, device="cuda")
dY = torch.randn(a.B, N, device="cuda")
dW = torch.empty(M, N, device="cuda")
for _ in range(a.iters):
    plan.sync(X, dY, dW)
torch.cuda.synchronize()
print(f"ok pack fc6 B={a.B} iters={a.iters}")
plan.close()
comm.close()
