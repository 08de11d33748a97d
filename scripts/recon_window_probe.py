#!/usr/bin/env python3
"""Reconstruction-only time of the VGG-19 bucket at n = world size (torchrun), after an untimed
gather, clean L2: does the operand buffer (NCCL symmetric window in push mode, cudaMalloc in
TAG_GATHER=nccl mode) change the reconstruction's speed?"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_06126_b200 import dist as tdist  # noqa: E402
from paper_2302_06126_b200 import synth, tag  # noqa: E402

rank, local_rank, world = tdist.init_from_env()
torch.cuda.set_device(local_rank)
comm = tdist.bootstrap_comm(tag, local_rank)
cfg = synth.CONFIGS[2]
plans, Xs, dYs, dWs = [], [], [], []
for L in cfg.layers:
    plans.append(tag.SfbPlan(comm, L.M, L.N, L.B))
    Xs.append(torch.randn(L.B, L.M, device="cuda").to(torch.bfloat16))
    dYs.append(torch.randn(L.B, L.N, device="cuda").to(torch.bfloat16))
    dWs.append(torch.empty(L.M, L.N, device="cuda"))
g = tag.SfbGroup(plans)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
ts = []
for it in range(23):
    g.gather(Xs, dYs)
    flush.zero_()
    flush.sum()
    torch.cuda.synchronize()
    torch.cuda._sleep(1_000_000)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.reconstruct(dWs)
    e1.record()
    torch.cuda.synchronize()
    if it >= 3:
        ts.append(e0.elapsed_time(e1))
t = tdist.max_over_ranks(statistics.median(ts))
if rank == 0:
    print(json.dumps({"n": world, "gather": plans[0].info()["gather"], "recon_us": round(t * 1e3, 2)}),
          flush=True)
g.close()
for p in plans:
    p.close()
comm.close()
