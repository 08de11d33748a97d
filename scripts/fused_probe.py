#!/usr/bin/env python3
"""Fused push+reconstruction timing probe (torchrun): the VGG-19 bucket, cold (L2 flushed, ranks
aligned by tag_comm_barrier), CUDA events around one tag_sfb_group_sync. TAG_FUSED_DEBUG=1/2/3
select the profiling variants of the fused kernel (no push / no wait / printf stamps)."""
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
for li, L in enumerate(cfg.layers):
    plans.append(tag.SfbPlan(comm, L.M, L.N, L.B))
    Xs.append(torch.randn(L.B, L.M, device="cuda").to(torch.bfloat16))
    dYs.append(torch.randn(L.B, L.N, device="cuda").to(torch.bfloat16))
    dWs.append(torch.empty(L.M, L.N, device="cuda"))
g = tag.SfbGroup(plans)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
s = torch.cuda.Stream()
ts = []
iters = int(os.environ.get("ITERS", "20"))
for it in range(iters + 3):
    flush.zero_()
    torch.cuda.synchronize()
    tdist.barrier()
    with torch.cuda.stream(s):
        torch.cuda._sleep(1_000_000)
        comm.barrier(s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        g.sync(Xs, dYs, dWs, s)
        e1.record(s)
    torch.cuda.synchronize()
    if it >= 3:
        ts.append(e0.elapsed_time(e1))
t = tdist.max_over_ranks(statistics.median(ts))
if rank == 0:
    print(json.dumps({"n": world, "dbg": os.environ.get("TAG_FUSED_DEBUG", "0"),
                      "no_fuse": bool(os.environ.get("TAG_NO_FUSE")), "step_us": round(t * 1e3, 2)}),
          flush=True)
g.close()
for p in plans:
    p.close()
comm.close()
