#!/usr/bin/env python3
"""Diagnostic (TAG_PUSH_DEBUG=3): cold bucket push of the VGG-19 FC factors, n ranks; the kernel
printf()s %globaltimer phase stamps (start, +data, +barrier) for a few CTAs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_06126_b200 import dist as tdist  # noqa: E402
from paper_2302_06126_b200 import synth, tag  # noqa: E402

rank, local_rank, world = tdist.init_from_env()
torch.cuda.set_device(local_rank)
comm = tdist.bootstrap_comm(tag, local_rank)
cfg = synth.CONFIGS[2]
plans, Xs, dYs = [], [], []
for li, L in enumerate(cfg.layers):
    plans.append(tag.SfbPlan(comm, L.M, L.N, L.B))
    Xs.append(torch.randn(L.B, L.M, device="cuda").to(torch.bfloat16))
    dYs.append(torch.randn(L.B, L.N, device="cuda").to(torch.bfloat16))
g = tag.SfbGroup(plans)
flush = torch.empty(64 * 1024 * 1024, device="cuda")
tok = torch.zeros(1, device="cuda")
for it in range(4):
    flush.zero_()
    torch.cuda.synchronize()
    tdist.barrier()
    torch.cuda._sleep(100000)
    torch.distributed.all_reduce(tok)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.gather(Xs, dYs)
    e1.record()
    torch.cuda.synchronize()
    print(f"rank {rank} iter {it} event_us {e0.elapsed_time(e1) * 1e3:.1f}", flush=True)
g.close()
for p in plans:
    p.close()
comm.close()
