#!/usr/bin/env python3
"""Fused push+reconstruction timing probe (torchrun): the VGG-19 bucket, cold (L2 flushed, ranks
aligned by tag_comm_barrier), CUDA events around one tag_sfb_group_sync. Diagnostics variants of
the library (scripts/build_variant.sh, loaded with TAG_LIB_PATH) select the profiling forms of the
fused kernel (no push / no wait / printf stamps); --label names the variant in the output."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_06126_b200 import dist as tdist  # noqa: E402
from paper_2302_06126_b200 import synth, tag  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--label", default="product")
ap.add_argument("--gather", default="auto")
ap.add_argument("--multicast", action="store_true")
args = ap.parse_args()
rank, local_rank, world = tdist.init_from_env()
torch.cuda.set_device(local_rank)
comm = tdist.bootstrap_comm(tag, local_rank, multicast=args.multicast)
cfg = synth.CONFIGS[2]
plans, Xs, dYs, dWs = [], [], [], []
for li, L in enumerate(cfg.layers):
    plans.append(tag.SfbPlan(comm, L.M, L.N, L.B, gather=args.gather))
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
    flush.sum()            # leave L2 holding clean lines (no write-back inside the timing)
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
p10 = tdist.max_over_ranks(sorted(ts)[len(ts) // 10])
if rank == 0:
    print(json.dumps({"n": world, "variant": args.label, "gather": args.gather,
                      "multicast": args.multicast,
                      "lib": os.environ.get("TAG_LIB_PATH", "libtag.so"),
                      "step_us": round(t * 1e3, 2),
                      "p10_us": round(p10 * 1e3, 2)}),
          flush=True)
g.close()
for p in plans:
    p.close()
comm.close()
