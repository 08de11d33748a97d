#!/usr/bin/env python3
"""Measure the two synchronisation curves the profiled selector reads (the paper's profiler,
P:331-334: transfers "starting from 1KB and doubled until 1GB"; SPEC fit_comm S:197-205):

  gather     x = bytes each rank receives, (n-1) * B(M+N) * 2   -> ns of tag_sfb_gather (NVLink push)
  allreduce  x = gradient bytes M * N * 4                        -> ns of tag_dense_allreduce
  ps         x = gradient bytes M * N * 4                        -> ns of tag_ps_sync (root 0)

Run under torchrun with n ranks; every point is device-timed on one call after a device barrier
(median of `--reps`, max over ranks). Rank 0 writes profiles/comm_n{n}.json."""
import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

from paper_2302_06126_b200 import dist as tdist  # noqa: E402
from paper_2302_06126_b200 import tag  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=9)
ap.add_argument("--max-gather", type=int, default=1 << 27)
ap.add_argument("--max-allreduce", type=int, default=1 << 30)
args = ap.parse_args()
rank, local_rank, world = tdist.init_from_env()
assert world > 1, "run under torchrun with >= 2 ranks"
torch.cuda.set_device(local_rank)
comm = tdist.bootstrap_comm(tag, local_rank)
s = torch.cuda.Stream()


def timed(fn):
    ts = []
    for _ in range(args.reps + 2):
        torch.cuda.synchronize()
        tdist.barrier()
        with torch.cuda.stream(s):
            torch.cuda._sleep(200_000)
            comm.barrier(s)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            fn()
            e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return tdist.max_over_ranks(statistics.median(ts[2:])) * 1e6     # ns


gather, allreduce, ps = [], [], []
x = 4096
while x <= args.max_gather:
    B = 8
    MN = max(16, (x // ((world - 1) * B * 2) // 16) * 16)     # M + N, each a multiple of 8
    M = N = MN // 2
    plan = tag.SfbPlan(comm, M, N, B)
    X = torch.randn(B, M, device="cuda").to(torch.bfloat16)
    dY = torch.randn(B, N, device="cuda").to(torch.bfloat16)
    ns = timed(lambda: plan.gather(X, dY, s))
    gather.append([(world - 1) * B * (M + N) * 2, int(round(ns))])
    plan.close()
    x *= 2
x = 4096
while x <= args.max_allreduce:
    M = 64
    N = max(8, (x // (M * 4) // 8) * 8)
    plan = tag.SfbPlan(comm, M, N, 1)
    dW = torch.randn(M, N, device="cuda")
    ns = timed(lambda: plan.dense_allreduce(dW, s))
    allreduce.append([M * N * 4, int(round(ns))])
    ns = timed(lambda: plan.ps_sync(dW, 0, s))
    ps.append([M * N * 4, int(round(ns))])
    plan.close()
    del dW
    x *= 2
if rank == 0:
    out = {"n": world, "gpu": torch.cuda.get_device_name(0), "gather": gather,
           "allreduce": allreduce, "ps": ps,
           "how": "scripts/profile_comm.py: one call after tag_comm_barrier, median of reps, max over ranks"}
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    path = os.path.join(ROOT, "gpurun_out" if os.path.isdir(os.path.join(ROOT, "gpurun_out")) else "profiles", f"comm_n{world}.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps(out))
comm.close()
