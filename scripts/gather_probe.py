#!/usr/bin/env python3
"""Gather-stage latency/bandwidth probe (torchrun, n ranks): back-to-back tag_sfb_gather calls of
one layer, CUDA-event timed over `iters` calls, max over ranks. TAG_GATHER=nccl selects the
ncclAllGather mode for comparison."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_06126_b200 import dist as tdist  # noqa: E402
from paper_2302_06126_b200 import tag  # noqa: E402

rank, local_rank, world = tdist.init_from_env()
torch.cuda.set_device(local_rank)
comm = tdist.bootstrap_comm(tag, local_rank)
out = {}
SIZES = [(4096, 1000, 32), (4096, 4096, 32), (25088, 4096, 32), (25088, 4096, 256),
         (512, 32000, 256)]
if os.environ.get("PROBE_SMALL"):
    SIZES = [(4096, 1000, 32), (25088, 4096, 32)]
flush = torch.empty(64 * 1024 * 1024, device="cuda")
for (M, N, B) in SIZES:
    plan = tag.SfbPlan(comm, M, N, B, "bf16", "bf16", "f32")
    X = torch.randn(B, M, device="cuda").to(torch.bfloat16)
    dY = torch.randn(B, N, device="cuda").to(torch.bfloat16)
    for _ in range(5):
        plan.gather(X, dY)
    torch.cuda.synchronize()
    tdist.barrier()
    iters = 50
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(200000)
    e0.record()
    for _ in range(iters):
        plan.gather(X, dY)
    e1.record()
    torch.cuda.synchronize()
    t = tdist.max_over_ranks(e0.elapsed_time(e1) / iters)
    ingress = (world - 1) * B * (M + N) * 2
    # cold: one gather after an L2 flush, device-aligned by a 1-element all-reduce
    cold = []
    tok = torch.zeros(1, device="cuda")
    for _ in range(10):
        flush.zero_()
        torch.cuda.synchronize()
        tdist.barrier()
        torch.cuda._sleep(100000)
        torch.distributed.all_reduce(tok)
        c0, c1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        c0.record()
        plan.gather(X, dY)
        c1.record()
        torch.cuda.synchronize()
        cold.append(c0.elapsed_time(c1))
    tc = tdist.max_over_ranks(sorted(cold)[len(cold) // 2])
    out[f"{M}x{N}xB{B}"] = {"us": round(t * 1e3, 2), "cold_us": round(tc * 1e3, 2),
                            "ingress_MB": ingress / 1e6,
                            "busbw_GBps": round(ingress / (t * 1e-3) / 1e9, 1),
                            "mode": plan.info()["gather"]}
    plan.close()
if rank == 0:
    print(json.dumps({"n": world, "gather": out}), flush=True)
comm.close()
