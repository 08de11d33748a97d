#!/usr/bin/env python3
"""Diagnostic (torchrun, n ranks): can the exchange of a wide layer overlap its reconstruction if
the layer is split by dY columns into two halves, the second half's factors pushed by a small
push-kernel grid on a side stream while the first half syncs (fused push + reconstruction on the
remaining SMs), then the second half reconstructed? Transformer output projection (512 x 32000,
256 tokens per rank). Run with a diagnostics build (TAG_LIB_PATH) that caps the push grid
(EXP_PUSH_GRID) and the reconstruction grid (EXP_RECON_SMS) so both kernels fit side by side.
Prints one JSON line (rank 0): whole-layer sync, split sequential, split overlapped (µs, max
over ranks), and whether the overlapped result equals the whole-layer one bit for bit."""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2302_06126_b200 import dist as tdist  # noqa: E402
from paper_2302_06126_b200 import synth, tag  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--label", default="")
ap.add_argument("--iters", type=int, default=15)
args = ap.parse_args()
rank, local_rank, world = tdist.init_from_env()
torch.cuda.set_device(local_rank)
comm = tdist.bootstrap_comm(tag, local_rank)
M, N, B = 512, 32000, 256
NA = 16000
X, dY = synth.factors(4, 0, rank, M, N, B, "normal", "softmax_onehot")
Xd = torch.from_numpy(X).to(torch.bfloat16).cuda()
dYd = torch.from_numpy(dY).to(torch.bfloat16).cuda()
dYa, dYb = dYd[:, :NA].contiguous(), dYd[:, NA:].contiguous()
whole = tag.SfbPlan(comm, M, N, B)
pa = tag.SfbPlan(comm, M, NA, B)
pb = tag.SfbPlan(comm, M, N - NA, B)
dW = torch.empty(M, N, device="cuda")
dWa = torch.empty(M, NA, device="cuda")
dWb = torch.empty(M, N - NA, device="cuda")
sA, sB = torch.cuda.Stream(), torch.cuda.Stream()
flush = torch.empty(64 * 1024 * 1024, device="cuda")


def timed(fn):
    ts = []
    for it in range(args.iters + 3):
        flush.zero_()
        flush.sum()
        torch.cuda.synchronize()
        tdist.barrier()
        with torch.cuda.stream(sA):
            torch.cuda._sleep(1_000_000)
            comm.barrier(sA)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(sA)
            fn(e0)
            e1.record(sA)
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
    return tdist.max_over_ranks(statistics.median(ts)) * 1e3


def whole_sync(e0):
    whole.sync(Xd, dYd, dW, sA)


def split_seq(e0):
    pa.sync(Xd, dYa, dWa, sA)
    pb.sync(Xd, dYb, dWb, sA)


def split_overlap(e0):
    sB.wait_event(e0)
    with torch.cuda.stream(sB):
        pb.gather(Xd, dYb, sB)                    # small push grid, side stream
        eb = torch.cuda.Event()
        eb.record(sB)
    pa.sync(Xd, dYa, dWa, sA)                     # fused push + reconstruction, other SMs
    sA.wait_event(eb)
    pb.reconstruct(dWb, sA)


t_whole = timed(whole_sync)
t_seq = timed(split_seq)
# only with a capped build: with both grids uncapped the two kernels cannot run side by side and
# a rank's fused kernel would wait for a peer whose fused kernel queues behind its push kernel
t_ovl = timed(split_overlap) if os.environ.get("TAG_LIB_PATH") else -1.0
torch.cuda.synchronize()
same = torch.equal(dW[:, :NA], dWa) and torch.equal(dW[:, NA:], dWb)
ok = all(tdist.all_gather_object(bool(same)))
if rank == 0:
    print(json.dumps({"n": world, "label": args.label, "lib": os.environ.get("TAG_LIB_PATH", ""),
                      "whole_us": round(t_whole, 2), "split_seq_us": round(t_seq, 2),
                      "split_overlap_us": round(t_ovl, 2), "bit_equal": ok}), flush=True)
for p in (whole, pa, pb):
    p.close()
comm.close()
