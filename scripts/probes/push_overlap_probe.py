#!/usr/bin/env python3
"""Driver of push_overlap_probe.cu (diagnostic): torchrun --nproc-per-node N. For P dedicated push
CTAs, the span of pushing one rank's VGG-19 bucket factors (2.72 MB) to every peer, alone and while
the other 148 - P SMs write 411 MB of HBM (fc6's fp32 dW); and the write span alone / with the push.
Median of 7 launches, max over ranks. Prints one JSON line (rank 0)."""
import ctypes
import json
import os
import statistics
import subprocess
import sys

import torch
import torch.distributed as dist

HERE = os.path.dirname(os.path.abspath(__file__))
rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
local = int(os.environ.get("LOCAL_RANK", 0))
torch.cuda.set_device(local)
dist.init_process_group("gloo")
import nvidia.nccl  # noqa: E402
nccl = list(nvidia.nccl.__path__)[0]
so = os.path.join(HERE, "libpushprobe.so")
if rank == 0 and not os.path.exists(so):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-std=c++17",
                           "-shared", "-Xcompiler", "-fPIC", f"-I{nccl}/include",
                           os.path.join(HERE, "push_overlap_probe.cu"), f"-L{nccl}/lib",
                           "-l:libnccl.so.2", "-Xlinker", f"-rpath,{nccl}/lib", "-o", so])
dist.barrier()
lib = ctypes.CDLL(so)
uid = ctypes.create_string_buffer(128)
if rank == 0:
    assert lib.probe_uid(uid) == 0
t = torch.frombuffer(bytearray(uid.raw), dtype=torch.uint8).clone()
dist.broadcast(t, 0)
uid = ctypes.create_string_buffer(bytes(t.tolist()), 128)
SLOT = 32 * (25088 + 4096 + 4096 + 4096 + 4096 + 1000) * 2
WRITE = 25088 * 4096 * 4
r = lib.probe_init(uid, world, rank, local, ctypes.c_size_t(SLOT), ctypes.c_size_t(WRITE))
assert r == 0, r
out = (ctypes.c_ulonglong * 4096)()
s = torch.cuda.current_stream().cuda_stream


def run(push, P, write, grid, reps=7):
    ps, ws = [], []
    for _ in range(reps + 2):
        dist.barrier()
        assert lib.probe_run(ctypes.c_size_t(push), P, ctypes.c_size_t(write), grid, out,
                             ctypes.c_void_p(s)) == 0
        st = [(out[2 * i], out[2 * i + 1]) for i in range(grid)]
        t0 = min(a for a, _ in st)
        ps.append((max(b for a, b in st[:P]) - t0) / 1e3 if P else 0.0)
        ws.append((max(b for a, b in st[P:]) - t0) / 1e3 if grid > P else 0.0)
    p, w = statistics.median(ps[2:]), statistics.median(ws[2:])
    tt = torch.tensor([p, w], dtype=torch.float64)
    dist.all_reduce(tt, op=dist.ReduceOp.MAX)
    return round(tt[0].item(), 2), round(tt[1].item(), 2)


res = {"n": world, "slot_MB": SLOT / 1e6, "egress_MB": SLOT * (world - 1) / 1e6,
       "write_MB": WRITE / 1e6, "write_alone_us": run(0, 0, WRITE, 148)[1], "rows": []}
for P in (4, 8, 12, 16, 24, 32, 48, 74, 148):
    alone = run(SLOT, P, 0, P)[0]
    both = run(SLOT, P, WRITE, 148) if P < 148 else (None, None)
    res["rows"].append({"P": P, "push_alone_us": alone, "push_with_write_us": both[0],
                        "write_with_push_us": both[1],
                        "egress_GBps_alone": round(SLOT * (world - 1) / (alone * 1e-6) / 1e9, 1)})
if rank == 0:
    print(json.dumps(res), flush=True)
