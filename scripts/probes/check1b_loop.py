#!/usr/bin/env python3
"""Stress probe (torchrun): the multi_gpu_check 1b sequence (new plan, 3 fused syncs at K = 256,
local_grad, dense_allreduce, synchronize, all_gather of a digest, close) repeated."""
import hashlib
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2302_06126_b200 import dist as tdist  # noqa: E402
from paper_2302_06126_b200 import synth, tag  # noqa: E402

rank, local_rank, world = tdist.init_from_env()
torch.cuda.set_device(local_rank)
comm = tdist.bootstrap_comm(tag, local_rank)
t0 = time.time()
n_it = int(os.environ.get("ITERS", 30))
it = -1
try:
    for it in range(n_it):
        for M, N in ((4096, 4096), (520, 264), (4096, 1000)):
            B = 256 // world if M != 4096 or N != 1000 else 32
            X, dY = synth.factors(64, it % 7, rank, M, N, B, "int3", "int3")
            plan = tag.SfbPlan(comm, M, N, B)
            Xd = torch.from_numpy(X).to(torch.bfloat16).cuda()
            dYd = torch.from_numpy(dY).to(torch.bfloat16).cuda()
            dW = torch.full((M, N), float("nan"), device="cuda")
            for _ in range(3):
                plan.sync(Xd, dYd, dW)
            dense = torch.empty_like(dW)
            plan.local_grad(Xd, dYd, dense)
            plan.dense_allreduce(dense)
            torch.cuda.synchronize()
            h = hashlib.sha256(dW.view(torch.uint8).cpu().numpy().tobytes()).hexdigest()
            hs = tdist.all_gather_object(h)
            assert len(set(hs)) == 1, "ranks differ"
            plan.close()
    msg = f"ok {n_it} rounds in {time.time() - t0:.1f}s"
except Exception as e:  # noqa: BLE001
    msg = f"FAIL at {it} after {time.time() - t0:.1f}s: {str(e).splitlines()[0]}"
print(f"rank {rank}: {msg}", flush=True)
os._exit(0)
