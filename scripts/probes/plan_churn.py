#!/usr/bin/env python3
"""Stress probe (torchrun): create a plan, sync a few times, destroy it — many times over, with
rank-dependent host delays — to exercise window initialisation / teardown races."""
import os
import random
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

from paper_2302_06126_b200 import dist as tdist  # noqa: E402
from paper_2302_06126_b200 import tag  # noqa: E402

rank, local_rank, world = tdist.init_from_env()
torch.cuda.set_device(local_rank)
comm = tdist.bootstrap_comm(tag, local_rank)
rnd = random.Random(rank)
shapes = [(4096, 4096, 256 // world), (4096, 1000, 32), (520, 264, 24), (25088, 4096, 32)]
t0 = time.time()
n_it = int(os.environ.get("ITERS", 40))
try:
    for it in range(n_it):
        M, N, B = shapes[it % len(shapes)]
        plan = tag.SfbPlan(comm, M, N, B)
        X = torch.randn(B, M, device="cuda").to(torch.bfloat16)
        dY = torch.randn(B, N, device="cuda").to(torch.bfloat16)
        dW = torch.empty(M, N, device="cuda")
        if rnd.random() < 0.5:
            torch.cuda._sleep(rnd.randint(0, 2_000_000))      # skew the ranks' streams
        for _ in range(3):
            plan.sync(X, dY, dW)
        torch.cuda.synchronize()
        plan.close()
    msg = f"ok {n_it} plan lifecycles in {time.time() - t0:.1f}s"
except Exception as e:  # noqa: BLE001
    msg = f"FAIL at {it} after {time.time() - t0:.1f}s: {str(e).splitlines()[0]}"
print(f"rank {rank}: {msg}", flush=True)
os._exit(0)
