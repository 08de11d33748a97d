"""The N > 1 host-side path on CPU: world_size-2 `gloo` process groups (no GPU).

Covers the torch.distributed plumbing libtag's bootstrap and bench.py rely on (128-byte id
broadcast, max-over-ranks, object all-gather), the multi-replica semantics of SFB with the
oracle as compute (every rank gathers every rank's factors and reconstructs a bit-identical
dW that equals the dense all-reduce route), rank-consistent selector decisions from libtag's
host-only selector, and bench.py's reference arm under torchrun.
"""
import json
import os
import socket
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

WORKER = r'''
import hashlib, json, os, sys
sys.path.insert(0, os.environ["ROOT"])
import numpy as np
import torch
import torch.distributed as dist
import oracle
from paper_2302_06126_b200 import dist as tdist, synth, tag

rank, local_rank, world = tdist.init_from_env("gloo")
res = {}
# 1. bootstrap id broadcast, max over ranks, object all-gather
uid = bytes(range(128)) if rank == 0 else bytes(128)
res["uid_ok"] = tdist.broadcast_bytes(uid, 128, 0) == bytes(range(128))
res["max"] = tdist.max_over_ranks(float(rank + 1))
res["gather"] = tdist.all_gather_object(rank * 10)
# 2. SFB over gloo with the oracle as compute (config 1 and a VGG-shaped fc8 slice)
for (cid, M, N, B, xd, dyd) in [(1, 64, 32, 4, "normal", "normal"), (2, 96, 1000, 32, "relu", "softmax_onehot")]:
    X, dY = synth.factors(cid, 0, rank, M, N, B, xd, dyd)
    gx = [torch.empty(B, M) for _ in range(world)]
    gy = [torch.empty(B, N) for _ in range(world)]
    dist.all_gather(gx, torch.from_numpy(X))          # the factor all-gather (a2)
    dist.all_gather(gy, torch.from_numpy(dY))
    Xall = np.stack([t.numpy() for t in gx])
    dYall = np.stack([t.numpy() for t in gy])
    dW = oracle.sfb_dw(Xall, dYall)                   # every rank reconstructs (a3)
    h = hashlib.sha256(dW.tobytes()).hexdigest()
    # dense route: sum of per-rank local gradients, then / (nB)
    S = torch.from_numpy(oracle.dense_sum(X[None], dY[None]))
    dist.all_reduce(S)
    dense = S.numpy() / (world * B)
    Xr, dYr = synth.all_factors(cid, 0, world, M, N, B, xd, dyd)
    ref = oracle.sfb_dw(Xr, dYr)
    res[f"sfb_{M}x{N}"] = dict(hashes=tdist.all_gather_object(h),
                               vs_ref=float(np.abs(dW - ref).max()),
                               vs_dense=float(np.linalg.norm(dW - dense) / np.linalg.norm(dense)))
# 3. selector: identical decisions on every rank (host-only libtag call, no GPU)
lays = [dict(M=L.M, N=L.N, B=L.B) for c in (2, 3, 4, 5) for L in synth.CONFIGS[c].layers]
got = tag.select([dict(l, factor_dtype="bf16", grad_dtype="f32") for l in lays], world,
                 900_000_000_000, 1421400000000000)
want = [oracle.selector.select(dict(l, e_w=2, e_g=4), dict(n=world, tau=900_000_000_000,
                                                            F=1421400000000000)) for l in lays]
res["selector"] = dict(same=all(g == got for g in tdist.all_gather_object(got)), oracle=got == want)
if rank == 0:
    print("RESULT " + json.dumps(res), flush=True)
dist.destroy_process_group()
'''


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _torchrun(args, env_extra=None, timeout=600):
    env = dict(os.environ, ROOT=ROOT, CUDA_VISIBLE_DEVICES="")
    env.update(env_extra or {})
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
           "--master-addr=127.0.0.1", f"--master-port={_port()}"] + args
    return subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, cwd=ROOT, env=env)


def test_gloo_world2_sfb_semantics(tmp_path, oracle_mod):
    worker = tmp_path / "worker.py"
    worker.write_text(WORKER)
    r = _torchrun([str(worker)])
    lines = [l for l in r.stdout.splitlines() if l.startswith("RESULT ")]
    assert r.returncode == 0 and lines, r.stdout[-2000:] + r.stderr[-3000:]
    res = json.loads(lines[-1][len("RESULT "):])
    assert res["uid_ok"] and res["max"] == 2.0 and res["gather"] == [0, 10]
    for k in ("sfb_64x32", "sfb_96x1000"):
        assert len(set(res[k]["hashes"])) == 1          # bitwise identical on both ranks
        assert res[k]["vs_ref"] == 0.0                   # gather order = rank-major (R12)
        assert res[k]["vs_dense"] <= 1e-13               # lossless vs the AllReduce route
    assert res["selector"]["same"] and res["selector"]["oracle"]


def test_bench_reference_arm_world2():
    """`bench.py --impl reference` under torchrun: rank 0 alone prints one JSON line, exit 0."""
    r = _torchrun(["bench.py", "--impl", "reference", "--gpus", "2", "--steps", "1",
                   "--warmup", "0", "--ref-mac", "2e8"])
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and len(lines) == 1, r.stdout[-2000:] + r.stderr[-3000:]
    line = json.loads(lines[0])
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["cpu_baseline"]["kind"] == "oracle" and line["value"] > 0
