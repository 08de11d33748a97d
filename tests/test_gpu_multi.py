"""Multi-GPU parity (n = 2 and 4) through torchrun + NCCL; skipped when the box has one GPU (then
tests/test_gpu_loopback.py runs the same code paths on a one-rank NCCL communicator and
test_gpu_recon.py the n-replica reconstruction as virtual n)."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("gather", ["push", "nccl", "multicast"])
@pytest.mark.parametrize("nproc", [2, 4])
def test_multi_gpu_sfb(cuda, nproc, gather):
    if torch.cuda.device_count() < nproc:
        pytest.skip(f"needs {nproc} GPUs, box has {torch.cuda.device_count()}")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={nproc}", "--master-addr=127.0.0.1", f"--master-port={_free_port()}",
           os.path.join(ROOT, "scripts", "multi_gpu_check.py")]
    if gather == "nccl":
        cmd += ["--gather", "nccl"]
    if gather == "multicast":
        cmd += ["--multicast"]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=ROOT)
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert r.returncode == 0 and lines, r.stdout[-3000:] + r.stderr[-3000:]
    res = json.loads(lines[-1])
    assert res["ok"] and res["n"] == nproc, res
    want = {"nccl": "nccl_allgather", "push": "nvlink_push",
            "multicast": "nvlink_push+multicast"}[gather]
    assert want in res["gather_modes"] or (gather == "multicast" and "nvlink_push" in
                                            res["gather_modes"]), res   # no NVLS: unicast
