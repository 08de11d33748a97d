#!/usr/bin/env python3
"""Probe: relative Frobenius error of the tensor-core reconstruction vs the fp64 oracle on the
exact operand values, as a function of K (bf16 operands; fp32 operands via 3xTF32 and SIMT)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure)
from paper_2302_06126_b200 import tag  # noqa: E402

comm = tag.Comm(1, 0, 0)
rs = np.random.default_rng(7)
M, N = 256, 512
out = {}
for K in (32, 256, 2048, 8192):
    X = rs.standard_normal((K, M)).astype(np.float32)
    dY = rs.standard_normal((K, N)).astype(np.float32)
    for wire in ("bf16", "f32"):
        wdt = torch.bfloat16 if wire == "bf16" else torch.float32
        Xd = torch.from_numpy(X).to(wdt).cuda()
        dYd = torch.from_numpy(dY).to(wdt).cuda()
        Xe = Xd.double().cpu().numpy()
        dYe = dYd.double().cpu().numpy()
        ref = oracle.sfb_dw(Xe[None], dYe[None])
        p = tag.SfbPlan(comm, M, N, K, wire, wire, "f32")
        dW = torch.empty((M, N), device="cuda")
        p.sync(Xd, dYd, dW)
        torch.cuda.synchronize()
        p.close()
        e = float(np.linalg.norm(dW.cpu().numpy() - ref) / np.linalg.norm(ref))
        out[f"{wire}_K{K}"] = e
print(json.dumps(out))
