#!/usr/bin/env python3
"""The paper's op profiler for the profiled selector (tag_sfb_select_profiled,
SURVEY §8(f) rank 4): on one GPU, for every layer of configs 2-5 and n in {2, 4, 8}, the measured
time of the SFB reconstruction at K = nB (tag_sfb_reconstruct from factors already in place:
virtual n replicas stacked rank-major) and of the dense path's local gradient at K = B
(tag_local_grad), each the median of `reps` CUDA-event-timed runs with L2 flushed in between.

    python scripts/profile_compute.py [--reps 15] [--out profiles/compute_profile.json]

Output: {"<config>": {"<layer>": {"<n>": {"recon_ns": .., "local_ns": ..}}}, "_doc": ...}.
bench.py passes these with the measured communication curves (profiles/comm_n<n>.json) to the
profiled selector and reports its decision beside the measured winner.
"""
import argparse
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2302_06126_b200 import synth, tag  # noqa: E402

TDT = {"f32": torch.float32, "bf16": torch.bfloat16}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=15)
    ap.add_argument("--out", default=os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "profiles", "compute_profile.json"))
    ap.add_argument("--configs", default="2,3,4,5")
    args = ap.parse_args()
    comm = tag.Comm(1, 0, 0)
    flush = torch.empty(64 * 1024 * 1024, device="cuda")

    def timed(fn):
        ts = []
        for it in range(args.reps + 2):
            flush.zero_()
            flush.sum()
            torch.cuda._sleep(200_000)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if it >= 2:
                ts.append(e0.elapsed_time(e1))
        return int(statistics.median(ts) * 1e6)          # ns

    res = {"_doc": "scripts/profile_compute.py: median CUDA-event ns, L2 flushed; recon at K = nB "
                   "(virtual n), local gradient at K = B; dtypes of each config",
           "gpu": torch.cuda.get_device_name(0)}
    for cid in [int(c) for c in args.configs.split(",")]:
        cfg = synth.CONFIGS[cid]
        out_t = TDT[cfg.out_dtype]
        for li, L in enumerate(cfg.layers):
            dW = torch.empty(L.M, L.N, dtype=out_t, device="cuda")
            X1 = torch.randn(L.B, L.M, device="cuda").to(TDT[cfg.in_dtype])
            dY1 = torch.randn(L.B, L.N, device="cuda").to(TDT[cfg.in_dtype])
            p1 = tag.SfbPlan(comm, L.M, L.N, L.B, cfg.in_dtype, cfg.wire_dtype, cfg.out_dtype)
            local_ns = timed(lambda: p1.local_grad(X1, dY1, dW))
            p1.close()
            for n in (2, 4, 8):
                K = n * L.B
                pk = tag.SfbPlan(comm, L.M, L.N, K, cfg.wire_dtype, cfg.wire_dtype, cfg.out_dtype)
                Xk = torch.randn(K, L.M, device="cuda").to(TDT[cfg.wire_dtype])
                dYk = torch.randn(K, L.N, device="cuda").to(TDT[cfg.wire_dtype])
                pk.gather(Xk, dYk)
                recon_ns = timed(lambda: pk.reconstruct(dW))
                pk.close()
                res.setdefault(str(cid), {}).setdefault(L.name, {})[str(n)] = {
                    "recon_ns": recon_ns, "local_ns": local_ns, "M": L.M, "N": L.N, "B": L.B}
                print(cid, L.name, n, recon_ns, local_ns, flush=True)
            del dW
    comm.close()
    with open(args.out, "w") as f:
        json.dump(res, f, indent=1)
    print("wrote", args.out)


if __name__ == "__main__":
    main()
