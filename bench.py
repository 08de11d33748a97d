#!/usr/bin/env python3
"""bench.py — per-layer SFB gradient synchronisation on B200 (TAG, arXiv 2302.06126).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 2] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU, NCCL)

Workload (BASELINE.json configs[1]): VGG-19 fc6 / fc7 / fc8 (25088x4096, 4096x4096, 4096x1000),
B = 32 rows per GPU, bf16 factors in and on the wire, fp32 dW out; n = N replicas. One STEP =
the whole hot path for every layer: pack (when a cast is needed) -> NCCL all-gather of the
factors (n > 1) -> tensor-core reconstruction of dW with the fused 1/(nB) scale; the selector is
evaluated per layer (host, exact integers). Synthetic seeded data (paper_2302_06126_b200/synth.py).

metric "dW GB/s": dW bytes materialised by all replicas per second = n * sum_layers M*N*4 / t_step
(each replica reconstructs the identical gradient). Device-timed with CUDA events on
the launching stream, max over ranks; L2 flushed (256 MiB write) between timed steps, outside the
timed interval. Per-layer sync us, stage split, roofline of the reconstruction kernel, the e2e
number through the host-buffer C-ABI call, clocks and the CPU-oracle baseline are in the same line.
"""
import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2302_06126_b200 import dist as tdist  # noqa: E402
from paper_2302_06126_b200 import synth  # noqa: E402
import torch.distributed as dist  # noqa: E402

METRIC = "per-layer SFB grad-sync us & dW GB/s (VGG-19 fc6/fc7/fc8, B=32/GPU)"
ESIZE = {"f32": 4, "bf16": 2}
SPIN_CYCLES = 1_000_000   # ~0.5 ms torch.cuda._sleep before each start event (not a libtag kernel)


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return pk, "measured (MEASURED_PEAKS.json)"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback (B200_PROFILING.md)"


class ClockSampler:
    """`nvidia-smi -lms 50` clocks / throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.rows = []
        self._p = None

    def __enter__(self):
        try:
            self._p = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                        "--format=csv,noheader,nounits", "-lms", "50"],
                                       stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            time.sleep(0.3)      # let the first sample land before the timed region starts
        except OSError:
            self._p = None
        return self

    def __exit__(self, *a):
        if self._p is None:
            return
        time.sleep(0.06)
        self._p.terminate()
        try:
            out, _ = self._p.communicate(timeout=5)
        except subprocess.TimeoutExpired:
            self._p.kill()
            out, _ = self._p.communicate()
        self.rows = [[c.strip() for c in ln.split(",")] for ln in out.splitlines() if ln.strip()]

    def summary(self):
        def num(x):
            try:
                return float(x)
            except ValueError:
                return None
        rows = [r for r in self.rows if len(r) >= 9]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        sm = [v for v in (num(r[1]) for r in rows) if v is not None]
        mx = [v for v in (num(r[2]) for r in rows) if v is not None]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(rows)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_oracle_baseline(cfg, n, budget_mac=1.25e10, reps=3):
    """Time the fp64 CPU oracle (as it stands) on a bounded sample of the same workload, SURVEY
    d-5: both routes — the dense route (per-replica products summed in rank order) and
    the SFB route (rank-1 outer-product accumulation) — on the first M_s input-feature
    rows of every layer's dW, M_s scaled so each route is ~budget_mac MACs; median of `reps` runs
    per route; the reported value is the SFB route's dW GB/s (the dense route's beside it)."""
    import oracle
    oracle.build()
    cores = os.cpu_count()
    os.environ.setdefault("OMP_NUM_THREADS", str(cores))
    full_mac = sum(L.M * L.N * n * L.B for L in cfg.layers)
    frac = min(1.0, budget_mac / full_mac)
    samples, desc, out_bytes = [], [], 0
    for li, L in enumerate(cfg.layers):
        Ms = max(8, int(L.M * frac))
        X, dY = synth.all_factors(cfg.cid, li, n, L.M, L.N, L.B, L.x_dist, L.dy_dist)
        Xs = torch.from_numpy(np.ascontiguousarray(X[:, :, :Ms])).to(torch.bfloat16).double().numpy()
        dYe = torch.from_numpy(dY).to(torch.bfloat16).double().numpy()
        samples.append((Xs, dYe))
        out_bytes += Ms * L.N * ESIZE[cfg.out_dtype]
        desc.append(f"{L.name}:{Ms}/{L.M} rows")
    secs = {}
    for route, fn in (("sfb", oracle.sfb_dw), ("dense", oracle.dense_dw)):
        ts = []
        for _ in range(reps):
            t0 = time.perf_counter()
            for Xs, dYe in samples:
                fn(Xs, dYe)
            ts.append(time.perf_counter() - t0)
        secs[route] = statistics.median(ts)
    return {"value": out_bytes / secs["sfb"] / 1e9, "unit": "GB/s", "cores": cores, "kind": "oracle",
            "cpu_model": cpu_model(), "seconds": round(secs["sfb"], 3),
            "dense_route": {"value": out_bytes / secs["dense"] / 1e9, "unit": "GB/s",
                            "seconds": round(secs["dense"], 3)},
            "stat": f"median of {reps} per route",
            "sample": f"fp64 SFB and dense routes, n={n}, K={n * cfg.layers[0].B}, dW rows "
                      + ", ".join(desc)}


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU oracle (this tier's reference arm) on the same config/metric."""
    if rank != 0:
        return
    n = world
    vals, secs = [], []
    cb = None
    for i in range(args.warmup + args.steps):
        cb = cpu_oracle_baseline(cfg, n, budget_mac=args.ref_mac, reps=1)
        if i >= args.warmup:
            vals.append(cb["value"])
            secs.append(cb["seconds"])
    v = statistics.median(vals)
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "GB/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "higher_is_better": True,
            "ms_per_step": round(statistics.median(secs) * 1e3, 3), "scaling": "weak",
            "vs_baseline": None, "dtype": "f64",
            "data": "synthetic", "config": config_json(cfg, n, args),
            "cpu_baseline": dict(cb, value=v),
            "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "note": "CPU fp64 oracle on the host cores, one replica's dW per step (bounded sample)"}
    print(json.dumps(line), flush=True)


def virtual_n_recon(tag, comm, cfg, nv, stream, flush_l2, start_events, peaks, iters=20):
    """Reconstruction-only timing at K = nv*B on one GPU (nv virtual replicas' factors stacked
    rank-major), fp32 and bf16 dW, each layer alone; fractions of the tensor and HBM roofs."""
    out = {}
    for out_dt in ("f32", "bf16"):
        res = {}
        for li, L in enumerate(cfg.layers):
            K = nv * L.B
            X, dY = synth.all_factors(cfg.cid, li, nv, L.M, L.N, L.B, L.x_dist, L.dy_dist)
            plan = tag.SfbPlan(comm, L.M, L.N, K, "bf16", "bf16", out_dt)
            Xd = torch.from_numpy(X.reshape(K, L.M)).to(torch.bfloat16).cuda()
            dYd = torch.from_numpy(dY.reshape(K, L.N)).to(torch.bfloat16).cuda()
            dW = torch.empty(L.M, L.N, dtype=torch.float32 if out_dt == "f32" else torch.bfloat16,
                             device="cuda")
            plan.gather(Xd, dYd, stream)
            for _ in range(3):
                plan.reconstruct(dW, stream)
            ts = []
            for _ in range(iters):
                evs = start_events(2)
                plan.reconstruct(dW, stream)
                evs[1].record(stream)
                torch.cuda.synchronize()
                ts.append(evs[0].elapsed_time(evs[1]))
            t = statistics.median(ts) * 1e-3
            # the same launch replayed back to back from CUDA graphs (1 and 10 launches, L2 flushed
            # before each replay): the slope is the per-launch device time without the ~2.5 us
            # CUDA-event floor and the launch gap a single-launch interval carries
            # (scripts/event_floor.py); the 10 launches rewrite the same dW, factors stay in L2
            graphs = {}
            for reps in (1, 10):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=stream):
                    for _ in range(reps):
                        plan.reconstruct(dW, stream)
                graphs[reps] = g
            gts = {1: [], 10: []}
            for _ in range(iters):
                for reps in (1, 10):
                    evs = start_events(2)
                    with torch.cuda.stream(stream):
                        graphs[reps].replay()
                    evs[1].record(stream)
                    torch.cuda.synchronize()
                    gts[reps].append(evs[0].elapsed_time(evs[1]))
            t_b2b = (statistics.median(gts[10]) - statistics.median(gts[1])) / 9 * 1e-3
            flops = 2.0 * L.M * L.N * K
            byts = K * (L.M + L.N) * 2 + L.M * L.N * ESIZE[out_dt]
            res[L.name] = {"K": K, "us": round(t * 1e6, 2),
                           "tensor_frac": round(flops / t / 1e12 / peaks["bf16_tflops"], 4),
                           "hbm_frac": round(byts / t / 1e9 / peaks["hbm_gbs"], 4),
                           "ideal_tensor_us": round(flops / (peaks["bf16_tflops"] * 1e12) * 1e6, 2),
                           "ideal_hbm_us": round(byts / (peaks["hbm_gbs"] * 1e9) * 1e6, 2),
                           "us_per_launch_b2b": round(t_b2b * 1e6, 2),
                           "tensor_frac_b2b": round(flops / t_b2b / 1e12 / peaks["bf16_tflops"], 4)}
            plan.close()
        out[f"dW_{out_dt}"] = res
    return out


def projected_n8(tag, comm, cfg, stream, flush_l2, start_events, dw_bytes, iters=20):
    """SURVEY d-1b "n = 8 without 8 GPUs": the bucket's reconstruction timed at K = 8B on this GPU
    (virtual replicas, one grouped launch) plus the factor gather read off the measured n = 4
    curve (profiles/comm_n4.json) at the n = 8 ingress (7 * B(M+N) * 2 bytes). Labelled
    projected, never measured."""
    prof = os.path.join(ROOT, "profiles", "comm_n4.json")
    if not os.path.exists(prof) or cfg.sgd:
        return None
    curve = json.load(open(prof))["gather"]
    plans, Xs, dYs, dWs = [], [], [], []
    for li, L in enumerate(cfg.layers):
        K = 8 * L.B
        X, dY = synth.all_factors(cfg.cid, li, 8, L.M, L.N, L.B, L.x_dist, L.dy_dist)
        plans.append(tag.SfbPlan(comm, L.M, L.N, K, "bf16", "bf16", cfg.out_dtype))
        Xs.append(torch.from_numpy(X.reshape(K, L.M)).to(torch.bfloat16).cuda())
        dYs.append(torch.from_numpy(dY.reshape(K, L.N)).to(torch.bfloat16).cuda())
        dWs.append(torch.empty(L.M, L.N, dtype=torch.float32 if cfg.out_dtype == "f32" else torch.bfloat16,
                               device="cuda"))
    g = tag.SfbGroup(plans)
    g.gather(Xs, dYs, stream)
    for _ in range(3):
        g.reconstruct(dWs, stream)
    ts = []
    for _ in range(iters):
        evs = start_events(2)
        g.reconstruct(dWs, stream)
        evs[1].record(stream)
        torch.cuda.synchronize()
        ts.append(evs[0].elapsed_time(evs[1]))
    g.close()
    for p in plans:
        p.close()
    rec_us = statistics.median(ts) * 1e3
    ingress = sum(7 * L.B * (L.M + L.N) * 2 for L in cfg.layers)
    i = 0
    while i + 2 < len(curve) and ingress > curve[i + 1][0]:
        i += 1
    (b0, t0), (b1, t1) = curve[i], curve[i + 1]
    gather_us = (t0 + (ingress - b0) * (t1 - t0) / (b1 - b0)) / 1e3
    step_us = rec_us + gather_us
    return {"label": "projected n = 8 (not measured): virtual-n bucket reconstruction + gather "
                     "from the n = 4 curve", "K": 8 * cfg.layers[0].B,
            "recon_bucket_us": round(rec_us, 2), "gather_ingress_MB": round(ingress / 1e6, 2),
            "gather_us_from_n4_curve": round(gather_us, 2), "step_us": round(step_us, 2),
            "value_GBps": round(8 * dw_bytes / (step_us * 1e-6) / 1e9, 1)}


def config_json(cfg, n, args):
    return {"workload": f"{cfg.name} sync (configs[{cfg.cid - 1}]), n={n}",
            "layers": [f"{L.name} {L.M}x{L.N}" for L in cfg.layers], "rows_per_gpu": cfg.layers[0].B,
            "n": n, "in/wire/out": f"{cfg.in_dtype}/{cfg.wire_dtype}/{cfg.out_dtype}",
            "parallelism": f"dp{n} (SFB all-gather + replicated reconstruction)",
            "l2": "flushed between timed steps (256 MiB write + 256 MiB read), outside the timed interval",
            "nccl_algo": os.environ.get("NCCL_ALGO", "default")}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="tag", choices=["tag", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-dense", action="store_true")
    ap.add_argument("--ref-mac", type=float, default=2.5e10)
    ap.add_argument("--no-virtual", action="store_true")
    ap.add_argument("--nccl-algo", default=None,
                    help="set NCCL_ALGO (e.g. ring) for this run, before any communicator exists")
    ap.add_argument("--per-layer-step", action="store_true",
                    help="time the step as one tag_sfb_sync per layer instead of one bucket")
    args = ap.parse_args()
    assert args.warmup >= 3 or args.impl == "reference", "need >= 3 warm-up steps"

    if args.nccl_algo:
        os.environ["NCCL_ALGO"] = args.nccl_algo
    rank, local_rank, world = tdist.init_from_env()
    cfg = synth.CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return

    from paper_2302_06126_b200 import tag
    torch.cuda.set_device(local_rank)
    n = world
    comm = tdist.bootstrap_comm(tag, local_rank)
    stream = torch.cuda.Stream()
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16}
    layers = []
    for li, L in enumerate(cfg.layers):
        X, dY = synth.factors(cfg.cid, li, rank, L.M, L.N, L.B, L.x_dist, L.dy_dist)
        sgd = cfg.sgd or {}
        plan = tag.SfbPlan(comm, L.M, L.N, L.B, cfg.in_dtype, cfg.wire_dtype, cfg.out_dtype,
                           fuse_sgd=bool(sgd), **sgd)
        Xh = torch.from_numpy(X).to(tdt[cfg.in_dtype]).pin_memory()
        dYh = torch.from_numpy(dY).to(tdt[cfg.in_dtype]).pin_memory()
        ent = dict(L=L, plan=plan, X=Xh.cuda(), dY=dYh.cuda(), Xh=Xh, dYh=dYh,
                   dW=torch.empty(L.M, L.N, dtype=tdt[cfg.out_dtype], device="cuda"))
        if sgd:   # E2: fp32 master weights and momentum, updated in the epilogue (no dW write)
            W0, v0 = synth.sgd_state(cfg.cid, li, L.M, L.N)
            ent["W"], ent["v"] = torch.from_numpy(W0).cuda(), torch.from_numpy(v0).cuda()
        layers.append(ent)
    peaks, peak_src = load_peaks()
    sel_layers = [dict(M=l["L"].M, N=l["L"].N, B=l["L"].B, factor_dtype=cfg.wire_dtype,
                       grad_dtype=cfg.out_dtype) for l in layers]
    choices = tag.select(sel_layers, n, 900_000_000_000,
                         int(peaks.get("bf16_tflops_sustained", 1400) * 1e12))
    # profiled selector (paper's profiler P:331-334): curves measured by scripts/profile_comm.py
    choices_prof = None
    profiled_compute = None
    prof_path = os.path.join(ROOT, "profiles", f"comm_n{n}.json")
    if n > 1 and os.path.exists(prof_path):
        prof = json.load(open(prof_path))
        # measured op times (scripts/profile_compute.py, the paper's op profiler P:323-329)
        # replace the linear compute model when this config and n were profiled
        rec = loc = None
        cp = os.path.join(ROOT, "profiles", "compute_profile.json")
        if os.path.exists(cp):
            ct = json.load(open(cp)).get(str(args.config), {})
            if all(str(n) in ct.get(l["L"].name, {}) for l in layers):
                rec = [ct[l["L"].name][str(n)]["recon_ns"] for l in layers]
                loc = [ct[l["L"].name][str(n)]["local_ns"] for l in layers]
        choices_prof = tag.select_profiled(sel_layers, n, prof["gather"], prof["allreduce"],
                                           int(peaks.get("bf16_tflops_sustained", 1400) * 1e12),
                                           prof.get("ps"), recon_ns=rec, local_ns=loc)
        profiled_compute = "measured op times (profiles/compute_profile.json)" if rec else \
            "linear model 2MNB/F"
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    flush_rd = torch.ones(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")

    def flush_l2():
        # write 256 MiB (> 126 MB L2), then read another 256 MiB so the dirty lines of the write
        # are drained to HBM before the timed interval starts (outside the events)
        flush.zero_()
        flush_rd.sum()
    nl = len(layers)

    sync_tok = torch.zeros(1, device="cuda")
    Xs, dYs, dWs = [l["X"] for l in layers], [l["dY"] for l in layers], [l["dW"] for l in layers]
    # the step is one bucket: one push kernel (n > 1) + one persistent reconstruction launch
    group = None if args.per_layer_step else tag.SfbGroup([l["plan"] for l in layers])

    def step():
        with torch.cuda.stream(stream):
            if group is not None and cfg.sgd:
                # E2: the optimizer step is fused into the same single launch, dW never stored
                group.sync_sgd(Xs, dYs, [l["W"] for l in layers], [l["v"] for l in layers], None,
                               stream)
            elif group is not None:
                # one call: at n > 1 a single fused kernel pushes the factors over NVLink and
                # reconstructs every layer (tag_sfb_group_sync); at n = 1 the reconstruction only
                group.sync(Xs, dYs, dWs, stream)
            else:
                for l in layers:
                    if cfg.sgd:
                        l["plan"].sync_sgd(l["X"], l["dY"], l["W"], l["v"], None, stream)
                    else:
                        l["plan"].sync(l["X"], l["dY"], l["dW"], stream)

    def start_events(k):
        flush_l2()
        torch.cuda.synchronize()
        tdist.barrier()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(k)]
        with torch.cuda.stream(stream):
            # a ~0.5 ms device spin ahead of the start event lets the host enqueue the whole step,
            # so the interval measures device time, not Python launch latency
            torch.cuda._sleep(SPIN_CYCLES)
            if n > 1:
                # device-side barrier of all ranks on this stream (libtag's LSA barrier kernel),
                # ordered before the start event, so inter-process launch skew is not timed
                comm.barrier(stream)
        evs[0].record(stream)
        return evs

    def timed_steps(nsteps):
        """Whole steps, [start, end] per step."""
        step_ms = []
        for _ in range(nsteps):
            evs = start_events(2)
            step()
            evs[1].record(stream)
            torch.cuda.synchronize()
            step_ms.append(evs[0].elapsed_time(evs[1]))
        return step_ms

    def timed_staged(nsteps):
        """The bucket split in two calls: gather (push kernel + LSA barrier) | reconstruct."""
        g_ms, r_ms = [], []
        for _ in range(nsteps):
            evs = start_events(3)
            with torch.cuda.stream(stream):
                group.gather(Xs, dYs, stream)
                evs[1].record(stream)
                group.reconstruct(dWs, stream)
                evs[2].record(stream)
            torch.cuda.synchronize()
            g_ms.append(evs[0].elapsed_time(evs[1]))
            r_ms.append(evs[1].elapsed_time(evs[2]))
        return g_ms, r_ms

    def timed_layers(nsteps):
        """Per-layer staged pass: gather | reconstruct of each layer on its own."""
        rec, syn = [[] for _ in range(nl)], [[] for _ in range(nl)]
        for _ in range(nsteps):
            evs = start_events(2 * nl + 1)
            with torch.cuda.stream(stream):
                for i, l in enumerate(layers):
                    if cfg.sgd:           # no stage split with the fused optimizer: whole sync
                        evs[2 * i + 1].record(stream)
                        l["plan"].sync_sgd(l["X"], l["dY"], l["W"], l["v"], None, stream)
                    else:
                        l["plan"].gather(l["X"], l["dY"], stream)
                        evs[2 * i + 1].record(stream)
                        l["plan"].reconstruct(l["dW"], stream)
                    evs[2 * i + 2].record(stream)
            torch.cuda.synchronize()
            for i in range(nl):
                rec[i].append(evs[2 * i + 1].elapsed_time(evs[2 * i + 2]))
                syn[i].append(evs[2 * i].elapsed_time(evs[2 * i + 2]))
        return rec, syn

    # ---------------------------------------------------------------- warm-up + timed region
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    tdist.barrier()
    launches0 = tag.kernel_launches()
    with ClockSampler(local_rank) as clk:
        steps_ms = timed_steps(args.steps)
    # libtag kernels inside the timed intervals: the per-step pre-start barrier kernel (n > 1) is
    # launched before each start event, so it is counted by the library but not timed
    launches = tag.kernel_launches() - launches0 - (args.steps if n > 1 else 0)
    torch.cuda.synchronize()
    tdist.barrier()
    nstaged = max(5, min(args.steps, 30))
    layer_recon_ms, layer_sync_ms = timed_layers(nstaged)
    staged_g_ms, staged_r_ms = (timed_staged(nstaged) if group is not None and not cfg.sgd
                                else ([], []))

    t_step_ms = tdist.max_over_ranks(statistics.mean(steps_ms))
    qs = statistics.quantiles(steps_ms, n=10) if len(steps_ms) >= 2 else [steps_ms[0]] * 9
    step_stats = {"p10_ms": round(tdist.max_over_ranks(qs[0]), 4),
                  "p50_ms": round(tdist.max_over_ranks(statistics.median(steps_ms)), 4),
                  "p90_ms": round(tdist.max_over_ranks(qs[8]), 4),
                  "mean_ms": round(t_step_ms, 4), "steps": len(steps_ms)}
    dw_bytes = sum(l["L"].M * l["L"].N * ESIZE[cfg.out_dtype] for l in layers)
    value = n * dw_bytes / (t_step_ms * 1e-3) / 1e9

    # roofline of the dominant kernel. Bucket mode: the step is ONE launch of recon_tc_kernel
    # (with the NVLink push fused in at n > 1), so its duration is the step's.
    # E2 reads and writes W and v (16 B per element) and stores no dW
    alg_bytes = sum(n * l["L"].B * (l["L"].M + l["L"].N) * ESIZE[cfg.wire_dtype]
                    + l["L"].M * l["L"].N * (16 if cfg.sgd else ESIZE[cfg.out_dtype])
                    for l in layers)
    if group is not None:
        kernel_ms = t_step_ms
        launches_per_step = 1
        recon_only_ms = (tdist.max_over_ranks(statistics.mean(staged_r_ms)) if staged_r_ms
                         else kernel_ms)
    else:
        kernel_ms = tdist.max_over_ranks(sum(statistics.mean(r) for r in layer_recon_ms))
        launches_per_step = nl
        recon_only_ms = kernel_ms
    achieved = alg_bytes / (kernel_ms * 1e-3) / 1e9
    traffic = None
    tp = os.path.join(ROOT, "profiles", "recon_traffic.json")
    if os.path.exists(tp):
        try:
            traffic = json.load(open(tp)).get(f"config{args.config}_n{n}")
        except Exception:
            traffic = None
    roofline = {"kernel": ("recon_tc_kernel<FUSED> (NVLink push + tcgen05 reconstruction, one launch "
                           "per bucket)" if (group is not None and n > 1) else
                           "recon_tc_kernel (grouped tcgen05 reconstruction, fused 1/(nB) epilogue)"),
                "bound": "hbm", "achieved": round(achieved, 1), "peak": peaks["hbm_gbs"],
                "unit": "GB/s", "frac": round(achieved / peaks["hbm_gbs"], 4),
                "traffic": traffic, "peak_source": peak_src,
                "algorithmic_bytes_per_step": alg_bytes, "launches_per_step": launches_per_step,
                "kernel_us": round(kernel_ms * 1e3, 2),
                "share_of_step": round(kernel_ms / t_step_ms, 3),
                "recon_only_us": round(recon_only_ms * 1e3, 2),
                "recon_only_hbm_frac": round(alg_bytes / (recon_only_ms * 1e-3) / 1e9 / peaks["hbm_gbs"], 4)}

    per_layer = {}
    for i, l in enumerate(layers):
        L = l["L"]
        t_sync = tdist.max_over_ranks(statistics.median(layer_sync_ms[i]))
        t_rec = tdist.max_over_ranks(statistics.median(layer_recon_ms[i]))
        flops = 2.0 * L.M * L.N * n * L.B
        rbytes = n * L.B * (L.M + L.N) * ESIZE[cfg.wire_dtype] + L.M * L.N * ESIZE[cfg.out_dtype]
        ag = (n - 1) * L.B * (L.M + L.N) * ESIZE[cfg.wire_dtype]
        per_layer[L.name] = {
            "sync_us": round(t_sync * 1e3, 2), "recon_us": round(t_rec * 1e3, 2),
            # staged gather stage (a1 + a2; n = 1: no exchange, only the event gap)
            ("gather_us" if n > 1 else "stage_gap_us"): round((t_sync - t_rec) * 1e3, 2),
            "dW_GBps": round(L.M * L.N * ESIZE[cfg.out_dtype] / (t_sync * 1e-3) / 1e9, 1),
            "recon_hbm_frac": round(rbytes / (t_rec * 1e-3) / 1e9 / peaks["hbm_gbs"], 4),
            "recon_tensor_frac": round(flops / (t_rec * 1e-3) / 1e12 / peaks["bf16_tflops"], 4),
            "allgather_busbw_GBps": round(ag / ((t_sync - t_rec) * 1e-3) / 1e9, 1) if n > 1 else None,
            "selector": {0: "allreduce", 1: "sfb", 2: "none"}[choices[i]],
            "selector_profiled": ({0: "allreduce", 1: "sfb", 2: "none", 3: "ps"}[choices_prof[i]]
                                  if choices_prof else None),
            "gather": l["plan"].info()["gather"] + ("+multicast" if l["plan"].info()["multicast"] else "")}
    if group is not None and n > 1 and staged_g_ms:
        t_gather = tdist.max_over_ranks(statistics.mean(staged_g_ms))
        ag_all = sum((n - 1) * l["L"].B * (l["L"].M + l["L"].N) * ESIZE[cfg.wire_dtype] for l in layers)
        per_layer["bucket_gather_staged"] = {"us": round(t_gather * 1e3, 2),
                                      "ingress_MB": round(ag_all / 1e6, 3),
                                      "busbw_GBps": round(ag_all / (t_gather * 1e-3) / 1e9, 1),
                                      "frac_of_900": round(ag_all / (t_gather * 1e-3) / 900e9, 4)}

    # ---------------------------------------------------------------- dense baseline (n > 1)
    # SURVEY d-1b: from (X_r, dY_r) to the synchronised result on every rank. Dense = local GEMM
    # (K = B) + ncclAllReduce with PreMulSum(1/(nB)) (+ the unfused SGD step for E2 configs, whose
    # SFB side fuses it). The AllReduce alone is timed too and reported as nccl-tests bus
    # bandwidth 2(n-1)/n * M*N*e_g / t against 900 GB/s and as a fraction of the ring ideal
    # 2(n-1)/n * G / 900 GB/s. NCCL picks its algorithm unless the run sets
    # NCCL_ALGO (bench --nccl-algo ring), which `nccl_algo` in the config records.
    if n > 1 and not args.no_dense:
        reps = max(3, min(args.steps, 10))

        def timed(fn):
            t = []
            for _ in range(reps):
                e0, e1 = start_events(2)
                with torch.cuda.stream(stream):
                    fn()
                e1.record(stream)
                torch.cuda.synchronize()
                t.append(e0.elapsed_time(e1))
            return tdist.max_over_ranks(statistics.median(t))
        for i, l in enumerate(layers):
            L, plan = l["L"], l["plan"]

            def dense():
                plan.local_grad(l["X"], l["dY"], l["dW"], stream)
                plan.dense_allreduce(l["dW"], stream)
                if cfg.sgd:
                    plan.sgd_step(l["dW"], l["W"], l["v"], stream)
            td = timed(dense)
            ta = timed(lambda: plan.dense_allreduce(l["dW"], stream))
            # Replicate-with-PS: the same local gradient, reduced to a round-robin PS
            # (root = layer index mod n) and broadcast back
            tp = timed(lambda: (plan.local_grad(l["X"], l["dY"], l["dW"], stream),
                                plan.ps_sync(l["dW"], i % n, stream)))
            G = L.M * L.N * ESIZE[cfg.out_dtype]
            ring_ideal_us = 2 * (n - 1) / n * G / 900e9 * 1e6
            pl = per_layer[L.name]
            pl["dense_us"] = round(td * 1e3, 2)
            pl["dense_includes_sgd_step"] = bool(cfg.sgd)
            pl["allreduce_us"] = round(ta * 1e3, 2)
            pl["allreduce_busbw_GBps"] = round(2 * (n - 1) / n * G / (ta * 1e-3) / 1e9, 1)
            pl["allreduce_frac_of_900"] = round(2 * (n - 1) / n * G / (ta * 1e-3) / 900e9, 4)
            pl["allreduce_frac_of_ring_ideal"] = round(ring_ideal_us / (ta * 1e3), 4)
            pl["ps_us"] = round(tp * 1e3, 2)
            pl["sfb_speedup_vs_dense"] = round(td / (pl["sync_us"] / 1e3), 2)
            pl["measured_winner"] = min([(pl["sync_us"], "sfb"), (td * 1e3, "allreduce"),
                                         (tp * 1e3, "ps")])[1]
            pl["selector_agrees"] = pl["selector"] == pl["measured_winner"]
            pl["selector_profiled_agrees"] = (pl["selector_profiled"] == pl["measured_winner"]
                                              if pl["selector_profiled"] else None)

    # ---------------------------------------------------------------- sharded variant (n > 1)
    # every rank still receives all factors but reconstructs only its
    # 1/n row-shard of each dW (ZeRO-style consumers); not the paper's replicated semantics, so
    # reported beside the headline, never as `value`.
    sharded = None
    if n > 1 and not cfg.sgd:
        shards = []
        for l in layers:
            rb, rc = l["plan"].shard_rows()
            shards.append(torch.empty(max(rc, 1), l["L"].N, dtype=tdt[cfg.out_dtype],
                                      device="cuda")[:rc])
        def sharded_step():
            with torch.cuda.stream(stream):
                if group is not None:        # one fused launch for the bucket's shards
                    group.sync_sharded(Xs, dYs, shards, stream)
                else:
                    for l, sh in zip(layers, shards):
                        l["plan"].sync_sharded(l["X"], l["dY"], sh, stream)
        for _ in range(3):
            sharded_step()
        ts = []
        for _ in range(max(5, min(args.steps, 20))):
            e0, e1 = start_events(2)
            sharded_step()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t_sh = tdist.max_over_ranks(statistics.mean(ts))
        sharded = {"ms_per_step": round(t_sh, 4),
                   "dW_GBps_all_ranks": round(dw_bytes / (t_sh * 1e-3) / 1e9, 1),
                   "note": "each rank reconstructs M/n rows of every layer (tag_sfb_group_sync_sharded)"}

    # f-2 for the fused-optimizer configs: the sharded SGD step (each rank updates its rows of W
    # and its momentum shard in the fused launch) + the W all-gather, per layer in sequence,
    # against the replicated fused SGD of the same layers (the headline step)
    if n > 1 and cfg.sgd:
        vsh = []
        for l in layers:
            rb, rc = l["plan"].shard_rows()
            vsh.append(torch.zeros(max(rc, 1), l["L"].N, device="cuda")[:rc])

        def sharded_sgd_step():
            with torch.cuda.stream(stream):
                for l, v in zip(layers, vsh):
                    l["plan"].sync_sharded_sgd(l["X"], l["dY"], l["W"], v, stream)
        for _ in range(3):
            sharded_sgd_step()
        ts = []
        for _ in range(max(5, min(args.steps, 20))):
            e0, e1 = start_events(2)
            sharded_sgd_step()
            e1.record(stream)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        t_sh = tdist.max_over_ranks(statistics.mean(ts))
        sharded = {"ms_per_step": round(t_sh, 4),
                   "replicated_fused_sgd_ms": round(t_step_ms, 4),
                   "note": "tag_sfb_sync_sharded_sgd per layer: sharded SGD-momentum in the fused "
                           "launch + W all-gather (momentum memory / n)"}

    # ---------------------------------------------------------------- e2e through host buffers
    dWh = [torch.empty(l["L"].M, l["L"].N, dtype=tdt[cfg.out_dtype]).pin_memory() for l in layers]
    h2d = sum(l["Xh"].numel() * l["Xh"].element_size() + l["dYh"].numel() * l["dYh"].element_size()
              for l in layers)
    d2h = sum(t.numel() * t.element_size() for t in dWh)
    for _ in range(2):
        with torch.cuda.stream(stream):
            for l, h in zip(layers, dWh):
                l["plan"].sync_host(l["Xh"], l["dYh"], h, stream)
    torch.cuda.synchronize()
    e2e_ms = []
    for _ in range(max(3, min(args.steps, 10))):
        torch.cuda.synchronize()
        tdist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        with torch.cuda.stream(stream):
            for l, h in zip(layers, dWh):
                l["plan"].sync_host(l["Xh"], l["dYh"], h, stream)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    t_e2e = tdist.max_over_ranks(statistics.mean(e2e_ms))
    e2e = {"value": round(n * dw_bytes / (t_e2e * 1e-3) / 1e9, 2), "unit": "GB/s",
           "ms_per_step": round(t_e2e, 4), "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
           "api": "tag_sfb_sync_host (pinned host X, dY in; full dW out)"}

    # ---------------------------------------------------------------- virtual n = 8 (1 GPU)
    # north_star's target point is fc6 at n = 8 (K = 256); with one GPU the reconstruction of that
    # point is timed on K = 8*32 stacked factor rows (identical contraction and alpha = 1/(8B))
    virt = proj8 = None
    if n == 1 and not args.no_virtual:
        virt = virtual_n_recon(tag, comm, cfg, 8, stream, flush_l2, start_events, peaks)
        proj8 = projected_n8(tag, comm, cfg, stream, flush_l2, start_events, dw_bytes)

    clocks = clk.summary()
    cpu = None
    if rank == 0 and n == 1 and not args.no_cpu_baseline:
        cpu = cpu_oracle_baseline(cfg, n)

    if rank == 0:
        line = {"metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world,
                "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step_ms, 4),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": cfg.wire_dtype, "data": "synthetic", "config": config_json(cfg, n, args),
                "per_layer": per_layer, "roofline": roofline, "e2e": e2e,
                "gpu_launches": launches, "clocks": clocks, "cpu_baseline": cpu,
                "virtual_n8_recon": virt, "projected_n8": proj8, "step_stats": step_stats,
                "sharded_variant": sharded, "selector_profiled_compute": profiled_compute,
                "lib": tag.version()}
        print(json.dumps(line), flush=True)
    if group is not None:
        group.close()
    for l in layers:
        l["plan"].close()
    comm.close()
    if tdist.env_ranks()[2] > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
