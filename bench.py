#!/usr/bin/env python
"""Benchmark of the B200 randomized-HALS path (rnmf::rhals_fit drop-in) — driver contract.

One *step* = one complete rhals_fit (sketch + sweeps + trace) on the workload.  `value` is HALS
sweeps/s of whole fits with X resident in HBM (X larger than L2, so no flush is needed); `e2e`
is the same metric through the public API with X in pinned host memory (H2D of X and D2H of
W, H and the trace inside every step).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--impl reference]

N > 1 (torchrun, one process per GPU): ONE fit of the config with X sharded by rows over the N
GPUs (paper_1711_02037_b200.distributed; strong scaling); `value` = sweeps/s of that fit, device
time max over ranks.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_1711_02037_b200 import workloads  # noqa: E402

METRIC = "rHALS end-to-end s and HALS iters/s at 1/2/4/8 B200; sketch/QᵀX HBM GB/s vs peak"


def load_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), float(d.get("bf16_tflops", 1681.0)), "measured"
    except Exception:
        return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self) -> dict:
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=2)
        except Exception:
            self.proc.kill()
        sms, maxs, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sms.append(float(parts[0]))
                maxs.append(float(parts[1]))
            except ValueError:
                continue
            for nm, v in zip(names, parts[2:6]):
                if v.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": float(np.median(sms)) if sms else None, "sm_max_mhz": max(maxs) if maxs else None,
                "reasons": sorted(reasons), "samples": len(sms)}


def load_traffic(cfg_name: str):
    """DRAM bytes per launch of the X-streaming kernels from the committed ncu --set full summary
    (profiles/latest_traffic.json, written by tools/ncu_summary.py); None if absent."""
    p = os.path.join(ROOT, "profiles", "latest_traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        return d.get(cfg_name)
    except Exception:
        return None


def make_workload(cfg_name: str, device):
    """X (device, fp32/fp64), injected Omega / unscaled init draws, solver options."""
    import torch

    from paper_1711_02037_b200 import api

    cfg = workloads.CONFIGS[cfg_name]
    if cfg_name == "C1":
        x = workloads.c1_matrix(0)
    elif cfg_name == "C2":
        x = workloads.faces_matrix(0)
    elif cfg_name == "C3":
        x = workloads.unmixing_matrix(0)
    elif cfg_name == "C4":
        x = None
    else:
        raise SystemExit(f"config {cfg_name} is multi-GPU only (200 GB); not runnable in this build")
    if x is None:
        xd = workloads.noisy_lowrank_device(0, cfg.m, cfg.n, 40, 0.5, 0.1, device=device)
    else:
        xd = torch.from_numpy(x).to(device)
    l = min(cfg.k + cfg.p, cfg.m, cfg.n)
    omega, w0, h0 = workloads.injected_inputs(0, cfg.m, cfg.n, cfg.k, l)
    opts = api.SolverOptions(rank=cfg.k, oversampling=cfg.p, power_iterations=cfg.q, max_iter=cfg.iters,
                             tol=1e-300, seed=0)
    return cfg, xd, omega, w0, h0, opts


def cpu_baseline(cfg_name: str, x_host: np.ndarray, cfg, omega, w0, h0, threads: int = 1):
    """Oracle (fp64 C++ restatement of the reference) on the box's host cores: sketch + 10 sweeps
    measured (trace_full_every = 10 makes that exactly one sweep/metrics period), extrapolated to
    the config's full sweep count: t(0) + (iters/10) * (t(10) - t(0))."""
    from oracle import oracle as orc

    orc.set_threads(threads)
    x64 = np.ascontiguousarray(x_host, dtype=np.float64)
    base = dict(rank=cfg.k, tol=1e-300, oversampling=cfg.p, power_iterations=cfg.q, seed=0, trace_full_every=10)
    t = time.perf_counter()
    orc.rhals_fit(x64, dict(base, max_iter=0), omega=omega, w0=w0, h0=h0)
    t0 = time.perf_counter() - t
    t = time.perf_counter()
    orc.rhals_fit(x64, dict(base, max_iter=10), omega=omega, w0=w0, h0=h0)
    t10 = time.perf_counter() - t
    est = t0 + (cfg.iters / 10.0) * max(t10 - t0, 0.0)
    return {
        "value": cfg.iters / est,
        "unit": "iters/s",
        "cores": threads,
        "kind": "port",
        "sample": f"{cfg_name} full matrix, fp64 oracle: rhals_fit with 0 and 10 sweeps measured "
                  f"({t0:.2f}s, {t10:.2f}s), extrapolated to {cfg.iters} sweeps = {est:.2f}s",
        "est_fit_s": est,
    }


def run_reference(args):
    """--impl reference: the reference algorithm's CPU implementation (the oracle port; the
    reference itself cannot be compiled here, no Eigen) on all host threads."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = workloads.CONFIGS[args.config]
    if args.config == "C1":
        x = workloads.c1_matrix(0)
    elif args.config == "C2":
        x = workloads.faces_matrix(0)
    elif args.config == "C3":
        x = workloads.unmixing_matrix(0)
    else:
        print(json.dumps({"impl": "reference", "unavailable": f"{args.config} does not fit host-side fp64 oracle"}))
        return
    l = min(cfg.k + cfg.p, cfg.m, cfg.n)
    omega, w0, h0 = workloads.injected_inputs(0, cfg.m, cfg.n, cfg.k, l)
    threads = os.cpu_count() or 1
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_baseline(args.config, x, cfg, omega, w0, h0, threads=threads)
        if i >= args.warmup:
            vals.append(r)
        if i + 1 >= args.warmup and len(vals) >= args.steps:
            break
    v = float(np.mean([r["value"] for r in vals]))
    est = float(np.mean([r["est_fit_s"] for r in vals]))
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "iters/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": est * 1e3, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "m": cfg.m, "n": cfg.n, "k": cfg.k, "p": cfg.p, "q": cfg.q,
                   "iters": cfg.iters},
        "cpu_baseline": {"value": v, "unit": "iters/s", "cores": threads, "kind": "port",
                         "sample": vals[0]["sample"] if vals else ""},
        "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # tf32x3: the X-streaming sketch GEMMs on tcgen05 tensor cores (3xTF32 split, chunked TMEM
    # accumulation promoted to fp32) -- measured more accurate than the FFMA kernels against the
    # fp64 oracle (tests/test_gpu_tf32x3.py, profiles/r01/mode_parity_c2.json); "exact" = FFMA
    ap.add_argument("--math", default="tf32x3", choices=["exact", "tf32x3", "tf32"])
    ap.add_argument("--sharded", action="store_true", help="row-sharded path even at N = 1 (testing)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "b200" else args.warmup
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    from paper_1711_02037_b200 import api

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=device)

    cfg, xd, omega, w0, h0, opts = make_workload(args.config, device)
    opts.math_mode = {"exact": api.MathMode.Exact, "tf32x3": api.MathMode.TF32x3, "tf32": api.MathMode.TF32}[args.math]
    esz = xd.element_size()
    m_total = cfg.m
    if world > 1 or args.sharded:
        from paper_1711_02037_b200 import distributed as pdist

        ctx = (pdist.ShardedContext(local) if world > 1 else
               pdist.ShardedContext(local, rank=0, world=1, comm_id=pdist.comm_unique_id()))
        off, cnt = pdist.shard_rows(m_total, world, rank)
        xd = xd[off:off + cnt].contiguous()
        w0 = np.ascontiguousarray(w0[off:off + cnt])

        def fit(x):
            return pdist.rhals_fit_sharded(x, opts, row_offset=off, m_total=m_total, ctx=ctx, omega=omega, w0=w0,
                                           h0=h0)
    else:
        ctx = api.Context(local)

        def fit(x):
            return api.rhals_fit(x, opts, omega=omega, w0=w0, h0=h0, ctx=ctx)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- device-resident X: `value`
    for _ in range(args.warmup):
        fit(xd)
    # X per GPU below 2x the 126 MB L2 (sharded / small configs): flush L2 between steps so no
    # step starts with X cached by the previous one (the library's device time excludes the flush)
    x_bytes_local = xd.numel() * esz
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=device) if x_bytes_local < 252e6 else None
    sampler = ClockSampler(local)
    barrier()
    sampler.start()
    t_wall = time.perf_counter()
    dev_ms, launches, stages = [], 0, []
    last = None
    for _ in range(args.steps):
        if flush is not None:
            flush.zero_()
        last = fit(xd)
        st = ctx.stage_times()
        dev_ms.append(st["total_ms"])
        launches += int(st["kernel_launches"])
        stages.append(st)
    barrier()
    wall_s = time.perf_counter() - t_wall
    clocks = sampler.stop()
    total_ms = float(np.sum(dev_ms))
    if world > 1:
        t = torch.tensor([total_ms], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        total_ms = float(t.item())
    ms_per_step = total_ms / args.steps
    sweeps = last.trace[-1].iter
    value = sweeps * args.steps / (total_ms / 1e3)  # one fit over all N GPUs

    # ---- e2e through the public API with host X (pinned)
    x_pin = torch.empty(xd.shape, dtype=xd.dtype, pin_memory=True)
    x_pin.copy_(xd)
    x_np = x_pin.numpy()
    for _ in range(1):
        fit(x_np)
    barrier()
    e2e_ms = []
    for _ in range(args.steps):
        ev0 = torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        res = fit(x_np)
        e2e_ms.append((time.perf_counter() - t0) * 1e3)
        _ = res.trace[-1].rel_err  # the step's result is on the host
    barrier()
    e2e_total = float(np.sum(e2e_ms))
    if world > 1:
        t = torch.tensor([e2e_total], device=device, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_total = float(t.item())
    e2e_value = sweeps * args.steps / (e2e_total / 1e3)
    m, n, k = xd.shape[0], cfg.n, cfg.k
    l = min(cfg.k + cfg.p, m, n)
    # whole job: every rank copies its X rows and W0 rows, Omega / H0 replicated; W rows + H back
    h2d = cfg.m * n * esz + 8 * cfg.m * k + world * 8 * (n * l + k * n)
    d2h = esz * (cfg.m * k + world * k * n) + world * 56 * (sweeps + 1)

    # the other sketch arithmetic (FFMA when the timed run used the tensor cores, and vice versa):
    # the same X passes once more for a second sketch roofline, outside the timed region
    alt_sketch = None
    if esz == 4 and world == 1 and args.math in ("exact", "tf32x3"):
        alt = "exact" if args.math == "tf32x3" else "tf32x3"
        opts.math_mode = api.MathMode.Exact if alt == "exact" else api.MathMode.TF32x3
        for _ in range(2):
            fit(xd)
        tst = ctx.stage_times()
        opts.math_mode = api.MathMode.TF32x3 if args.math == "tf32x3" else api.MathMode.Exact
        tb = tst["xw_bytes"] + tst["xtw_bytes"]
        tms = tst["xw_kernel_ms"] + tst["xtw_kernel_ms"]
        alt_sketch = {"math_mode": alt, "sketch_gbs": tb / (tms / 1e3) / 1e9 if tms > 0 else None,
                      "xw_gbs": tst["xw_bytes"] / (tst["xw_kernel_ms"] / 1e3) / 1e9 if tst["xw_kernel_ms"] > 0 else None,
                      "xtw_gbs": tst["xtw_bytes"] / (tst["xtw_kernel_ms"] / 1e3) / 1e9 if tst["xtw_kernel_ms"] > 0 else None,
                      "fit_ms": tst["total_ms"]}

    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return

    # ---- roofline of the X-streaming kernels and stage shares
    hbm_peak, _, peak_kind = load_peaks()
    agg = {key: float(np.mean([s[key] for s in stages])) for key in stages[0]}
    # roofline of the sketch GEMM kernels: algorithmic X bytes per launch / the kernels' own
    # device time (CUDA events on the library stream around the kernel launches alone);
    # the *_span_gbs figures include operand preparation and the split-K reduction
    xw_gbs = agg["xw_bytes"] / (agg["xw_kernel_ms"] / 1e3) / 1e9 if agg["xw_kernel_ms"] > 0 else 0.0
    xtw_gbs = agg["xtw_bytes"] / (agg["xtw_kernel_ms"] / 1e3) / 1e9 if agg["xtw_kernel_ms"] > 0 else 0.0
    sk_bytes = agg["xw_bytes"] + agg["xtw_bytes"]
    sk_ms = agg["xw_kernel_ms"] + agg["xtw_kernel_ms"]
    sk_gbs = sk_bytes / (sk_ms / 1e3) / 1e9 if sk_ms > 0 else 0.0
    sk_span_ms = agg["xw_ms"] + agg["xtw_ms"]
    sk_span_gbs = sk_bytes / (sk_span_ms / 1e3) / 1e9 if sk_span_ms > 0 else 0.0
    met_gbs = agg["metrics_bytes"] / (agg["metrics_ms"] / 1e3) / 1e9 if agg["metrics_ms"] > 0 else 0.0
    traffic = load_traffic(args.config)
    shares = {name: agg[name] / agg["total_ms"] for name in
              ("scan_ms", "sketch_ms", "qr_ms", "init_ms", "sweeps_ms", "metrics_ms", "h2d_ms", "d2h_ms")}
    line = {
        "metric": METRIC,
        "value": value,
        "unit": "iters/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": ms_per_step,
        "higher_is_better": True,
        "scaling": "strong",
        "vs_baseline": None,
        "dtype": "f32" if esz == 4 else "f64",
        "data": "synthetic (seeded stand-in for the paper's dataset; see paper_1711_02037_b200/workloads.py)",
        "config": {"workload": cfg.name, "m": cfg.m, "n": n, "k": k, "p": cfg.p, "q": cfg.q, "iters": cfg.iters,
                   "tol": 1e-300, "math_mode": args.math,
                   "parallelism": f"rows{world}" if world > 1 else "single-gpu",
                   "l2": (f"X per GPU = {m * n * esz / 1e6:.0f} MB > 126 MB L2 (no flush needed)" if flush is None
                          else f"X per GPU = {m * n * esz / 1e6:.0f} MB: L2 flushed (256 MB write) between steps")},
        "end_to_end_s": ms_per_step / 1e3,
        "e2e": {"value": e2e_value, "unit": "iters/s", "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
                "ms_per_step": e2e_total / args.steps},
        "gpu_launches": launches,
        "roofline": {"bound": "hbm",
                     "kernel": ("X-streaming sketch GEMMs " + ("(tc_xw_kernel Y=X*S, tc_xtw_kernel X^T*Q; tcgen05 3xTF32)"
                                if args.math != "exact" else "(xw_tma_kernel Y=X*S, xtw_tma_kernel X^T*Q; FFMA)")),
                     "achieved": sk_gbs, "peak": hbm_peak, "unit": "GB/s", "frac": sk_gbs / hbm_peak,
                     "peak_kind": peak_kind,
                     "traffic": traffic.get("sketch_bytes_per_launch") if traffic else None,
                     "traffic_source": traffic.get("source") if traffic else None,
                     "per_kernel": {"xw_gbs": xw_gbs, "xtw_gbs": xtw_gbs, "sketch_span_gbs": sk_span_gbs,
                                    "xw_kernel_us": 1e3 * agg["xw_kernel_ms"] / max(agg["xw_launches"], 1),
                                    "xtw_kernel_us": 1e3 * agg["xtw_kernel_ms"] / max(agg["xtw_launches"], 1),
                                    "xw_bytes_per_launch": agg["xw_bytes"] / max(agg["xw_launches"], 1),
                                    "xtw_bytes_per_launch": agg["xtw_bytes"] / max(agg["xtw_launches"], 1),
                                    "metrics_pass_gbs": met_gbs,
                                    "metrics_bytes_per_eval": agg["metrics_bytes"] / max(agg["metrics_passes"], 1),
                                    "ncu_dram_bytes_per_launch": traffic.get("kernels") if traffic else None}},
        "roofline_other_sketch_math": (dict(alt_sketch, frac=alt_sketch["sketch_gbs"] / hbm_peak, peak=hbm_peak)
                                       if alt_sketch and alt_sketch["sketch_gbs"] else None),
        "stage_ms": {key: agg[key] for key in ("scan_ms", "sketch_ms", "qr_ms", "init_ms", "sweeps_ms", "metrics_ms",
                                               "xw_ms", "xtw_ms", "xw_kernel_ms", "xtw_kernel_ms", "h2d_ms", "d2h_ms",
                                               "total_ms")},
        "stage_share": shares,
        "sweep_us": 1e3 * agg["sweeps_ms"] / max(sweeps, 1),
        # sweeps/s steady state (sweep kernel only, no full-space metrics) and amortised
        # (whole fit), and the W-phase column step (sweep time / k, an upper bound: it includes the
        # per-sweep H phase and compressed evaluation)
        "sweeps_per_s_steady": sweeps / (agg["sweeps_ms"] / 1e3) if agg["sweeps_ms"] > 0 else None,
        "sweeps_per_s_amortised": sweeps / (agg["total_ms"] / 1e3) if agg["total_ms"] > 0 else None,
        "column_step_us_upper": 1e3 * agg["sweeps_ms"] / max(sweeps, 1) / k,
        "final_rel_err": last.trace[-1].rel_err,
        "wall_s_timed": wall_s,
        "clocks": clocks,
    }
    if not args.no_cpu_baseline and world == 1:
        try:
            x_host = xd.cpu().numpy()
            line["cpu_baseline"] = cpu_baseline(args.config, x_host, cfg, omega, w0, h0, threads=1)
        except Exception as exc:  # reported, never silently dropped
            line["cpu_baseline"] = {"value": None, "error": repr(exc)}
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
