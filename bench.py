#!/usr/bin/env python
"""Benchmark of the B200 randomized-HALS path (rnmf::rhals_fit drop-in) — driver contract.

One *step* = one complete rhals_fit (sketch + sweeps + trace) on the workload.  `value` is HALS
sweeps/s of whole fits with X resident in HBM (X larger than L2, so no flush is needed); `e2e`
is the same metric through the public API with X in pinned host memory (H2D of X and D2H of
W, H and the trace inside every step).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl reference]

Default workload: BASELINE config C4 (200,000 x 20,000, rank 40 + noise, fp32, k 40, p 20, q 2,
200 sweeps), the largest config that fits one GPU and the one BASELINE.md names for the 1 -> 8
GPU curve.  C1-C3 are selectable (--config), C5 runs in full at >= 4 GPUs and on labelled row
slices below that (slice_rows).  C4 / C5 X is generated on the device per shard (seeded per
row block, shard-count independent: workloads.noisy_lowrank_shard).

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


def slice_rows(cfg_name: str, world: int):
    """Rows of the config a `world`-GPU run factorises.  C5 (200 GB fp32) does not fit one GPU:
    BASELINE.json runs it at 8 and 4 GPUs in full and at 2 GPUs on a 100,000-row slice; a single
    GPU takes a 40,000-row slice (16 GB) -- both labelled in `config`."""
    cfg = workloads.CONFIGS[cfg_name]
    if cfg_name == "C5" and world < 4:
        return 100000 if world >= 2 else 40000
    return cfg.m


def host_matrix(cfg_name: str):
    if cfg_name == "C1":
        return workloads.c1_matrix(0)
    if cfg_name == "C2":
        return workloads.faces_matrix(0)
    if cfg_name == "C3":
        return workloads.unmixing_matrix(0)
    return None


def make_workload(cfg_name: str, device, world: int = 1, rank: int = 0, sharded: bool = False):
    """This rank's X rows on the device (C4/C5: generated per shard by the seeded per-block
    generator, no rank builds the whole matrix), the injected Omega / unscaled init draws (this
    rank's W0 rows), the solver options and (row offset, rows, total rows)."""
    import torch

    from paper_1711_02037_b200 import api

    cfg = workloads.CONFIGS[cfg_name]
    m_total = slice_rows(cfg_name, world)
    if world > 1 or sharded:
        from paper_1711_02037_b200 import distributed as pdist

        off, cnt = pdist.shard_rows(m_total, world, rank)
    else:
        off, cnt = 0, m_total
    x = host_matrix(cfg_name)
    if x is None:
        xd = workloads.config_shard(cfg_name, off, cnt, device=device)
    else:
        xd = torch.from_numpy(np.ascontiguousarray(x[off:off + cnt])).to(device)
    l = min(cfg.k + cfg.p, m_total, cfg.n)
    omega, w0, h0 = workloads.injected_inputs(0, m_total, cfg.n, cfg.k, l)
    w0 = np.ascontiguousarray(w0[off:off + cnt])
    opts = api.SolverOptions(rank=cfg.k, oversampling=cfg.p, power_iterations=cfg.q, max_iter=cfg.iters,
                             tol=1e-300, seed=0)
    return cfg, xd, omega, w0, h0, opts, (off, cnt, m_total)


# ---- CPU baseline: the fp64 oracle (restatement of the reference rhals_fit) on host cores --------
# C1-C3: the whole fit is timed (every sweep).  C4 / C5 need ~100 GB / ~1.2 TB of fp64 reference
# temporaries (the m x n residual of p/src/rhals.cpp:141): the oracle runs on row slices of the
# config (full n, k, l, q; the same per-block generator) at two heights m1 < m2, each with 0 and
# 10 sweeps (10 sweeps = one full-space metrics period), and the full fit is extrapolated with
# t(m, s) = A(m) + (s / 10) P(m), A and P linear in m (sketch / metrics / W-phase work is linear
# in m at fixed n; the H phase is independent of m).  Labelled "extrapolated".
# slice heights: tall enough that the m-dependent part of a 10-sweep period (W phase, metrics)
# stands out of the m-independent H phase and of host timing jitter (1,000 / 3,000-row slices gave
# 85 - 550 s for the same C4 fit), short enough for ~15 - 25 s of CPU work in total
SLICE_ROWS = {"C4": (2000, 10000), "C5": (500, 2500)}


def _oracle_fit_s(orc, x64, cfg, omega, w0, h0, sweeps, reps=1):
    """Wall time of one oracle fit; the minimum of `reps` runs (host jitter only ever adds time)."""
    base = dict(rank=cfg.k, tol=1e-300, oversampling=cfg.p, power_iterations=cfg.q, seed=0, trace_full_every=10,
                max_iter=sweeps)
    best = float("inf")
    for _ in range(reps):
        t = time.perf_counter()
        orc.rhals_fit(x64, base, omega=omega, w0=w0, h0=h0)
        best = min(best, time.perf_counter() - t)
    return best


def cpu_sample(cfg_name: str, threads: int, x_host=None, m_full=None, reps=1):
    """One bounded CPU sample of the config -> dict(value iters/s of the full config, est_fit_s,
    wall_s actually spent, sample description, extrapolated flag)."""
    from oracle import oracle as orc

    orc.set_threads(threads)
    cfg = workloads.CONFIGS[cfg_name]
    t_all = time.perf_counter()
    if cfg_name in SLICE_ROWS:
        import torch

        m_full = cfg.m if m_full is None else m_full
        pts = {}
        for ms in SLICE_ROWS[cfg_name]:
            dev = "cuda" if torch.cuda.is_available() else "cpu"  # the bench's own rows 0..ms-1 on a GPU box
            x64 = workloads.config_shard(cfg_name, 0, ms, device=dev).cpu().numpy().astype(np.float64)
            l = min(cfg.k + cfg.p, ms, cfg.n)
            om, w0, h0 = workloads.injected_inputs(0, ms, cfg.n, cfg.k, l)
            pts[ms] = (_oracle_fit_s(orc, x64, cfg, om, w0, h0, 0, reps), _oracle_fit_s(orc, x64, cfg, om, w0, h0, 10, reps))
            del x64
            torch.cuda.empty_cache() if torch.cuda.is_available() else None
        (m1, m2) = SLICE_ROWS[cfg_name]
        a_slope = (pts[m2][0] - pts[m1][0]) / (m2 - m1)
        p_slope = ((pts[m2][1] - pts[m2][0]) - (pts[m1][1] - pts[m1][0])) / (m2 - m1)
        a_full = pts[m1][0] + a_slope * (m_full - m1)
        p_full = (pts[m1][1] - pts[m1][0]) + p_slope * (m_full - m1)
        est = a_full + (cfg.iters / 10.0) * max(p_full, 0.0)
        sample = (f"{cfg_name} row slices m={m1},{m2} (full n={cfg.n}, k={cfg.k}, l={cfg.k + cfg.p}, q={cfg.q}), "
                  f"fp64 oracle with 0 / 10 sweeps (min of {reps}): " +
                  ", ".join(f"m={ms}: {t0:.2f}s / {t10:.2f}s" for ms, (t0, t10) in pts.items()) +
                  f"; extrapolated to {m_full} rows x {cfg.iters} sweeps = {est:.1f}s")
        extrap = True
    else:
        x = host_matrix(cfg_name) if x_host is None else x_host
        x64 = np.ascontiguousarray(x, dtype=np.float64)
        l = min(cfg.k + cfg.p, cfg.m, cfg.n)
        om, w0, h0 = workloads.injected_inputs(0, cfg.m, cfg.n, cfg.k, l)
        est = _oracle_fit_s(orc, x64, cfg, om, w0, h0, cfg.iters)
        sample = f"{cfg_name} full matrix, fp64 oracle rhals_fit, all {cfg.iters} sweeps timed ({est:.2f}s)"
        extrap = False
    return {"value": cfg.iters / est, "unit": "iters/s", "cores": threads, "kind": "port", "sample": sample,
            "est_fit_s": est, "wall_s": time.perf_counter() - t_all, "extrapolated": extrap}


def run_reference(args):
    """--impl reference: the reference algorithm's CPU implementation (the fp64 oracle port; the
    reference itself cannot be compiled here: no Eigen) on all host threads, on this arm's config.
    Each step is one bounded sample (C1-C3: one whole fit; C4/C5: the row-slice samples above)."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cfg = workloads.CONFIGS[args.config]
    threads = os.cpu_count() or 1
    x = host_matrix(args.config)
    vals = []
    for i in range(args.warmup + args.steps):
        r = cpu_sample(args.config, threads, x, m_full=slice_rows(args.config, args.gpus))
        if i >= args.warmup:
            vals.append(r)
    # median over the steps: one step disturbed by another process on the host does not move it
    v = float(np.median([r["value"] for r in vals]))
    est = float(np.median([r["est_fit_s"] for r in vals]))
    wall = float(np.mean([r["wall_s"] for r in vals]))
    m_total = slice_rows(args.config, args.gpus)
    line = {
        "impl": "reference", "metric": METRIC, "value": v, "unit": "iters/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup,
        # wall time of one measured sample; the full-config fit time it implies is est_fit_s
        "ms_per_step": wall * 1e3, "est_fit_s": est, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name + (f" rows 0..{m_total - 1}" if m_total != cfg.m else ""), "m": m_total,
                   "n": cfg.n, "k": cfg.k, "p": cfg.p, "q": cfg.q, "iters": cfg.iters, "tol": 1e-300,
                   "math_mode": "fp64 (CPU)", "parallelism": f"{threads} host threads"},
        "cpu_baseline": {"value": v, "unit": "iters/s", "cores": threads, "kind": "port",
                         "sample": vals[0]["sample"] if vals else "", "extrapolated": vals[0]["extrapolated"]},
        "e2e": {"value": v, "unit": "iters/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    # C4 (200,000 x 20,000, k 40, 200 sweeps, 16 GB fp32): the largest BASELINE config that fits one
    # GPU and the config BASELINE.md names for the 1 -> 8 GPU curve
    ap.add_argument("--config", default="C4", choices=sorted(workloads.CONFIGS))
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    # tf32x3: the X-streaming sketch GEMMs on tcgen05 tensor cores (3xTF32 split, chunked TMEM
    # accumulation promoted to fp32) -- measured more accurate than the FFMA kernels against the
    # fp64 oracle (tests/test_gpu_tf32x3.py, profiles/r01/mode_parity_c2.json); "exact" = FFMA
    ap.add_argument("--math", default="tf32x3", choices=["exact", "tf32x3", "tf32"])
    ap.add_argument("--sharded", action="store_true", help="row-sharded path even at N = 1 (testing)")
    # two extra fits in the other sketch arithmetic after the timed region (a second sketch roofline
    # on the line); off by default so the launch list of the bench command holds the timed math only
    ap.add_argument("--alt-math", action="store_true")
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

    cfg, xd, omega, w0, h0, opts, (off, cnt, m_total) = make_workload(args.config, device, world, rank, args.sharded)
    opts.math_mode = {"exact": api.MathMode.Exact, "tf32x3": api.MathMode.TF32x3, "tf32": api.MathMode.TF32}[args.math]
    esz = xd.element_size()
    if world > 1 or args.sharded:
        from paper_1711_02037_b200 import distributed as pdist

        ctx = (pdist.ShardedContext(local) if world > 1 else
               pdist.ShardedContext(local, rank=0, world=1, comm_id=pdist.comm_unique_id()))

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
    l = min(cfg.k + cfg.p, m_total, n)
    # whole job: every rank copies its X rows and W0 rows, Omega / H0 replicated; W rows + H back
    h2d = m_total * n * esz + 8 * m_total * k + world * 8 * (n * l + k * n)
    d2h = esz * (m_total * k + world * k * n) + world * 56 * (sweeps + 1)

    # the other sketch arithmetic (FFMA when the timed run used the tensor cores, and vice versa):
    # the same X passes once more for a second sketch roofline, outside the timed region
    alt_sketch = None
    if args.alt_math and esz == 4 and world == 1 and args.math in ("exact", "tf32x3"):
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
        "config": {"workload": cfg.name + (f" rows 0..{m_total - 1} (slice)" if m_total != cfg.m else ""),
                   "m": m_total, "n": n, "k": k, "p": cfg.p, "q": cfg.q, "iters": cfg.iters,
                   "tol": 1e-300, "math_mode": args.math,
                   "parallelism": (f"rows{world}" if world > 1 else
                                   "single-gpu, row-sharded code path (world 1)" if args.sharded else "single-gpu"),
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
            del x_pin, x_np
            # the extrapolated configs take the minimum of two runs per point (differences of
            # differences amplify host jitter: single runs gave 400 - 1000 s for the same C4 fit)
            line["cpu_baseline"] = cpu_sample(args.config, os.cpu_count() or 1, m_full=m_total,
                                              reps=2 if args.config in SLICE_ROWS else 1)
        except Exception as exc:  # reported, never silently dropped
            line["cpu_baseline"] = {"value": None, "error": repr(exc)}
    print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
