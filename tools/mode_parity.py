#!/usr/bin/env python
"""Trace parity of each math mode against the fp64 oracle on a BASELINE config (injected Omega /
init draws on both sides) plus the per-stage device times of the GPU fit."""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--rows", type=int, default=0, help="row slice of the config matrix (0 = full)")
    ap.add_argument("--iters", type=int, default=0)
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    import bench
    from oracle import oracle as orc
    from paper_1711_02037_b200 import api, workloads

    import torch

    cfg, xd, omega, w0, h0, opts = bench.make_workload(args.config, torch.device("cuda", 0))
    if args.iters:
        opts.max_iter = args.iters
    x = xd.cpu().numpy()
    if args.rows:
        x = np.ascontiguousarray(x[: args.rows])
        w0 = w0[: args.rows]
        xd = torch.from_numpy(x).cuda()
    orc.set_threads(args.threads)
    t = time.time()
    ref = orc.rhals_fit(x.astype(np.float64), dict(rank=opts.rank, max_iter=opts.max_iter, tol=opts.tol,
                                                    oversampling=opts.oversampling,
                                                    power_iterations=opts.power_iterations, seed=opts.seed),
                        omega=omega, w0=w0, h0=h0)
    t_or = time.time() - t
    out = {"config": args.config, "shape": list(x.shape), "oracle_s": t_or, "modes": {}}
    ctx = api.Context(0)
    for mode in (api.MathMode.Exact, api.MathMode.TF32x3, api.MathMode.TF32):
        opts.math_mode = mode
        res = api.rhals_fit(xd, opts, omega=omega, w0=w0, h0=h0, ctx=ctx)
        res = api.rhals_fit(xd, opts, omega=omega, w0=w0, h0=h0, ctx=ctx)
        st = ctx.stage_times()
        dev = {}
        for f in ("rel_err", "objective_compressed", "objective", "pgrad", "pgrad_full"):
            g = np.array([getattr(r, f) for r in res.trace])
            o = np.array([r[f] for r in ref.trace])
            rel = np.abs(g - o) / np.maximum(np.abs(o), 1e-300)
            dev[f] = float(np.max(rel))
            dev[f + "_worst_record"] = int(np.argmax(rel))
        out["modes"][mode.name] = {
            "max_rel_dev": dev,
            "final_rel_err_abs_diff": abs(res.trace[-1].rel_err - ref.trace[-1]["rel_err"]),
            "final_rel_err": res.trace[-1].rel_err,
            "total_ms": st["total_ms"], "sketch_ms": st["sketch_ms"], "xw_ms": st["xw_ms"], "xtw_ms": st["xtw_ms"],
            "qr_ms": st["qr_ms"], "sweeps_ms": st["sweeps_ms"], "metrics_ms": st["metrics_ms"],
        }
    out["oracle_final_rel_err"] = ref.trace[-1]["rel_err"]
    # sketch quality per mode: principal angles between range(Q_gpu) and range(Q_oracle), and the
    # relative projection residual ||X - Q Q^T X|| / ||X||
    l = omega.shape[1]
    so = api.SketchOptions(target_rank=opts.rank, oversampling=opts.oversampling,
                           power_iterations=opts.power_iterations)
    qo, _ = orc.rqb(x.astype(np.float64), opts.rank, opts.oversampling, opts.power_iterations, omega=omega)
    x64 = x.astype(np.float64)
    nx = np.linalg.norm(x64)
    out["sketch"] = {"oracle_proj_resid": float(np.linalg.norm(x64 - qo @ (qo.T @ x64)) / nx)}
    for mode in (api.MathMode.Exact, api.MathMode.TF32x3, api.MathMode.TF32):
        sk = api.rqb(xd, so, omega=omega, ctx=ctx, math_mode=mode)
        q = sk.q.double().cpu().numpy() if hasattr(sk.q, "cpu") else np.asarray(sk.q, dtype=np.float64)
        sv = np.linalg.svd(q.T @ qo, compute_uv=False)
        sines = np.sqrt(np.maximum(0.0, 1.0 - np.clip(sv, 0, 1) ** 2))
        out["sketch"][mode.name] = {
            "sin_angles_top5": sorted(sines.tolist())[-5:],
            "proj_resid": float(np.linalg.norm(x64 - q @ (q.T @ x64)) / nx),
            "orth_err": float(np.linalg.norm(q.T @ q - np.eye(l))),
        }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
