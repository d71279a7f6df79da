#!/usr/bin/env python
"""Run N fits of a BASELINE config on cuda:0 and print the stage times (for ncu / RNMF_PROF runs)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C4")
    ap.add_argument("--fits", type=int, default=1)
    ap.add_argument("--iters", type=int, default=0, help="override sweep count")
    ap.add_argument("--math", default="tf32x3")
    args = ap.parse_args()
    import torch

    import bench
    from paper_1711_02037_b200 import api

    cfg, xd, omega, w0, h0, opts, _ = bench.make_workload(args.config, torch.device("cuda", 0))
    if args.iters:
        opts.max_iter = args.iters
    opts.math_mode = {"exact": api.MathMode.Exact, "tf32x3": api.MathMode.TF32x3, "tf32": api.MathMode.TF32}[args.math]
    ctx = api.Context(0)
    for _ in range(args.fits):
        res = api.rhals_fit(xd, opts, omega=omega, w0=w0, h0=h0, ctx=ctx)
        st = ctx.stage_times()
        print(json.dumps({"rel_err": res.trace[-1].rel_err, "sweeps": res.trace[-1].iter,
                          **{k: v for k, v in st.items() if k.endswith("_ms")}}))


if __name__ == "__main__":
    main()
