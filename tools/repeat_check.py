#!/usr/bin/env python
"""Bitwise run-to-run check of whole BASELINE-config fits on cuda:0 (development aid): N fits of the
same inputs must give identical W, H and trace bits in TF32X3 mode."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C2,C3,C4")
    ap.add_argument("--fits", type=int, default=4)
    args = ap.parse_args()
    import torch

    import bench
    from paper_1711_02037_b200 import api

    ok = True
    for name in args.configs.split(","):
        cfg, xd, omega, w0, h0, opts, _ = bench.make_workload(name, torch.device("cuda", 0))
        opts.math_mode = api.MathMode.TF32x3
        ctx = api.Context(0)
        ref = None
        for i in range(args.fits):
            res = api.rhals_fit(xd, opts, omega=omega, w0=w0, h0=h0, ctx=ctx)
            cur = (res.factors.w.clone(), res.factors.h.clone(),
                   [(t.objective, t.rel_err, t.pgrad, t.pgrad_full, t.objective_compressed) for t in res.trace])
            if ref is None:
                ref = cur
            else:
                same = bool(torch.equal(ref[0], cur[0])) and bool(torch.equal(ref[1], cur[1])) and ref[2] == cur[2]
                nd = sum(1 for a, b in zip(ref[2], cur[2]) if a != b)
                print(f"{name} fit {i}: {'identical' if same else 'DIFFERENT'} (trace records differing: {nd})")
                ok &= same
        del xd, ctx
        torch.cuda.empty_cache()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
