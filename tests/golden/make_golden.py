#!/usr/bin/env python
"""Generates tests/golden/*.npz|json from the CPU oracle (which is itself pinned to the
reference's known answers and property suites, tests/test_oracle_reference_suites.py).

The reference cannot be built in this container (no Eigen), so these are oracle regression
fixtures: they pin the oracle against drift and let the GPU tests compare against committed
numbers.  Re-run only when the oracle's restatement changes:  python tests/golden/make_golden.py
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import oracle  # noqa: E402
from paper_1711_02037_b200 import workloads  # noqa: E402

CASES = {
    # name: (rows, cols, rank, noise, xseed, opts, inject_seed or None)
    "noisy_f64_injected": (96, 72, 4, 0.1, 5, dict(rank=4, max_iter=30, tol=1e-300, oversampling=6, power_iterations=2, seed=7), 3),
    "reg_injected": (80, 60, 3, 0.05, 9, dict(rank=3, max_iter=25, tol=1e-300, oversampling=5, power_iterations=1, seed=2, reg=(0.3, 0.2, 0.05, 0.02)), 4),
    "default_streams": (70, 50, 3, 0.05, 13, dict(rank=3, max_iter=20, tol=1e-300, oversampling=8, seed=42, trace_full_every=3), None),
    "early_stop_tol": (60, 45, 3, 0.05, 17, dict(rank=3, max_iter=200, tol=1e-3, oversampling=8, seed=5), None),
    "q0_cadence7": (64, 40, 2, 0.02, 21, dict(rank=2, max_iter=15, tol=1e-300, oversampling=4, power_iterations=0, seed=9, trace_full_every=7), 6),
}


def main():
    rng_fx = {
        "mt19937_64_seed5489_10000th": int(oracle.rng_u64(5489, 10000)[-1]),
        "u64": {str(s): [int(v) for v in oracle.rng_u64(s, 8)] for s in (0, 1, 42, 2**63 + 5)},
        "uniform": {str(s): oracle.rng_uniform(s, 8).tolist() for s in (0, 1, 42, 701532786141963250)},
        "gaussian": {str(s): oracle.rng_gaussian(s, 9).tolist() for s in (0, 42, 7)},
        "split": {f"{s}:{t}": oracle.rng_split_seed(s, t) for s in (0, 5, 42, 99) for t in (1, 2, 3)},
    }
    with open(os.path.join(HERE, "rng.json"), "w") as f:
        json.dump(rng_fx, f, indent=1)
    for name, (m, n, r, noise, xs, o, inj) in CASES.items():
        x = oracle.synth_lowrank(m, n, r, noise, xs)
        l = min(o["rank"] + o["oversampling"], m, n)
        om = w0 = h0 = None
        if inj is not None:
            om, w0, h0 = workloads.injected_inputs(inj, m, n, o["rank"], l)
        res = oracle.rhals_fit(x, o, omega=om, w0=w0, h0=h0)
        fields = ["iter", "objective", "rel_err", "pgrad", "pgrad_full", "objective_compressed"]
        trace = np.array([[t[f] for f in fields] for t in res.trace], dtype=np.float64)
        extra = {} if inj is None else dict(omega=om, w0=w0, h0=h0)
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), x=x, w=res.w, h=res.h, trace=trace,
                            opts=json.dumps(o), **extra)
        print(name, x.shape, len(res.trace), res.trace[-1]["rel_err"])


if __name__ == "__main__":
    main()
