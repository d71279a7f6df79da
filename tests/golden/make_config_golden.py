#!/usr/bin/env python
"""Oracle fixtures for the BASELINE configs at (or near) full size -- TEST INFRASTRUCTURE.

The fp64 CPU oracle (oracle/rnmf_oracle.cpp, pinned by tests/test_oracle_reference_suites.py and
tests/golden/make_golden.py) takes minutes on these shapes, too long to re-run inside the GPU
test suite, so its traces are computed once here and committed.  The GPU tests
(tests/test_gpu_configs.py) regenerate the same X, Omega, W0, H0 from the seeded workload
generators, check the regenerated X against the stored checksums, run the sm_100a path and compare
its trace with the stored oracle trace at the north-star tolerances.

Cases (BASELINE.json configs; injected Omega / init draws as bench.py uses them):
  C2       faces-like 32256 x 2410, k 16, p 20, q 2, 200 sweeps (the full config)
  C3       unmixing-like 1,048,576 x 256, k 10, p 10, q 2, 300 sweeps (the full config)
  C4slice  rows 0..19,999 of the C4 distribution: 20,000 x 20,000, rank 40 + noise, k 40, p 20,
           q 2, 200 sweeps (C4's n, k, l; the full 200,000-row C4 needs ~100 GB of fp64 oracle
           temporaries and hours of CPU)

  python tests/golden/make_config_golden.py [C2 C3 C4slice] [--threads N]
"""
import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from paper_1711_02037_b200 import workloads  # noqa: E402

FIELDS = ["iter", "objective", "rel_err", "pgrad", "pgrad_full", "objective_compressed"]


def case(name):
    """(X fp32 host, k, p, q, iters, injection seed) of a fixture case."""
    if name == "C2":
        return workloads.faces_matrix(0), 16, 20, 2, 200, 0
    if name == "C3":
        return workloads.unmixing_matrix(0), 10, 10, 2, 300, 0
    if name == "C4slice":
        return workloads.noisy_lowrank_matrix(0, 20000, 20000, 40, 0.5, 0.1), 40, 20, 2, 200, 0
    raise KeyError(name)


def x_checksum(x):
    x64 = x.astype(np.float64)
    return np.array([x64.sum(), (x64 * x64).sum(), float(x.shape[0]), float(x.shape[1])])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cases", nargs="*", default=["C2", "C3", "C4slice"])
    ap.add_argument("--threads", type=int, default=os.cpu_count() or 1)
    args = ap.parse_args()
    from oracle import oracle

    oracle.build()
    oracle.set_threads(args.threads)
    for name in args.cases:
        t0 = time.perf_counter()
        x, k, p, q, iters, inj = case(name)
        m, n = x.shape
        l = min(k + p, m, n)
        om, w0, h0 = workloads.injected_inputs(inj, m, n, k, l)
        opts = dict(rank=k, max_iter=iters, tol=1e-300, oversampling=p, power_iterations=q, seed=0)
        res = oracle.rhals_fit(x.astype(np.float64), opts, omega=om, w0=w0, h0=h0)
        trace = np.array([[t[f] for f in FIELDS] for t in res.trace], dtype=np.float64)
        np.savez_compressed(os.path.join(HERE, f"config_{name}.npz"), trace=trace, opts=json.dumps(opts),
                            x_checksum=x_checksum(x), w_colnorm=np.linalg.norm(res.w, axis=0),
                            h_rownorm=np.linalg.norm(res.h, axis=1), threads=args.threads,
                            oracle_s=time.perf_counter() - t0)
        print(name, x.shape, len(res.trace), res.trace[-1]["rel_err"], f"{time.perf_counter() - t0:.1f}s", flush=True)


if __name__ == "__main__":
    main()
