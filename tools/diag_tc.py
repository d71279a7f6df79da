"""Development aid: TF32X3 vs EXACT compress on small shapes against the oracle."""
import os
import sys

import numpy as np

sys.path.insert(0, os.getcwd())
from oracle import oracle  # noqa: E402
from paper_1711_02037_b200 import api as gpu, workloads  # noqa: E402

for (m, n, k, q) in [(5, 3, 2, 1), (5, 3, 2, 0), (6, 4, 2, 0), (129, 33, 4, 1)]:
    x = oracle.synth_lowrank(m, n, min(k, m, n), 0.1, 40 + m + n)
    l = min(k + 4, m, n)
    om, w0, h0 = workloads.injected_inputs(5, m, n, k, l)
    od = dict(rank=k, max_iter=8, tol=1e-300, oversampling=4, power_iterations=q, seed=2)
    ref = oracle.compress(x, od, omega=om, w0=w0, h0=h0)
    for mode in ("Exact", "TF32x3"):
        o = gpu.SolverOptions(rank=k, max_iter=8, tol=1e-300, oversampling=4, power_iterations=q, seed=2)
        o.math_mode = getattr(gpu.MathMode, mode)
        cp = gpu.compress(x.astype(np.float32), o, omega=om, w0=w0, h0=h0)
        Q, B, Wt = (np.asarray(v, dtype=np.float64) for v in (cp.q, cp.b, cp.wt))
        P = Q @ Q.T; Pr = ref.q @ ref.q.T
        print(m, n, k, q, mode, "proj %.2e" % np.abs(P - Pr).max(), "QtX-B %.2e" % np.abs(Q.T @ x - B).max(),
              "QtW-Wt %.2e" % np.abs(Q.T @ w0 - Wt).max(), "orth %.2e" % np.abs(Q.T @ Q - np.eye(l)).max())
        if m < 10:
            print(Q)
