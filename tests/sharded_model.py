"""Test infrastructure: a numpy model of the row-sharded rhals_fit decomposition that
the C++/CUDA library implements (include/rnmf_gpu.h, "multi-GPU"), with torch.distributed
all-reduces standing in for the NCCL / NVLink exchanges.  Every rank holds rows
[off, off + m_r) of X; the model sums exactly the partial products the library sums across GPUs
and replicates what it replicates:

  sketch   Gram of every CholeskyQR pass, X^T Q, B = Q^T X           -> all-reduce
  init     sum(X), sum(X^2) (scan), W~ = Q^T W, ||W(:,j)||^2         -> all-reduce
  W phase  per column [Q^T W(:,j); ||W(:,j)||^2]                     -> all-reduce
  H phase  B, W~, S, T = B H^T, V = H H^T, residc, grad_H            replicated
  pgrad    projected ||grad_W||^2 (rows)                            -> all-reduce
  metrics  objective, projected ||grad_W||^2, W^T X, W^T W          -> all-reduce

The reference algorithm it decomposes is p/src/rhals.cpp:23-213 / p/src/sketch.cpp:52-71, as
restated by oracle/rnmf_oracle.cpp; the CPU tests check model(world=2) == oracle(world=1).
"""
from __future__ import annotations

import numpy as np

DIV_FLOOR = 1e-12  # kDivisionFloor, p/src/hals.cpp


def _allreduce(a, dist):
    import torch

    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64))
    dist.all_reduce(t)
    return t.numpy()


def _cholqr2_sharded(y, dist):
    """CholeskyQR2 with the Gram summed over the ranks (row-sharded Y)."""
    for _ in range(2):
        g = _allreduce(y.T @ y, dist)
        r = np.linalg.cholesky(g).T  # upper, G = R^T R
        y = np.linalg.solve(r.T, y.T).T
    return y


def _qr_replicated(a):
    q, _ = np.linalg.qr(a)
    return q


def _proj_sq(g, at):
    gp = np.where(at > 0.0, g, np.minimum(g, 0.0))
    return float(np.sum(gp * gp))


def sharded_rhals_fit(x_local, m_total, rank_off, opts, omega, w0_local, h0, dist):
    """Returns (W_local, H, trace) of the row-sharded fit; trace = list of dicts as oracle.rhals_fit."""
    k = int(opts["rank"])
    q_iters = int(opts.get("power_iterations", 2))
    max_iter = int(opts["max_iter"])
    tfe = int(opts.get("trace_full_every", 10))
    tol = float(opts.get("tol", 1e-4))
    m, n = x_local.shape
    # scan: sum / sum of squares over all rows
    s = _allreduce(np.array([x_local.sum(), (x_local * x_local).sum()]), dist)
    x_norm = np.sqrt(s[1])
    # rqb
    y = x_local @ omega
    for _ in range(q_iters):
        q = _cholqr2_sharded(y, dist)
        p = _allreduce(x_local.T @ q, dist)
        z = _qr_replicated(p)
        y = x_local @ z
    q = _cholqr2_sharded(y, dist)
    b = _allreduce(q.T @ x_local, dist)
    # random_init scale sqrt(mean(X)/k)
    scale = np.sqrt(s[0] / (m_total * n) / k)
    w = w0_local * scale
    h = h0 * scale
    wt = _allreduce(q.T @ w, dist)

    def metrics():
        resid = x_local - w @ h
        obj = _allreduce(np.array([np.sum(resid * resid)]), dist)[0]
        gw = -2.0 * (x_local @ h.T - w @ (h @ h.T))
        pgw = _allreduce(np.array([_proj_sq(gw, w)]), dist)[0]
        wtx = _allreduce(w.T @ x_local, dist)
        wtw = _allreduce(w.T @ w, dist)
        gh = -2.0 * (wtx - wtw @ h)
        return obj, pgw + _proj_sq(gh, h)

    def compressed_pgrad(st_r):
        residc = b - wt @ h
        objc = float(np.sum(residc * residc))
        gw = -2.0 * (q @ (residc @ h.T))
        pgw = _allreduce(np.array([_proj_sq(gw, w)]), dist)[0]
        if st_r is not None:
            st, r = st_r
            gh = 2.0 * (st @ h - r.T)
        else:
            gh = -2.0 * (wt.T @ residc)
        return objc, pgw + _proj_sq(gh, h)

    trace = []
    obj, pgf = metrics()
    objc, pg0 = compressed_pgrad(None)
    trace.append(dict(iter=0, objective=obj, rel_err=np.sqrt(obj) / x_norm, pgrad=pg0, pgrad_full=pgf,
                      objective_compressed=objc))
    for it in range(1, max_iter + 1):
        if not pg0 > 0.0:
            break
        # W phase (rhals_update_W, p/src/rhals.cpp:107-114 / :23-32)
        t = b @ h.T
        v = h @ h.T
        for j in range(k):
            denom = max(v[j, j], DIV_FLOOR)
            wt[:, j] = wt[:, j] + (t[:, j] - wt @ v[:, j]) / denom
            w[:, j] = np.maximum(q @ wt[:, j], 0.0)
            red = _allreduce(np.concatenate([q.T @ w[:, j], [w[:, j] @ w[:, j]]]), dist)
            wt[:, j] = red[:-1]
        wn = _allreduce(np.sum(w * w, axis=0), dist)
        # H phase (rhals_h_phase, p/src/rhals.cpp:49-58), replicated
        r = b.T @ wt
        st = wt.T @ wt
        for j in range(k):
            num = r[:, j] - st[:, j] @ h
            h[j] = np.maximum(0.0, h[j] + num / max(wn[j], DIV_FLOOR))
        objc, pgc = compressed_pgrad((st, r))
        full = it % tfe == 0 or it == max_iter
        if full:
            obj, pgf = metrics()
        stop = pgc < tol * pg0
        if stop and not full:
            obj, pgf = metrics()
        trace.append(dict(iter=it, objective=obj, rel_err=np.sqrt(obj) / x_norm, pgrad=pgc, pgrad_full=pgf,
                          objective_compressed=objc))
        if stop:
            break
    return w, h, trace
