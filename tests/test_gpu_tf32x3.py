"""GPU parity of math_mode TF32X3 (X-streaming sketch GEMMs on tcgen05 tensor cores, 3xTF32 split
with chunked TMEM accumulation promoted to fp32 registers) against the fp64 oracle, at the same
fp32 tolerances as the EXACT (FFMA) verification mode: per-record trace within 1e-3 relative and
final rel_err within 1e-4 absolute (BASELINE.json north_star).  EXACT stays the verification mode;
these tests show the tensor-core sketch does not loosen the bar.

Sizes cover both tcgen05 kernels' code paths: several 128-row tiles and ragged tails (m, n not
multiples of 128 / 32), several K chunks (n > 64, rows per split > 64), c = l below, at and above
one 16-column UMMA step.
"""
import numpy as np
import pytest

from paper_1711_02037_b200 import workloads

from test_gpu_parity import F32_FINAL_ATOL, F32_TRACE_RTOL, _odict, assert_trace_close

pytestmark = pytest.mark.gpu


def _max_dev(trace, ref, field):
    return max(abs(getattr(g, field) - o[field]) / max(abs(o[field]), 1e-300) for g, o in zip(trace, ref))


def assert_pgrad_no_worse(gpu, x32, o, ref, om, w0, h0, res):
    """The projected-gradient fields cancel to ~1e-4 of their terms near convergence, so their
    deviation is set by the trajectory, not the sketch arithmetic: TF32X3 must stay within 1e-3
    or within 2x of what the EXACT (FFMA) verification mode shows on the same inputs."""
    o.math_mode = gpu.MathMode.Exact
    ex = gpu.rhals_fit(x32, o, omega=om, w0=w0, h0=h0)
    for f in ("pgrad", "pgrad_full"):
        d_tc, d_ex = _max_dev(res.trace, ref.trace, f), _max_dev(ex.trace, ref.trace, f)
        assert d_tc <= max(F32_TRACE_RTOL, 2.0 * d_ex), (f, d_tc, d_ex)


@pytest.mark.parametrize("m,n,k,p", [(700, 300, 6, 8), (2051, 517, 10, 10), (4100, 1000, 16, 20), (333, 1200, 5, 11),
                                     (2500, 900, 40, 20)])
def test_tf32x3_fit_parity(gpu, oracle, m, n, k, p):
    x = oracle.synth_lowrank(m, n, k, 0.05, 100 + m)
    o = gpu.SolverOptions(rank=k, max_iter=30, tol=1e-300, oversampling=p, power_iterations=2, seed=7)
    l = min(k + p, m, n)
    om, w0, h0 = workloads.injected_inputs(2, m, n, k, l)
    ref = oracle.rhals_fit(x, _odict(o), omega=om, w0=w0, h0=h0)
    o.math_mode = gpu.MathMode.TF32x3
    x32 = x.astype(np.float32)
    res = gpu.rhals_fit(x32, o, omega=om, w0=w0, h0=h0)
    assert_trace_close(res.trace, ref.trace, F32_TRACE_RTOL, F32_FINAL_ATOL)
    assert_pgrad_no_worse(gpu, x32, o, ref, om, w0, h0, res)


def test_tf32x3_faces_config_parity(gpu, oracle):
    """BASELINE config 2 shape and data (faces-like 32256 x 2410, k 16, p 20, q 2), 30 sweeps."""
    x = workloads.faces_matrix(0)
    m, n = x.shape
    o = gpu.SolverOptions(rank=16, max_iter=30, tol=1e-300, oversampling=20, power_iterations=2, seed=0)
    om, w0, h0 = workloads.injected_inputs(0, m, n, 16, 36)
    ref = oracle.rhals_fit(x.astype(np.float64), _odict(o), omega=om, w0=w0, h0=h0)
    o.math_mode = gpu.MathMode.TF32x3
    res = gpu.rhals_fit(x, o, omega=om, w0=w0, h0=h0)
    assert_trace_close(res.trace, ref.trace, F32_TRACE_RTOL, F32_FINAL_ATOL)
    assert_pgrad_no_worse(gpu, x, o, ref, om, w0, h0, res)


def test_tf32x3_rqb_projector(gpu, oracle):
    """The tensor-core sketch spans the same subspace as the fp64 oracle's (QQ^T X agrees)."""
    x = oracle.synth_lowrank(1500, 700, 12, 0.05, 5)
    om = np.random.default_rng(3).standard_normal((700, 20))
    r = gpu.rqb(x.astype(np.float32), gpu.SketchOptions(target_rank=12, oversampling=8, power_iterations=2), omega=om,
                math_mode=gpu.MathMode.TF32x3)
    qo, bo = oracle.rqb(x, 12, 8, 2, omega=om)
    q = r.q.astype(np.float64)
    b = r.b.astype(np.float64)
    np.testing.assert_allclose(q.T @ q, np.eye(20), atol=1e-5)
    np.testing.assert_allclose(q @ b, qo @ bo, atol=2e-5 * np.abs(x).max())


@pytest.mark.parametrize("m,n,k", [(1, 1, 1), (5, 3, 2), (1000, 7, 3), (7, 1000, 3), (129, 33, 4), (64, 4000, 8)])
def test_tf32x3_edge_shapes(gpu, oracle, m, n, k):
    """Tiny and ragged shapes through the tensor-core sketch and metrics kernels (partial 128-row
    tiles, fewer columns than one 32-wide stage, l clamped to min(m, n))."""
    o = gpu.SolverOptions(rank=k, max_iter=8, tol=1e-300, oversampling=4, power_iterations=1, seed=2)
    if k > min(m, n):
        o.rank = min(m, n)
    l = min(o.rank + 4, m, n)
    # X of rank >= l: with rank(X) < l the trailing sketch directions are rounding noise (the C1
    # situation, checked two-stage in test_gpu_parity) and the trace is not comparable pointwise
    x = oracle.synth_lowrank(m, n, l, 0.1, 40 + m + n)
    om, w0, h0 = workloads.injected_inputs(5, m, n, o.rank, l)
    ref = oracle.rhals_fit(x, _odict(o), omega=om, w0=w0, h0=h0)
    o.math_mode = gpu.MathMode.TF32x3
    res = gpu.rhals_fit(x.astype(np.float32), o, omega=om, w0=w0, h0=h0)
    assert len(res.trace) == len(ref.trace)
    assert abs(res.trace[-1].rel_err - ref.trace[-1]["rel_err"]) <= 1e-4 + 1e-3 * ref.trace[-1]["rel_err"]


@pytest.mark.parametrize("m,n,k,p", [(20000, 3000, 40, 20), (30011, 777, 16, 20), (9000, 5000, 10, 6), (6000, 4000, 64, 32),
                                     (12000, 2500, 33, 15)])
def test_tf32x3_bitwise_repeatable(gpu, m, n, k, p):
    """Three fits of the same inputs give identical bits (W, H and every trace field).  The
    tensor-core kernels hand tiles between the TMA, split, UMMA and epilogue warps through
    mbarriers and tensor memory; a missed wait or a slot reused too early would show up here as
    run-to-run differences.  Shapes: many persistent tiles per CTA, ragged tails, l = 60 / 36 / 16 / 96 / 48
    (tensor-memory and shared-memory lo layouts, both fused metrics kernels)."""
    x = workloads.noisy_lowrank_matrix(3, m, n, k, 0.5, 0.1)
    o = gpu.SolverOptions(rank=k, max_iter=12, tol=1e-300, oversampling=p, power_iterations=2, seed=5,
                          trace_full_every=3)
    o.math_mode = gpu.MathMode.TF32x3
    runs = [gpu.rhals_fit(x, o) for _ in range(3)]
    for r in runs[1:]:
        np.testing.assert_array_equal(runs[0].factors.w, r.factors.w)
        np.testing.assert_array_equal(runs[0].factors.h, r.factors.h)
        for a, b in zip(runs[0].trace, r.trace):
            assert (a.objective, a.rel_err, a.pgrad, a.pgrad_full, a.objective_compressed) == \
                   (b.objective, b.rel_err, b.pgrad, b.pgrad_full, b.objective_compressed)
