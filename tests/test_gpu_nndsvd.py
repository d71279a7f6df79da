"""InitScheme::Svd (NNDSVD init, p/src/hals.cpp:126-170) on the GPU against the fp64 oracle, plus the
reference's own recovery test that uses it (p/tests/test_rhals.cpp:126-143)."""
import numpy as np
import pytest


def _x(seed=21, m=600, n=300, r=8, noise=0.01):
    rng = np.random.default_rng(seed)
    w = np.abs(rng.standard_normal((m, r))) * (1.0 + np.arange(r))  # distinct singular values
    h = np.abs(rng.standard_normal((r, n)))
    return w @ h + noise * np.abs(rng.standard_normal((m, n)))


def _opts(api, **kw):
    base = dict(rank=6, oversampling=6, power_iterations=2, max_iter=0, tol=1e-300, seed=13, trace_full_every=5,
                init=api.InitScheme.Svd)
    base.update(kw)
    return api.SolverOptions(**base)


def _odict(o):
    return dict(rank=o.rank, oversampling=o.oversampling, power_iterations=o.power_iterations, max_iter=o.max_iter,
                tol=o.tol, seed=o.seed, trace_full_every=o.trace_full_every, init=int(o.init))


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,rtol", [(np.float64, 1e-7), (np.float32, 2e-3)])
def test_nndsvd_init_matches_oracle(gpu, oracle, dtype, rtol):
    api = gpu
    x = _x()
    o = _opts(api)
    res = api.rhals_fit(x.astype(dtype), o)  # max_iter 0: the init itself
    ref = oracle.rhals_fit(x, _odict(o))
    w, h = np.asarray(res.factors.w, np.float64), np.asarray(res.factors.h, np.float64)
    assert w.min() > 0.0 and h.min() > 0.0  # zeros were replaced by mean(X)/100
    np.testing.assert_allclose(w, ref.w, rtol=rtol, atol=rtol * np.abs(ref.w).max())
    np.testing.assert_allclose(h, ref.h, rtol=rtol, atol=rtol * np.abs(ref.h).max())


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,rtol", [(np.float64, 1e-7), (np.float32, 1e-3)])
def test_nndsvd_fit_trace_matches_oracle(gpu, oracle, dtype, rtol):
    api = gpu
    x = _x(seed=5)
    o = _opts(api, max_iter=30)
    res = api.rhals_fit(x.astype(dtype), o)
    ref = oracle.rhals_fit(x, _odict(o))
    assert len(res.trace) == len(ref.trace)
    for g, r in zip(res.trace, ref.trace):
        for f in ("objective", "rel_err", "pgrad", "pgrad_full", "objective_compressed"):
            np.testing.assert_allclose(getattr(g, f), r[f], rtol=rtol, atol=1e-12, err_msg=f"{f} @ {g.iter}")
    assert abs(res.trace[-1].rel_err - ref.trace[-1]["rel_err"]) < 1e-4


@pytest.mark.gpu
def test_nndsvd_exact_lowrank_recovery(gpu, oracle):
    """p/tests/test_rhals.cpp:126-143 'rhals_fit: exact low-rank recovery' through the GPU path."""
    api = gpu
    x = oracle.synth_lowrank(200, 100, 5, 0.0, 29)
    o = api.SolverOptions(rank=5, max_iter=300, tol=1e-24, init=api.InitScheme.Svd, oversampling=10,
                          power_iterations=2, seed=11)
    res = api.rhals_fit(x, o)
    w, h = np.asarray(res.factors.w), np.asarray(res.factors.h)
    assert res.trace[-1].rel_err <= 1e-6
    assert w.min() >= 0.0 and h.min() >= 0.0
    rel = np.linalg.norm(x - w @ h) / np.linalg.norm(x)
    assert rel == pytest.approx(res.trace[-1].rel_err, rel=1e-9)


@pytest.mark.gpu
def test_nndsvd_rejects_overrides(gpu):
    api = gpu
    x = _x(m=100, n=80)
    with pytest.raises(api.ParameterError, match="init overrides require InitScheme::Random"):
        api.rhals_fit(x, _opts(api), w0=np.ones((100, 6)), h0=np.ones((6, 80)))
