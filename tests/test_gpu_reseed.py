"""reseed_dead (p/src/rhals.cpp:182-186, reseed_dead_components p/src/hals.cpp:96-105) on the GPU:
the kernel stamps every component's liveness per sweep and hands a sweep with a dead W column or H
row to the host, which draws the reseed values from the reference stream in the reference order;
traces and factors against the fp64 oracle.  Mirrors p/tests/test_hals.cpp:405-418 for rHALS."""
import numpy as np
import pytest


def _odict(o):
    r = o.reg
    return dict(rank=o.rank, oversampling=o.oversampling, power_iterations=o.power_iterations, max_iter=o.max_iter,
                tol=o.tol, seed=o.seed, trace_full_every=o.trace_full_every, reseed_dead=int(o.reseed_dead),
                order=int(o.order), reg=(r.alpha_w, r.alpha_h, r.beta_w, r.beta_h))


def _check(api, oracle, x, o, rtol):
    res = api.rhals_fit(x, o)
    ref = oracle.rhals_fit(x.astype(np.float64), _odict(o))
    assert len(res.trace) == len(ref.trace)
    for g, r in zip(res.trace, ref.trace):
        for f in ("objective", "rel_err", "pgrad", "pgrad_full", "objective_compressed"):
            np.testing.assert_allclose(getattr(g, f), r[f], rtol=rtol, atol=1e-12, err_msg=f"{f} @ {g.iter}")
    for got, want in ((res.factors.w, ref.w), (res.factors.h, ref.h)):
        np.testing.assert_allclose(np.asarray(got, np.float64), want, rtol=10 * rtol,
                                   atol=10 * rtol * max(np.abs(want).max(), 1e-300))
    return res


@pytest.mark.gpu
def test_dead_components_stay_dead_unless_reseeded(gpu, oracle):
    api = gpu
    x = oracle.synth_lowrank(60, 40, 2, 0.0, 67)
    base = dict(rank=3, max_iter=4, tol=1e-300, seed=8, oversampling=4, reg=api.RegConfig(0.0, 0.0, 1e6, 0.0))
    dead = api.rhals_fit(x, api.SolverOptions(**base))
    assert np.abs(dead.factors.w).max() == 0.0
    alive = api.rhals_fit(x, api.SolverOptions(**base, reseed_dead=True))
    assert np.abs(alive.factors.w).max() > 0.0
    # parity of the every-sweep reseed on a full-rank X (an exactly rank-2 X makes the trailing
    # sketch columns rounding noise, see the two-stage C1 tests)
    xn = oracle.synth_lowrank(60, 40, 2, 0.05, 67)
    _check(api, oracle, xn, api.SolverOptions(**base, reseed_dead=True), 1e-8)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype,rtol", [(np.float64, 1e-8), (np.float32, 1e-3)])
@pytest.mark.parametrize("order", ["Grouped", "Shuffled"])
def test_partial_reseed_matches_oracle(gpu, oracle, dtype, rtol, order):
    """A strong l1 penalty on H kills some rows mid-run; they are reseeded and the fit continues."""
    api = gpu
    rng = np.random.default_rng(4)
    x = np.abs(rng.standard_normal((300, 3))) @ np.abs(rng.standard_normal((3, 150)))
    x += 0.01 * np.abs(rng.standard_normal(x.shape))
    o = api.SolverOptions(rank=6, max_iter=17, tol=1e-300, seed=2, oversampling=4, trace_full_every=4,
                          reseed_dead=True, order=getattr(api.UpdateOrder, order),
                          reg=api.RegConfig(0.0, 0.0, 0.0, 2.0))
    _check(api, oracle, x.astype(dtype), o, rtol)
