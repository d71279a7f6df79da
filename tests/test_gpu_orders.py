"""UpdateOrder::Interleaved / Shuffled (p/src/rhals.cpp:34-45,73-78; sweep_order p/src/hals.cpp:83-94)
on the GPU against the fp64 oracle: per-component fresh T/V, the H row update after each W column,
the shuffle stream drawn like the reference, grad_H from the residual (invalid scratch)."""
import numpy as np
import pytest


def _x(seed=9, m=500, n=220, r=7):
    rng = np.random.default_rng(seed)
    return np.abs(rng.standard_normal((m, r))) @ np.abs(rng.standard_normal((r, n))) + \
        0.05 * np.abs(rng.standard_normal((m, n)))


@pytest.mark.gpu
@pytest.mark.parametrize("order", ["Interleaved", "Shuffled"])
@pytest.mark.parametrize("dtype,rtol", [(np.float64, 1e-8), (np.float32, 1e-3)])
def test_fresh_orders_match_oracle(gpu, oracle, order, dtype, rtol):
    api = gpu
    x = _x()
    o = api.SolverOptions(rank=6, oversampling=6, power_iterations=1, max_iter=23, tol=1e-300, seed=17,
                          trace_full_every=5, order=getattr(api.UpdateOrder, order), reg=api.RegConfig(0.01, 0.02, 0.0, 0.001))
    res = api.rhals_fit(x.astype(dtype), o)
    ref = oracle.rhals_fit(x, dict(rank=6, oversampling=6, power_iterations=1, max_iter=23, tol=1e-300, seed=17,
                                   trace_full_every=5, order=int(o.order), reg=(0.01, 0.02, 0.0, 0.001)))
    assert len(res.trace) == len(ref.trace)
    for g, r in zip(res.trace, ref.trace):
        for f in ("objective", "rel_err", "pgrad", "pgrad_full", "objective_compressed"):
            np.testing.assert_allclose(getattr(g, f), r[f], rtol=rtol, atol=1e-12, err_msg=f"{f} @ {g.iter}")
    np.testing.assert_allclose(np.asarray(res.factors.h, np.float64), ref.h, rtol=10 * rtol,
                               atol=10 * rtol * np.abs(ref.h).max())


@pytest.mark.gpu
def test_shuffled_differs_from_interleaved(gpu):
    api = gpu
    x = _x(m=200, n=100)
    tr = {}
    for order in ("Interleaved", "Shuffled"):
        o = api.SolverOptions(rank=5, max_iter=6, tol=1e-300, seed=3, oversampling=5,
                              order=getattr(api.UpdateOrder, order))
        tr[order] = [r.objective_compressed for r in api.rhals_fit(x, o).trace]
    assert tr["Interleaved"][0] == tr["Shuffled"][0]
    assert tr["Interleaved"][1:] != tr["Shuffled"][1:]
