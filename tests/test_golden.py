"""Golden fixtures (tests/golden/, made by tests/golden/make_golden.py from the pinned oracle).

CPU: the oracle still reproduces every fixture (guards the checker against drift) and the Rng
known answers.  GPU: the sm_100a path reproduces the fixture traces and factors, including the
early-stop iteration, the trace_full_every cadence, q = 0 and regularisation."""
import glob
import json
import os

import numpy as np
import pytest

HERE = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")
FIELDS = ["iter", "objective", "rel_err", "pgrad", "pgrad_full", "objective_compressed"]
# config_*.npz are the full-size config traces of tests/test_gpu_configs.py (no X stored)
CASES = sorted(os.path.basename(p)[:-4] for p in glob.glob(os.path.join(HERE, "*.npz"))
               if not os.path.basename(p).startswith("config_"))


def load(name):
    d = np.load(os.path.join(HERE, name + ".npz"))
    o = json.loads(str(d["opts"]))
    inj = {k: d[k] for k in ("omega", "w0", "h0") if k in d.files}
    return d["x"], o, inj, d["trace"], d["w"], d["h"]


def test_rng_fixture(oracle):
    fx = json.load(open(os.path.join(HERE, "rng.json")))
    assert fx["mt19937_64_seed5489_10000th"] == 9981545732273789042
    for s, vals in fx["u64"].items():
        assert [int(v) for v in oracle.rng_u64(int(s), len(vals))] == vals
    for s, vals in fx["uniform"].items():
        assert oracle.rng_uniform(int(s), len(vals)).tolist() == vals
    for s, vals in fx["gaussian"].items():
        assert oracle.rng_gaussian(int(s), len(vals)).tolist() == vals
    for key, v in fx["split"].items():
        s, t = key.split(":")
        assert oracle.rng_split_seed(int(s), int(t)) == v


@pytest.mark.parametrize("name", CASES)
def test_oracle_reproduces_fixture(oracle, name):
    x, o, inj, trace, w, h = load(name)
    r = oracle.rhals_fit(x, o, **inj)
    got = np.array([[t[f] for f in FIELDS] for t in r.trace])
    assert got.shape == trace.shape
    np.testing.assert_allclose(got, trace, rtol=1e-12, atol=0)
    np.testing.assert_allclose(r.w, w, rtol=1e-12, atol=1e-300)
    np.testing.assert_allclose(r.h, h, rtol=1e-12, atol=1e-300)


def _gpu_opts(api, o):
    kw = dict(o)
    if "reg" in kw:
        kw["reg"] = api.RegConfig(*kw["reg"])
    return api.SolverOptions(**kw)


@pytest.mark.gpu
@pytest.mark.parametrize("name", CASES)
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_gpu_matches_fixture(gpu, name, dtype):
    x, o, inj, trace, w, h = load(name)
    res = gpu.rhals_fit(x.astype(dtype), _gpu_opts(gpu, o), **inj)
    got = np.array([[getattr(t, f) for f in FIELDS] for t in res.trace])
    if dtype == np.float64:
        assert got.shape == trace.shape, "stop iteration / trace length differs"
        for col, f in enumerate(FIELDS[1:], start=1):
            rtol = 1e-8 if f in ("objective", "rel_err", "objective_compressed") else 1e-6
            np.testing.assert_allclose(got[:, col], trace[:, col], rtol=rtol, err_msg=f)
        np.testing.assert_allclose(res.factors.w, w, rtol=1e-7, atol=1e-9 * np.abs(w).max())
        np.testing.assert_allclose(res.factors.h, h, rtol=1e-7, atol=1e-9 * np.abs(h).max())
    else:
        n = min(len(got), len(trace))
        if name != "early_stop_tol":
            assert got.shape == trace.shape
        for col, f in ((2, "rel_err"), (5, "objective_compressed"), (1, "objective")):
            np.testing.assert_allclose(got[:n, col], trace[:n, col], rtol=1e-3, err_msg=f)
        assert abs(got[-1, 2] - trace[-1, 2]) <= 1e-4
