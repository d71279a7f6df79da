"""Pins the CPU oracle against the reference's own test suites (CPU only, no GPU).

The reference cannot be built here (no Eigen), so the oracle is pinned by re-running
the reference's known-answer and property tests against it, case by case:
  p/tests/test_core.cpp, test_sketch.cpp, test_hals.cpp, test_rhals.cpp, acceptance.cpp (criteria
  that fit a CPU test budget).  Each test names the reference case it restates.
"""
import numpy as np
import pytest

from paper_1711_02037_b200._abi import DataError, ParameterError, ShapeError


def o_opts(o, **kw):
    return o.options(**kw)


# ---------------------------------------------------------------- Rng  (p/include/rnmf/types.hpp:55-102)
def test_rng_known_answers(oracle):
    # C++ standard [rand.predef]: the 10000th output of default-seeded (5489) mt19937_64
    assert int(oracle.rng_u64(5489, 10000)[-1]) == 9981545732273789042
    # SURVEY §8c known answers
    assert int(oracle.rng_u64(0, 1)[0]) == 2947667278772165694
    assert oracle.rng_uniform(0, 3).tolist() == [0.15979336337046079, 0.99214520962982877, 0.039569025844865657]
    assert oracle.rng_gaussian(42, 3).tolist() == [-0.48121769980184498, -0.57453687389830577, 0.49458385623521361]
    assert oracle.rng_split_seed(0, 3) == 1961750202426094747
    assert oracle.rng_split_seed(42, 3) == 701532786141963250
    assert oracle.rng_uniform(701532786141963250, 2).tolist() == [0.08240196158514701, 0.4392180609409867]


def test_rng_split_consumption_independent(oracle):  # test_core.cpp "rng: split streams ..."
    a = oracle.rng_uniform(oracle.rng_split_seed(9, 4), 1)[0]
    assert a == oracle.rng_uniform(oracle.rng_split_seed(9, 4), 1)[0]
    assert oracle.rng_uniform(oracle.rng_split_seed(9, 1), 1)[0] != oracle.rng_uniform(oracle.rng_split_seed(9, 2), 1)[0]


def test_uniform_matrix_range_determinism_mean(oracle):  # test_core.cpp "uniform_matrix: ..."
    a = oracle.uniform_matrix(11, 1000, 10)
    b = oracle.uniform_matrix(11, 1000, 10)
    assert (a == b).all() and a.min() >= 0.0 and a.max() < 1.0 and 0.45 < a.mean() < 0.55
    with pytest.raises(ShapeError):
        oracle.uniform_matrix(11, 0, 3)
    with pytest.raises(ShapeError):
        oracle.uniform_matrix(11, 3, 0)
    # row-major draw order (p/src/core.cpp:20-32)
    assert (oracle.uniform_matrix(11, 3, 4).ravel() == oracle.rng_uniform(11, 12)).all()


def test_gaussian_matrix_determinism_moments(oracle):  # test_core.cpp "gaussian_matrix: ..."
    a = oracle.gaussian_matrix(5, 2000, 10)
    assert (a == oracle.gaussian_matrix(5, 2000, 10)).all()
    assert abs(a.mean()) < 0.05 and 0.9 < a.var() < 1.1


# ---------------------------------------------------------------- QR  (p/src/core.cpp:7-16)
def test_economic_qr_reconstruction(oracle):  # test_core.cpp "economic_qr: reconstruction ..."
    a = oracle.gaussian_matrix(3, 50, 10)
    q, r = oracle.economic_qr(a)
    assert q.shape == (50, 10) and r.shape == (10, 10)
    assert np.linalg.norm(q @ r - a) <= 1e-12 * max(1.0, np.linalg.norm(a))
    assert np.abs(q.T @ q - np.eye(10)).max() <= 1e-12
    assert (np.tril(r, -1) == 0).all()


def test_economic_qr_orthonormal_input(oracle):  # test_core.cpp "orthonormal input gives signed identity R"
    q0, _ = oracle.economic_qr(oracle.gaussian_matrix(4, 6, 3))
    q, r = oracle.economic_qr(q0)
    for j in range(3):
        assert abs(abs(r[j, j]) - 1.0) <= 1e-12
        sign = 1.0 if r[j, j] > 0 else -1.0
        assert np.abs(q[:, j] * sign - q0[:, j]).max() <= 1e-12
        for i in range(j):
            assert abs(r[i, j]) <= 1e-12


def test_economic_qr_345(oracle):  # test_core.cpp "economic_qr: 3-4-5 column"
    q, _ = oracle.economic_qr(np.array([[3.0, 0], [4, 0], [0, 1]]))
    sign = 1.0 if q[0, 0] > 0 else -1.0
    assert abs(sign * q[0, 0] - 0.6) <= 1e-12 and abs(sign * q[1, 0] - 0.8) <= 1e-12 and abs(q[2, 0]) <= 1e-12


def test_economic_qr_rejects_wide(oracle):
    with pytest.raises(ShapeError):
        oracle.economic_qr(np.zeros((2, 3)))


# ---------------------------------------------------------------- sketch  (p/src/sketch.cpp:30-71)
def _decay_matrix(oracle, seed):
    """test_sketch.cpp decay_matrix: 100 x 80, singular values 2^-1, 2^-2, ... (one Rng stream)."""
    draws = oracle.rng_gaussian(seed, 100 * 80 + 80 * 80)
    u, _ = oracle.economic_qr(draws[: 100 * 80].reshape(100, 80))
    v, _ = oracle.economic_qr(draws[100 * 80:].reshape(80, 80))
    s = 2.0 ** -np.arange(1, 81)
    return u @ np.diag(s) @ v.T


def test_rqb_exact_rank1(oracle):  # test_sketch.cpp "rqb: exact rank-1 capture"
    d = oracle.rng_uniform(2, 13)
    u, v = d[:8] + 0.5, d[8:] + 0.5
    a = np.outer(u, v)
    q, b = oracle.rqb(a, 1, 2, 0, 1, 1)
    assert q.shape == (8, 3) and b.shape == (3, 5)
    assert np.linalg.norm(a - q @ b) <= 1e-12 * np.linalg.norm(a)
    assert np.abs(q.T @ q - np.eye(3)).max() <= 1e-10


def test_rqb_decaying_spectrum(oracle):  # test_sketch.cpp "rqb: decaying spectrum error against SVD oracle"
    a = _decay_matrix(oracle, 31)
    s11 = np.linalg.svd(a, compute_uv=False)[10]
    assert abs(s11 - 2.0 ** -11) <= 1e-10 * 2.0 ** -11
    q, b = oracle.rqb(a, 10, 10, 2, 1, 77)
    assert np.linalg.norm(a - q @ b, 2) <= 10 * s11


def test_rqb_power_iterations_help(oracle):  # test_sketch.cpp "rqb: power iterations tighten the error"
    a = _decay_matrix(oracle, 19)
    q0, b0 = oracle.rqb(a, 10, 10, 0, 1, 5)
    q2, b2 = oracle.rqb(a, 10, 10, 2, 1, 5)
    assert np.linalg.norm(a - q2 @ b2, 2) <= np.linalg.norm(a - q0 @ b0, 2)


def test_rqb_idempotence_clamp_errors_determinism(oracle):
    a = oracle.synth_lowrank(40, 30, 6, 0.05, 9)
    q, b = oracle.rqb(a, 6, 5, 2, 1, 3)
    qb = q @ b
    assert np.linalg.norm(q @ (q.T @ qb) - qb) <= 1e-12 * np.linalg.norm(qb)
    small = oracle.synth_lowrank(10, 8, 2, 0.0, 4)
    q, b = oracle.rqb(small, 2, 20, 2, 1, 1)  # 22 > 8 clamps to 8
    assert q.shape[1] == 8 and b.shape[0] == 8
    with pytest.raises(ParameterError):
        oracle.rqb(small, 0, 20, 2, 1, 1)
    with pytest.raises(ParameterError):
        oracle.rqb(small, 9, 20, 2, 1, 1)
    bad = small.copy()
    bad[3, 4] = np.nan
    with pytest.raises(DataError):
        oracle.rqb(bad, 2, 20, 2, 1, 1)
    a = oracle.synth_lowrank(30, 25, 4, 0.0, 8)
    q1, b1 = oracle.rqb(a, 4, 6, 2, 1, 123)
    q2, b2 = oracle.rqb(a, 4, 6, 2, 1, 123)
    assert (q1 == q2).all() and (b1 == b2).all()


# ---------------------------------------------------------------- HALS helpers  (p/src/hals.cpp)
def test_update_hand_examples(oracle):  # test_hals.cpp hand examples
    x = np.array([[2.0, 4], [1, 2]])
    w = oracle.update_W(x, np.array([[1.0], [1]]), np.array([[1.0, 2]]))
    assert abs(w[0, 0] - 2.0) <= 2e-14 and abs(w[1, 0] - 1.0) <= 1e-14
    w = oracle.update_W(x, np.zeros((2, 1)), np.array([[1.0, 2]]), (0, 0, 10.0, 0))
    assert w[0, 0] == 0.0 and w[1, 0] == 0.0
    x = np.array([[2.0, 1], [4, 2]])
    h = oracle.update_H(x, np.array([[1.0], [2]]), np.array([[1.0, 1]]))
    assert abs(h[0, 0] - 2.0) <= 2e-14 and abs(h[0, 1] - 1.0) <= 1e-14


def test_objective_and_pgrad_hand_values(oracle):  # test_hals.cpp "objective: hand values", "pgrad 16"
    x = np.array([[1.0, 2], [3, 4]])
    w, h = np.ones((2, 1)), np.ones((1, 2))
    assert abs(oracle.objective(x, w, h) - 14.0) <= 14.0 * 1e-15
    assert oracle.objective(w @ h, w, h) == 0.0
    assert abs(oracle.projected_gradient_norm(np.eye(2), w, h) - 16.0) <= 16.0 * 1e-13


def _naive_pgrad(x, w, h):
    """test_hals.cpp naive_pgrad, vectorised: grad_W = 2(W HH^T - X H^T), grad_H = 2(W^T W H - W^T X)."""
    gw = 2 * (w @ (h @ h.T) - x @ h.T)
    gh = 2 * ((w.T @ w) @ h - w.T @ x)
    pw = np.where(w > 0, gw, np.minimum(0, gw))
    ph = np.where(h > 0, gh, np.minimum(0, gh))
    return (pw ** 2).sum() + (ph ** 2).sum()


def test_pgrad_matches_naive_with_boundary(oracle):  # test_hals.cpp "matches a naive oracle with boundary entries"
    draws = oracle.rng_uniform(14, 20 * (21 + 18))
    for trial in range(20):
        x = oracle.synth_lowrank(7, 6, 3, 0.1, 100 + trial)
        d = draws[trial * 39:(trial + 1) * 39]
        w = d[:21].reshape(7, 3).copy()
        h = d[21:].reshape(3, 6).copy()
        w[w < 0.3] = 0.0
        h[h < 0.3] = 0.0
        lib = oracle.projected_gradient_norm(x, w, h)
        assert lib == pytest.approx(_naive_pgrad(x, w, h), rel=1e-10)


def _oracle_update_W(x, w, h):
    w = w.copy()
    for j in range(w.shape[1]):
        r = x - sum(np.outer(w[:, i], h[i]) for i in range(w.shape[1]) if i != j)
        w[:, j] = np.maximum(r @ h[j] / (h[j] @ h[j]), 0)
    return w


def _oracle_update_H(x, w, h):
    h = h.copy()
    for j in range(h.shape[0]):
        r = x - sum(np.outer(w[:, i], h[i]) for i in range(h.shape[0]) if i != j)
        h[j] = np.maximum(r.T @ w[:, j] / (w[:, j] @ w[:, j]), 0)
    return h


def test_residual_oracle_equivalence(oracle):  # acceptance.cpp criterion 10 (100 seeds)
    worst = 0.0
    for seed in range(100):
        d = oracle.rng_uniform(3000 + seed, 20 + 10 + 8)
        x, w0, h0 = d[:20].reshape(5, 4) + 0.5, d[20:30].reshape(5, 2) + 0.25, d[30:].reshape(2, 4) + 0.25
        w1 = oracle.update_W(x, w0, h0)
        assert np.linalg.norm(w1[:, 0]) > 0 and np.linalg.norm(w1[:, 1]) > 0
        worst = max(worst, np.abs(w1 - _oracle_update_W(x, w0, h0)).max())
        h1 = oracle.update_H(x, w1, h0)
        worst = max(worst, np.abs(h1 - _oracle_update_H(x, w1, h0)).max())
    assert worst <= 1e-12


def test_init_factors_and_errors(oracle):  # test_hals.cpp "init_factors: ..."
    x = oracle.synth_lowrank(12, 9, 3, 0.1, 17)
    for scheme in (0, 1):
        a = oracle.init_factors(x, 3, scheme, 5)
        b = oracle.init_factors(x, 3, scheme, 5)
        assert a[0].shape == (12, 3) and a[1].shape == (3, 9)
        assert a[0].min() >= 0 and a[1].min() >= 0
        assert (a[0] == b[0]).all() and (a[1] == b[1]).all()
    # random_init: W then H uniform from Rng(seed), scaled by sqrt(mean/k) (p/src/hals.cpp:118-124)
    w, h = oracle.init_factors(x, 3, 0, 5)
    u = oracle.rng_uniform(5, 12 * 3 + 3 * 9)
    scale = np.sqrt(x.mean() / 3)
    np.testing.assert_allclose(w, u[:36].reshape(12, 3) * scale, rtol=1e-15)
    np.testing.assert_allclose(h, u[36:].reshape(3, 9) * scale, rtol=1e-15)
    bad = np.ones((3, 3))
    bad[1, 2] = -0.5
    with pytest.raises(DataError):
        oracle.init_factors(bad, 2, 0, 1)


def test_svd_init_rank1(oracle):  # test_hals.cpp "init_factors: svd scheme recovers a positive rank-1 pair"
    d = oracle.rng_uniform(8, 15)
    u, v = d[:9] + 0.5, d[9:] + 0.5
    w, h = oracle.init_factors(np.outer(u, v), 1, 1, 1)
    assert np.linalg.norm(w[:, 0] / np.linalg.norm(w[:, 0]) - u / np.linalg.norm(u)) <= 1e-8
    assert np.linalg.norm(h[0] / np.linalg.norm(h[0]) - v / np.linalg.norm(v)) <= 1e-8


def test_hals_fit_recovery_and_orders(oracle):  # test_hals.cpp hals_fit cases
    x = oracle.synth_lowrank(50, 40, 2, 0.0, 23)
    r = oracle.hals_fit(x, o_opts(oracle, rank=2, max_iter=500, tol=1e-20, init=1, seed=9))
    assert r.trace[-1]["rel_err"] <= 1e-6
    rel = np.linalg.norm(x - r.w @ r.h) / np.linalg.norm(x)
    assert rel == pytest.approx(r.trace[-1]["rel_err"], rel=1e-9)
    x = oracle.synth_lowrank(25, 18, 4, 0.1, 31)
    for order in (1, 0, 2):
        r = oracle.hals_fit(x, o_opts(oracle, rank=4, max_iter=40, tol=1e-300, order=order, seed=2))
        slack = 1e-12 * r.trace[0]["objective"]
        for a, b in zip(r.trace, r.trace[1:]):
            assert b["objective"] <= a["objective"] + slack


# ---------------------------------------------------------------- rHALS  (p/src/rhals.cpp)
def test_compress_contract(oracle):  # test_rhals.cpp "compress: shape contract, sketch quality, determinism"
    x = oracle.synth_lowrank(40, 30, 4, 0.0, 5)
    o = o_opts(oracle, rank=4, oversampling=10, power_iterations=2, seed=13)
    cp = oracle.compress(x, o)
    assert cp.q.shape == (40, 14) and cp.b.shape == (14, 30) and cp.wt.shape == (14, 4)
    assert np.linalg.norm(x - cp.q @ cp.b) <= 1e-10 * np.linalg.norm(x)
    assert np.abs(cp.wt - cp.q.T @ cp.w).max() <= 1e-14
    cp2 = oracle.compress(x, o)
    assert (cp.b == cp2.b).all() and (cp.w == cp2.w).all()


def test_compress_init_matches_init_factors(oracle):  # test_rhals.cpp "compress: initialization matches hals_fit"
    x = oracle.synth_lowrank(20, 15, 3, 0.0, 7)
    cp = oracle.compress(x, o_opts(oracle, rank=3, oversampling=8, seed=99))
    w, h = oracle.init_factors(x, 3, 0, 99)
    assert (cp.w == w).all() and (cp.h == h).all()


def _identity_problem(oracle, x, rank, seed):
    w, h = oracle.init_factors(x, rank, 0, seed)
    return oracle.CompressedProblem(np.eye(x.shape[0]), x.copy(), w.copy(), w.copy(), h.copy())


def test_identity_basis_reduction(oracle):  # test_rhals.cpp "rhals updates reduce to deterministic ones"
    x = oracle.synth_lowrank(6, 5, 2, 0.1, 21)
    for reg in ((0, 0, 0, 0), (0.5, 0.25, 0.1, 0.05)):
        cp = _identity_problem(oracle, x, 2, 3)
        w_det = oracle.update_W(x, cp.w, cp.h, reg)
        oracle.rhals_update_W(cp, reg)
        assert np.abs(cp.w - w_det).max() <= 1e-12 and np.abs(cp.wt - cp.w).max() <= 1e-12
        h_det = oracle.update_H(x, cp.w, cp.h, reg)
        oracle.rhals_update_H(cp, reg)
        assert np.abs(cp.h - h_det).max() <= 1e-12 and cp.h.min() >= 0


def test_rank1_sketched_equivalence(oracle):  # test_rhals.cpp "rhals updates match the deterministic rule on the sketched matrix"
    d = oracle.rng_uniform(2, 10)
    x = np.outer(d[:6] + 0.5, d[6:] + 0.5)
    cp = oracle.compress(x, o_opts(oracle, rank=1, oversampling=2, power_iterations=2, seed=31))
    oracle.rhals_update_W(cp)
    assert np.abs(cp.w - cp.q @ cp.wt).max() <= 1e-12
    xs = cp.q @ cp.b
    probe = cp.copy()
    oracle.rhals_update_H(probe)
    h_det = oracle.update_H(xs, cp.w, cp.h)
    assert np.abs(probe.h - h_det).max() <= 1e-10
    probe = cp.copy()
    probe.h = h_det
    oracle.rhals_update_W(probe)
    assert np.abs(probe.w - oracle.update_W(xs, cp.w, h_det)).max() <= 1e-10


def test_update_w_nonneg_and_consistent(oracle):  # test_rhals.cpp "rhals_update_W keeps W nonnegative and W~ consistent"
    x = oracle.synth_lowrank(30, 20, 3, 0.05, 17)
    cp = oracle.compress(x, o_opts(oracle, rank=3, oversampling=8, seed=3))
    for _ in range(5):
        oracle.rhals_update_W(cp)
        oracle.rhals_update_H(cp)
        assert cp.w.min() >= 0 and cp.h.min() >= 0
        assert np.linalg.norm(cp.wt - cp.q.T @ cp.w) <= 1e-12 * max(1.0, np.linalg.norm(cp.w))


def test_rhals_exact_recovery_svd_init(oracle):  # test_rhals.cpp "rhals_fit: exact low-rank recovery"
    x = oracle.synth_lowrank(200, 100, 5, 0.0, 29)
    r = oracle.rhals_fit(x, o_opts(oracle, rank=5, max_iter=300, tol=1e-24, init=1, oversampling=10,
                                   power_iterations=2, seed=11))
    assert r.trace[-1]["rel_err"] <= 1e-6
    rel = np.linalg.norm(x - r.w @ r.h) / np.linalg.norm(x)
    assert rel == pytest.approx(r.trace[-1]["rel_err"], rel=1e-9)


def test_rhals_tracks_hals(oracle):  # test_rhals.cpp "rhals_fit: tracks the deterministic solver"
    x = oracle.synth_lowrank(120, 80, 4, 0.0, 37)
    o = o_opts(oracle, rank=4, max_iter=200, tol=1e-24, init=1, oversampling=12, seed=5)
    assert abs(oracle.hals_fit(x, o).trace[-1]["rel_err"] - oracle.rhals_fit(x, o).trace[-1]["rel_err"]) <= 1e-3


def test_rhals_compressed_objective_nonincreasing(oracle):  # test_rhals.cpp "(soft)"
    x = oracle.synth_lowrank(50, 35, 4, 0.05, 43)
    r = oracle.rhals_fit(x, o_opts(oracle, rank=4, max_iter=60, tol=1e-300, oversampling=10, seed=7))
    slack = 1e-8 * r.trace[0]["objective_compressed"]
    for a, b in zip(r.trace, r.trace[1:]):
        assert b["objective_compressed"] <= a["objective_compressed"] + slack


def test_rhals_trace_bookkeeping(oracle):  # test_rhals.cpp "rhals_fit: trace bookkeeping"
    x = oracle.synth_lowrank(60, 45, 3, 0.05, 51)
    r = oracle.rhals_fit(x, o_opts(oracle, rank=3, max_iter=25, tol=1e-300, oversampling=8, trace_full_every=10, seed=2))
    t = r.trace
    assert len(t) == 26
    for a, b in zip(t, t[1:]):
        assert b["iter"] == a["iter"] + 1 and b["elapsed_s"] >= a["elapsed_s"]
    assert t[10]["rel_err"] != t[9]["rel_err"]
    assert t[11]["rel_err"] == t[10]["rel_err"]
    assert t[25]["rel_err"] != t[24]["rel_err"]


def test_rhals_max_iter_zero(oracle):  # test_rhals.cpp "rhals_fit: max_iter 0 returns the initialization"
    x = oracle.synth_lowrank(14, 10, 2, 0.0, 3)
    r = oracle.rhals_fit(x, o_opts(oracle, rank=2, max_iter=0, oversampling=6, seed=55))
    assert len(r.trace) == 1
    w, h = oracle.init_factors(x, 2, 0, 55)
    assert (r.w == w).all() and (r.h == h).all()


def test_rhals_alternative_orders(oracle):  # test_rhals.cpp "alternative orders still descend ..."
    x = oracle.synth_lowrank(40, 28, 3, 0.05, 61)
    for order in (0, 2):
        r = oracle.rhals_fit(x, o_opts(oracle, rank=3, max_iter=30, tol=1e-300, order=order, oversampling=8, seed=4))
        assert r.w.min() >= 0 and r.h.min() >= 0
        assert r.trace[-1]["objective_compressed"] < r.trace[0]["objective_compressed"]


def test_rhals_l1_sparsifies(oracle):  # test_rhals.cpp "rhals_fit: l1 regularization sparsifies W"
    x = oracle.synth_lowrank(40, 30, 4, 0.1, 71)
    o = dict(rank=4, max_iter=60, tol=1e-300, oversampling=10, seed=6)
    plain = oracle.rhals_fit(x, o_opts(oracle, **o))
    lasso = oracle.rhals_fit(x, o_opts(oracle, **o, reg=(0, 0, 0.9, 0)))
    assert (lasso.w == 0).sum() >= (plain.w == 0).sum() and lasso.w.min() >= 0


def test_complete_basis_reduction(oracle):  # acceptance.cpp criterion 9
    x = oracle.synth_lowrank(30, 20, 3, 0.1, 17)
    q, _ = oracle.economic_qr(oracle.gaussian_matrix(23, 30, 30))
    w, h = oracle.init_factors(x, 3, 0, 5)
    cp = oracle.CompressedProblem(q, q.T @ x, q.T @ w, w.copy(), h.copy())
    w1 = oracle.update_W(x, w, h)
    h1 = oracle.update_H(x, w1, h)
    oracle.rhals_update_W(cp)
    oracle.rhals_update_H(cp)
    assert np.abs(cp.w - w1).max() <= 1e-12 * max(1.0, np.abs(w1).max())
    assert np.abs(cp.h - h1).max() <= 1e-12 * max(1.0, np.abs(h1).max())


def test_errors_in_reference_order(oracle):  # p/src/hals.cpp:36-53: data errors before parameter errors
    x = np.ones((6, 5))
    x[2, 3] = -1
    with pytest.raises(DataError, match=r"negative entries at \(2,3\)"):
        oracle.rhals_fit(x, o_opts(oracle, rank=0))
    x[1, 1] = np.inf
    with pytest.raises(DataError, match=r"non-finite entries at \(1,1\)"):
        oracle.rhals_fit(x, o_opts(oracle, rank=2))
    y = np.ones((6, 5))
    for kw in (dict(rank=0), dict(rank=6), dict(rank=2, max_iter=-1), dict(rank=2, tol=0.0),
               dict(rank=2, reg=(-1, 0, 0, 0)), dict(rank=2, trace_full_every=0), dict(rank=2, oversampling=-1)):
        with pytest.raises(ParameterError):
            oracle.rhals_fit(y, o_opts(oracle, **kw))


def test_oracle_rqb_streaming_block_independence(oracle):
    """p/tests/test_sketch.cpp:143-166 on the oracle's restatement of rqb_streaming."""
    a = oracle.synth_lowrank(300, 200, 5, 0.0, 5)
    a /= np.linalg.norm(a)
    qm, bm = oracle.rqb(a, 5, 10, 2, seed=21)
    prev = None
    for bs in (1, 7, 64, 1024):
        q, b = oracle.rqb_streaming(a, 5, 10, 2, seed=21, block_size=bs)
        assert np.linalg.norm(q @ b - qm @ bm) <= 1e-10
        if prev is not None:
            assert np.linalg.norm(q @ b - prev) <= 1e-10
        prev = q @ b


def test_oracle_rqb_streaming_errors(oracle):
    a = oracle.synth_lowrank(50, 80, 3, 0.0, 1)
    a[3, 70] = np.inf
    with pytest.raises(DataError, match=r"non-finite values in columns \[64, 80\)"):
        oracle.rqb_streaming(a, 3, 2, 1, block_size=32)
    with pytest.raises(ParameterError, match="block size"):
        oracle.rqb_streaming(a, 3, 2, 1, block_size=0)


def test_rnmfmat1_writer_layout(tmp_path):
    """RNMFMAT1 (p/include/rnmf/data_io.hpp:12-15): magic, LE u64 rows / cols, row-major LE f64."""
    from paper_1711_02037_b200 import api

    a = np.arange(6, dtype=np.float64).reshape(2, 3)
    p = tmp_path / "a.bin"
    api.write_matrix_bin(str(p), a)
    raw = p.read_bytes()
    assert raw[:8] == b"RNMFMAT1" and len(raw) == 24 + 48
    assert int.from_bytes(raw[8:16], "little") == 2 and int.from_bytes(raw[16:24], "little") == 3
    assert np.array_equal(np.frombuffer(raw[24:], dtype="<f8").reshape(2, 3), a)
