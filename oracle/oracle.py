"""TEST INFRASTRUCTURE ONLY — ctypes binding of the CPU oracle (oracle/_build/liboracle.so).

The oracle is an fp64 C++ restatement of the reference rnmf randomized-HALS path
(see rnmf_oracle.h for what it restates and how it is pinned).  Only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs import this
module; the product package never does.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

from paper_1711_02037_b200 import _abi
from paper_1711_02037_b200._abi import (
    ProblemShapeC,
    RegConfigC,
    SolverOptionsC,
    TraceRecordC,
    err_buffer,
    raise_for_status,
)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_build", "liboracle.so")

_D = ctypes.POINTER(ctypes.c_double)
_I64 = ctypes.c_int64
_lib = None
_CAP = ctypes.c_size_t(_abi.ERR_CAP)


def build(force: bool = False) -> str:
    srcs = [os.path.join(_HERE, "rnmf_oracle.cpp"), os.path.join(_HERE, "rnmf_oracle.h")]
    if force or not os.path.exists(LIB_PATH) or any(
        os.path.getmtime(s) > os.path.getmtime(LIB_PATH) for s in srcs
    ):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = ctypes.CDLL(LIB_PATH)
        _lib.oracle_rng_split_seed.restype = ctypes.c_uint64
        _lib.oracle_rng_split_seed.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        _lib.oracle_set_threads.argtypes = [ctypes.c_int]
        _lib.oracle_set_threads.restype = None
    return _lib


def set_threads(n: int) -> None:
    lib().oracle_set_threads(int(n))


def _dp(a):
    if a is None:
        return None
    return a.ctypes.data_as(_D)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.float64))


def options(**kw) -> SolverOptionsC:
    o = SolverOptionsC()
    o.rank = 0
    o.max_iter = 200
    o.tol = 1e-4
    o.init = 0
    o.order = 1
    o.stopping = 0
    o.reseed_dead = 0
    o.reg = RegConfigC(0.0, 0.0, 0.0, 0.0)
    o.seed = 0
    o.trace_full_every = 10
    o.oversampling = 20
    o.power_iterations = 2
    o.math_mode = 0
    for k, v in kw.items():
        if k == "reg":
            v = RegConfigC(*v) if not isinstance(v, RegConfigC) else v
        setattr(o, k, int(v) if isinstance(v, (bool, np.bool_)) else v)
    return o


def _opts(opts):
    if isinstance(opts, SolverOptionsC):
        return opts
    if isinstance(opts, dict):
        return options(**opts)
    # api.SolverOptions-like object
    return opts.to_c()


def trace_to_dicts(buf, n) -> list[dict]:
    return [
        {name: getattr(buf[i], name) for name, _ in TraceRecordC._fields_} for i in range(n)
    ]


# ---- Rng / fills -----------------------------------------------------------------------------
def rng_split_seed(seed: int, stream: int) -> int:
    return int(lib().oracle_rng_split_seed(seed, stream))


def rng_u64(seed: int, count: int) -> np.ndarray:
    out = np.empty(count, dtype=np.uint64)
    lib().oracle_rng_u64(ctypes.c_uint64(seed), _I64(count), out.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    return out


def rng_uniform(seed: int, count: int) -> np.ndarray:
    out = np.empty(count)
    lib().oracle_rng_uniform(ctypes.c_uint64(seed), _I64(count), _dp(out))
    return out


def rng_gaussian(seed: int, count: int) -> np.ndarray:
    out = np.empty(count)
    lib().oracle_rng_gaussian(ctypes.c_uint64(seed), _I64(count), _dp(out))
    return out


def uniform_matrix(seed: int, rows: int, cols: int) -> np.ndarray:
    out = np.empty((max(rows, 0), max(cols, 0)))
    e = err_buffer()
    st = lib().oracle_uniform_matrix(ctypes.c_uint64(seed), _I64(rows), _I64(cols), _dp(out), e, _CAP)
    raise_for_status(st, e)
    return out


def gaussian_matrix(seed: int, rows: int, cols: int) -> np.ndarray:
    out = np.empty((max(rows, 0), max(cols, 0)))
    e = err_buffer()
    st = lib().oracle_gaussian_matrix(ctypes.c_uint64(seed), _I64(rows), _I64(cols), _dp(out), e, _CAP)
    raise_for_status(st, e)
    return out


# ---- core ------------------------------------------------------------------------------------
def economic_qr(a):
    a = _f64(a)
    m, l = a.shape
    q = np.empty((m, l))
    r = np.empty((l, l))
    e = err_buffer()
    st = lib().oracle_economic_qr(_dp(a), _I64(m), _I64(l), _dp(q), _dp(r), e, _CAP)
    raise_for_status(st, e)
    return q, r


def synth_lowrank(rows: int, cols: int, rank: int, noise: float, seed: int) -> np.ndarray:
    out = np.empty((rows, cols))
    e = err_buffer()
    st = lib().oracle_synth_lowrank(_I64(rows), _I64(cols), _I64(rank), ctypes.c_double(noise),
                                    ctypes.c_uint64(seed), _dp(out), e, _CAP)
    raise_for_status(st, e)
    return out


# ---- sketch ----------------------------------------------------------------------------------
def sketch_width(rows, cols, target_rank, oversampling=20, power_iterations=2, block_size=1024):
    l = _I64(0)
    e = err_buffer()
    st = lib().oracle_sketch_width(_I64(rows), _I64(cols), _I64(target_rank), _I64(oversampling),
                                   _I64(power_iterations), _I64(block_size), ctypes.byref(l), e,
                                   _CAP)
    raise_for_status(st, e)
    return l.value


def rqb(a, target_rank, oversampling=20, power_iterations=2, test_matrix=1, seed=0, omega=None):
    a = _f64(a)
    m, n = a.shape
    l = sketch_width(m, n, target_rank, oversampling, power_iterations)
    q = np.empty((m, l))
    b = np.empty((l, n))
    om = _f64(omega) if omega is not None else None
    lo = _I64(0)
    e = err_buffer()
    st = lib().oracle_rqb(_dp(a), _I64(m), _I64(n), _I64(target_rank), _I64(oversampling),
                          _I64(power_iterations), ctypes.c_int(int(test_matrix)), ctypes.c_uint64(seed),
                          _dp(om), _dp(q), _dp(b), ctypes.byref(lo), e, _CAP)
    raise_for_status(st, e)
    return q, b


def rqb_streaming(a, target_rank, oversampling=20, power_iterations=2, test_matrix=1, seed=0, block_size=1024,
                  omega=None):
    """rqb_streaming (p/src/sketch.cpp:73-116) over the in-memory matrix a, column blocks of block_size."""
    a = _f64(a)
    m, n = a.shape
    lo = _I64(0)
    e = err_buffer()
    args = (_I64(m), _I64(n), _I64(target_rank), _I64(oversampling), _I64(power_iterations),
            ctypes.c_int(int(test_matrix)), _I64(block_size), ctypes.c_uint64(seed))
    st = lib().oracle_rqb_streaming(_dp(a), *args, None, None, None, ctypes.byref(lo), e, _CAP)
    raise_for_status(st, e)
    l = lo.value
    q = np.empty((m, l))
    b = np.empty((l, n))
    om = _f64(omega) if omega is not None else None
    st = lib().oracle_rqb_streaming(_dp(a), *args, _dp(om), _dp(q), _dp(b), ctypes.byref(lo), e, _CAP)
    raise_for_status(st, e)
    return q, b


# ---- deterministic helpers -----------------------------------------------------------------
def init_factors(x, rank, scheme=0, seed=0):
    x = _f64(x)
    m, n = x.shape
    w = np.empty((m, max(rank, 0)))
    h = np.empty((max(rank, 0), n))
    e = err_buffer()
    st = lib().oracle_init_factors(_dp(x), _I64(m), _I64(n), _I64(rank), ctypes.c_int(int(scheme)),
                                   ctypes.c_uint64(seed), _dp(w), _dp(h), e, _CAP)
    raise_for_status(st, e)
    return w, h


def _reg(reg):
    if reg is None:
        return RegConfigC(0.0, 0.0, 0.0, 0.0)
    if isinstance(reg, RegConfigC):
        return reg
    if isinstance(reg, (tuple, list)):
        return RegConfigC(*reg)
    return RegConfigC(reg.alpha_w, reg.alpha_h, reg.beta_w, reg.beta_h)


def update_W(x, w, h, reg=None):
    x, w, h = _f64(x), _f64(w), _f64(h)
    m, n = x.shape
    k = w.shape[1]
    if h.shape[0] != k or w.shape[0] != m or h.shape[1] != n:
        raise _abi.ShapeError(f"update_W: inconsistent shapes X={m}x{n}, W={w.shape[0]}x{w.shape[1]}, H={h.shape[0]}x{h.shape[1]}")
    out = np.empty_like(w)
    e = err_buffer()
    r = _reg(reg)
    st = lib().oracle_update_W(_dp(x), _I64(m), _I64(n), _I64(k), _dp(w), _dp(h), ctypes.byref(r), _dp(out), e, _CAP)
    raise_for_status(st, e)
    return out


def update_H(x, w, h, reg=None):
    x, w, h = _f64(x), _f64(w), _f64(h)
    m, n = x.shape
    k = w.shape[1]
    if h.shape[0] != k or w.shape[0] != m or h.shape[1] != n:
        raise _abi.ShapeError(f"update_H: inconsistent shapes X={m}x{n}, W={w.shape[0]}x{w.shape[1]}, H={h.shape[0]}x{h.shape[1]}")
    out = np.empty_like(h)
    e = err_buffer()
    r = _reg(reg)
    st = lib().oracle_update_H(_dp(x), _I64(m), _I64(n), _I64(k), _dp(w), _dp(h), ctypes.byref(r), _dp(out), e, _CAP)
    raise_for_status(st, e)
    return out


def objective(x, w, h):
    x, w, h = _f64(x), _f64(w), _f64(h)
    out = ctypes.c_double(0)
    e = err_buffer()
    st = lib().oracle_objective(_dp(x), _I64(x.shape[0]), _I64(x.shape[1]), _I64(w.shape[1]), _dp(w), _dp(h), ctypes.byref(out), e, _CAP)
    raise_for_status(st, e)
    return out.value


def projected_gradient_norm(x, w, h):
    x, w, h = _f64(x), _f64(w), _f64(h)
    out = ctypes.c_double(0)
    e = err_buffer()
    st = lib().oracle_projected_gradient_norm(_dp(x), _I64(x.shape[0]), _I64(x.shape[1]), _I64(w.shape[1]), _dp(w), _dp(h), ctypes.byref(out), e, _CAP)
    raise_for_status(st, e)
    return out.value


@dataclass
class FitResult:
    w: np.ndarray
    h: np.ndarray
    trace: list


def hals_fit(x, opts) -> FitResult:
    x = _f64(x)
    o = _opts(opts)
    m, n = x.shape
    k = max(int(o.rank), 0)
    w = np.empty((m, k))
    h = np.empty((k, n))
    cap = max(int(o.max_iter), 0) + 1
    buf = (TraceRecordC * cap)()
    ln = _I64(0)
    e = err_buffer()
    st = lib().oracle_hals_fit(_dp(x), _I64(m), _I64(n), ctypes.byref(o), _dp(w), _dp(h), buf, _I64(cap), ctypes.byref(ln), e, _CAP)
    raise_for_status(st, e)
    return FitResult(w, h, trace_to_dicts(buf, ln.value))


# ---- randomized HALS -------------------------------------------------------------------------
@dataclass
class CompressedProblem:
    q: np.ndarray
    b: np.ndarray
    wt: np.ndarray
    w: np.ndarray
    h: np.ndarray

    def copy(self):
        return CompressedProblem(self.q.copy(), self.b.copy(), self.wt.copy(), self.w.copy(), self.h.copy())

    def shape_c(self) -> ProblemShapeC:
        return ProblemShapeC(*self.q.shape, *self.b.shape, *self.wt.shape, *self.w.shape, *self.h.shape)


def compress(x, opts, omega=None, w0=None, h0=None) -> CompressedProblem:
    x = _f64(x)
    o = _opts(opts)
    m, n = x.shape
    k = max(int(o.rank), 0)
    try:
        l = sketch_width(m, n, k, o.oversampling, o.power_iterations)
    except _abi.ParameterError:
        l = 1  # let the oracle raise in the reference order (data errors first)
    q, b = np.empty((m, l)), np.empty((l, n))
    wt, w, h = np.empty((l, k)), np.empty((m, k)), np.empty((k, n))
    lo = _I64(0)
    e = err_buffer()
    om, a0, b0 = (_f64(v) if v is not None else None for v in (omega, w0, h0))
    st = lib().oracle_compress(_dp(x), _I64(m), _I64(n), ctypes.byref(o), _dp(om), _dp(a0), _dp(b0),
                               _dp(q), _dp(b), _dp(wt), _dp(w), _dp(h), ctypes.byref(lo), e, _CAP)
    raise_for_status(st, e)
    return CompressedProblem(q, b, wt, w, h)


def rhals_update_W(cp: CompressedProblem, reg=None) -> None:
    for name in ("q", "b", "wt", "w", "h"):
        setattr(cp, name, _f64(getattr(cp, name)))
    r = _reg(reg)
    e = err_buffer()
    s = cp.shape_c()
    st = lib().oracle_rhals_update_W(ctypes.byref(s), _dp(cp.q), _dp(cp.b), _dp(cp.wt), _dp(cp.w), _dp(cp.h), ctypes.byref(r), e, _CAP)
    raise_for_status(st, e)


def rhals_update_H(cp: CompressedProblem, reg=None) -> None:
    for name in ("q", "b", "wt", "w", "h"):
        setattr(cp, name, _f64(getattr(cp, name)))
    r = _reg(reg)
    e = err_buffer()
    s = cp.shape_c()
    st = lib().oracle_rhals_update_H(ctypes.byref(s), _dp(cp.q), _dp(cp.b), _dp(cp.wt), _dp(cp.w), _dp(cp.h), ctypes.byref(r), e, _CAP)
    raise_for_status(st, e)


def rhals_fit(x, opts, omega=None, w0=None, h0=None) -> FitResult:
    x = _f64(x)
    o = _opts(opts)
    m, n = x.shape
    k = max(int(o.rank), 0)
    w, h = np.empty((m, k)), np.empty((k, n))
    cap = max(int(o.max_iter), 0) + 1
    buf = (TraceRecordC * cap)()
    ln = _I64(0)
    e = err_buffer()
    om, a0, b0 = (_f64(v) if v is not None else None for v in (omega, w0, h0))
    st = lib().oracle_rhals_fit(_dp(x), _I64(m), _I64(n), ctypes.byref(o), _dp(om), _dp(a0), _dp(b0),
                                _dp(w), _dp(h), buf, _I64(cap), ctypes.byref(ln), e, _CAP)
    raise_for_status(st, e)
    return FitResult(w, h, trace_to_dicts(buf, ln.value))


def rhals_fit_compressed(x, opts, cp: CompressedProblem) -> FitResult:
    x = _f64(x)
    o = _opts(opts)
    m, n = x.shape
    cp = cp.copy()
    for name in ("q", "b", "wt", "w", "h"):
        setattr(cp, name, _f64(getattr(cp, name)))
    cap = max(int(o.max_iter), 0) + 1
    buf = (TraceRecordC * cap)()
    ln = _I64(0)
    e = err_buffer()
    s = cp.shape_c()
    st = lib().oracle_rhals_fit_compressed(_dp(x), _I64(m), _I64(n), ctypes.byref(o), ctypes.byref(s),
                                           _dp(cp.q), _dp(cp.b), _dp(cp.wt), _dp(cp.w), _dp(cp.h),
                                           buf, _I64(cap), ctypes.byref(ln), e, _CAP)
    raise_for_status(st, e)
    return FitResult(cp.w, cp.h, trace_to_dicts(buf, ln.value))
