"""Python mirror of the reference rnmf C++ API for the randomized-HALS hot path, running on B200.

Reference interface (p/ = /root/reference/proj/):
  rnmf::rhals_fit(X, SolverOptions) -> FitResult{FactorPair{W, H}, trace}   p/include/rnmf/rhals.hpp:40
  rnmf::compress(X, SolverOptions) -> CompressedProblem{q, b, wt, w, h}    p/include/rnmf/rhals.hpp:22
  rnmf::rhals_update_W(cp, reg) / rhals_update_H(cp, reg)                  p/include/rnmf/rhals.hpp:27,33
  rnmf::rqb(A, SketchOptions) -> SketchResult{q, b}                        p/include/rnmf/sketch.hpp:64

Every call goes through the C ABI of lib/librnmf_gpu.so (include/rnmf_gpu.h); all arithmetic runs
in the sm_100a kernels.  Matrices may be numpy arrays (host memory, results returned as numpy) or
torch CUDA tensors (device memory, results returned as torch tensors on the same device).  The
element type follows X: float64 -> the fp64 path, float32 -> the fp32 path.
"""
from __future__ import annotations

import ctypes
import dataclasses
import sys
from dataclasses import dataclass, field
from typing import Any, List, Optional

import numpy as np

from . import _abi
from ._abi import (
    DataError,
    InitScheme,
    IoError,
    MathMode,
    ParameterError,
    ProblemShapeC,
    RegConfigC,
    ShapeError,
    SolverOptionsC,
    StageTimesC,
    StoppingRule,
    TestMatrixKind,
    TraceRecordC,
    UpdateOrder,
    err_buffer,
    raise_for_status,
)
from . import _lib as _lib_mod
from ._lib import lib

__all__ = [
    "RegConfig", "SolverOptions", "SketchOptions", "TraceRecord", "FactorPair", "FitResult",
    "CompressedProblem", "SketchResult", "Context", "rhals_fit", "rhals_fit_compressed", "compress",
    "rhals_update_W", "rhals_update_H", "rqb", "last_stage_times", "device_count", "version",
    "ShapeError", "ParameterError", "DataError", "IoError", "InitScheme", "UpdateOrder",
    "StoppingRule", "TestMatrixKind", "MathMode", "ColumnSource", "MatrixColumnSource", "FileColumnSource",
    "rqb_streaming", "write_matrix_bin",
]

_CAP = ctypes.c_size_t(_abi.ERR_CAP)


# ---- option / result types (p/include/rnmf/hals.hpp:15-63, sketch.hpp:9-22) ----------------------
@dataclass
class RegConfig:
    alpha_w: float = 0.0
    alpha_h: float = 0.0
    beta_w: float = 0.0
    beta_h: float = 0.0

    def to_c(self) -> RegConfigC:
        return RegConfigC(self.alpha_w, self.alpha_h, self.beta_w, self.beta_h)


@dataclass
class SolverOptions:
    rank: int = 0
    max_iter: int = 200
    tol: float = 1e-4
    init: InitScheme = InitScheme.Random
    order: UpdateOrder = UpdateOrder.Grouped
    stopping: StoppingRule = StoppingRule.ProjectedGradient
    reg: RegConfig = field(default_factory=RegConfig)
    seed: int = 0
    reseed_dead: bool = False
    trace_full_every: int = 10
    oversampling: int = 20
    power_iterations: int = 2
    math_mode: MathMode = MathMode.Exact  # GPU-only (include/rnmf_gpu.h)

    def to_c(self) -> SolverOptionsC:
        o = SolverOptionsC()
        o.rank = int(self.rank)
        o.max_iter = int(self.max_iter)
        o.tol = float(self.tol)
        o.init = int(self.init)
        o.order = int(self.order)
        o.stopping = int(self.stopping)
        o.reseed_dead = int(bool(self.reseed_dead))
        o.reg = self.reg.to_c() if isinstance(self.reg, RegConfig) else RegConfigC(*self.reg)
        o.seed = int(self.seed) & 0xFFFFFFFFFFFFFFFF
        o.trace_full_every = int(self.trace_full_every)
        o.oversampling = int(self.oversampling)
        o.power_iterations = int(self.power_iterations)
        o.math_mode = int(self.math_mode)
        return o


@dataclass
class SketchOptions:
    target_rank: int = 0
    oversampling: int = 20
    power_iterations: int = 2
    test_matrix: TestMatrixKind = TestMatrixKind.Gaussian
    block_size: int = 1024
    seed: int = 0


@dataclass
class TraceRecord:
    iter: int = 0
    elapsed_s: float = 0.0
    objective: float = 0.0
    rel_err: float = 0.0
    pgrad: float = 0.0
    pgrad_full: float = 0.0
    objective_compressed: float = 0.0


@dataclass
class FactorPair:
    w: Any
    h: Any


@dataclass
class FitResult:
    factors: FactorPair
    trace: List[TraceRecord]


@dataclass
class CompressedProblem:
    q: Any
    b: Any
    wt: Any
    w: Any
    h: Any


@dataclass
class SketchResult:
    q: Any
    b: Any


# ---- context -----------------------------------------------------------------------------------
def device_count() -> int:
    return int(lib().rnmf_gpu_device_count())


def version() -> str:
    buf = ctypes.create_string_buffer(256)
    lib().rnmf_version(buf, ctypes.c_size_t(256))
    return buf.value.decode()


class Context:
    """Owns a CUDA stream and device workspaces on one GPU (rnmf_gpu_context)."""

    def __init__(self, device: int = 0):
        self.device = int(device)
        h = ctypes.c_void_p()
        e = err_buffer()
        st = lib().rnmf_gpu_context_create(self.device, ctypes.byref(h), e, _CAP)
        raise_for_status(st, e)
        self._h = h

    @property
    def handle(self) -> ctypes.c_void_p:
        if self._h is None:
            raise RuntimeError("context destroyed")
        return self._h

    def close(self) -> None:
        if getattr(self, "_h", None) is not None:
            lib().rnmf_gpu_context_destroy(self._h)
            self._h = None

    def __del__(self):  # pragma: no cover - interpreter teardown
        try:
            self.close()
        except Exception:
            pass

    def stage_times(self) -> dict:
        t = StageTimesC()
        lib().rnmf_gpu_last_stage_times(self.handle, ctypes.byref(t))
        return t.as_dict()


_default_ctx: dict = {}


def _ctx_for(device: int, ctx: Optional[Context]) -> Context:
    if ctx is not None:
        return ctx
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


def last_stage_times(ctx: Optional[Context] = None, device: int = 0) -> dict:
    return _ctx_for(device, ctx).stage_times()


# ---- array plumbing ----------------------------------------------------------------------------
class _Mat:
    """A matrix argument: host numpy or device torch tensor, C-contiguous."""

    def __init__(self, a, dtype=None, name="matrix"):
        self.torch = _is_torch(a)
        if self.torch:
            import torch

            if not a.is_cuda:
                a = a.detach().cpu().numpy()
                self.torch = False
            else:
                if dtype is not None and a.dtype != (torch.float32 if dtype == np.float32 else torch.float64):
                    a = a.to(torch.float32 if dtype == np.float32 else torch.float64)
                if a.dtype not in (torch.float32, torch.float64):
                    a = a.to(torch.float64)
                a = a.contiguous()
                self.arr = a
                self.np_dtype = np.float32 if a.dtype == torch.float32 else np.float64
                self.device = a.device.index if a.device.index is not None else torch.cuda.current_device()
                self.shape = tuple(a.shape)
                return
        arr = np.asarray(a)
        if dtype is not None:
            arr = arr.astype(dtype, copy=False)
        elif arr.dtype not in (np.float32, np.float64):
            arr = arr.astype(np.float64)
        self.arr = np.ascontiguousarray(arr)
        self.np_dtype = self.arr.dtype.type
        self.device = None
        self.shape = self.arr.shape
        if self.arr.ndim != 2:
            raise ShapeError(f"{name}: expected a 2-D matrix, got shape {self.shape}")

    @property
    def ptr(self) -> int:
        return self.arr.data_ptr() if self.torch else self.arr.ctypes.data

    @property
    def dtype_code(self) -> int:
        return _abi.RNMF_F32 if self.np_dtype == np.float32 else _abi.RNMF_F64

    @property
    def location(self) -> int:
        return _abi.RNMF_DEVICE if self.torch else _abi.RNMF_HOST

    def empty(self, rows, cols):
        if self.torch:
            import torch

            return torch.empty((rows, cols), dtype=self.arr.dtype, device=self.arr.device)
        return np.empty((rows, cols), dtype=self.np_dtype)


def _is_torch(a) -> bool:
    mod = type(a).__module__
    return mod.startswith("torch")


def _ptr(a) -> int:
    return a.data_ptr() if _is_torch(a) else a.ctypes.data


def _f64_host(a, rows, cols, name):
    if a is None:
        return None
    if _is_torch(a):
        a = a.detach().cpu().numpy()
    arr = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    if arr.shape != (rows, cols):
        raise ShapeError(f"{name}: expected {rows}x{cols}, got {'x'.join(map(str, arr.shape))}")
    return arr


def _dptr(arr):
    return None if arr is None else arr.ctypes.data_as(ctypes.POINTER(ctypes.c_double))


def _sync_torch(m: _Mat) -> None:
    if m.torch:
        import torch

        torch.cuda.synchronize(m.arr.device)


def _trace_list(buf, n) -> List[TraceRecord]:
    return [
        TraceRecord(**{name: getattr(buf[i], name) for name, _ in TraceRecordC._fields_}) for i in range(n)
    ]


# ---- the hot path --------------------------------------------------------------------------------
def rhals_fit(x, opts: SolverOptions, *, omega=None, w0=None, h0=None, ctx: Optional[Context] = None) -> FitResult:
    """rnmf::rhals_fit (p/src/rhals.cpp:121-213) on the GPU.

    omega (n x l), w0 (m x k), h0 (k x n): optional host draws replacing the reference's internal
    random streams (the unscaled init draws are scaled by sqrt(mean(X)/k) as in random_init)."""
    X = _Mat(x, name="X")
    m, n = X.shape
    c = _ctx_for(X.device or 0, ctx)
    o = opts.to_c()
    k = max(int(opts.rank), 0)
    l = _sketch_width_nothrow(m, n, k, opts.oversampling)
    om = _f64_host(omega, n, l, "omega") if omega is not None else None
    a0 = _f64_host(w0, m, k, "w0") if w0 is not None else None
    b0 = _f64_host(h0, k, n, "h0") if h0 is not None else None
    w = X.empty(m, k)
    h = X.empty(k, n)
    cap = max(int(opts.max_iter), 0) + 1
    buf = (TraceRecordC * cap)()
    ln = ctypes.c_int64(0)
    e = err_buffer()
    _sync_torch(X)
    st = lib().rnmf_gpu_rhals_fit(
        c.handle, X.ptr, X.dtype_code, X.location, m, n, ctypes.byref(o), _dptr(om), _dptr(a0), _dptr(b0),
        _ptr(w), _ptr(h), buf, cap, ctypes.byref(ln), e, _CAP)
    raise_for_status(st, e)
    return FitResult(FactorPair(w, h), _trace_list(buf, ln.value))


def hals_fit(x, opts: SolverOptions, *, w0=None, h0=None, ctx: Optional[Context] = None) -> FitResult:
    """rnmf::hals_fit (p/src/hals.cpp:268-323) on the GPU: the deterministic full-space HALS solver
    (UpdateOrder::Grouped), every sweep recorded with the full-space metrics.  w0 / h0 as in
    rhals_fit."""
    X = _Mat(x, name="X")
    m, n = X.shape
    c = _ctx_for(X.device or 0, ctx)
    o = opts.to_c()
    k = max(int(opts.rank), 0)
    a0 = _f64_host(w0, m, k, "w0") if w0 is not None else None
    b0 = _f64_host(h0, k, n, "h0") if h0 is not None else None
    w = X.empty(m, k)
    h = X.empty(k, n)
    cap = max(int(opts.max_iter), 0) + 1
    buf = (TraceRecordC * cap)()
    ln = ctypes.c_int64(0)
    e = err_buffer()
    _sync_torch(X)
    st = lib().rnmf_gpu_hals_fit(c.handle, X.ptr, X.dtype_code, X.location, m, n, ctypes.byref(o), _dptr(a0),
                                 _dptr(b0), _ptr(w), _ptr(h), buf, cap, ctypes.byref(ln), e, _CAP)
    raise_for_status(st, e)
    return FitResult(FactorPair(w, h), _trace_list(buf, ln.value))


def _sketch_width_nothrow(m, n, k, p):
    bound = min(m, n)
    return max(1, min(k + max(p, 0), bound)) if bound > 0 else 1


def compress(x, opts: SolverOptions, *, omega=None, w0=None, h0=None, ctx: Optional[Context] = None) -> CompressedProblem:
    """rnmf::compress (p/src/rhals.cpp:84-105) on the GPU."""
    X = _Mat(x, name="X")
    m, n = X.shape
    c = _ctx_for(X.device or 0, ctx)
    o = opts.to_c()
    k = max(int(opts.rank), 0)
    l = _sketch_width_nothrow(m, n, k, opts.oversampling)
    om = _f64_host(omega, n, l, "omega") if omega is not None else None
    a0 = _f64_host(w0, m, k, "w0") if w0 is not None else None
    b0 = _f64_host(h0, k, n, "h0") if h0 is not None else None
    q, b, wt, w, h = X.empty(m, l), X.empty(l, n), X.empty(l, k), X.empty(m, k), X.empty(k, n)
    lo = ctypes.c_int64(0)
    e = err_buffer()
    _sync_torch(X)
    st = lib().rnmf_gpu_compress(c.handle, X.ptr, X.dtype_code, X.location, m, n, ctypes.byref(o), _dptr(om),
                                 _dptr(a0), _dptr(b0), _ptr(q), _ptr(b), _ptr(wt), _ptr(w), _ptr(h),
                                 ctypes.byref(lo), e, _CAP)
    raise_for_status(st, e)
    return CompressedProblem(q, b, wt, w, h)


def rqb(a, opts: SketchOptions, *, omega=None, ctx: Optional[Context] = None,
        math_mode: int = MathMode.Exact) -> SketchResult:
    """rnmf::rqb (p/src/sketch.cpp:52-71) on the GPU.  `math_mode` selects the arithmetic of the
    X-streaming GEMMs (MathMode; Exact = FMA in the working precision)."""
    A = _Mat(a, name="A")
    m, n = A.shape
    c = _ctx_for(A.device or 0, ctx)
    if opts.block_size < 1:
        # sketch_width's block-size check (p/src/sketch.cpp:40-42); the GPU sketch is in-memory
        raise ParameterError("sketch: block size must be at least 1")
    lo = ctypes.c_int64(0)
    e = err_buffer()
    st = lib().rnmf_gpu_rqb(c.handle, A.ptr, A.dtype_code, A.location, m, n, int(opts.target_rank),
                            int(opts.oversampling), int(opts.power_iterations), int(opts.test_matrix),
                            ctypes.c_uint64(int(opts.seed) & 0xFFFFFFFFFFFFFFFF), None, 0, None, None,
                            ctypes.byref(lo), e, _CAP)
    raise_for_status(st, e)
    l = lo.value
    om = _f64_host(omega, n, l, "omega") if omega is not None else None
    q, b = A.empty(m, l), A.empty(l, n)
    _sync_torch(A)
    st = lib().rnmf_gpu_rqb(c.handle, A.ptr, A.dtype_code, A.location, m, n, int(opts.target_rank),
                            int(opts.oversampling), int(opts.power_iterations), int(opts.test_matrix),
                            ctypes.c_uint64(int(opts.seed) & 0xFFFFFFFFFFFFFFFF), _dptr(om), int(math_mode), _ptr(q), _ptr(b),
                            ctypes.byref(lo), e, _CAP)
    raise_for_status(st, e)
    return SketchResult(q, b)


# ---- column-streamed sketch (rqb_streaming, p/src/sketch.cpp:73-116) -----------------------------
class ColumnSource:
    """rnmf::ColumnSource (p/include/rnmf/sketch.hpp:26-33): rows(), cols() and
    read_columns(first, count, dst) filling dst (rows x count float64, row-major) with columns
    [first, first + count)."""

    def rows(self) -> int:
        raise NotImplementedError

    def cols(self) -> int:
        raise NotImplementedError

    def read_columns(self, first: int, count: int, dst: np.ndarray) -> None:
        raise NotImplementedError


class MatrixColumnSource(ColumnSource):
    """rnmf::MatrixColumnSource (p/include/rnmf/sketch.hpp:41-51): an in-memory matrix."""

    def __init__(self, a):
        self.a = np.asarray(a, dtype=np.float64)
        if self.a.ndim != 2:
            raise ShapeError("MatrixColumnSource: expected a 2-D matrix")

    def rows(self) -> int:
        return int(self.a.shape[0])

    def cols(self) -> int:
        return int(self.a.shape[1])

    def read_columns(self, first: int, count: int, dst: np.ndarray) -> None:
        if first < 0 or count < 1 or first + count > self.cols():
            raise ParameterError(f"read_columns: range [{first}, {first + count}) out of bounds for {self.cols()} columns")
        dst[:, :] = self.a[:, first:first + count]


class FileColumnSource(ColumnSource):
    """rnmf::FileColumnSource (p/include/rnmf/data_io.hpp:32-45) over an RNMFMAT1 binary file.
    rqb_streaming reads it natively (rnmf_gpu_rqb_streaming_file); the header is validated there
    with the reference's messages."""

    def __init__(self, path: str):
        self.path = str(path)


def write_matrix_bin(path: str, a) -> None:
    """RNMFMAT1 writer (p/include/rnmf/data_io.hpp:12-15, write_matrix with MatrixFormat::Bin):
    magic, rows / cols as little-endian u64, row-major little-endian float64 payload."""
    a = np.ascontiguousarray(a, dtype="<f8")
    with open(path, "wb") as f:
        f.write(b"RNMFMAT1")
        f.write(np.array([a.shape[0], a.shape[1]], dtype="<u8").tobytes())
        f.write(a.tobytes())


def rqb_streaming(src, opts: SketchOptions, *, omega=None, ctx: Optional[Context] = None) -> SketchResult:
    """rnmf::rqb_streaming (p/src/sketch.cpp:73-116) on the GPU, fp64: the source is read in column
    blocks of opts.block_size, 2 + power_iterations passes, each block streamed to the device while
    the host reads the next.  Returns host float64 Q (m x l) and B (l x n)."""
    c = _ctx_for(0, ctx)
    e = err_buffer()
    lo = ctypes.c_int64(0)
    seed = ctypes.c_uint64(int(opts.seed) & 0xFFFFFFFFFFFFFFFF)
    if isinstance(src, FileColumnSource):
        path = src.path.encode()
        mo, no = ctypes.c_int64(0), ctypes.c_int64(0)
        args = (int(opts.target_rank), int(opts.oversampling), int(opts.power_iterations), int(opts.test_matrix),
                int(opts.block_size), seed)
        st = lib().rnmf_gpu_rqb_streaming_file(c.handle, path, *args, None, None, None, ctypes.byref(mo),
                                               ctypes.byref(no), ctypes.byref(lo), e, _CAP)
        raise_for_status(st, e)
        m, n, l = mo.value, no.value, lo.value
        om = _f64_host(omega, n, l, "omega") if omega is not None else None
        q = np.empty((m, l), dtype=np.float64)
        b = np.empty((l, n), dtype=np.float64)
        st = lib().rnmf_gpu_rqb_streaming_file(c.handle, path, *args, _dptr(om), _dptr(q), _dptr(b),
                                               ctypes.byref(mo), ctypes.byref(no), ctypes.byref(lo), e, _CAP)
        raise_for_status(st, e)
        return SketchResult(q, b)
    if not isinstance(src, ColumnSource):
        src = MatrixColumnSource(src)
    m, n = int(src.rows()), int(src.cols())
    failure = []

    def _read(_user, first, count, dst):
        try:
            view = np.ctypeslib.as_array(dst, shape=(m * count,)).reshape(m, count)
            src.read_columns(int(first), int(count), view)
            return 0
        except BaseException as exc:  # reported through the status, re-raised below
            failure.append(exc)
            return 1

    reader = _lib_mod.COLUMN_READER(_read)
    args = (int(opts.target_rank), int(opts.oversampling), int(opts.power_iterations), int(opts.test_matrix),
            int(opts.block_size), seed)
    st = lib().rnmf_gpu_rqb_streaming(c.handle, reader, None, m, n, *args, None, None, None, ctypes.byref(lo), e, _CAP)
    raise_for_status(st, e)
    l = lo.value
    om = _f64_host(omega, n, l, "omega") if omega is not None else None
    q = np.empty((m, l), dtype=np.float64)
    b = np.empty((l, n), dtype=np.float64)
    st = lib().rnmf_gpu_rqb_streaming(c.handle, reader, None, m, n, *args, _dptr(om), _dptr(q), _dptr(b),
                                      ctypes.byref(lo), e, _CAP)
    if failure and not isinstance(failure[0], Exception):
        raise failure[0]
    if st != 0 and failure and isinstance(failure[0], (ShapeError, ParameterError, DataError, IoError)):
        raise failure[0]
    raise_for_status(st, e)
    return SketchResult(q, b)


def _cp_mats(cp: CompressedProblem):
    q = _Mat(cp.q, name="Q")
    dt = q.np_dtype
    mats = [q] + [_Mat(getattr(cp, nm), dtype=dt, name=nm) for nm in ("b", "wt", "w", "h")]
    locs = {mm.location for mm in mats}
    if len(locs) != 1:
        raise ParameterError("compressed problem mixes host and device matrices")
    return mats


def _shape_of(mats) -> ProblemShapeC:
    s = []
    for mm in mats:
        s.extend(mm.shape)
    return ProblemShapeC(*s)


def _write_back(cp: CompressedProblem, name: str, mat: _Mat):
    """Store an updated matrix back into cp (in place when cp already holds that exact buffer)."""
    cur = getattr(cp, name)
    if cur is mat.arr:
        return
    if _is_torch(cur) and mat.torch and cur.shape == mat.arr.shape:
        cur.copy_(mat.arr)
    elif isinstance(cur, np.ndarray) and not mat.torch and cur.shape == mat.arr.shape and cur.flags.writeable:
        cur[...] = mat.arr
    else:
        setattr(cp, name, mat.arr)


def rhals_update_W(cp: CompressedProblem, reg: Optional[RegConfig] = None, *, ctx: Optional[Context] = None) -> None:
    """rnmf::rhals_update_W (p/src/rhals.cpp:107-114): W~ and W updated in place."""
    mats = _cp_mats(cp)
    q, b, wt, w, h = mats
    c = _ctx_for(q.device or 0, ctx)
    r = (reg or RegConfig()).to_c()
    s = _shape_of(mats)
    e = err_buffer()
    for mm in mats:
        _sync_torch(mm)
    st = lib().rnmf_gpu_rhals_update_W(c.handle, q.dtype_code, q.location, ctypes.byref(s), q.ptr, b.ptr, wt.ptr,
                                       w.ptr, h.ptr, ctypes.byref(r), e, _CAP)
    raise_for_status(st, e)
    _write_back(cp, "wt", wt)
    _write_back(cp, "w", w)


def rhals_update_H(cp: CompressedProblem, reg: Optional[RegConfig] = None, *, ctx: Optional[Context] = None) -> None:
    """rnmf::rhals_update_H (p/src/rhals.cpp:116-119): H updated in place."""
    mats = _cp_mats(cp)
    q, b, wt, w, h = mats
    c = _ctx_for(q.device or 0, ctx)
    r = (reg or RegConfig()).to_c()
    s = _shape_of(mats)
    e = err_buffer()
    for mm in mats:
        _sync_torch(mm)
    st = lib().rnmf_gpu_rhals_update_H(c.handle, q.dtype_code, q.location, ctypes.byref(s), q.ptr, b.ptr, wt.ptr,
                                       w.ptr, h.ptr, ctypes.byref(r), e, _CAP)
    raise_for_status(st, e)
    _write_back(cp, "h", h)


def rhals_fit_compressed(x, opts: SolverOptions, cp: CompressedProblem, *, ctx: Optional[Context] = None) -> FitResult:
    """The sweep/trace loop of rhals_fit (p/src/rhals.cpp:128-213) from a given compressed problem.
    cp.wt, cp.w, cp.h are updated; the returned factors alias cp.w / cp.h."""
    X = _Mat(x, name="X")
    m, n = X.shape
    mats = [_Mat(getattr(cp, nm), dtype=X.np_dtype, name=nm) for nm in ("q", "b", "wt", "w", "h")]
    if any(mm.location != X.location for mm in mats):
        raise ParameterError("X and the compressed problem must share a location")
    q, b, wt, w, h = mats
    c = _ctx_for(X.device or 0, ctx)
    o = opts.to_c()
    s = _shape_of(mats)
    cap = max(int(opts.max_iter), 0) + 1
    buf = (TraceRecordC * cap)()
    ln = ctypes.c_int64(0)
    e = err_buffer()
    _sync_torch(X)
    st = lib().rnmf_gpu_rhals_fit_compressed(c.handle, X.ptr, X.dtype_code, X.location, m, n, ctypes.byref(o),
                                             ctypes.byref(s), q.ptr, b.ptr, wt.ptr, w.ptr, h.ptr, buf, cap,
                                             ctypes.byref(ln), e, _CAP)
    raise_for_status(st, e)
    _write_back(cp, "wt", wt)
    _write_back(cp, "w", w)
    _write_back(cp, "h", h)
    return FitResult(FactorPair(cp.w, cp.h), _trace_list(buf, ln.value))
