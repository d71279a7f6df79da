"""ctypes mirror of include/rnmf_gpu.h (the C-ABI drop-in boundary).

The enums, option/trace structs and exception classes follow the reference rnmf library:
  * exceptions        p/include/rnmf/types.hpp:22-39
  * InitScheme / UpdateOrder / StoppingRule   p/include/rnmf/hals.hpp:9-11
  * RegConfig / SolverOptions / TraceRecord   p/include/rnmf/hals.hpp:15-56
  * TestMatrixKind / SketchOptions            p/include/rnmf/sketch.hpp:7-17
"""
from __future__ import annotations

import ctypes
import enum

# ---- status codes ------------------------------------------------------------------------
RNMF_OK = 0
RNMF_SHAPE_ERROR = 1
RNMF_PARAMETER_ERROR = 2
RNMF_DATA_ERROR = 3
RNMF_IO_ERROR = 4
RNMF_CUDA_ERROR = 5

RNMF_F32 = 0
RNMF_F64 = 1
RNMF_HOST = 0
RNMF_DEVICE = 1


class InitScheme(enum.IntEnum):
    Random = 0
    Svd = 1


class UpdateOrder(enum.IntEnum):
    Interleaved = 0
    Grouped = 1
    Shuffled = 2


class StoppingRule(enum.IntEnum):
    ProjectedGradient = 0
    Objective = 1


class TestMatrixKind(enum.IntEnum):
    Uniform = 0
    Gaussian = 1


class MathMode(enum.IntEnum):
    """GPU-only arithmetic of the X-streaming GEMMs (see include/rnmf_gpu.h)."""

    Exact = 0
    TF32x3 = 1
    TF32 = 2


# ---- exceptions (same class hierarchy as the reference) ------------------------------------
class ShapeError(ValueError):
    """rnmf::ShapeError (std::invalid_argument), types.hpp:22."""


class ParameterError(ValueError):
    """rnmf::ParameterError (std::invalid_argument), types.hpp:27."""


class DataError(RuntimeError):
    """rnmf::DataError (std::runtime_error), types.hpp:32."""


class IoError(RuntimeError):
    """rnmf::IoError (std::runtime_error), types.hpp:37."""


class CudaError(RuntimeError):
    """CUDA/NCCL failure inside the B200 library (no reference equivalent)."""


_ERRORS = {
    RNMF_SHAPE_ERROR: ShapeError,
    RNMF_PARAMETER_ERROR: ParameterError,
    RNMF_DATA_ERROR: DataError,
    RNMF_IO_ERROR: IoError,
    RNMF_CUDA_ERROR: CudaError,
}


def raise_for_status(status: int, err: ctypes.Array) -> None:
    if status == RNMF_OK:
        return
    msg = err.value.decode("utf-8", "replace")
    raise _ERRORS.get(status, CudaError)(msg)


# ---- POD structs ----------------------------------------------------------------------------
class RegConfigC(ctypes.Structure):
    _fields_ = [
        ("alpha_w", ctypes.c_double),
        ("alpha_h", ctypes.c_double),
        ("beta_w", ctypes.c_double),
        ("beta_h", ctypes.c_double),
    ]


class SolverOptionsC(ctypes.Structure):
    _fields_ = [
        ("rank", ctypes.c_int64),
        ("max_iter", ctypes.c_int64),
        ("tol", ctypes.c_double),
        ("init", ctypes.c_int32),
        ("order", ctypes.c_int32),
        ("stopping", ctypes.c_int32),
        ("reseed_dead", ctypes.c_int32),
        ("reg", RegConfigC),
        ("seed", ctypes.c_uint64),
        ("trace_full_every", ctypes.c_int64),
        ("oversampling", ctypes.c_int64),
        ("power_iterations", ctypes.c_int64),
        ("math_mode", ctypes.c_int32),
        ("reserved0", ctypes.c_int32),
    ]


class TraceRecordC(ctypes.Structure):
    _fields_ = [
        ("iter", ctypes.c_int64),
        ("elapsed_s", ctypes.c_double),
        ("objective", ctypes.c_double),
        ("rel_err", ctypes.c_double),
        ("pgrad", ctypes.c_double),
        ("pgrad_full", ctypes.c_double),
        ("objective_compressed", ctypes.c_double),
    ]


class ProblemShapeC(ctypes.Structure):
    _fields_ = [
        ("q_rows", ctypes.c_int64),
        ("q_cols", ctypes.c_int64),
        ("b_rows", ctypes.c_int64),
        ("b_cols", ctypes.c_int64),
        ("wt_rows", ctypes.c_int64),
        ("wt_cols", ctypes.c_int64),
        ("w_rows", ctypes.c_int64),
        ("w_cols", ctypes.c_int64),
        ("h_rows", ctypes.c_int64),
        ("h_cols", ctypes.c_int64),
    ]


class StageTimesC(ctypes.Structure):
    _fields_ = [
        ("scan_ms", ctypes.c_double),
        ("sketch_ms", ctypes.c_double),
        ("qr_ms", ctypes.c_double),
        ("init_ms", ctypes.c_double),
        ("sweeps_ms", ctypes.c_double),
        ("metrics_ms", ctypes.c_double),
        ("total_ms", ctypes.c_double),
        ("h2d_ms", ctypes.c_double),
        ("d2h_ms", ctypes.c_double),
        ("sketch_bytes", ctypes.c_double),
        ("metrics_bytes", ctypes.c_double),
        ("sketch_passes", ctypes.c_int64),
        ("metrics_passes", ctypes.c_int64),
        ("sweeps", ctypes.c_int64),
        ("kernel_launches", ctypes.c_int64),
        ("xw_ms", ctypes.c_double),
        ("xtw_ms", ctypes.c_double),
        ("xw_launches", ctypes.c_int64),
        ("xtw_launches", ctypes.c_int64),
        ("xw_bytes", ctypes.c_double),
        ("xtw_bytes", ctypes.c_double),
        ("xw_kernel_ms", ctypes.c_double),
        ("xtw_kernel_ms", ctypes.c_double),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


ERR_CAP = 1024


def err_buffer() -> ctypes.Array:
    return ctypes.create_string_buffer(ERR_CAP)
