"""Loader for the in-tree sm_100a library lib/librnmf_gpu.so (no fallback: fails loudly)."""
from __future__ import annotations

import ctypes
import os

from ._abi import ProblemShapeC, RegConfigC, SolverOptionsC, StageTimesC, TraceRecordC

HERE = os.path.dirname(os.path.abspath(__file__))
# RNMF_GPU_LIB: development override (e.g. a build with the sweep-kernel cycle profile compiled in)
LIB_PATH = os.environ.get("RNMF_GPU_LIB") or os.path.join(HERE, "lib", "librnmf_gpu.so")
HEADER_PATH = os.path.join(os.path.dirname(HERE), "include", "rnmf_gpu.h")

_lib = None

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int
_sz = ctypes.c_size_t
_cp = ctypes.c_char_p
_dp = ctypes.POINTER(ctypes.c_double)
_i64p = ctypes.POINTER(ctypes.c_int64)
# rnmf_column_reader: int (*)(void* user, int64_t first, int64_t count, double* dst)
COLUMN_READER = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_int64, ctypes.c_int64,
                                 ctypes.POINTER(ctypes.c_double))

_SIGS = {
    "rnmf_version": (_i32, [_cp, _sz]),
    "rnmf_default_options": (None, [ctypes.POINTER(SolverOptionsC)]),
    "rnmf_gpu_device_count": (_i32, []),
    "rnmf_gpu_context_create": (_i32, [_i32, ctypes.POINTER(_vp), _cp, _sz]),
    "rnmf_gpu_context_destroy": (None, [_vp]),
    "rnmf_gpu_last_stage_times": (_i32, [_vp, ctypes.POINTER(StageTimesC)]),
    "rnmf_gpu_rhals_fit": (
        _i32,
        [_vp, _vp, _i32, _i32, _i64, _i64, ctypes.POINTER(SolverOptionsC), _dp, _dp, _dp, _vp, _vp,
         ctypes.POINTER(TraceRecordC), _i64, _i64p, _cp, _sz],
    ),
    "rnmf_gpu_hals_fit": (
        _i32,
        [_vp, _vp, _i32, _i32, _i64, _i64, ctypes.POINTER(SolverOptionsC), _dp, _dp, _vp, _vp,
         ctypes.POINTER(TraceRecordC), _i64, _i64p, _cp, _sz],
    ),
    "rnmf_gpu_comm_unique_id": (_i32, [ctypes.c_char_p, _cp, _sz]),
    "rnmf_gpu_context_create_sharded": (_i32, [_i32, _i32, _i32, ctypes.c_char_p, ctypes.POINTER(_vp), _cp, _sz]),
    "rnmf_gpu_rhals_fit_sharded": (
        _i32,
        [_vp, _vp, _i32, _i32, _i64, _i64, _i64, _i64, ctypes.POINTER(SolverOptionsC), _dp, _dp, _dp, _vp, _vp,
         ctypes.POINTER(TraceRecordC), _i64, _i64p, _cp, _sz],
    ),
    "rnmf_gpu_rhals_fit_compressed": (
        _i32,
        [_vp, _vp, _i32, _i32, _i64, _i64, ctypes.POINTER(SolverOptionsC), ctypes.POINTER(ProblemShapeC),
         _vp, _vp, _vp, _vp, _vp, ctypes.POINTER(TraceRecordC), _i64, _i64p, _cp, _sz],
    ),
    "rnmf_gpu_compress": (
        _i32,
        [_vp, _vp, _i32, _i32, _i64, _i64, ctypes.POINTER(SolverOptionsC), _dp, _dp, _dp, _vp, _vp, _vp, _vp,
         _vp, _i64p, _cp, _sz],
    ),
    "rnmf_gpu_rqb": (
        _i32,
        [_vp, _vp, _i32, _i32, _i64, _i64, _i64, _i64, _i64, _i32, ctypes.c_uint64, _dp, _i32, _vp, _vp, _i64p,
         _cp, _sz],
    ),
    "rnmf_gpu_rqb_streaming": (
        _i32,
        [_vp, COLUMN_READER, _vp, _i64, _i64, _i64, _i64, _i64, _i32, _i64, ctypes.c_uint64, _dp, _dp, _dp, _i64p,
         _cp, _sz],
    ),
    "rnmf_gpu_rqb_streaming_file": (
        _i32,
        [_vp, _cp, _i64, _i64, _i64, _i32, _i64, ctypes.c_uint64, _dp, _dp, _dp, _i64p, _i64p, _i64p, _cp, _sz],
    ),
    "rnmf_gpu_rhals_update_W": (
        _i32,
        [_vp, _i32, _i32, ctypes.POINTER(ProblemShapeC), _vp, _vp, _vp, _vp, _vp, ctypes.POINTER(RegConfigC),
         _cp, _sz],
    ),
    "rnmf_gpu_rhals_update_H": (
        _i32,
        [_vp, _i32, _i32, ctypes.POINTER(ProblemShapeC), _vp, _vp, _vp, _vp, _vp, ctypes.POINTER(RegConfigC),
         _cp, _sz],
    ),
}

EXPORTED = tuple(_SIGS)


def lib():
    """The loaded CUDA library.  Raises if it was not built (there is no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -m paper_1711_02037_b200.build` "
                "(the B200 path has no CPU fallback)"
            )
        l = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(l, name)
            fn.restype = res
            fn.argtypes = args
        _lib = l
    return _lib
