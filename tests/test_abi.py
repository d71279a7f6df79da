"""CPU-side checks of the drop-in boundary: the C-ABI library loads, exports every entry point
include/rnmf_gpu.h declares, reports its version/defaults, and fails loudly without a GPU
(there is no CPU fallback)."""
import ctypes
import re

import pytest

from paper_1711_02037_b200 import _abi, _lib


def _declared_functions():
    text = open(_lib.HEADER_PATH).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rnmf_[A-Za-z0-9_]+)\s*\(", text)))


def test_header_declares_expected_api():
    names = _declared_functions()
    for n in ("rnmf_gpu_rhals_fit", "rnmf_gpu_compress", "rnmf_gpu_rqb", "rnmf_gpu_rhals_update_W",
              "rnmf_gpu_rhals_update_H", "rnmf_gpu_rhals_fit_compressed", "rnmf_gpu_context_create"):
        assert n in names


def test_library_exports_every_declared_symbol():
    lib = _lib.lib()
    for n in _declared_functions():
        assert hasattr(lib, n), f"{n} declared in include/rnmf_gpu.h but not exported"
    assert set(_declared_functions()) == set(_lib.EXPORTED)


def test_struct_layouts_match_header():
    # 8-byte aligned PODs; sizes pinned so a header change is caught on both sides
    assert ctypes.sizeof(_abi.RegConfigC) == 32
    assert ctypes.sizeof(_abi.SolverOptionsC) == 8 * 3 + 4 * 4 + 32 + 8 * 4 + 4 * 2
    assert ctypes.sizeof(_abi.TraceRecordC) == 56
    assert ctypes.sizeof(_abi.ProblemShapeC) == 80


def test_version_and_defaults():
    from paper_1711_02037_b200 import api

    assert api.version().startswith("rnmf-b200")
    o = _abi.SolverOptionsC()
    _lib.lib().rnmf_default_options(ctypes.byref(o))
    # p/include/rnmf/hals.hpp:22-38
    assert (o.rank, o.max_iter, o.tol, o.init, o.order, o.stopping, o.reseed_dead, o.seed,
            o.trace_full_every, o.oversampling, o.power_iterations) == (0, 200, 1e-4, 0, 1, 0, 0, 0, 10, 20, 2)
    d = api.SolverOptions().to_c()
    for f, _ in _abi.SolverOptionsC._fields_:
        if f == "reg":
            continue
        assert getattr(d, f) == getattr(o, f), f


def test_no_gpu_fails_loudly():
    from paper_1711_02037_b200 import api

    if api.device_count() > 0:
        pytest.skip("a GPU is visible")
    with pytest.raises(_abi.CudaError, match="no CPU fallback"):
        api.Context(0)
    import numpy as np

    with pytest.raises(_abi.CudaError):
        api.rhals_fit(np.ones((10, 8)), api.SolverOptions(rank=2))
