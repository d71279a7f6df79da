"""The header-only C++ face (include/rnmf_gpu.hpp): compiles and links against the library on CPU;
on a B200 the demo runs a fit, rqb vs rqb_streaming and the exception mapping."""
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_1711_02037_b200", "lib")


def _build(tmp_path):
    exe = tmp_path / "wrapper_demo"
    cmd = ["g++", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "include"),
           os.path.join(ROOT, "tests", "cpp", "wrapper_demo.cpp"), "-L", LIBDIR, "-lrnmf_gpu",
           f"-Wl,-rpath,{LIBDIR}", "-o", str(exe)]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    return exe


def test_cpp_wrapper_compiles_and_links(tmp_path):
    if not os.path.exists(os.path.join(LIBDIR, "librnmf_gpu.so")):
        pytest.skip("library not built")
    assert _build(tmp_path).exists()


@pytest.mark.gpu
def test_cpp_wrapper_runs(tmp_path):
    out = subprocess.run([str(_build(tmp_path))], check=True, capture_output=True, text=True).stdout
    kv = dict(re.findall(r"(\w+)=(\S+)", out))
    assert int(kv["records"]) == 31
    assert 0.0 < float(kv["final_rel_err"]) < 0.1
    assert float(kv["qb_dev"]) < 1e-9
    assert kv["data_error"] == "1" and kv["parameter_error"] == "1"
