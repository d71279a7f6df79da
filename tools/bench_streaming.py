#!/usr/bin/env python
"""Measure the GPU column-streamed sketch (rqb_streaming, fp64) on the C2-shaped matrix: in-memory
source (Python ColumnSource callback) and RNMFMAT1 file source, against the fp64 oracle's
restatement on the host.  Prints one JSON line.  Development / reporting aid (not the driver bench)."""
import json
import os
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    from oracle import oracle as orc
    from paper_1711_02037_b200 import api, workloads

    x = workloads.faces_matrix(0).astype(np.float64)
    m, n = x.shape
    o = api.SketchOptions(target_rank=16, oversampling=20, power_iterations=2, seed=0, block_size=1024)
    passes = 2 + o.power_iterations
    src_bytes = passes * x.nbytes
    ctx = api.Context(0)
    api.rqb_streaming(x, o, ctx=ctx)  # warm-up (allocations, pinned staging)
    t = time.perf_counter()
    r = api.rqb_streaming(x, o, ctx=ctx)
    t_mem = time.perf_counter() - t
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "x.bin")
        api.write_matrix_bin(path, x)
        api.rqb_streaming(api.FileColumnSource(path), o, ctx=ctx)
        t = time.perf_counter()
        rf = api.rqb_streaming(api.FileColumnSource(path), o, ctx=ctx)
        t_file = time.perf_counter() - t
    threads = os.cpu_count() or 1
    orc.set_threads(threads)
    t = time.perf_counter()
    qo, bo = orc.rqb_streaming(x, 16, 20, 2, seed=0, block_size=1024)
    t_orc = time.perf_counter() - t
    dev = float(np.abs(r.q @ r.b - qo @ bo).max() / np.abs(x).max())
    print(json.dumps({
        "workload": f"rqb_streaming C2 shape {m}x{n} fp64, l=36, q=2, block 1024 columns ({passes} passes)",
        "gpu_memory_source_s": t_mem, "gpu_memory_source_gbs": src_bytes / t_mem / 1e9,
        "gpu_file_source_s": t_file, "gpu_file_source_gbs": src_bytes / t_file / 1e9,
        "oracle_s": t_orc, "oracle_threads": threads, "speedup_vs_oracle": t_orc / t_mem,
        "max_abs_dev_qb_vs_oracle_rel": dev, "file_equals_memory": bool(np.array_equal(rf.q, r.q)),
    }))


if __name__ == "__main__":
    main()
