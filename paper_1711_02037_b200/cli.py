"""`rnmf`-compatible command line for the B200 path: the `fit` and `bench` subcommands of the
reference CLI (p/tools/rnmf_main.cpp:126-295, 330-382) with the same options, output files,
manifests, trace CSV schema (`iter,elapsed_s,objective,rel_err,pgrad`, :76-87) and bench CSV schema
(`method,mean_time_s,speedup_vs_hals,iterations,rel_err`, :288-295), running `hals` / `rhals` on
the GPU through the C ABI.  Matrices are read and written in the reference formats (RNMFMAT1 .bin,
.csv; p/src/data_io.cpp).  GPU-only options: --math (X-pass arithmetic, default exact: fp64
input, the verification mode) and --device.

    python -m paper_1711_02037_b200.cli fit --input x.bin --rank 20 --method rhals \
        --out-w w.csv --out-h h.csv --trace trace.csv
    python -m paper_1711_02037_b200.cli bench --input x.bin --rank 20 --out bench.csv

Exit codes as the reference (:386-395): 0 ok, 2 ParameterError / ShapeError / usage, 1 otherwise.
"""
from __future__ import annotations

import argparse
import datetime
import os
import sys
import time

import numpy as np

from . import api

_MAGIC = b"RNMFMAT1"


def _fmt(v: float) -> str:
    return "%.17g" % v


def _fnv1a64_file(path: str) -> str:
    h = 14695981039346656037
    with open(path, "rb") as f:
        while True:
            buf = f.read(1 << 16)
            if not buf:
                break
            for b in buf:
                h = ((h ^ b) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return "%016x" % h


def _now() -> str:
    return datetime.datetime.now(datetime.timezone.utc).strftime("%Y-%m-%dT%H:%M:%SZ")


def format_from_extension(path: str) -> str:
    ext = os.path.splitext(path)[1]
    if ext in (".bin", ".csv"):
        return ext[1:]
    raise api.ParameterError(f"cannot infer matrix format from '{path}' (expected .csv or .bin)")


def read_matrix(path: str) -> np.ndarray:
    """read_matrix (p/src/data_io.cpp:65-150): RNMFMAT1 or CSV, with the reference's DataError /
    IoError conditions."""
    fmt = format_from_extension(path)
    try:
        f = open(path, "rb")
    except OSError:
        raise api.IoError(f"cannot open '{path}'")
    with f:
        data = f.read()
    if fmt == "bin":
        if data[:8] != _MAGIC:
            raise api.DataError(f"'{path}': bad magic at byte 0 (expected \"RNMFMAT1\")")
        if len(data) < 24:
            raise api.DataError(f"'{path}': truncated header, file ends before byte 24")
        rows, cols = (int(v) for v in np.frombuffer(data[8:24], dtype="<u8"))
        if rows > (1 << 40) or cols > (1 << 40):
            raise api.DataError(f"'{path}': implausible dimensions {rows}x{cols}")
        expected = rows * cols * 8
        got = min(len(data) - 24, expected)
        if got != expected:
            raise api.DataError(f"'{path}': truncated payload, expected {expected} bytes after the header, "
                                f"got {got} (file ends at byte {24 + got})")
        if len(data) > 24 + expected:
            raise api.DataError(f"'{path}': trailing data after byte {24 + expected}")
        a = np.frombuffer(data[24:24 + expected], dtype="<f8").reshape(rows, cols).astype(np.float64)
    else:
        rows_v, cols = [], -1
        lines = data.decode().split("\n")
        for no, line in enumerate(lines, 1):
            line = line.rstrip("\r")
            if line == "" and no == len(lines):
                break
            cells = line.split(",")
            vals = []
            for ci, cell in enumerate(cells):
                try:
                    if cell.strip() != cell or cell == "":
                        raise ValueError
                    vals.append(float(cell))
                except ValueError:
                    raise api.DataError(f"'{path}': line {no}, column {ci + 1}: cannot parse cell '{cell}'")
            if cols < 0:
                cols = len(vals)
            elif len(vals) != cols:
                raise api.DataError(f"'{path}': line {no}: expected {cols} columns, got {len(vals)} (ragged row)")
            rows_v.append(vals)
        if not rows_v:
            raise api.DataError(f"'{path}': empty CSV file")
        a = np.array(rows_v, dtype=np.float64)
    bad = np.argwhere(~np.isfinite(a))
    if bad.size:
        i, j = bad[0]
        raise api.DataError(f"'{path}' contains non-finite entries at ({i},{j})")
    return a


def write_matrix(path: str, a) -> None:
    """write_matrix (p/src/data_io.cpp:38-63,158-165): RNMFMAT1 or CSV with %.17g cells."""
    fmt = format_from_extension(path)
    a = np.asarray(a, dtype=np.float64)
    try:
        if fmt == "bin":
            api.write_matrix_bin(path, a)
        else:
            with open(path, "w") as f:
                for row in a:
                    f.write(",".join(_fmt(v) for v in row) + "\n")
    except OSError:
        raise api.IoError(f"cannot open '{path}' for writing")


def write_manifest(path: str, entries) -> None:
    try:
        with open(path, "w") as f:
            for key, value in entries:
                f.write(f"{key}={value}\n")
    except OSError:
        raise api.IoError(f"cannot open '{path}' for writing")


def write_trace_csv(path: str, trace) -> None:
    """write_trace_csv (p/tools/rnmf_main.cpp:76-87)."""
    try:
        with open(path, "w") as f:
            f.write("iter,elapsed_s,objective,rel_err,pgrad\n")
            for r in trace:
                f.write(f"{int(r.iter)},{_fmt(r.elapsed_s)},{_fmt(r.objective)},{_fmt(r.rel_err)},{_fmt(r.pgrad)}\n")
    except OSError:
        raise api.IoError(f"cannot open '{path}' for writing")


_INIT = {"random": api.InitScheme.Random, "svd": api.InitScheme.Svd}
_ORDER = {"grouped": api.UpdateOrder.Grouped, "interleaved": api.UpdateOrder.Interleaved,
          "shuffled": api.UpdateOrder.Shuffled}
_MATH = {"exact": api.MathMode.Exact, "tf32x3": api.MathMode.TF32x3, "tf32": api.MathMode.TF32}


def solver_options(a) -> api.SolverOptions:
    """solver_options (p/tools/rnmf_main.cpp:145-158) plus the GPU math mode."""
    o = api.SolverOptions(rank=a.rank, max_iter=a.max_iter, tol=a.tol, seed=a.seed, oversampling=a.oversample,
                          power_iterations=a.power)
    o.init = _INIT[a.init]
    o.order = _ORDER[a.order]
    o.reg = api.RegConfig(getattr(a, "alpha_w", 0.0), getattr(a, "alpha_h", 0.0), getattr(a, "beta_w", 0.0),
                          getattr(a, "beta_h", 0.0))
    o.math_mode = _MATH[a.math]
    return o


def _input(x: np.ndarray, math: str):
    # exact: fp64 as the reference; tensor-core modes run on fp32 X
    return x if math == "exact" else x.astype(np.float32)


def _solve(method: str, x, opts, ctx):
    return api.rhals_fit(x, opts, ctx=ctx) if method == "rhals" else api.hals_fit(x, opts, ctx=ctx)


def run_fit(a) -> int:
    """run_fit (p/tools/rnmf_main.cpp:184-207)."""
    started = _now()
    x = read_matrix(a.input)
    opts = solver_options(a)
    ctx = api.Context(a.device)
    res = _solve(a.method, _input(x, a.math), opts, ctx)
    manifest = [("command", "fit"), ("input", a.input), ("rank", str(a.rank)), ("method", a.method),
                ("oversample", str(a.oversample)), ("power", str(a.power)), ("max_iter", str(a.max_iter)),
                ("tol", _fmt(a.tol)), ("init", a.init), ("order", a.order), ("alpha_w", _fmt(a.alpha_w)),
                ("alpha_h", _fmt(a.alpha_h)), ("beta_w", _fmt(a.beta_w)), ("beta_h", _fmt(a.beta_h)),
                ("seed", str(a.seed)), ("out_w", a.out_w), ("out_h", a.out_h), ("trace", a.trace or ""),
                ("input_digest", _fnv1a64_file(a.input)), ("started_at", started), ("version", api.version()),
                ("device", "b200"), ("math", a.math)]
    write_matrix(a.out_w, np.asarray(res.factors.w, dtype=np.float64))
    write_manifest(a.out_w + ".manifest", manifest)
    write_matrix(a.out_h, np.asarray(res.factors.h, dtype=np.float64))
    write_manifest(a.out_h + ".manifest", manifest)
    if a.trace:
        write_trace_csv(a.trace, res.trace)
        write_manifest(a.trace + ".manifest", manifest)
    last = res.trace[-1]
    print(f"fit: method={a.method} iters={last.iter} rel_err={_fmt(last.rel_err)} elapsed_s={_fmt(last.elapsed_s)}")
    return 0


def split_methods(csv: str):
    out = []
    for item in csv.split(","):
        if item not in ("hals", "rhals"):
            raise api.ParameterError(f"unknown method '{item}' (expected hals or rhals)")
        out.append(item)
    return out


def run_bench(a) -> int:
    """run_bench (p/tools/rnmf_main.cpp:229-314): mean wall time of `repeat` fits per method and the
    speed-up against hals."""
    started = _now()
    if a.repeat < 1:
        raise api.ParameterError("--repeat must be at least 1")
    methods = split_methods(a.methods)
    x = _input(read_matrix(a.input), a.math)
    a.alpha_w = a.alpha_h = a.beta_w = a.beta_h = 0.0
    opts = solver_options(a)
    ctx = api.Context(a.device)
    rows = []
    hals_mean = None
    for method in methods:
        total = 0.0
        res = None
        for _ in range(a.repeat):
            t0 = time.perf_counter()
            res = _solve(method, x, opts, ctx)
            total += time.perf_counter() - t0
        mean = total / a.repeat
        rows.append((method, mean, res.trace[-1].iter, res.trace[-1].rel_err))
        if method == "hals":
            hals_mean = mean
    try:
        with open(a.out, "w") as f:
            f.write("method,mean_time_s,speedup_vs_hals,iterations,rel_err\n")
            for method, mean, iters, rel in rows:
                sp = _fmt(hals_mean / mean) if hals_mean is not None else ""
                f.write(f"{method},{_fmt(mean)},{sp},{iters},{_fmt(rel)}\n")
    except OSError:
        raise api.IoError(f"cannot open '{a.out}' for writing")
    write_manifest(a.out + ".manifest",
                   [("command", "bench"), ("input", a.input), ("rank", str(a.rank)), ("methods", a.methods),
                    ("repeat", str(a.repeat)), ("max_iter", str(a.max_iter)), ("tol", _fmt(a.tol)),
                    ("init", a.init), ("order", a.order), ("oversample", str(a.oversample)),
                    ("power", str(a.power)), ("seed", str(a.seed)), ("out", a.out),
                    ("input_digest", _fnv1a64_file(a.input)), ("started_at", started), ("version", api.version()),
                    ("device", "b200"), ("math", a.math)])
    return 0


def _parser():
    ap = argparse.ArgumentParser(prog="rnmf-b200",
                                 description="randomized and deterministic HALS NMF on a B200 GPU")
    sub = ap.add_subparsers(dest="cmd", required=True)

    def common(p):
        p.add_argument("--input", required=True)
        p.add_argument("--rank", type=int, required=True)
        p.add_argument("--oversample", type=int, default=20)
        p.add_argument("--power", type=int, default=2)
        p.add_argument("--max-iter", dest="max_iter", type=int, default=200)
        p.add_argument("--tol", type=float, default=1e-4)
        p.add_argument("--init", default="random", choices=["random", "svd"])
        p.add_argument("--order", default="grouped", choices=["interleaved", "grouped", "shuffled"])
        p.add_argument("--seed", type=int, default=0)
        p.add_argument("--math", default="exact", choices=sorted(_MATH))
        p.add_argument("--device", type=int, default=0)

    fit = sub.add_parser("fit", help="factorize a nonnegative matrix")
    common(fit)
    fit.add_argument("--method", default="hals", choices=["hals", "rhals"])
    for name in ("alpha-w", "alpha-h", "beta-w", "beta-h"):
        fit.add_argument("--" + name, dest=name.replace("-", "_"), type=float, default=0.0)
    fit.add_argument("--out-w", dest="out_w", required=True)
    fit.add_argument("--out-h", dest="out_h", required=True)
    fit.add_argument("--trace", default="")

    bench = sub.add_parser("bench", help="time solvers against each other")
    common(bench)
    bench.add_argument("--methods", default="hals,rhals")
    bench.add_argument("--repeat", type=int, default=3)
    bench.add_argument("--out", required=True)
    return ap


def main(argv=None) -> int:
    ap = _parser()
    try:
        args = ap.parse_args(argv)
    except SystemExit as e:  # usage errors exit 2 as CLI11's ParseError path
        return int(e.code or 0)
    try:
        return run_fit(args) if args.cmd == "fit" else run_bench(args)
    except (api.ParameterError, api.ShapeError) as e:
        print(f"error: {e}", file=sys.stderr)
        return 2
    except Exception as e:  # DataError, IoError, CUDA errors
        print(f"error: {e}", file=sys.stderr)
        return 1


if __name__ == "__main__":
    sys.exit(main())
