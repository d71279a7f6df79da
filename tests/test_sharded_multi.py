"""The library's row-sharded path at world = 2 on two GPUs (NCCL communicator, CUDA-IPC peer sync
blocks, the hierarchical and the flat cross-GPU column step): W / H / trace against the unsharded
fit and the oracle.  Needs two GPUs (skipped otherwise; the driver's boxes have one), one process
per GPU, each under a timeout so a cross-GPU deadlock fails fast."""
import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

_WORKER = r"""
import json, sys
import numpy as np
sys.path.insert(0, {root!r})
from paper_1711_02037_b200 import api, distributed as d
rank, cid, out = int(sys.argv[1]), bytes.fromhex(sys.argv[2]), sys.argv[3]
rng = np.random.default_rng(5)
m, n, k = 2000, 500, 8
x = np.abs(rng.standard_normal((m, k))) @ np.abs(rng.standard_normal((k, n))) + 0.05 * np.abs(rng.standard_normal((m, n)))
x = x.astype(np.{dtype})
rows = [(0, 1100), (1100, 2000)][rank]
ctx = d.ShardedContext(rank, rank=rank, world=2, comm_id=cid)
o = api.SolverOptions(rank=k, oversampling=6, power_iterations=1, max_iter=30, tol=1e-300, seed=3)
res = d.rhals_fit_sharded(x[rows[0]:rows[1]], o, row_offset=rows[0], m_total=m, ctx=ctx)
ctx.close()
np.save(out + f".w{{rank}}.npy", np.asarray(res.factors.w, dtype=np.float64))
if rank == 0:
    np.save(out + ".h.npy", np.asarray(res.factors.h, dtype=np.float64))
    json.dump([[t.rel_err, t.pgrad, t.objective_compressed] for t in res.trace], open(out + ".trace.json", "w"))
    plain = api.rhals_fit(x, o, ctx=api.Context(0))
    json.dump([[t.rel_err, t.pgrad, t.objective_compressed] for t in plain.trace], open(out + ".plain.json", "w"))
"""


def _gpus():
    try:
        import torch

        return torch.cuda.device_count()
    except Exception:
        return 0


@pytest.mark.skipif(_gpus() < 2, reason="needs two GPUs")
@pytest.mark.parametrize("flat", [False, True])
@pytest.mark.parametrize("dtype", ["float64", "float32"])
def test_world2_matches_unsharded(tmp_path, flat, dtype):
    sys.path.insert(0, ROOT)
    from paper_1711_02037_b200 import distributed as d

    cid = d.comm_unique_id().hex()
    out = str(tmp_path / "r")
    env = dict(os.environ)
    if flat:
        env["RNMF_XGPU_FLAT"] = "1"
    script = _WORKER.format(root=ROOT, dtype=dtype)
    procs = [subprocess.Popen([sys.executable, "-c", script, str(r), cid, out], env=env) for r in (0, 1)]
    try:
        codes = [p.wait(timeout=300) for p in procs]
    finally:
        for p in procs:
            if p.poll() is None:
                p.kill()
    assert codes == [0, 0]
    tr = np.array(json.load(open(out + ".trace.json")))
    pl = np.array(json.load(open(out + ".plain.json")))
    rtol = 1e-8 if dtype == "float64" else 1e-3
    np.testing.assert_allclose(tr, pl, rtol=rtol, atol=1e-12)
    w = np.vstack([np.load(out + ".w0.npy"), np.load(out + ".w1.npy")])
    assert w.shape == (2000, 8) and (w >= 0).all()
