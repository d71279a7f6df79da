"""Row-sharded rhals_fit over the GPUs of one node, one process per GPU.

X is split by rows: rank r holds rows [offset_r, offset_r + m_r) (`shard_rows`).  The exchange steps
run inside the C++/CUDA library (include/rnmf_gpu.h, "multi-GPU"): NCCL all-reduces of the Gram
matrices of the sketch QRs, of X^T Q, Q^T X, W^T W, W^T X and the metrics scalars, and, inside the
persistent sweep kernel, integer atomics into every GPU's column accumulators over NVLink.  This
module only distributes the NCCL id through torch.distributed (any backend) and marshals arguments,
mirroring `api.rhals_fit`.

    import torch.distributed as dist
    dist.init_process_group("nccl")            # torchrun: RANK / WORLD_SIZE / LOCAL_RANK
    ctx = ShardedContext(local_rank)            # collective
    off, cnt = shard_rows(m, ctx.world, ctx.rank)
    res = rhals_fit_sharded(x[off:off + cnt], opts, row_offset=off, m_total=m, ctx=ctx)  # collective
"""
from __future__ import annotations

import ctypes
from typing import Optional

from ._abi import TraceRecordC
from ._lib import lib
from .api import (
    _CAP, Context, FactorPair, FitResult, SolverOptions, _dptr, _f64_host, _Mat, _ptr, _sketch_width_nothrow,
    _sync_torch, _trace_list, err_buffer, raise_for_status,
)

COMM_ID_BYTES = 128


def shard_rows(m: int, world: int, rank: int) -> tuple[int, int]:
    """Balanced contiguous row blocks: rank r owns [m*r//world, m*(r+1)//world)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    lo, hi = m * rank // world, m * (rank + 1) // world
    return lo, hi - lo


def comm_unique_id() -> bytes:
    """A fresh NCCL unique id (rank 0 creates it, every rank needs the same bytes)."""
    buf = ctypes.create_string_buffer(COMM_ID_BYTES)
    e = err_buffer()
    raise_for_status(lib().rnmf_gpu_comm_unique_id(buf, e, _CAP), e)
    return buf.raw


def broadcast_comm_id(group=None) -> bytes:
    """Rank 0's unique id on every rank of the initialised torch.distributed group."""
    import torch.distributed as dist

    obj = [comm_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    return obj[0]


class ShardedContext(Context):
    """rnmf_gpu_context_create_sharded: a context on `device` that is rank `rank` of `world`
    (collective over the ranks; rank/world default to torch.distributed's)."""

    def __init__(self, device: int = 0, rank: Optional[int] = None, world: Optional[int] = None,
                 comm_id: Optional[bytes] = None, group=None):
        if rank is None or world is None or comm_id is None:
            import torch.distributed as dist

            rank = dist.get_rank(group) if rank is None else rank
            world = dist.get_world_size(group) if world is None else world
            comm_id = broadcast_comm_id(group) if comm_id is None else comm_id
        if len(comm_id) != COMM_ID_BYTES:
            raise ValueError("communicator id must be 128 bytes")
        self.device, self.rank, self.world = int(device), int(rank), int(world)
        h = ctypes.c_void_p()
        e = err_buffer()
        st = lib().rnmf_gpu_context_create_sharded(self.device, self.rank, self.world, comm_id, ctypes.byref(h), e,
                                                   _CAP)
        raise_for_status(st, e)
        self._h = h


def rhals_fit_sharded(x_local, opts: SolverOptions, *, row_offset: int, m_total: int, ctx: ShardedContext,
                      omega=None, w0=None, h0=None) -> FitResult:
    """rhals_fit of the m_total x n matrix whose rows [row_offset, row_offset + m_local) are `x_local`
    (numpy host array or CUDA tensor on ctx's GPU).  Collective: every rank calls it with the same
    options.  omega / h0 as in api.rhals_fit (same on every rank); w0 = this rank's rows of the
    unscaled W draw.  Returns W (this rank's rows), H (replicated) and the trace (identical on all
    ranks)."""
    X = _Mat(x_local, name="X")
    m, n = X.shape
    o = opts.to_c()
    k = max(int(opts.rank), 0)
    l = _sketch_width_nothrow(int(m_total), n, k, opts.oversampling)
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
    st = lib().rnmf_gpu_rhals_fit_sharded(
        ctx.handle, X.ptr, X.dtype_code, X.location, m, int(row_offset), int(m_total), n, ctypes.byref(o), _dptr(om),
        _dptr(a0), _dptr(b0), _ptr(w), _ptr(h), buf, cap, ctypes.byref(ln), e, _CAP)
    raise_for_status(st, e)
    return FitResult(FactorPair(w, h), _trace_list(buf, ln.value))
