"""Row-sharded multi-GPU plumbing on torch.distributed.

One process per GPU. W (m_total x n) is split into contiguous row panels;
rank p holds rows [row0, row0 + rows) of W and of U, V is replicated. The
device path (csrc/host_core.cu, RowSplit) allreduces every reduction over
panel rows with NCCL; this module only does the host-side set-up: the row
partition and the rendezvous of the NCCL unique id (made on rank 0, broadcast
over the process group -- gloo on CPU, nccl on GPU).
"""
from __future__ import annotations


def row_partition(m: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced split: (row0, rows) of rank `rank`; the first
    m % world ranks get one extra row."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("row_partition: bad rank / world")
    if m < world:
        raise ValueError("row_partition: fewer rows than ranks")
    base, extra = divmod(m, world)
    row0 = rank * base + min(rank, extra)
    return row0, base + (1 if rank < extra else 0)


def broadcast_unique_id(group=None) -> bytes:
    """Rank 0 makes an NCCL unique id; every rank returns the same 128 bytes."""
    import torch
    import torch.distributed as dist

    from . import api

    rank = dist.get_rank(group)
    backend = dist.get_backend(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    buf = torch.zeros(128, dtype=torch.uint8, device=dev)
    if rank == 0:
        buf.copy_(torch.frombuffer(bytearray(api.nccl_unique_id()), dtype=torch.uint8))
    dist.broadcast(buf, src=dist.get_global_rank(group, 0) if group is not None else 0, group=group)
    return bytes(buf.cpu().numpy().tobytes())


def init_comm(ctx, group=None) -> None:
    """Attach an NCCL communicator over the process group to `ctx` (collective)."""
    import torch.distributed as dist

    uid = broadcast_unique_id(group)
    ctx.init_comm(dist.get_world_size(group), dist.get_rank(group), uid)


def init_host_comm(ctx, group=None) -> None:
    """Attach host-staged collectives over a gloo process group to `ctx`: the
    device buffer of every reduction is copied to the host and all-reduced with
    torch.distributed (so several ranks can share one GPU in tests; NCCL through
    init_comm is the product path)."""
    import numpy as np
    import torch
    import torch.distributed as dist

    def allreduce(arr, op):
        t = torch.from_numpy(arr)  # shares memory with the library's host copy
        dist.all_reduce(t, op=dist.ReduceOp.SUM if op == 0 else dist.ReduceOp.MAX, group=group)
        np.copyto(arr, t.numpy())

    ctx.init_host_comm(dist.get_world_size(group), dist.get_rank(group), allreduce)


def shard_operator(w_local, m_total: int, row0: int, ctx, device: bool = False, ld=None):
    """DenseOperator over this rank's row panel (host array or device tensor),
    marked as rows [row0, row0 + rows) of m_total."""
    from . import api

    if device:
        rows, n = w_local.shape[1], w_local.shape[0]  # column-major panel = row-major (n, rows) tensor
        op = api.DenseOperator(w_local, ctx=ctx, device=True, shape=(rows, n), ld=ld or rows)
    else:
        op = api.DenseOperator(w_local, ctx=ctx)
    op.set_row_shard(m_total, row0)
    return op


def shard_csc(colptr, rowidx, vals, row0: int, rows: int):
    """Rows [row0, row0 + rows) of a CSC matrix as a local CSC over the same
    columns (row indices relative to row0, positions in their original order)
    -- the observation a rank passes to mc_svt_sharded. Also returns the
    positions taken (indices into the global CSC arrays)."""
    import numpy as np

    colptr = np.asarray(colptr, dtype=np.int64)
    rowidx = np.asarray(rowidx)
    keep = (rowidx >= row0) & (rowidx < row0 + rows)
    pos = np.nonzero(keep)[0]
    col_of = np.repeat(np.arange(len(colptr) - 1), np.diff(colptr))
    counts = np.bincount(col_of[pos], minlength=len(colptr) - 1)
    local_ptr = np.zeros(len(colptr), dtype=np.int64)
    np.cumsum(counts, out=local_ptr[1:])
    return local_ptr, (rowidx[pos] - row0).astype(np.int32), np.asarray(vals)[pos], pos
