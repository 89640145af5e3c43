"""Multi-GPU plumbing for the 1D block-cyclic tiled QR.

torch.distributed carries only the one-time exchange of CUDA IPC blobs (argument
marshalling); the V/T broadcast itself is done by the panel tasks' peer stores inside the
executor kernel (include/tqr.h, multi-GPU section).
"""
from __future__ import annotations


def exchange_blobs(blob: bytes, group=None) -> bytes:
    """All-gather one fixed-size blob per rank (any torch.distributed backend, incl. gloo);
    returns the concatenation in rank order."""
    import torch.distributed as dist
    world = dist.get_world_size(group)
    out = [None] * world
    dist.all_gather_object(out, bytes(blob), group=group)
    if any(len(x) != len(blob) for x in out):
        raise RuntimeError("ranks exchanged blobs of different sizes")
    return b"".join(out)


def connect(plan, group=None):
    """Connect a multi-rank Plan to its peers (collective over `group`)."""
    plan.comm_connect(exchange_blobs(plan.comm_export(), group))
    return plan


def owned_columns(q: int, nranks: int, rank: int):
    """Global tile columns held by `rank`, in storage order (storage column jl <-> rank + jl*nranks)."""
    return list(range(rank, q, nranks))
