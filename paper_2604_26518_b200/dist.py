"""Host-side plumbing for multi-process runs (one process per GPU): slab
extraction, NCCL unique-id distribution over torch.distributed, and
max-over-ranks timing.  Only marshalling -- the exchanges themselves run in
libgmt (gmt_create_dist: ncclSend/Recv halos, ncclAllGather, ncclAllReduce).
"""
from __future__ import annotations

import numpy as np

from . import gmt


def slab_layout(res: int, levels: int, nranks: int, rank: int) -> dict:
    """gmt_slab_layout (host only): z0, nz, Ld, L of this rank's slab."""
    return gmt.gmt_slab_layout(res, levels, nranks, rank)


def slab_of(field: np.ndarray, levels: int, nranks: int, rank: int) -> np.ndarray:
    """This rank's N/P z-planes of a full (N, N, N) material field, or of a
    full vector [m, c, z, y, x], contiguous."""
    n = field.shape[-1]
    lay = slab_layout(n, levels, nranks, rank)
    z0, nz = lay["z0"], lay["nz"]
    if field.ndim == 3:
        return np.ascontiguousarray(field[z0:z0 + nz])
    return np.ascontiguousarray(field[:, :, z0:z0 + nz])


def share_unique_id(pg=None) -> bytes:
    """Rank 0 creates the NCCL unique id; every rank returns the same bytes."""
    import torch.distributed as dist
    obj = [gmt.gmt_nccl_unique_id() if dist.get_rank(pg) == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=pg)
    return obj[0]


def max_over_ranks(x: float, device=None, pg=None) -> float:
    """Max of a per-rank scalar (e.g. device-timed milliseconds)."""
    import torch
    import torch.distributed as dist
    t = torch.tensor([float(x)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=pg)
    return float(t.item())


def gather_slabs(local: np.ndarray, pg=None) -> np.ndarray:
    """Reassemble per-rank z-slabs (of a material or a [m,c,z,y,x] vector)
    along z on every rank (host objects; for tests and result collection)."""
    import torch.distributed as dist
    parts = [None] * dist.get_world_size(pg)
    dist.all_gather_object(parts, local, group=pg)
    return np.concatenate(parts, axis=0 if local.ndim == 3 else 2)
