"""torch.distributed plumbing for the slab contexts: bootstrap of the NCCL id
(rtm_create_dist) and of the CUDA-IPC records of a peer context (rtm_create_peer, no NCCL), and
the host rank barrier the library calls.  No field arithmetic here: this module only moves the
opaque 128-byte id / 512-byte records between processes over a process group (any backend;
gloo works without a GPU) and installs ``group.barrier`` as the library's rank barrier.
"""
from __future__ import annotations

from . import rtm as _r


def exchange_neighbour_records(rec: bytes, rank: int, world: int, group=None):
    """All-gather every rank's record over ``group``; return (lo, hi) = the records of rank-1
    and rank+1 (None where that neighbour does not exist)."""
    import torch.distributed as dist
    got = [None] * world
    dist.all_gather_object(got, rec, group=group)
    for k, r in enumerate(got):
        if not isinstance(r, (bytes, bytearray)):
            raise RuntimeError(f"rank {k} sent no record")
    lo = bytes(got[rank - 1]) if rank > 0 else None
    hi = bytes(got[rank + 1]) if rank < world - 1 else None
    return lo, hi


def create_peer(nx, ny, nz, dx, dt, coeffs, rank, world, device, group=None,
                halo_mode=3, host_ordered=False):
    """rtm_create_peer + IPC bootstrap over ``group`` + the group's barrier as the library's
    rank barrier; sets the halo mode (collective).  Returns the context handle."""
    import torch.distributed as dist
    h = _r.rtm_create_peer(nx, ny, nz, dx, dt, coeffs, rank, world, device)
    try:
        lo, hi = exchange_neighbour_records(_r.rtm_ipc_export(h), rank, world, group)
        _r.rtm_ipc_import(h, lo, hi)
        _r.rtm_set_host_barrier(h, lambda: dist.barrier(group=group))
        _r.rtm_set_option(h, _r.RTM_OPT_HOST_ORDERED, int(host_ordered))
        _r.rtm_set_option(h, _r.RTM_OPT_HALO_MODE, halo_mode)  # collective: flags + barrier
    except Exception:
        _r.rtm_destroy(h)
        raise
    return h


def broadcast_unique_id(rank: int, group=None) -> bytes:
    """The NCCL id of rtm_create_dist: created on rank 0, broadcast over ``group``."""
    import torch.distributed as dist
    box = [_r.rtm_get_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(box, src=0, group=group)
    return box[0]
