"""Sequence sharding plumbing: build the library's NCCL communicator from
a torch.distributed process group. torch only carries the 128-byte NCCL unique id from rank 0 to
the other ranks; the halo exchange itself is inside libcascade_b200 (casc_apply_seqsharded)."""
from __future__ import annotations

import torch

from . import api


def broadcast_unique_id(group=None, device=None) -> bytes:
    """Rank 0 creates the NCCL unique id (casc_nccl_unique_id); every rank of `group` returns it.
    The broadcast goes through the group's own backend (a CUDA tensor for nccl, CPU for gloo)."""
    import torch.distributed as dist
    rank = dist.get_rank(group)
    if rank == 0:
        t = torch.frombuffer(bytearray(api.nccl_unique_id()), dtype=torch.uint8).clone()
    else:
        t = torch.zeros(128, dtype=torch.uint8)
    if dist.get_backend(group) == "nccl":
        t = t.to(device if device is not None else torch.device("cuda", torch.cuda.current_device()))
    src = dist.get_global_rank(group, 0) if group is not None else 0
    dist.broadcast(t, src=src, group=group)
    return bytes(t.cpu().numpy().tobytes())


def comm_from_process_group(group=None, device=None) -> api.Comm:
    """The library communicator over the ranks of `group` (one rank per process and GPU; the
    caller has selected this rank's device)."""
    import torch.distributed as dist
    uid = broadcast_unique_id(group, device)
    return api.comm_init(dist.get_rank(group), dist.get_world_size(group), uid)
