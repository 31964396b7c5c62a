"""Tensor-parallel plumbing: bootstrap the NCCL communicator used by ALLREDUCE_SUM nodes.

torch.distributed (any backend) only carries the 128-byte ncclUniqueId from rank 0 to the others
(P:L857-878 TP setting); the communicator itself is created and owned through the
C ABI (cgx_nccl_comm_init) and the collective is captured inside each rank's graph.
"""
from __future__ import annotations

from . import cgx


def broadcast_unique_id(group=None) -> bytes:
    import torch.distributed as dist
    obj = [cgx.nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                               group=group)
    return obj[0]


def nccl_bootstrap(device: int, group=None) -> int:
    """Create this rank's ncclComm_t (returned as an integer handle; destroy with
    cgx.nccl_comm_destroy)."""
    import torch.distributed as dist
    uid = broadcast_unique_id(group)
    return cgx.nccl_comm_init(dist.get_world_size(group), dist.get_rank(group), uid, device)
