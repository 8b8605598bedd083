"""Multi-GPU plumbing: one process per GPU, NCCL over NVLink / NVSwitch.

The basic scheme's slab decomposition (csrc/solver.cu, nccl mode) needs one
NCCL communicator shared by the ranks; torch.distributed (any backend) is
only used to hand rank 0's NCCL unique id to the other ranks.  The material
points (config 2) need no communicator at all: every rank evaluates its own
batch.
"""

import ctypes
from dataclasses import dataclass
from typing import Callable, Optional

from . import _lib


@dataclass(frozen=True)
class Comm:
    """Rank, world size and the NCCL unique id of a communicator to create.

    ``transport`` = "nccl" (default: ncclAlltoAll transposes, the north
    star's path) or "p2p" (opt-in: fused pack / unpack kernels over NVLink
    peer memory through CUDA IPC handles swapped with ``allgather``, bytes
    -> list of every rank's bytes; tested on sibling slabs of one GPU and at
    world size 1 -- a multi-process run needs a multi-GPU box).
    """

    rank: int
    world: int
    uid: bytes
    allgather: Optional[Callable[[bytes], list]] = None
    transport: str = "nccl"


def nccl_unique_id():
    """A fresh ncclUniqueId (128 bytes) from libautomat's NCCL."""
    lib = _lib.load(require_device=False)
    buf = ctypes.create_string_buffer(128)
    _lib.check(lib.am_nccl_unique_id(buf), "nccl_unique_id")
    return buf.raw


def comm_from_torch(group=None, transport="nccl"):
    """Build a Comm over an initialised torch.distributed process group:
    rank 0 creates the NCCL id, the group broadcasts it (and later the IPC
    handles of the P2P transport)."""
    import torch.distributed as dist

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    obj = [nccl_unique_id() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)

    def allgather(b):
        out = [None] * world
        dist.all_gather_object(out, b, group=group)
        return out

    return Comm(rank=rank, world=world, uid=obj[0], allgather=allgather, transport=transport)


def slab_range(n, world, rank):
    """x planes [x0, x0 + n/world) owned by `rank` (the decomposition of solver.cu)."""
    if n % world:
        raise ValueError(f"{world} ranks must divide the grid size {n}")
    w = n // world
    return rank * w, (rank + 1) * w
