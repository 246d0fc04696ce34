"""Multi-GPU plumbing for the grid-resistance path.

One process per GPU (torchrun), the relation replicated on every rank.  The
library splits the work itself (skygpu_pipeline shard_rank / shard_world):

* rank-grid skyline engine (large skylines, BASELINE config 5): by grid ROW
  (row % world == rank), keep flags MAX-reduced;
* cell-occupancy resistance engine (huge skylines): by STEP g of the scan
  (longest-processing-time over the per-step cost, cells.cu
  cells_step_plan), every candidate on every rank, den MAX-reduced;
* pair engines: by SKYLINE TUPLE — interleaved 256-tuple chunks r, r + world,
  ... (k_shard_iota; interleaving balances the early-exit work, SURVEY.md
  §7.4 item 5), den MAX-reduced.

init_library_nccl() gives the library its OWN NCCL communicator (the unique
id made by rank 0 and broadcast over torch.distributed): the exchanges are
then ncclAllReduce(MAX) queued on the library's stream, no host sync.
install_collective() is the older route through a torch.distributed callback.
Without either, only the resistance stage is sharded and the caller reduces
the map (combine_denominators).
"""
from __future__ import annotations

import numpy as np

CHUNK = 256


def shard_owner(index: np.ndarray | int, world: int):
    """Rank owning skyline position `index` (mirrors k_shard_iota)."""
    return (np.asarray(index) // CHUNK) % world


def owned_positions(S: int, rank: int, world: int) -> np.ndarray:
    """Ascending skyline positions owned by `rank` (the kernel's candidate list)."""
    idx = np.arange(S, dtype=np.int64)
    return idx[shard_owner(idx, world) == rank]


def init_library_nccl(group=None):
    """Give libskygpu its own NCCL group over the torch.distributed world:
    rank 0 makes the unique id, a broadcast ships it (any backend: gloo on
    CPU works), every rank joins on the library's current device."""
    import torch.distributed as dist

    from . import skypar

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    uid = skypar.nccl_unique_id() if rank == 0 else bytes(128)
    obj = [uid]
    dist.broadcast_object_list(obj, src=0, group=group)
    skypar.nccl_init(obj[0], world, rank)
    return rank, world


def combine_denominators(partial, group=None):
    """Max-reduce sharded denominators in place (0 = not owned by this rank).

    `partial` is a torch tensor (int32) on the backend's device."""
    import torch.distributed as dist

    dist.all_reduce(partial, op=dist.ReduceOp.MAX, group=group)
    return partial


def gres_sharded(values, ids=None, plan=None, cap=25, rank: int = 0, world: int = 1, group=None,
                 device=None):
    """Skyline + sharded grid resistance on this rank's GPU, combined with a
    MAX all-reduce; returns (positions, full denominators, g_max)."""
    import torch

    from . import skypar

    res = skypar.pipeline(values, ids, plan, cap=cap, shard_rank=rank, shard_world=world)
    den = torch.from_numpy(res.den.astype(np.int32))
    if world > 1:
        den = den.to(device) if device is not None else den
        combine_denominators(den, group)
        den = den.cpu()
    return res.positions, den.numpy(), res.g_max


class _DeviceBuffer:
    """A raw device buffer seen by torch through __cuda_array_interface__."""

    def __init__(self, ptr: int, count: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (count,), "typestr": typestr,
                                         "data": (ptr, False), "version": 3}


def install_collective(group=None):
    """Route libskygpu's sharded-call exchange (uint8 keep flags, int32
    denominators; MAX) through torch.distributed — NCCL over NVLink/NVSwitch
    on GPUs."""
    import torch
    import torch.distributed as dist

    from . import skypar

    def allreduce_max(ptr, count, elem_bytes, stream):
        # the library's buffer lives on the library's device, not necessarily
        # torch's current one: build the view there and refuse a copy (a copy
        # would be reduced while the library's buffer stays partial)
        dev = torch.device("cuda", skypar.current_device())
        t = torch.as_tensor(_DeviceBuffer(ptr, count, "|u1" if elem_bytes == 1 else "<i4"),
                            device=dev)
        if t.data_ptr() != ptr:
            return 1
        with torch.cuda.device(dev):
            dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
            torch.cuda.current_stream(dev).synchronize()  # in place before the library continues
        return 0

    skypar.set_collective(allreduce_max)
