"""Multi-GPU plumbing for the grid-resistance path.

One process per GPU (torchrun), the relation replicated on every rank.  The
gres work is sharded by SKYLINE TUPLE: rank r owns the interleaved 256-tuple
chunks r, r + world, r + 2*world, ... of the skyline (libskygpu's
k_shard_iota; interleaving balances the early-exit work, SURVEY.md §7.4
item 5).  Each rank writes the denominators of its own tuples and 0 for the
others, so one MAX all-reduce (NCCL over NVLink on GPUs, gloo on CPU) yields
the full map — the only exchange on the path.
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
