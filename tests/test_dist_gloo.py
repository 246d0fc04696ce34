"""Multi-process (world_size 2 and 3, gloo on CPU) check of the N>1 host
logic: the shard ownership rule partitions the skyline, each rank's partial
denominators (0 = not owned) combine by one MAX all-reduce into exactly the
oracle's full map.  The per-rank partial map is produced from the CPU oracle
restricted to the rank's owned tuples — the contract libskygpu's sharded
kernel satisfies on the GPU (tests/test_gpu_parity.py::test_shards_*)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_02274_b200 import dist as skydist


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, kind, n, d, seed, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import pyoracle as po

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        v = po.generate(kind, n, d, seed)
        pos, _ = po.skyline_sfs(v)
        full, gm, _ = po.grid_resistance(v[pos], pos, 25)
        S = len(pos)
        mine = skydist.owned_positions(S, rank, world)
        partial = np.zeros(S, dtype=np.int32)
        partial[mine] = full[mine]
        t = torch.from_numpy(partial)
        skydist.combine_denominators(t)
        q.put((rank, bool((t.numpy() == full).all()), len(mine), S))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_gres_combines_with_max_allreduce(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, "ant", 6000, 4, 5, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in out)
    assert sum(k for _, _, k, _ in out) == out[0][3]  # ownership partitions the skyline


def test_shard_owner_partitions_and_balances():
    S = 10_000
    for world in (1, 2, 4, 8):
        owners = skydist.shard_owner(np.arange(S), world)
        counts = np.bincount(owners, minlength=world)
        assert counts.sum() == S and counts.max() - counts.min() <= skydist.CHUNK
        for r in range(world):
            assert (skydist.owned_positions(S, r, world) == np.nonzero(owners == r)[0]).all()
