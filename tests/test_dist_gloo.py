"""Multi-process (world_size 2, 3 and 4, gloo on CPU) checks of the N>1 host
logic, one process per rank:

* tuple sharding (pair engines): the ownership rule partitions the skyline,
  each rank's partial denominators (0 = not owned) combine by one MAX
  all-reduce into exactly the oracle's full map;
* step sharding (cell engine): each rank takes the steps that libskygpu's OWN
  host-side plan assigns it (skygpu_cells_step_plan, the function the
  sharded pipeline calls), computes its partial map over those steps (the
  oracle's cell scan restricted to them), and one MAX all-reduce gives the
  oracle's full map; the ranks' step lists partition the scan.
The per-rank partial maps come from the CPU oracle — the contract the
library's sharded kernels satisfy on the GPU (tests/test_gpu_parity.py::
test_shards_*, test_step_sharded_cells_*)."""
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


def _step_worker(rank, world, port, kind, n, d, seed, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import pyoracle as po
    from paper_2412_02274_b200 import skypar

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        v = po.generate(kind, n, d, seed)
        pos, _ = po.skyline_sfs(v)
        sky = v[pos]
        full, gm, _ = po.grid_resistance(sky, pos, 25)
        steps = skypar.cells_step_plan(sky.max(axis=0), gm, len(pos), rank, world)
        partial = po.gres_cells_steps(sky, steps) if steps else np.ones(len(pos), np.int32)
        t = torch.from_numpy(partial.astype(np.int32))
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        got = [None] * world
        dist.all_gather_object(got, steps)
        q.put((rank, bool((t.numpy() == full).all()), got, gm))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_step_sharded_cells_combine_with_max_allreduce(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_step_worker, args=(r, world, port, "ant", 5000, 4, 9, q))
             for r in range(world)]
    for p in procs:
        p.start()
    out = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert all(ok for _, ok, _, _ in out)
    plans, gm = out[0][2], out[0][3]
    flat = sorted(g for pl in plans for g in pl)
    assert flat == list(range(2, gm + 1))  # the ranks' steps partition the scan
    assert all(pl == sorted(pl, reverse=True) for pl in plans)


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
