"""GPU parity: libskygpu (through its C-ABI) against the reference's golden
outputs and against the CPU oracle on seeded inputs.  Bit-exact: skyline id
sets and order, g_max, every denominator."""
import numpy as np
import pytest

import paper_2412_02274_b200 as sk
from conftest import golden_input, golden_names, load_golden, spec_cap
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu


def plan_of(g, d):
    sp = g["spec"]
    return sk.make_plan(sp["strategy"], sp["p"], d)


def check_pipeline_against_golden(g, engine=sk.GRES_AUTO):
    v, ids = golden_input(g, sk.generate)
    n, d = v.shape
    plan = plan_of(g, d)
    if "error" in g:
        with pytest.raises(ValueError) as ei:
            sk.parallel_skyline(v, ids, plan)
        assert str(ei.value) == g["error"]
        return
    sky = sk.parallel_skyline(v, ids, plan, cores=4)
    assert sorted(sky.ids.tolist()) == g["skyline_ids"]
    assert sky.ids.tolist() == g["skyline_order"]
    if "gres_error" in g:
        with pytest.raises(ValueError) as ei:
            sk.grid_resistance(sky.values, sky.ids, plan, cap=spec_cap(g), check_skyline=True)
        assert str(ei.value) == g["gres_error"]
        return
    res = sk.pipeline(v, ids, plan, cap=spec_cap(g), engine=engine)
    assert ids[res.positions].tolist() == g["skyline_order"]
    assert res.g_max == g["g_max"]
    got = dict(zip(ids[res.positions].tolist(), res.den.tolist()))
    assert [got[i] for i in g["skyline_ids"]] == g["den"]
    # the standalone grid_resistance entry point on the reference's skyline
    gr = sk.grid_resistance(sky.values, sky.ids, plan, cap=spec_cap(g), cores=2)
    assert gr.g_max == g["g_max"]
    assert [gr.denominators[i] for i in g["skyline_ids"]] == g["den"]


@pytest.mark.parametrize("name", golden_names(exclude=("C4_", "C5_", "C1_", "C2_", "C3_")))
def test_small_goldens(name):
    check_pipeline_against_golden(load_golden(name))


@pytest.mark.parametrize("name", ["C1_uni_100k_d4", "C1_uni_100k_d4_sliced16", "C2_ant_1M_d3",
                                  "C3_corr_1M_d6", "C5_prefix_2k_d7", "C5_prefix_10k_d7",
                                  "C5_prefix_20k_d7", "C4_uni_10M_d5", "C4_uni_10M_d5_grid64",
                                  "C4_uni_10M_d5_sliced64"])
def test_config_goldens(name):
    check_pipeline_against_golden(load_golden(name))


@pytest.mark.parametrize("gen,n,d,seed", [
    ("uni", 3000, 1, 1), ("ant", 3000, 2, 2), ("lattice", 5000, 3, 3), ("uni", 20000, 6, 4),
    ("ant", 4000, 8, 5), ("uni", 2000, 9, 6), ("ant", 1500, 12, 7), ("lattice", 3000, 10, 8),
    ("corr", 50000, 4, 9), ("ant", 100000, 4, 10)])
def test_random_against_oracle(gen, n, d, seed):
    v = sk.generate(gen, n, d, seed)
    ids = np.arange(n, dtype=np.int64)
    pos, _ = po.skyline_sfs(v, ids)
    res = sk.pipeline(v, ids, cap=25)
    assert res.positions.tolist() == pos.tolist()
    den, gm, _ = po.grid_resistance(v[pos], ids[pos], 25)
    assert res.g_max == gm
    assert res.den.tolist() == den.tolist()


def test_unsorted_and_negative_ids_follow_sum_id_order():
    rng = np.random.default_rng(3)
    v = np.floor(rng.random((4000, 3)) * 8) / 8  # many sum ties -> id order matters
    ids = rng.permutation(10**6)[:4000].astype(np.int64) - 500000
    pos, _ = po.skyline_sfs(v, ids)
    sky = sk.parallel_skyline(v, ids)
    assert sky.positions.tolist() == pos.tolist()


def test_reps_filtering_keeps_result():
    v = sk.generate("ant", 5000, 3, 21)
    base = sk.parallel_skyline(v)
    order = np.lexsort((np.arange(5000), v.sum(axis=1)))
    reps = (v[order[:10]], order[:10])
    withr = sk.parallel_skyline(v, None, sk.make_plan("angular", 16, 3), reps=reps, cores=4)
    assert sorted(withr.ids.tolist()) == sorted(base.ids.tolist())


@pytest.mark.parametrize("world", [2, 3, 8])
def test_shards_max_reduce_to_full_map(world):
    v = sk.generate("ant", 20000, 5, 31)
    full = sk.pipeline(v, cap=25)
    acc = np.zeros_like(full.den)
    for r in range(world):
        part = sk.pipeline(v, cap=25, shard_rank=r, shard_world=world)
        assert part.positions.tolist() == full.positions.tolist()
        assert ((part.den == 0) | (part.den == full.den)).all()
        acc = np.maximum(acc, part.den)
    assert acc.tolist() == full.den.tolist()


@pytest.mark.parametrize("world", [2, 3, 8])
def test_step_sharded_cells_max_reduce_to_full_map(world):
    """Cell engine, sharded by STEP (cells_step_plan): each shard's map is its
    largest dominated step (1 if none); the MAX over shards is the full map,
    and each shard ran exactly its planned steps."""
    v = sk.generate("ant", 60000, 5, 41)
    full = sk.pipeline(v, cap=25, engine=sk.GRES_CELLS)
    assert full.stats["gres_engine"] == sk.GRES_CELLS
    acc = np.zeros_like(full.den)
    for r in range(world):
        part = sk.pipeline(v, cap=25, engine=sk.GRES_CELLS, shard_rank=r, shard_world=world)
        assert part.positions.tolist() == full.positions.tolist()
        assert (part.den >= 1).all() and (part.den <= full.den).all()
        acc = np.maximum(acc, part.den)
    assert acc.tolist() == full.den.tolist()


def test_library_nccl_group_of_one():
    """The library's own NCCL path on one GPU: a group of one joins, sharded
    calls with world 1 run unchanged, the group is released."""
    from paper_2412_02274_b200 import skypar
    uid = skypar.nccl_unique_id()
    assert len(uid) == 128
    skypar.nccl_init(uid, 1, 0)
    try:
        v = sk.generate("ant", 300000, 7, 3)
        a = sk.pipeline(v, cap=25, shard_rank=0, shard_world=1)
    finally:
        skypar.nccl_release()
    b = sk.pipeline(v, cap=25)
    assert a.positions.tolist() == b.positions.tolist() and a.den.tolist() == b.den.tolist()


def test_api_kats():
    # proj/tests/test_gres.cpp:26-34, 61-73, 91-97, 163-170, 172-177
    assert sk.snap_to_grid([0.30, 0.62], 5).tolist() == [0.2, 0.6]
    assert sk.snap_to_grid([0.0, 0.0], 7).tolist() == [0.0, 0.0]
    with pytest.raises(ValueError, match="intervals must be >= 1"):
        sk.snap_to_grid([0.3], 0)
    assert sk.max_grid_intervals(np.array([[0.2], [0.7]]), None) == 2
    assert sk.max_grid_intervals(np.array([[0.2, 0.9], [0.24, 0.9]]), None) == 25
    assert sk.max_grid_intervals(np.array([[0.2, 0.9], [0.24, 0.9]]), 10) == 10
    with pytest.raises(ValueError, match="all tuples are identical"):
        sk.max_grid_intervals(np.array([[0.3, 0.3], [0.3, 0.3]]), 25)
    with pytest.raises(ValueError, match="overflows the integer range"):
        sk.max_grid_intervals(np.array([[0.5], [0.5 + 1e-12]]), None)
    assert sk.max_grid_intervals(np.array([[0.5], [0.5 + 1e-12]]), 25) == 25
    r = sk.grid_resistance(np.array([[0.5, 0.5]]), cap=25)
    assert r.den.tolist() == [1]
    r = sk.grid_resistance(np.array([[0.30, 0.40], [0.40, 0.30]]), cap=None)
    assert r.g_max >= 2 and r.den.tolist() == [1, 1]
    r = sk.grid_resistance(np.zeros((0, 2)), cap=25)
    assert r.den.size == 0 and r.g_max == 1
    with pytest.raises(ValueError, match="cores must be >= 1"):
        sk.grid_resistance(np.array([[0.5, 0.5]]), cores=0)
    with pytest.raises(ValueError, match="cores must be >= 1"):
        sk.parallel_skyline(np.array([[0.5, 0.5]]), cores=0)
    with pytest.raises(ValueError, match=r"input is not a skyline \(tuple 0 dominates tuple 1\)"):
        sk.grid_resistance(np.array([[0.1, 0.1], [0.5, 0.5]]), check_skyline=True)
    assert sk.parallel_skyline(np.zeros((0, 3))).ids.size == 0


def test_generic_dims_and_duplicates():
    rng = np.random.default_rng(5)
    base = np.floor(rng.random((300, 11)) * 4) / 4
    v = np.vstack([base, base[:50]])  # exact duplicates are all retained
    ids = np.arange(len(v), dtype=np.int64)
    pos, _ = po.skyline_sfs(v, ids)
    res = sk.pipeline(v, ids, cap=None)
    assert res.positions.tolist() == pos.tolist()
    den, gm, _ = po.grid_resistance(v[pos], ids[pos], None)
    assert res.g_max == gm and res.den.tolist() == den.tolist()


@pytest.mark.parametrize("name", ["C1_uni_100k_d4", "C2_ant_1M_d3", "C5_prefix_2k_d7",
                                  "C5_prefix_10k_d7", "rand_ant_n1500_d5_angular",
                                  "rand_lattice_n1500_d7_none", "uncapped_lattice_d3"])
def test_cell_engine_matches_golden(name):
    """The cell-occupancy gres engine (cells.cu) gives the reference's map."""
    g = load_golden(name)
    v, ids = golden_input(g, sk.generate)
    res = sk.pipeline(v, ids, plan_of(g, v.shape[1]), cap=spec_cap(g), engine=sk.GRES_CELLS)
    assert res.g_max == g["g_max"]
    got = dict(zip(ids[res.positions].tolist(), res.den.tolist()))
    assert [got[i] for i in g["skyline_ids"]] == g["den"]
    if res.g_max >= 2:
        assert res.stats["gres_engine"] == sk.GRES_CELLS


@pytest.mark.parametrize("world", [2, 5])
def test_cell_engine_shards(world):
    v = sk.generate("ant", 30000, 6, 41)
    full = sk.pipeline(v, cap=25, engine=sk.GRES_PAIRS)
    acc = np.zeros_like(full.den)
    for r in range(world):
        part = sk.pipeline(v, cap=25, engine=sk.GRES_CELLS, shard_rank=r, shard_world=world)
        acc = np.maximum(acc, part.den)
    assert acc.tolist() == full.den.tolist()


@pytest.mark.parametrize("gen,d", [("ant", 1), ("ant", 2), ("ant", 3), ("uni", 4),
                                   ("lattice", 3), ("corr", 4)])
def test_cell_engine_smem_matches_pairs(gen, d):
    """The shared-memory cell kernel (all steps in one launch, d <= 4) and
    the per-step HBM variant give the pair engine's map."""
    v = sk.generate(gen, 20000, d, 50 + d)
    full = sk.pipeline(v, cap=25, engine=sk.GRES_PAIRS)
    auto = sk.pipeline(v, cap=25)
    assert auto.positions.tolist() == full.positions.tolist()
    assert auto.den.tolist() == full.den.tolist()
    if auto.g_max >= 2:
        assert auto.stats["gres_engine"] == sk.GRES_CELLS and auto.stats["gres_cells"] == 0
        assert auto.stats["gres_kernel_launches"] == 1


@pytest.mark.parametrize("case", ["witness_fires", "coarse_gaps", "values_above_one",
                                  "value_exactly_one", "cap_31", "cap_2"])
def test_speculative_gres_launch(case):
    """The pipeline's speculative capped scan (g_max = cap from the device
    gap witness, codes within cap + 1) and its fallback when either does not
    hold: the map is the oracle's in every case."""
    rng = np.random.default_rng(71)
    cap = {"cap_31": 31, "cap_2": 2}.get(case, 25)
    if case == "coarse_gaps":          # min positive gap 0.1 -> g_max = 10 < cap
        v = rng.integers(0, 10, size=(3000, 3)) / 10.0
    elif case == "values_above_one":   # codes beyond cap + 1
        v = 3.0 * sk.generate("ant", 3000, 3, 5)
    elif case == "value_exactly_one":
        v = sk.generate("ant", 3000, 3, 6)
        v[0] = [1.0, 0.0, 0.0]
    else:
        v = sk.generate("ant", 3000, 3, 7)
    ids = np.arange(len(v), dtype=np.int64)
    res = sk.pipeline(v, ids, cap=cap)
    pos, _ = po.skyline_sfs(v, ids)
    assert res.positions.tolist() == pos.tolist()
    den, gm, _ = po.grid_resistance(v[pos], ids[pos], cap)
    assert res.g_max == gm and res.den.tolist() == den.tolist()


def test_cell_engine_hbm_variant_small_d(monkeypatch):
    monkeypatch.setenv("SKYGPU_CELLS_SMEM", "0")
    v = sk.generate("ant", 50000, 3, 61)
    full = sk.pipeline(v, cap=25, engine=sk.GRES_PAIRS)
    cells = sk.pipeline(v, cap=25, engine=sk.GRES_CELLS)
    assert cells.stats["gres_engine"] == sk.GRES_CELLS and cells.stats["gres_cells"] > 0
    assert cells.den.tolist() == full.den.tolist()


@pytest.mark.parametrize("gen,d,scale", [("ant", 2, None), ("ant", 3, None), ("uni", 4, None),
                                         ("ant", 5, None), ("lattice", 6, None), ("ant", 7, None),
                                         ("corr", 8, None), ("ant", 7, (1.0, 0.3, 0.6, 1.0, 0.5, 0.9, 0.2)),
                                         ("ant", 4, (0.1, 1.0, 0.4, 0.7)), ("lattice", 5, (4.0,) * 5)])
def test_min_grid_cell_engine_matches_pairs(monkeypatch, gen, d, scale):
    """The min-grid form of the HBM cell engine (one byte per cell: the
    smallest code of the min'd attribute under it) against the pair engine,
    over every d it takes, unequal extents (the min'd attribute is the widest,
    not attribute 0), ties/duplicates (lattice) and codes far above cap
    (values up to 4: extents ~100)."""
    monkeypatch.setenv("SKYGPU_CELLS_SMEM", "0")
    v = sk.generate(gen, 30000, d, 70 + d)
    if scale is not None:
        v = v * np.asarray(scale)
    full = sk.pipeline(v, cap=25, engine=sk.GRES_PAIRS)
    cells = sk.pipeline(v, cap=25, engine=sk.GRES_CELLS)
    assert cells.positions.tolist() == full.positions.tolist()
    # (the min-grid takes codes of the min'd attribute up to 62, the bitset
    # form up to 63 on attribute 0; beyond both the pair engine answers)
    if full.g_max >= 2 and np.floor(v[full.positions].max() * full.g_max) <= 62:
        assert cells.stats["gres_engine"] == sk.GRES_CELLS and cells.stats["gres_cells"] > 0
    assert cells.den.tolist() == full.den.tolist()


@pytest.mark.parametrize("world", [2, 3])
def test_cell_engine_smem_shards(world):
    v = sk.generate("ant", 30000, 3, 43)
    full = sk.pipeline(v, cap=25, engine=sk.GRES_PAIRS)
    acc = np.zeros_like(full.den)
    for r in range(world):
        part = sk.pipeline(v, cap=25, shard_rank=r, shard_world=world)
        assert part.stats["gres_cells"] == 0
        acc = np.maximum(acc, part.den)
    assert acc.tolist() == full.den.tolist()


# ------------------------------------------------ one-pass rank-grid skyline engine
@pytest.mark.parametrize("name", ["C1_uni_100k_d4", "C2_ant_1M_d3", "C3_corr_1M_d6",
                                  "C5_prefix_2k_d7", "C5_prefix_10k_d7",
                                  "rand_lattice_n1500_d7_none", "rand_ant_n1500_d5_angular",
                                  "uncapped_lattice_d3"])
def test_grid_engine_matches_golden(name):
    """skyline_grid.cu (forced) gives the reference's skyline, order and map."""
    g = load_golden(name)
    v, ids = golden_input(g, sk.generate)
    res = sk.pipeline(v, ids, plan_of(g, v.shape[1]), cap=spec_cap(g), sky_engine=sk.SKY_GRID)
    assert res.stats["sky_engine"] == sk.SKY_GRID
    assert ids[res.positions].tolist() == g["skyline_order"]
    assert res.g_max == g["g_max"]
    got = dict(zip(ids[res.positions].tolist(), res.den.tolist()))
    assert [got[i] for i in g["skyline_ids"]] == g["den"]


@pytest.mark.parametrize("gen,n,d,seed", [
    ("uni", 3000, 1, 1), ("ant", 3000, 2, 2), ("lattice", 5000, 3, 3), ("uni", 20000, 6, 4),
    ("ant", 4000, 8, 5), ("corr", 50000, 4, 9), ("ant", 100000, 4, 10)])
def test_grid_engine_random_against_oracle(gen, n, d, seed):
    v = sk.generate(gen, n, d, seed)
    ids = np.arange(n, dtype=np.int64)
    pos, _ = po.skyline_sfs(v, ids)
    res = sk.pipeline(v, ids, cap=25, skip_gres=True, sky_engine=sk.SKY_GRID)
    assert res.positions.tolist() == pos.tolist()


def test_grid_engine_ties_and_unsorted_ids():
    rng = np.random.default_rng(3)
    v = np.floor(rng.random((6000, 4)) * 6) / 6  # sum ties, duplicates
    ids = rng.permutation(10**6)[:6000].astype(np.int64) - 500000
    pos, _ = po.skyline_sfs(v, ids)
    res = sk.pipeline(v, ids, skip_gres=True, sky_engine=sk.SKY_GRID)
    assert res.positions.tolist() == pos.tolist()
    # FP-tie case: {<2e-20,1>, <1e-20,1>} have equal sums; the predecessor
    # rule keeps both (the reference's SFS order), brute force would not
    v2 = np.array([[2e-20, 1.0], [1e-20, 1.0]])
    for eng in (sk.SKY_GRID, sk.SKY_ROUNDS):
        r2 = sk.pipeline(v2, np.array([0, 1]), skip_gres=True, sky_engine=eng)
        assert sorted(r2.positions.tolist()) == sorted(po.skyline_sfs(v2, np.array([0, 1]))[0].tolist())


@pytest.mark.timeout(120)
@pytest.mark.parametrize("gen,n,d", [("uni", 90000, 3), ("corr", 40000, 4), ("uni", 250000, 2),
                                     ("uni", 120000, 5)])
def test_grid_engine_items_that_die_at_once(gen, n, d):
    """Dense dominance (tiny skylines): nearly every K6 item loses all of its
    candidates within a stage or two, so the consumer warps' "everything dead"
    early-outs and the producer's stop run constantly.  Round 2 found a
    deadlock exactly there (lanes of one warp read the shared alive masks for
    themselves, disagreed, and waited at different warp barriers:
    profiles/r02_k6_deadlock_gdb.txt) — the masks are now read once per warp.
    Repeated: the interleaving differs from run to run."""
    v = sk.generate(gen, n, d, 11)
    ids = 7 + 5 * np.arange(n, dtype=np.int64)
    pos, _ = po.skyline_sfs(v, ids)
    for _ in range(6):
        res = sk.pipeline(v, ids, skip_gres=True, sky_engine=sk.SKY_GRID)
        assert res.stats["sky_engine"] == sk.SKY_GRID
        assert res.positions.tolist() == pos.tolist()


@pytest.mark.parametrize("n", [200_000, 1_000_000])
def test_grid_engine_auto_on_large_skyline(n):
    """C5-style data (skyline ~ input) switches to the rank grid after round 1;
    both engines agree bit-exactly (order included)."""
    v = sk.generate("ant", n, 7, 1)
    a = sk.pipeline(v, cap=25, skip_gres=True)
    assert a.stats["sky_engine"] == sk.SKY_GRID
    b = sk.pipeline(v, cap=25, skip_gres=True, sky_engine=sk.SKY_ROUNDS)
    assert b.stats["sky_engine"] == sk.SKY_ROUNDS
    assert a.positions.tolist() == b.positions.tolist()


# ------------------------------------------------ exact reference accounting
def _oracle_accounting(v, ids, pids, p, reps):
    """The reference's counters restated with the oracle's SFS
    (core.cpp:48-73) and filter (partition.cpp:287-302) semantics."""
    per = np.zeros(p, dtype=np.int64)
    local = []
    for g in range(p):
        idx = np.flatnonzero(pids == g)
        keep = []
        for i in idx:
            k = 0
            dom = False
            for r in (reps if reps is not None else []):
                k += 1
                if np.all(r <= v[i]) and np.any(r < v[i]):
                    dom = True
                    break
            per[g] += k
            if not dom:
                keep.append(i)
        keep = np.array(keep, dtype=np.int64)
        if len(keep):
            pos, t = po.skyline_sfs(v[keep], ids[keep])
            per[g] += t
            local.extend(keep[pos].tolist())
    local = np.array(local, dtype=np.int64)
    pos, fin = po.skyline_sfs(v[local], ids[local]) if len(local) else (np.zeros(0, np.int64), 0)
    return per, fin, len(local), local[pos] if len(local) else local


@pytest.mark.parametrize("gen,n,d,p,seed,nreps", [
    ("ant", 3000, 3, 1, 1, 0), ("ant", 4000, 3, 8, 2, 0), ("uni", 5000, 4, 5, 3, 0),
    ("lattice", 3000, 3, 4, 4, 0), ("ant", 2000, 5, 6, 5, 3), ("uni", 2000, 2, 3, 6, 10)])
def test_sfs_accounting_matches_reference_counters(gen, n, d, p, seed, nreps):
    v = sk.generate(gen, n, d, seed)
    rng = np.random.default_rng(seed)
    ids = rng.permutation(10 * n)[:n].astype(np.int64)
    pids = rng.integers(-1, p, n).astype(np.int64)  # -1 = dropped before phase 1
    reps = None
    if nreps:
        order = np.lexsort((ids, v.sum(axis=1)))
        reps = v[order[:nreps]]
    got = sk.sfs_accounting(v, ids, pids, p, reps)
    per, fin, into, pos = _oracle_accounting(v, ids, pids, p, reps)
    assert got.per_partition.tolist() == per.tolist()
    assert got.final_tests == fin
    assert got.into_final == into
    assert got.positions.tolist() == pos.tolist()


def test_sfs_accounting_anti_diagonal_kat():
    # proj/tests/test_core.cpp:116-133: n mutually incomparable tuples -> n(n-1)/2
    n = 64
    v = np.array([[i, n - 1 - i] for i in range(n)], dtype=np.float64)
    got = sk.sfs_accounting(v, np.arange(n), np.zeros(n, dtype=np.int64), 1)
    assert got.per_partition.tolist() == [n * (n - 1) // 2]
    assert got.final_tests == n * (n - 1) // 2 and len(got.positions) == n


# ------------------------------------------------ streamed host input (H2D overlap)
def _host_vs_device(v, ids, plan=None, cap=25):
    """pipeline() from host arrays (>= 48 MB of input: the streamed, chunk-
    overlapped path) vs the same call on device pointers (one-shot path)."""
    import torch
    host = sk.pipeline(v, ids, plan, cap=cap)
    n, d = v.shape
    dv = torch.from_numpy(np.ascontiguousarray(v)).cuda()
    di = torch.from_numpy(np.ascontiguousarray(ids)).cuda()
    pos = torch.empty(n, dtype=torch.int64, device="cuda")
    den = torch.empty(n, dtype=torch.int32, device="cuda")
    from paper_2412_02274_b200 import skypar
    S, gm, _ = skypar.pipeline_raw(dv.data_ptr(), di.data_ptr(), n, d,
                                   plan or sk.make_plan("none", 1, d), cap, 0, 0, 1,
                                   skypar.DEVICE_PTRS, pos.data_ptr(), den.data_ptr())
    torch.cuda.synchronize()
    assert host.positions.tolist() == pos[:S].cpu().tolist()
    assert host.g_max == gm and host.den.tolist() == den[:S].cpu().tolist()
    return host


@pytest.mark.parametrize("gen,n,d,seed", [("ant", 2_000_000, 3, 3), ("uni", 1_500_000, 5, 4),
                                          ("corr", 1_600_000, 4, 5), ("lattice", 2_000_000, 3, 6)])
def test_streamed_host_input_matches_device_path(gen, n, d, seed):
    v = sk.generate(gen, n, d, seed)
    rng = np.random.default_rng(seed)
    ids = rng.permutation(3 * n)[:n].astype(np.int64)  # unsorted ids: (sum, id) ties matter
    res = _host_vs_device(v, ids)
    pos, _ = po.skyline_sfs(v, ids)
    assert res.positions.tolist() == pos.tolist()


def test_streamed_fp_tie_across_chunks():
    """A head tuple dominating a tail tuple of EQUAL sum but larger id does
    not precede it: the reference keeps both."""
    n = 2_100_000
    rng = np.random.default_rng(9)
    v = 2.0 + rng.random((n, 2))           # filler, dominated by the pair below
    v[0] = [1e-20, 1.0]                    # head: dominates t, same sum 1.0
    v[n - 1] = [2e-20, 1.0]                # tail
    ids = np.arange(n, dtype=np.int64) + 10
    ids[0], ids[n - 1] = 9, 5              # t has the smaller id -> t first
    res = _host_vs_device(v, ids)
    pos, _ = po.skyline_sfs(v, ids)
    assert res.positions.tolist() == pos.tolist()
    assert sorted(res.positions.tolist()) == [0, n - 1]


def test_streamed_seed_dominated_by_tail():
    """The seed (skyline of the head's first prefix) is not final: a tail
    tuple can dominate a seed tuple, and a seed tuple still rules out the
    head tuples it dominates."""
    n = 2_100_000
    rng = np.random.default_rng(11)
    v = 0.7 + 0.3 * rng.random((n, 3))
    v[3] = [0.5, 0.5, 0.5]                 # head seed, dominated by the tail tuple below
    v[7] = [0.6, 0.55, 0.6]                # head, dominated by both
    v[n - 2] = [0.4, 0.45, 0.4]            # tail
    v[n - 1] = [0.1, 0.9, 0.65]            # tail, incomparable with the rest
    ids = np.arange(n, dtype=np.int64)
    res = _host_vs_device(v, ids)
    pos, _ = po.skyline_sfs(v, ids)
    assert res.positions.tolist() == pos.tolist()
    assert 3 not in res.positions.tolist() and n - 2 in res.positions.tolist()


@pytest.mark.parametrize("cap", ["1000", "6000", "20000"])
@pytest.mark.parametrize("gen,d", [("ant", 3), ("uni", 4), ("corr", 6), ("lattice", 2)])
def test_device_sized_rounds_and_their_redo(monkeypatch, gen, d, cap):
    """The round sized on the device (prefix count never read before K5)
    and the ride-along final round; a lowered capacity (SKYGPU_DEV_CAP) makes
    the prefix or the survivors miss it, which must redo the round the
    synchronous way with the same result."""
    monkeypatch.setenv("SKYGPU_DEV_CAP", cap)
    v = sk.generate(gen, 300_000, d, 31)
    ids = np.arange(len(v), dtype=np.int64)
    res = sk.pipeline(v, ids, cap=25)
    pos, _ = po.skyline_sfs(v, ids)
    assert res.positions.tolist() == pos.tolist()
    den, gm, _ = po.grid_resistance(v[pos], ids[pos], 25)
    assert res.g_max == gm and res.den.tolist() == den.tolist()


@pytest.mark.parametrize("gen,ids_kind", [("ant", "permuted"), ("lattice", "permuted"),
                                           ("lattice", "strided"), ("lattice", "one_swap"),
                                           ("uni", "duplicate")])
def test_late_ids_speculation(gen, ids_kind):
    """Host inputs below the streaming size: the ids travel behind the values
    and the skyline runs on the speculation that they are strictly increasing
    (ties by position); any other ids re-run the call once they are in.  The
    lattice generator makes (sum, id) ties plentiful, so a wrong tie order
    would show."""
    n = 200_000
    v = sk.generate(gen, n, 3, 17)
    rng = np.random.default_rng(17)
    if ids_kind == "permuted":
        ids = rng.permutation(n).astype(np.int64)
    elif ids_kind == "strided":
        ids = 5 + 3 * np.arange(n, dtype=np.int64)
    elif ids_kind == "one_swap":
        ids = np.arange(n, dtype=np.int64)
        ids[n - 2], ids[n - 1] = ids[n - 1], ids[n - 2]
    else:  # a repeated id: not strictly increasing
        ids = np.arange(n, dtype=np.int64)
        ids[n // 2] = ids[n // 2 - 1]
    res = sk.pipeline(v, ids, cap=25)
    pos, _ = po.skyline_sfs(v, ids)
    assert res.positions.tolist() == pos.tolist()
    den, gm, _ = po.grid_resistance(v[pos], ids[pos], 25)
    assert res.g_max == gm and res.den.tolist() == den.tolist()


@pytest.mark.parametrize("gen,d,ids_kind", [("ant", 3, "permuted"), ("lattice", 3, "permuted"),
                                             ("ant", 7, "one_swap"), ("ant", 7, "sorted")])
def test_late_ids_streamed(gen, d, ids_kind):
    """Streamed host inputs (>= 48 MB): every value chunk first, the ids last;
    the head seed, the seeded filter and the rank-grid engine (ant d = 7)
    order ties by position until the ids are in and checked."""
    n = 2_000_000 if d == 3 else 1_000_000
    v = sk.generate(gen, n, d, 23)
    rng = np.random.default_rng(23)
    ids = np.arange(n, dtype=np.int64)
    if ids_kind == "permuted":
        ids = rng.permutation(n).astype(np.int64)
    elif ids_kind == "one_swap":
        ids[0], ids[1] = ids[1], ids[0]
    res = _host_vs_device(v, ids)
    if d == 3:
        pos, _ = po.skyline_sfs(v, ids)
        assert res.positions.tolist() == pos.tolist()


# ------------------------------------------------ sharded calls with an installed collective
def _emulated_two_ranks(run):
    """Emulate a 2-rank group on one GPU: rank 1 runs first and its MAX
    all-reduce inputs are recorded; rank 0 then runs with a collective that
    MAX-combines each buffer with rank 1's recording of the same call index.
    Returns rank 0's result (what every rank would hold)."""
    import torch
    from paper_2412_02274_b200 import skypar
    from paper_2412_02274_b200.dist import _DeviceBuffer

    def view(ptr, count, eb):
        return torch.as_tensor(_DeviceBuffer(ptr, count, "|u1" if eb == 1 else "<i4"),
                               device="cuda")

    recorded = []

    def record(ptr, count, eb, stream):
        torch.cuda.synchronize()
        recorded.append(view(ptr, count, eb).clone())
        return 0

    calls = iter(range(100))

    def combine(ptr, count, eb, stream):
        torch.cuda.synchronize()
        t = view(ptr, count, eb)
        t.copy_(torch.maximum(t, recorded[next(calls)]))
        torch.cuda.synchronize()
        return 0

    try:
        skypar.set_collective(record)
        run(1)
        skypar.set_collective(combine)
        out = run(0)
    finally:
        skypar.set_collective(None)
    return out, recorded


def test_sharded_rank_grid_skyline_exchange():
    """The rank-grid engine split by grid row: each rank decides its rows,
    the keep flags are MAX-reduced (skyline only here: in the one-GPU
    emulation rank 1 never sees rank 0's flags, so its gres input differs)."""
    v = sk.generate("ant", 300_000, 7, 2)
    full = sk.pipeline(v, cap=25, skip_gres=True)
    assert full.stats["sky_engine"] == sk.SKY_GRID
    out, recorded = _emulated_two_ranks(
        lambda rank: sk.pipeline(v, cap=25, skip_gres=True, shard_rank=rank, shard_world=2))
    keep1 = recorded[0].cpu().numpy()
    assert len(recorded) == 1 and 0 < keep1.sum() < len(full.positions)  # rank 1: its rows only
    assert out.positions.tolist() == full.positions.tolist()


def test_sharded_gres_exchange_returns_full_map():
    v = sk.generate("ant", 50_000, 4, 3)
    full = sk.pipeline(v, cap=25)
    out, recorded = _emulated_two_ranks(
        lambda rank: sk.pipeline(v, cap=25, shard_rank=rank, shard_world=2))
    assert len(recorded) == 1 and recorded[0].dtype.itemsize == 4  # only the den exchange
    assert (recorded[0].cpu().numpy() == 0).any()  # rank 1 left rank 0's tuples at 0
    assert out.positions.tolist() == full.positions.tolist()
    assert out.den.tolist() == full.den.tolist()


# ------------------------------------------------ device-side input preparation
def _np_normalize(v):
    """harness.cpp:161-177 in numpy: std::min/std::max keep the FIRST of equal
    candidates, so a zero minimum carries the sign of the first zero."""
    out = np.zeros_like(v)
    for j in range(v.shape[1]):
        col = v[:, j]
        lo, hi = np.inf, -np.inf
        for x in col:  # literal left-to-right std::min / std::max
            lo = x if x < lo else lo
            hi = x if hi < x else hi
        out[:, j] = (col - lo) / (hi - lo) if hi > lo else 0.0
    return out


@pytest.mark.parametrize("seed", [1, 2])
def test_normalize_bit_identical(seed):
    rng = np.random.default_rng(seed)
    v = rng.random((3000, 5)) * [1, 10, 1e-300, 7, 1]
    v[:, 3] = 7.0                      # constant attribute -> 0
    v[5, 4], v[10, 4], v[20, 4] = 0.0, -0.0, 0.0   # zero minimum, first zero +0.0
    v[2, 0] = -0.0                     # zero minimum, first zero -0.0
    v[7, 0] = 0.0
    got = sk.normalize(v)
    want = _np_normalize(v)
    assert got.tobytes() == want.tobytes()


@pytest.mark.parametrize("gen,n,d,k", [("ant", 5000, 3, 10), ("uni", 3000, 4, 100),
                                       ("lattice", 2000, 3, 25), ("ant", 50, 2, 100)])
def test_select_representatives_matches_reference_rule(gen, n, d, k):
    v = sk.generate(gen, n, d, 7)
    rng = np.random.default_rng(7)
    ids = rng.permutation(5 * n)[:n].astype(np.int64)
    pos, tests = sk.select_representatives(v, ids, k)
    s = np.array([sum(row) for row in v.tolist()])  # left-to-right sums
    picked = np.lexsort((ids, s))[:min(k, n)]
    want, want_tests = [], 0
    for i in picked:  # partition.cpp:229-245
        dom = False
        for j in picked:
            if j == i:
                continue
            want_tests += 1
            if np.all(v[j] <= v[i]) and np.any(v[j] < v[i]):
                dom = True
                break
        if not dom:
            want.append(int(i))
    assert pos.tolist() == want and tests == want_tests


def test_pipeline_normalize_flag_equals_normalized_input():
    v = sk.generate("ant", 20000, 3, 4) * [3.0, 0.5, 100.0]
    a = sk.pipeline(v, cap=25, normalize=True)
    b = sk.pipeline(_np_normalize(v), cap=25)
    assert a.positions.tolist() == b.positions.tolist()
    assert a.g_max == b.g_max and a.den.tolist() == b.den.tolist()
