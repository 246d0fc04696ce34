"""assign_partitions (partition.cpp:183-213): the CPU oracle's restatement
pinned to the reference's own ids (tests/golden/partition/pids_cases.json.gz,
made by oracle/refdrive --mode pids through the unmodified reference), and the
device assign_partitions (skygpu_assign_partitions) against both; plus the
plan-partitioned local-skyline pruning engine (SKYGPU_SKY_PARTS) against the
reference goldens."""
import gzip
import json
import os

import numpy as np
import pytest

from conftest import GOLDEN, golden_input, golden_names, load_golden, spec_cap
from oracle import pyoracle as po

with gzip.open(os.path.join(GOLDEN, "partition", "pids_cases.json.gz"), "rt") as _f:
    CASES = json.load(_f)["cases"]
CASE_IDS = [f"{c['gen']}_n{c['n']}_d{c['d']}_{c['strategy']}{c['p']}" for c in CASES]


def _input(c):
    return po.generate(c["gen"], c["n"], c["d"], c["seed"])


def _angular_boundary(v, slices):
    """per tuple: True when some angle's (2 angle / pi) * m lies within 1e-9 of
    an integer (where a last-ulp atan2 difference may flip the slice)"""
    n, d = v.shape
    out = np.zeros(n, dtype=bool)
    tail = np.zeros((n, d + 1))
    for j in range(d - 1, -1, -1):
        tail[:, j] = tail[:, j + 1] + v[:, j] * v[:, j]
    for j in range(d - 1):
        f = (2.0 * np.arctan2(np.sqrt(tail[:, j + 1]), v[:, j]) / np.pi) * slices
        out |= np.abs(f - np.round(f)) < 1e-9
    return out


@pytest.mark.parametrize("k", range(len(CASES)), ids=CASE_IDS)
def test_oracle_pids_match_reference(k):
    c = CASES[k]
    v = _input(c)
    got = po.assign_partitions(v, None, c["strategy"], c["slices"], c["partitions"])
    assert got.tolist() == c["pids"]
    assert got.min() >= 0 and got.max() < c["partitions"]


def test_oracle_sliced_ties_follow_ids():
    # equal attribute-0 values order by id (partition.cpp:197-203): reversing
    # the ids reverses the order inside every tie group
    v = np.array([[0.5, 0.1], [0.5, 0.2], [0.5, 0.3], [0.1, 0.9]])
    assert po.assign_partitions(v, None, "sliced", 1, 4).tolist() == [1, 2, 3, 0]
    ids = np.array([9, 8, 7, 6], dtype=np.int64)
    assert po.assign_partitions(v, ids, "sliced", 1, 4).tolist() == [3, 2, 1, 0]


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(CASES)), ids=CASE_IDS)
def test_device_pids_match_reference(k):
    import paper_2412_02274_b200 as sk
    c = CASES[k]
    v = _input(c)
    plan = sk.make_plan(c["strategy"], c["p"], c["d"])
    assert (plan.slices, plan.partitions) == (c["slices"], c["partitions"])
    got = sk.assign_partitions(v, plan)
    ref = np.asarray(c["pids"])
    diff = got != ref
    if c["strategy"] == "angular":
        # the device atan2 may differ from glibc's in the last ulp: only at a
        # slice boundary, never elsewhere
        assert not (diff & ~_angular_boundary(v, c["slices"])).any(), np.flatnonzero(diff)[:10]
    else:
        assert not diff.any(), np.flatnonzero(diff)[:10]


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["grid", "angular", "sliced"])
@pytest.mark.parametrize("gen,d", [("uni", 4), ("ant", 7), ("lattice", 3)])
def test_device_pids_match_oracle_shuffled_ids(strategy, gen, d):
    import paper_2412_02274_b200 as sk
    v = po.generate(gen, 20000, d, 5)
    ids = np.random.default_rng(3).permutation(40000)[:20000].astype(np.int64)
    plan = sk.make_plan(strategy, 64, d)
    got = sk.assign_partitions(v, plan, ids)
    ref = po.assign_partitions(v, ids, strategy, plan.slices, plan.partitions)
    diff = got != ref
    if strategy == "angular":
        diff &= ~_angular_boundary(v, plan.slices)
    assert not diff.any()


@pytest.mark.gpu
def test_device_pids_grid_out_of_range_error():
    import paper_2412_02274_b200 as sk
    v = np.array([[0.2, 0.3], [0.4, 1.5], [2.0, 0.1]])
    with pytest.raises(ValueError, match=r"grid_cell: value 1\.500000 in attribute 2 outside \[0,1\]"):
        sk.assign_partitions(v, sk.make_plan("grid", 4, 2))


# ---------------------------------------------------------------- pruning
PRUNE_CASES = golden_names(prefixes=("rand_", "kat_", "reps", "uncapped_", "huge_", "big_",
                                     "C1_", "C2_", "C3_", "C5_prefix_"))


@pytest.mark.gpu
@pytest.mark.parametrize("name", PRUNE_CASES)
def test_local_prune_matches_reference_golden(name):
    import paper_2412_02274_b200 as sk
    g = load_golden(name)
    if "error" in g or g["spec"].get("reps", 0):
        pytest.skip("contract error / representatives case")
    v, ids = golden_input(g, sk.generate)
    sp = g["spec"]
    plan = sk.make_plan(sp["strategy"], sp["p"], sp["d"])
    res = sk.pipeline(v, ids, plan, cap=spec_cap(g), local_prune=True,
                      skip_gres="gres_error" in g)
    assert ids[res.positions].tolist() == g["skyline_order"]
    if "g_max" in g:
        assert res.g_max == g["g_max"]
        got = dict(zip(ids[res.positions].tolist(), res.den.tolist()))
        assert [got[i] for i in g["skyline_ids"]] == g["den"]
    assert res.stats["tuples_into_final"] <= res.stats["tuples_into_parallel"] <= len(v)
    assert res.stats["tuples_into_final"] >= len(g["skyline_ids"])


@pytest.mark.gpu
@pytest.mark.parametrize("strategy", ["none", "grid", "angular", "sliced"])
@pytest.mark.parametrize("gen,n,d", [("uni", 200000, 4), ("ant", 200000, 3), ("ant", 50000, 7),
                                     ("lattice", 100000, 3)])
def test_local_prune_plan_invariance(strategy, gen, n, d):
    # acceptance_main.cpp:145-184: every plan gives the same skyline and map;
    # the pruned engine must equal the unpruned one (and the oracle)
    import paper_2412_02274_b200 as sk
    v = sk.generate(gen, n, d, 9)
    ids = np.arange(n, dtype=np.int64)
    plan = sk.make_plan(strategy, 64, d)
    base = sk.pipeline(v, ids, plan, cap=25)
    pr = sk.pipeline(v, ids, plan, cap=25, local_prune=True)
    assert pr.positions.tolist() == base.positions.tolist()
    assert pr.den.tolist() == base.den.tolist()
    pos, _ = po.skyline_sfs(v, ids)
    assert pr.positions.tolist() == pos.tolist()
    if strategy != "none":
        assert pr.stats["tuples_into_final"] < n  # the partitions pruned something


@pytest.mark.gpu
@pytest.mark.parametrize("gen,n,d,pruned", [("ant", 300000, 7, False), ("uni", 400000, 4, True)])
def test_local_prune_probe_gate(gen, n, d, pruned):
    """From 2^18 tuples a probe (every (n >> 13)-th tuple) runs first; when the
    windows dominate under a quarter of it (skyline-heavy data) the full pass
    prunes nothing and the merge engine decides everything.  Either way the
    result is the unpruned engine's."""
    import paper_2412_02274_b200 as sk
    v = sk.generate(gen, n, d, 5)
    plan = sk.make_plan("angular", 64, d)
    base = sk.pipeline(v, None, plan, cap=25)
    pr = sk.pipeline(v, None, plan, cap=25, local_prune=True)
    assert pr.positions.tolist() == base.positions.tolist()
    assert pr.den.tolist() == base.den.tolist()
    if pruned:
        assert pr.stats["tuples_into_final"] < n // 2
    else:
        assert pr.stats["tuples_into_final"] == n


@pytest.mark.gpu
def test_local_prune_shuffled_and_late_ids():
    # ties by id with ids not in position order (the late-ids redo path)
    import paper_2412_02274_b200 as sk
    v = po.generate("lattice", 120000, 3, 4)
    ids = np.random.default_rng(8).permutation(10 ** 6)[:120000].astype(np.int64)
    for strategy in ("angular", "sliced"):
        plan = sk.make_plan(strategy, 16, 3)
        pr = sk.pipeline(v, ids, plan, cap=25, local_prune=True)
        pos, _ = po.skyline_sfs(v, ids)
        assert pr.positions.tolist() == pos.tolist()
        den, gm, _ = po.grid_resistance(v[pos], ids[pos], 25)
        assert pr.g_max == gm and pr.den.tolist() == den.tolist()


# ---------------------------------------------------------------- skyline_bnl
BNL_CASES = [n for n in golden_names() if "bruteforce_ids" in load_golden(n)]


@pytest.mark.gpu
@pytest.mark.parametrize("name", BNL_CASES)
def test_skyline_bnl_matches_reference_bruteforce(name):
    # core.cpp:25-46: BNL's set is the brute-force skyline (test_core.cpp:92-103,
    # acceptance_main.cpp:55-69 compare id sets) — incl. kat_fp_tie, where the
    # SFS order keeps a tuple an equal-sum successor dominates
    import paper_2412_02274_b200 as sk
    g = load_golden(name)
    v, ids = golden_input(g, sk.generate)
    res = sk.skyline_bnl(v, ids)
    assert sorted(res.ids.tolist()) == g["bruteforce_ids"]
    assert res.stats["skyline_size"] == len(g["bruteforce_ids"])


@pytest.mark.gpu
@pytest.mark.parametrize("gen,n,d", [("lattice", 3000, 2), ("lattice", 20000, 3), ("uni", 100000, 4),
                                     ("ant", 20000, 5)])  # (the numpy check is quadratic in S)
def test_skyline_bnl_matches_oracle_bruteforce_sets(gen, n, d):
    import paper_2412_02274_b200 as sk
    v = sk.generate(gen, n, d, 12)
    ids = np.random.default_rng(1).permutation(n).astype(np.int64)
    res = sk.skyline_bnl(v, ids)
    sfs_pos, _ = po.skyline_sfs(v, ids)
    # the brute-force set = SFS set minus equal-sum dominated (oracle check on SFS's set)
    keep = []
    for p in sfs_pos:
        dom = np.all(v[sfs_pos] <= v[p], axis=1) & np.any(v[sfs_pos] < v[p], axis=1)
        keep.append(not dom.any())
    expect = sorted(ids[sfs_pos[np.asarray(keep, dtype=bool)]].tolist())
    assert sorted(res.ids.tolist()) == expect


@pytest.mark.gpu
def test_skyline_bnl_edge_cases():
    import paper_2412_02274_b200 as sk
    assert sk.skyline_bnl(np.zeros((0, 3))).positions.size == 0
    # identical tuples do not dominate each other (test_core.cpp:84-90)
    assert sorted(sk.skyline_bnl(np.ones((5, 2))).ids.tolist()) == [0, 1, 2, 3, 4]
    # anti-diagonal: every tuple kept (test_core.cpp:116-125)
    n = 64
    v = np.array([[i, n - 1 - i] for i in range(n)], dtype=np.float64)
    assert sk.skyline_bnl(v).positions.size == n
    # equal float64 sums, the later (larger id) tuple dominates: BNL drops the earlier
    v = np.array([[2e-20, 1.0], [1e-20, 1.0], [0.5, 0.5]])
    assert sorted(sk.skyline_bnl(v).ids.tolist()) == [1, 2]
