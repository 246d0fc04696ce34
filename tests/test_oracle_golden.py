"""Pin the CPU oracle (oracle/skyoracle.c) against the reference's own outputs
(tests/golden, made by the unmodified reference library) and the reference's
known-answer tests.  CPU only."""
import numpy as np
import pytest

from conftest import golden_input, golden_names, load_golden, spec_cap
from oracle import pyoracle as po

SMALL = golden_names(exclude=("C4_", "C5_prefix_10k", "C5_prefix_20k"))


@pytest.mark.parametrize("name", SMALL)
def test_oracle_matches_reference_golden(name):
    g = load_golden(name)
    v, ids = golden_input(g, po.generate)
    if "error" in g:
        assert g["spec"]["strategy"] == "grid"  # the only contract error in the fixtures
        bad = [(i, j) for i in range(len(v)) for j in range(v.shape[1]) if not 0.0 <= v[i, j] <= 1.0]
        i, j = bad[0]
        assert g["error"].startswith(f"grid_cell: value {v[i, j]:.6f} in attribute {j + 1} outside [0,1]")
        return
    pos, _ = po.skyline_sfs(v, ids)
    assert sorted(ids[pos].tolist()) == g["skyline_ids"]
    assert ids[pos].tolist() == g["skyline_order"]
    if "bruteforce_ids" in g:
        assert sorted(po.skyline_bruteforce(v).tolist()) == g["bruteforce_ids"]
    if "gres_error" in g:
        assert "not a skyline" in g["gres_error"]
        return
    sky = v[pos]
    den, gm, _ = po.grid_resistance(sky, ids[pos], spec_cap(g))
    assert gm == g["g_max"]
    got = dict(zip(ids[pos].tolist(), den.tolist()))
    assert [got[i] for i in g["skyline_ids"]] == g["den"]
    assert g["rows"] == list(range(gm, 1, -1))
    if "bruteforce_den" in g:
        assert g["bruteforce_den"] == g["den"]  # stability (acceptance criterion 3)
    if gm >= 2 and sky.shape[1] <= 5 and np.all(sky < 1.0) and len(sky) <= 20000:
        cells = po.gres_cells(sky, gm)  # independent S-independent check
        assert (cells == den).all()


def test_mt19937_64_pin():
    # proj/tests/test_datagen.cpp:43-58: the 10000th draw of mt19937_64(5489)
    assert po.mt64_nth(5489, 10000) == 9981545732273789042


def test_snap_kats():
    # proj/tests/test_gres.cpp:26-34
    assert po.snap(np.array([0.0, 0.0]), 7).tolist() == [0.0, 0.0]
    assert po.snap(np.array([0.30, 0.62]), 5).tolist() == [0.2, 0.6]


def test_max_grid_intervals_kats():
    # proj/tests/test_gres.cpp:61-73
    assert po.max_grid_intervals(np.array([[0.2], [0.7]]), None) == 2
    assert po.max_grid_intervals(np.array([[0.2, 0.9], [0.24, 0.9]]), None) == 25
    assert po.max_grid_intervals(np.array([[0.2, 0.9], [0.24, 0.9]]), 10) == 10
    with pytest.raises(ValueError, match="identical"):
        po.max_grid_intervals(np.array([[0.3, 0.3], [0.3, 0.3]]), 25)
    tiny = np.array([[0.5], [0.5 + 1e-12]])
    with pytest.raises(ValueError, match="overflows"):
        po.max_grid_intervals(tiny, None)
    assert po.max_grid_intervals(tiny, 25) == 25


def test_plan_sizing_kats():
    # partition.cpp:24-31,53-83 and SURVEY.md §8(a) a6
    assert po.make_plan("grid", 64, 5) == (2, 32)
    assert po.make_plan("angular", 64, 5) == (3, 81)
    assert po.make_plan("sliced", 64, 5) == (1, 64)
    assert po.make_plan("angular", 64, 7) == (2, 64)
    assert po.make_plan("grid", 16, 3) == (2, 8)
    assert po.make_plan("grid", 16, 4) == (2, 16)
    assert po.make_plan("grid", 16, 6) == (2, 64)
    assert po.make_plan("angular", 16, 3) == (4, 16)
    assert po.make_plan("angular", 16, 4) == (2, 8)
    assert po.make_plan("angular", 16, 6) == (2, 32)
    assert po.make_plan("none", 16, 3) == (1, 1)


def test_anti_diagonal_sfs_counts():
    # proj/tests/test_core.cpp:116-133: SFS does n(n-1)/2 tests on incomparable tuples
    n = 64
    v = np.array([[i, n - 1 - i] for i in range(n)], dtype=np.float64)
    pos, tests = po.skyline_sfs(v)
    assert len(pos) == n and tests == n * (n - 1) // 2


def test_fp_tie_predecessor_rule():
    # SFS/parallel keep both, brute force keeps one
    v = np.array([[2e-20, 1.0], [1e-20, 1.0]])
    pos, _ = po.skyline_sfs(v)
    assert sorted(pos.tolist()) == [0, 1]
    assert po.skyline_bruteforce(v).tolist() == [1]


@pytest.mark.parametrize("seed", [1, 2, 3])
def test_cells_equals_sfs_scan(seed):
    v = po.generate("ant", 3000, 4, seed)
    pos, _ = po.skyline_sfs(v)
    den, gm, _ = po.grid_resistance(v[pos], pos, 25)
    assert (po.gres_cells(v[pos], gm) == den).all()
