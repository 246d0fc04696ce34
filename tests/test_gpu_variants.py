"""The process-static alternatives of the library (SKYGPU_* switches, read
once per process) against the reference goldens: each runs in its own
subprocess.  Covers the one-CTA A' regrouping (SKYGPU_CELL_ORDER=1), the
quantile-grid K5 pruning (SKYGPU_QGRID=1), the plan-cell K5 scan order
(SKYGPU_SCAN_CELLS=plan, the paper's grid/angular/sliced partitions as the
scan order) and the per-lane ALU rank-grid decide kernel
(SKYGPU_GRID_KERNEL=alu) — all three skyline engine choices each."""
import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))
CASES = ",".join(["C1_uni_100k_d4", "C2_ant_1M_d3", "C5_prefix_10k_d7", "rand_ant_n1500_d5_angular",
                  "rand_lattice_n1500_d4_angular", "rand_uni_n1500_d3_grid",
                  "rand_lattice_n1500_d3_sliced", "uncapped_lattice_d3", "huge_values_ties"])


def _run(env, *extra):
    e = dict(os.environ)
    e.update(env)
    out = subprocess.check_output([sys.executable, os.path.join(HERE, "_env_variant.py"), CASES,
                                   *extra], env=e, text=True, timeout=900)
    return json.loads(out.strip().splitlines()[-1])


@pytest.mark.parametrize("env", [{"SKYGPU_CELL_ORDER": "1"}, {"SKYGPU_QGRID": "1"},
                                 {"SKYGPU_SCAN_CELLS": "plan"},
                                 {"SKYGPU_QGRID": "1", "SKYGPU_CELL_ORDER": "1"},
                                 {"SKYGPU_PDL": "0"}, {"SKYGPU_CELLS_UNFUSED": "1"},
                                 {"SKYGPU_CELLS_SMEM": "0"}, {"SKYGPU_GRES_TILED": "1"},
                                 {"SKYGPU_INTRA": "1"}, {"SKYGPU_INTRA": "2"},
                                 {"SKYGPU_FUSED_SELECT": "0"}, {"SKYGPU_NO_SPEC_FINAL": "1"},
                                 {"SKYGPU_NO_DEV_ROUND": "1"}, {"SKYGPU_OVERLAP": "0"},
                                 {"SKYGPU_PREFIX": "1500", "SKYGPU_SOLO": "4",
                                  "SKYGPU_DIR_PER_CELL": "32"},
                                 {"SKYGPU_IDS_LATE": "0"}, {"SKYGPU_GRID_SORT": "1"},
                                 {"SKYGPU_GRID_RECSCATTER": "0"},
                                 {"SKYGPU_GRID_ROW": "128",
                                                            "SKYGPU_GRID_K0": "16"}])
def test_env_variant_matches_goldens(env):
    r = _run(env)
    assert r["bad"] == [], r


def test_grid_decide_alu_and_tma_kernels_agree(tmp_path):
    """The two K6 kernels (TMA bitset default, per-lane ALU) on a C5-shaped
    1M-tuple relation (rank-grid engine): identical skyline, ids and order."""
    path = str(tmp_path / "pos.npy")
    a = _run({"SKYGPU_GRID_KERNEL": "alu"}, "1000000", path)
    assert a["bad"] == [], a
    b = _run({}, "1000000", path)
    assert b["bad"] == [], b


_BITSET = """
import sys, numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2412_02274_b200 as sk
bad = []
for gen, n, d in (("ant", 40000, 7), ("ant", 30000, 5), ("lattice", 20000, 6), ("uni", 40000, 4)):
    v = sk.generate(gen, n, d, 3)
    a = sk.pipeline(v, cap=25, engine=sk.GRES_PAIRS)
    b = sk.pipeline(v, cap=25, engine=sk.GRES_CELLS)
    if a.den.tolist() != b.den.tolist() or (b.g_max >= 2 and b.stats["gres_cells"] == 0):
        bad.append(f"{gen}{n}d{d}")
print(bad)
"""


@pytest.mark.parametrize("env", [{"SKYGPU_CELLS_BITSET": "1"}, {"SKYGPU_CELLS_SORT": "1"},
                                 {"SKYGPU_MG_NOCOL": "1"}, {"SKYGPU_MG_NOPRIV": "1"},
                                 {"SKYGPU_MG_PAIRSMEM": "1"}, {"SKYGPU_MG_LOADFIRST_MB": "100000"},
                                 {"SKYGPU_MG_NOPRIV": "1", "SKYGPU_MG_LOADFIRST_MB": "0"},
                                 {"SKYGPU_MG_RED_MB": "0"}, {"SKYGPU_MG_RED_MB": "100000"},
                                 {"SKYGPU_MG_RED_MB": "100000", "SKYGPU_MG_NOPRIV": "1"},
                                 {"SKYGPU_MG_PRIV_CELLS": "40960", "SKYGPU_MG_RED_MB": "0"}])
def test_cell_engine_variants(env):
    """The HBM cell engine's alternatives against the pair engine's map:
    SKYGPU_CELLS_BITSET=1 the u32/u64 bitset-row form (the min-grid form is
    the default), SKYGPU_CELLS_SORT=1 the min-grid over a locality order (the
    top step's rows), SKYGPU_MG_NOCOL=1 the slab pass without the dim-3 running
    minimum (one more sweep), SKYGPU_MG_NOPRIV=1 every step marked in HBM (no
    shared-memory privatised marks), SKYGPU_MG_PAIRSMEM=1 the shared-memory staged form of
    the two-dim sweep."""
    e = dict(os.environ, SKYGPU_CELLS_SMEM="0", **env)
    out = subprocess.check_output([sys.executable, "-c", _BITSET, os.path.dirname(HERE)], env=e,
                                  text=True, timeout=900)
    assert out.strip().splitlines()[-1] == "[]", out
