"""Full-scale BASELINE config 5 (anti-correlated n = 10,000,000, d = 7,
angular p = 64, cap 25) — the reference itself cannot run it (its SFS merge
is quadratic in the 6.5 M-tuple skyline: days), so the GPU result is pinned
three ways:

  * the skyline by two independent GPU engines: the one-pass rank grid
    (auto) and the prefix rounds (forced) — same ids in the same order;
  * every denominator by the CPU oracle's own cell-occupancy restatement of
    the scan (oracle/skyoracle.c so_gres_cells) over
    the GPU's skyline, and on sampled shards by the GPU pair engine;
  * the skyline's membership on samples by the predecessor rule in numpy.
Prefixes of the same stream are pinned to the reference's goldens
(test_gpu_parity.test_config_goldens: C5_prefix_2k/10k/20k)."""
import numpy as np
import pytest

import paper_2412_02274_b200 as sk
from oracle import pyoracle as po

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N, D = 10_000_000, 7


@pytest.fixture(scope="module")
def c5():
    v = sk.generate("ant", N, D, 1)
    plan = sk.make_plan("angular", 64, D)
    full = sk.pipeline(v, None, plan, cap=25)
    return v, plan, full


def test_c5_engines_and_stats(c5):
    v, plan, full = c5
    assert full.stats["sky_engine"] == sk.SKY_GRID and full.stats["gres_engine"] == sk.GRES_CELLS
    assert len(full.positions) == 6_538_958 and full.g_max == 25
    # the generator's bits: the oracle's restatement of datagen.cpp
    assert np.array_equal(po.generate("ant", 20000, D, 1), v[:20000])


def test_c5_rank_grid_equals_prefix_rounds(c5):
    v, plan, full = c5
    rounds = sk.pipeline(v, None, plan, cap=25, skip_gres=True, sky_engine=sk.SKY_ROUNDS)
    assert rounds.stats["sky_engine"] == sk.SKY_ROUNDS
    assert np.array_equal(rounds.positions, full.positions)


def test_c5_cells_equal_pairs_on_shards(c5):
    v, plan, full = c5
    world, checked = 1000, 0
    for r in (0, 1, 997):
        part = sk.pipeline(v, None, plan, cap=25, engine=sk.GRES_PAIRS, shard_rank=r,
                           shard_world=world)
        assert np.array_equal(part.positions, full.positions)
        m = part.den != 0
        checked += int(m.sum())
        assert np.array_equal(part.den[m], full.den[m])
    assert checked > 10000


def test_c5_resistance_equals_cpu_oracle_cells(c5):
    v, plan, full = c5
    sky = v[full.positions]
    den = po.gres_cells(sky, full.g_max)
    assert np.array_equal(den, full.den)


def test_c5_skyline_membership_by_predecessor_rule(c5):
    v, plan, full = c5
    sums = v[:, 0].copy()
    for j in range(1, D):
        sums = sums + v[:, j]  # left to right, as std::accumulate (core.cpp:21-23)
    ids = np.arange(N)
    mask = np.zeros(N, dtype=bool)
    mask[full.positions] = True
    rng = np.random.default_rng(5)

    def dominated_by_predecessor(t):
        pred = (sums < sums[t]) | ((sums == sums[t]) & (ids < t))
        le = np.all(v <= v[t], axis=1) & np.any(v < v[t], axis=1)
        return bool(np.any(pred & le))

    for t in rng.choice(np.flatnonzero(mask), 40, replace=False):
        assert not dominated_by_predecessor(t)
    for t in rng.choice(np.flatnonzero(~mask), 40, replace=False):
        assert dominated_by_predecessor(t)
