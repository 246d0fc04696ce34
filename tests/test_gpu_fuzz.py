"""Seeded random sweep of the pipeline against the CPU oracle (GPU).

Every speculative or device-sized path of the library (device-sized rounds
and their redo, the ride-along final round, late ids, the speculative capped
gres scan, the streamed head, the engines each flag forces) must give the
reference's answer on any input.  Each case draws a generator, size, arity,
plan, cap, id order, value scale, engine flags and pointer kind from one seed
and compares positions, g_max and every denominator with the oracle
(oracle/skyoracle.c, pinned to the reference's goldens).
"""
import numpy as np
import pytest

import paper_2412_02274_b200 as sk
from paper_2412_02274_b200 import skypar
from oracle import pyoracle as po

pytestmark = pytest.mark.gpu

GENS = ["uni", "ant", "corr", "lattice"]


def _case(seed):
    rng = np.random.default_rng(1000 + seed)
    gen = GENS[rng.integers(len(GENS))]
    d = int(rng.choice([1, 2, 3, 3, 4, 5, 6, 7, 9]))
    n = int(rng.choice([1, 2, 7, 300, 5000, 40000, 90000, 250000]))
    if gen == "ant" and d >= 4:
        n = min(n, 5000 if d >= 5 else 20000)  # (skyline ~ n: keep the oracle quick)
    v = sk.generate(gen, n, d, int(rng.integers(1 << 30)))
    scale = rng.choice(["unit", "unit", "above_one", "ones"])
    if scale == "above_one":
        v = v * 3.0
    elif scale == "ones" and n > 2:
        v[rng.integers(n)] = 1.0  # a value of exactly 1.0 (top code = cap)
    ids_kind = rng.choice(["arange", "arange", "permuted", "strided", "swap"])
    ids = np.arange(n, dtype=np.int64)
    if ids_kind == "permuted":
        ids = rng.permutation(n).astype(np.int64) - n // 2
    elif ids_kind == "strided":
        ids = 7 + 5 * ids
    elif ids_kind == "swap" and n > 1:
        i = int(rng.integers(n - 1))
        ids[i], ids[i + 1] = ids[i + 1], ids[i]
    strategies = ["none", "sliced"] + (["angular"] if d >= 2 else []) + \
        (["grid"] if scale != "above_one" else [])
    strat = strategies[rng.integers(len(strategies))]
    plan = sk.make_plan(strat, int(rng.choice([1, 4, 16, 64])), d)
    cap = [None, 2, 5, 25, 25, 31, 40][rng.integers(7)]
    if cap is None and not (gen == "lattice" or n <= 7):
        cap = 25  # (uncapped: g_max = 1/min gap, ~10^6+ steps on continuous data)
    engine = [sk.GRES_AUTO, sk.GRES_AUTO, sk.GRES_PAIRS, sk.GRES_CELLS][rng.integers(4)]
    sky_engine = [sk.SKY_AUTO, sk.SKY_AUTO, sk.SKY_ROUNDS, sk.SKY_GRID][rng.integers(4)]
    device_ptrs = bool(rng.integers(4) == 0)
    return gen, n, d, v, ids, plan, cap, engine, sky_engine, device_ptrs, scale, strat, ids_kind


def _run(v, ids, plan, cap, engine, sky_engine, device_ptrs):
    if not device_ptrs:
        res = sk.pipeline(v, ids, plan, cap=cap, engine=engine, sky_engine=sky_engine)
        return res.positions.tolist(), res.g_max, res.den.tolist()
    import torch
    n, d = v.shape
    dv = torch.from_numpy(np.ascontiguousarray(v)).cuda()
    di = torch.from_numpy(np.ascontiguousarray(ids)).cuda()
    pos = torch.empty(max(n, 1), dtype=torch.int64, device="cuda")
    den = torch.empty(max(n, 1), dtype=torch.int32, device="cuda")
    S, gm, _ = skypar.pipeline_raw(dv.data_ptr(), di.data_ptr(), n, d, plan, cap or 0, engine, 0,
                                   1, skypar.DEVICE_PTRS | sky_engine, pos.data_ptr(),
                                   den.data_ptr())
    torch.cuda.synchronize()
    return pos[:S].cpu().tolist(), gm, den[:S].cpu().tolist()


@pytest.mark.parametrize("seed", range(200))
def test_random_pipeline_against_oracle(seed):
    (gen, n, d, v, ids, plan, cap, engine, sky_engine, device_ptrs, scale, strat,
     ids_kind) = _case(seed)
    what = f"{gen} n={n} d={d} {strat} cap={cap} eng={engine}/{sky_engine} " \
           f"dev={device_ptrs} {scale} ids={ids_kind}"
    pos, _ = po.skyline_sfs(v, ids)
    try:
        den, gm, _ = po.grid_resistance(v[pos], ids[pos], cap)
    except ValueError:  # uncapped bound overflow: the library must say the same
        with pytest.raises(ValueError):
            _run(v, ids, plan, cap, engine, sky_engine, device_ptrs)
        return
    got_pos, got_gm, got_den = _run(v, ids, plan, cap, engine, sky_engine, device_ptrs)
    assert got_pos == pos.tolist(), what
    assert got_gm == gm, what
    assert got_den == den.tolist(), what
