"""Small invocations of every engine and speculation path, for
compute-sanitizer (memcheck / racecheck / synccheck / initcheck).

Run as  compute-sanitizer --tool <t> python scripts/sanitize_cases.py [case...]
(scripts/gpu_sanitize.sh runs every tool over every case and keeps the logs).
Each case cross-checks two engines of the library against each other on the
same input (no oracle here: the sanitizer's verdict is the point), and exits
non-zero on a mismatch.  Environment switches (SKYGPU_*) are read once per
process, so cases that need one are run in their own process by the shell
script (``--env-case``)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2412_02274_b200 as sk  # noqa: E402
from paper_2412_02274_b200 import skypar  # noqa: E402


def same(a, b, what):
    if not np.array_equal(np.asarray(a), np.asarray(b)):
        raise SystemExit(f"MISMATCH {what}")


def case_rounds():
    # prefix-round engine (K1..K5), capped and uncapped gres, three plans
    for gen, n, d in (("ant", 30000, 3), ("uni", 40000, 5), ("corr", 30000, 6), ("ant", 8000, 9)):
        v = sk.generate(gen, n, d, 3)
        for strat, p in (("angular", 16), ("grid", 8), ("sliced", 16), ("none", 1)):
            r = sk.pipeline(v, None, sk.make_plan(strat, p, d), cap=25, sky_engine=sk.SKY_ROUNDS)
            r2 = sk.pipeline(v, None, sk.make_plan(strat, p, d), cap=25, sky_engine=sk.SKY_ROUNDS,
                             engine=sk.GRES_PAIRS)
            same(r.positions, r2.positions, f"rounds {gen} {strat}")
            same(r.den, r2.den, f"gres auto vs pairs {gen} {strat}")
    v = sk.generate("uni", 3000, 3, 5)
    sk.pipeline(v, None, sk.make_plan("none", 1, 3), cap=None)  # uncapped: float64 gres path


def case_grid():
    # rank-grid engine (K6) against the prefix rounds
    for gen, n, d in (("ant", 60000, 7), ("ant", 80000, 4), ("ant", 50000, 5)):
        v = sk.generate(gen, n, d, 7)
        a = sk.pipeline(v, None, sk.make_plan("angular", 16, d), cap=25, sky_engine=sk.SKY_GRID,
                        skip_gres=True)
        b = sk.pipeline(v, None, sk.make_plan("angular", 16, d), cap=25, sky_engine=sk.SKY_ROUNDS,
                        skip_gres=True)
        same(a.positions, b.positions, f"grid vs rounds {gen} d={d}")


def case_gres():
    # pair engine vs HBM cell engine vs the small-grid shared-memory cell engine
    for gen, n, d in (("ant", 40000, 7), ("ant", 40000, 3), ("uni", 60000, 4)):
        v = sk.generate(gen, n, d, 11)
        pl = sk.make_plan("angular", 8, d)
        a = sk.pipeline(v, None, pl, cap=25, engine=sk.GRES_PAIRS)
        b = sk.pipeline(v, None, pl, cap=25, engine=sk.GRES_CELLS)
        same(a.den, b.den, f"pairs vs cells {gen} d={d}")
        # the gres entry point alone (host values of the skyline)
        s = v[a.positions]
        g = sk.grid_resistance(s, a.positions, pl, cap=25)
        same(g.den, a.den, f"grid_resistance {gen} d={d}")


def case_shards():
    # a 2-way sharded call per shard with the exchange left out: every shard's
    # partial map must be <= the full one and their MAX must equal it
    v = sk.generate("ant", 40000, 7, 13)
    pl = sk.make_plan("angular", 16, 7)
    full = sk.pipeline(v, None, pl, cap=25, engine=sk.GRES_CELLS)
    parts = []
    skypar.set_collective(lambda ptr, count, eb, stream: 0)  # identity exchange
    try:
        for r in range(2):
            parts.append(sk.pipeline(v, None, pl, cap=25, engine=sk.GRES_CELLS, shard_rank=r,
                                     shard_world=2, sky_engine=sk.SKY_ROUNDS))
    finally:
        skypar.set_collective(None)
    same(np.maximum(parts[0].den, parts[1].den), full.den, "shard MAX")


def case_ingest():
    v = sk.generate("uni", 5000, 4, 17)
    nv = skypar.normalize(v * 3.0 + 1.0)
    pos, _ = skypar.select_representatives(nv, None, 10)
    r = sk.pipeline(nv, None, sk.make_plan("grid", 16, 4), cap=25, normalize=True)
    txt = "\n".join(",".join(repr(float(x)) for x in row) for row in v[:2000]).encode()
    vals, ids = skypar.read_csv_bytes(b"a,b,c,d\n" + txt + b"\n", "x.csv")
    same(vals, v[:2000], "csv round trip")
    res, _ = skypar.pipeline_csv(b"a,b,c,d\n" + txt + b"\n", "x.csv", "angular", 8)
    assert len(pos) > 0 and len(r.positions) > 0 and len(res.positions) > 0


def case_accounting():
    v = sk.generate("ant", 20000, 3, 19)
    pids = (np.arange(len(v)) % 8).astype(np.int64)
    acc = skypar.sfs_accounting(v, None, pids, 8)
    r = sk.pipeline(v, None, sk.make_plan("none", 1, 3), cap=25, skip_gres=True)
    same(np.sort(acc.positions), np.sort(r.positions), "accounting skyline")


CASES = {"rounds": case_rounds, "grid": case_grid, "gres": case_gres, "shards": case_shards,
         "ingest": case_ingest, "accounting": case_accounting}

if __name__ == "__main__":
    skypar.set_device(0)
    names = sys.argv[1:] or list(CASES)
    for nm in names:
        CASES[nm]()
        print(f"case {nm} ok", flush=True)
