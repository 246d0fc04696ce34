"""Full-scale C5 check (10 M anti-correlated tuples, d = 7): no CPU can run
the reference here, so the GPU result is cross-checked by INDEPENDENT GPU
algorithms on the same input:
  skyline: the rank-grid engine (default) vs the prefix-round engine
           (exact same ids AND order);
  gres:    the cell-occupancy engine (default at this S) vs the pair-dominance
           engine on sampled shards of the skyline (interleaved chunks).
Both engines are parity-tested against the reference's goldens at small sizes.
"""
import json
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import paper_2412_02274_b200 as sk  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 10_000_000
shards = [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1", "2"])]
world = 1000
v = sk.generate("ant", n, 7, 1)
plan = sk.make_plan("angular", 64, 7)
out = {"n": n, "d": 7, "plan": "angular p=64", "cap": 25}
t0 = time.time()
full = sk.pipeline(v, None, plan, cap=25)
out["auto"] = {"S": int(len(full.positions)), "g_max": full.g_max,
               "sky_engine": full.stats["sky_engine"], "gres_engine": full.stats["gres_engine"],
               "wall_s": round(time.time() - t0, 2),
               "den_hist": {int(g): int(c) for g, c in zip(*np.unique(full.den, return_counts=True))}}
t0 = time.time()
rounds = sk.pipeline(v, None, plan, cap=25, skip_gres=True, sky_engine=sk.SKY_ROUNDS)
out["rounds"] = {"S": int(len(rounds.positions)), "sky_engine": rounds.stats["sky_engine"],
                 "sfs_rounds": rounds.stats["sfs_rounds"], "wall_s": round(time.time() - t0, 2)}
out["skyline_equal"] = bool(np.array_equal(rounds.positions, full.positions))
checked = mism = 0
for r in shards:
    t0 = time.time()
    part = sk.pipeline(v, None, plan, cap=25, engine=sk.GRES_PAIRS, shard_rank=r, shard_world=world)
    assert np.array_equal(part.positions, full.positions)
    m = part.den != 0
    checked += int(m.sum())
    mism += int((part.den[m] != full.den[m]).sum())
    out.setdefault("pairs_shards", []).append({"rank": r, "world": world, "tuples": int(m.sum()),
                                               "gres_tests": part.stats["gres_tests"],
                                               "wall_s": round(time.time() - t0, 2)})
out["gres_checked"] = checked
out["gres_mismatches"] = mism
out["ok"] = out["skyline_equal"] and mism == 0 and checked > 0
print(json.dumps(out), flush=True)
sys.exit(0 if out["ok"] else 1)
