"""Dump (or compare against a dump of) the C5 skyline positions of the
current K6 kernel choice (SKYGPU_GRID_KERNEL) — A/B equality check."""
import sys
import time

sys.path.insert(0, '.')
import numpy as np  # noqa: E402

import paper_2412_02274_b200 as sk  # noqa: E402

n = int(sys.argv[2]) if len(sys.argv) > 2 else 10_000_000
v = sk.generate("ant", n, 7, 1)
plan = sk.make_plan("angular", 64, 7)
res = sk.pipeline(v, None, plan, cap=25, skip_gres=True)
t0 = time.time()
res = sk.pipeline(v, None, plan, cap=25, skip_gres=True)
print("S", len(res.positions), "engine", res.stats["sky_engine"], "tests", res.stats["skyline_tests"],
      "wall", round(time.time() - t0, 3))
path = sys.argv[1]
if path.startswith("cmp:"):
    ref = np.load(path[4:])
    ok = np.array_equal(ref, res.positions)
    print("EQUAL" if ok else "MISMATCH", len(ref), len(res.positions))
    sys.exit(0 if ok else 1)
np.save(path, res.positions)
