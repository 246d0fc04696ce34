"""CPU side: the oracle's independent cell-occupancy restatement of the scan
(oracle/skyoracle.c so_gres_cells) over the GPU's
full-scale C5 skyline; every denominator must match."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, '.')
from oracle import pyoracle as po  # noqa: E402

z = np.load(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/c5_full_gpu.npz")
n = 10_000_000
mask = np.unpackbits(z["mask"])[:n].astype(bool)
v = po.generate("ant", n, 7, 1)
sky = v[mask]
t0 = time.time()
den = po.gres_cells(sky, int(z["g_max"]))
out = {"n": n, "d": 7, "S": int(mask.sum()), "g_max": int(z["g_max"]),
       "cpu_oracle_s": round(time.time() - t0, 1),
       "mismatches": int((den != z["den"].astype(np.int32)).sum()),
       "den_hist": {int(g): int(c) for g, c in zip(*np.unique(den, return_counts=True))}}
# the skyline itself, sampled against the predecessor rule:
# a kept tuple has no dominating predecessor in (sum, id) order, a dropped one has
sums = v[:, 0].copy()
for j in range(1, v.shape[1]):
    sums = sums + v[:, j]  # left to right, as std::accumulate
rng = np.random.default_rng(0)
ids = np.arange(n)


def dominated_by_predecessor(t):
    pred = (sums < sums[t]) | ((sums == sums[t]) & (ids < t))
    le = np.all(v <= v[t], axis=1) & np.any(v < v[t], axis=1)
    return bool(np.any(pred & le))


kept = rng.choice(np.flatnonzero(mask), 200, replace=False)
dropped = rng.choice(np.flatnonzero(~mask), 200, replace=False)
out["sampled_kept_ok"] = int(sum(not dominated_by_predecessor(t) for t in kept))
out["sampled_dropped_ok"] = int(sum(dominated_by_predecessor(t) for t in dropped))
print(json.dumps(out))
ok = out["mismatches"] == 0 and out["sampled_kept_ok"] == 200 and out["sampled_dropped_ok"] == 200
sys.exit(0 if ok else 1)
