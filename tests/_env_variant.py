"""Helper of test_gpu_variants.py: run golden cases through the pipeline in a
process whose environment selects an alternative kernel / scan layout
(process-static SKYGPU_* switches), print one JSON line of mismatches."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import paper_2412_02274_b200 as sk  # noqa: E402
from conftest import golden_input, load_golden, spec_cap  # noqa: E402

bad = []
for name in sys.argv[1].split(","):
    g = load_golden(name)
    v, ids = golden_input(g, sk.generate)
    plan = sk.make_plan(g["spec"]["strategy"], g["spec"]["p"], v.shape[1])
    for eng in (sk.SKY_AUTO, sk.SKY_ROUNDS, sk.SKY_GRID):
        res = sk.pipeline(v, ids, plan, cap=spec_cap(g), sky_engine=eng)
        got = dict(zip(ids[res.positions].tolist(), res.den.tolist()))
        if (ids[res.positions].tolist() != g["skyline_order"] or res.g_max != g["g_max"]
                or [got[i] for i in g["skyline_ids"]] != g["den"]):
            bad.append(f"{name}/engine{eng}")
if len(sys.argv) > 2:  # full C5-shaped check: this kernel choice vs a dump
    n = int(sys.argv[2])
    v = sk.generate("ant", n, 7, 1)
    res = sk.pipeline(v, None, sk.make_plan("angular", 64, 7), cap=25, skip_gres=True)
    path = sys.argv[3]
    if os.path.exists(path):
        if not np.array_equal(np.load(path), res.positions):
            bad.append(f"ant{n}d7 positions differ from {path}")
    else:
        np.save(path, res.positions)
print(json.dumps({"env": {k: v for k, v in os.environ.items() if k.startswith("SKYGPU_")},
                  "bad": bad}))
