"""One pipeline call of a bench workload, its stats printed as JSON — run
under ncu (scripts/gpu_itest.sh) so that a kernel's executed instructions per
launch can be divided by the dominance tests the same call counted."""
import json
import sys

sys.path.insert(0, ".")
import bench  # noqa: E402
import paper_2412_02274_b200 as sk  # noqa: E402

w = sys.argv[1]
gen, n, d, seed, strat, p, cap = bench.WORKLOADS[w]
v = sk.generate(gen, n, d, seed)
kw = {}
if len(sys.argv) > 2:
    kw["engine"] = int(sys.argv[2])
res = sk.pipeline(v, None, sk.make_plan(strat, p, d), cap=cap, **kw)
print(json.dumps({"workload": w, "S": len(res.positions), **{k: res.stats[k] for k in
      ("skyline_tests", "gres_tests", "sky_engine", "gres_engine", "code_bits")}}))
