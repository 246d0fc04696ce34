import sys, time, json
sys.path.insert(0, '.')
import numpy as np
import paper_2412_02274_b200 as sk
for n in [int(x) for x in sys.argv[1:]]:
    v = sk.generate("ant", n, 7, 1)
    t0 = time.time()
    r = sk.pipeline(v, cap=25, skip_gres=True)
    t1 = time.time()
    st = r.stats
    print(json.dumps({"n": n, "S": len(r.positions), "wall_s": round(t1 - t0, 3), "sky_ms": st["ms_skyline"],
                      "tests": st["skyline_tests"], "rounds": st["sfs_rounds"]}), flush=True)
    if t1 - t0 > 60: break
