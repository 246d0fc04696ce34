"""C5 scaling probe: skyline (and optionally gres) of ant d=7 prefixes."""
import json
import sys
import time

sys.path.insert(0, '.')
import paper_2412_02274_b200 as sk  # noqa: E402

gres = "--gres" in sys.argv
eng = {"auto": sk.SKY_AUTO, "grid": sk.SKY_GRID, "rounds": sk.SKY_ROUNDS}[
    next((a.split("=")[1] for a in sys.argv if a.startswith("--engine=")), "auto")]
for n in [int(x) for x in sys.argv[1:] if not x.startswith("--")]:
    v = sk.generate("ant", n, 7, 1)
    for rep in range(2):
        t0 = time.time()
        r = sk.pipeline(v, cap=25, skip_gres=not gres, sky_engine=eng)
        t1 = time.time()
        st = r.stats
        print(json.dumps({"n": n, "rep": rep, "S": len(r.positions), "wall_s": round(t1 - t0, 3),
                          "sky_ms": round(st["ms_skyline"], 2), "sky_kernel_ms": round(st["ms_sky_kernel"], 2),
                          "gres_ms": round(st["ms_gres"], 2), "g_max": r.g_max,
                          "engine": st["sky_engine"], "gres_engine": st["gres_engine"],
                          "tests": st["skyline_tests"], "rounds": st["sfs_rounds"]}), flush=True)
        if t1 - t0 > 60:
            break
