# K6 grid-shape sweep on C5 (skyline only)
for row in 512 256 128 64 32; do for k0 in 64 128; do
SKYGPU_GRID_ROW=$row SKYGPU_GRID_K0=$k0 timeout 300 python - <<'PY'
import os, sys, time, json
sys.path.insert(0, ".")
import paper_2412_02274_b200 as sk
v = sk.generate("ant", 10_000_000, 7, 1)
pl = sk.make_plan("angular", 64, 7)
for i in range(3):
    r = sk.pipeline(v, None, pl, cap=25, skip_gres=True)
st = r.stats
print(os.environ["SKYGPU_GRID_ROW"], os.environ["SKYGPU_GRID_K0"], "S", len(r.positions), "sky_ms", round(st["ms_skyline"], 3),
      "k6_ms", round(st["ms_sky_kernel"], 3), "units", st["sky_units"], "tests", st["skyline_tests"], flush=True)
PY
done; done
