"""Extended seeded sweep of tests/test_gpu_fuzz (beyond the suite's 200 seeds):
python scripts/fuzz_sweep.py LO HI — every case against the CPU oracle; prints
the failing seeds.  Run per chunk under `timeout` (a hang shows as a missing
summary line)."""
import os, sys, time
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, root); sys.path.insert(0, os.path.join(root, "tests"))
import test_gpu_fuzz as t
lo, hi = int(sys.argv[1]), int(sys.argv[2])
bad = []
t0 = time.time()
for seed in range(lo, hi):
    print("seed", seed, flush=True)
    try:
        t.test_random_pipeline_against_oracle(seed)
    except BaseException as e:  # noqa: BLE001
        bad.append(seed)
        print("FAIL", seed, repr(e)[:300], flush=True)
print(f"SUMMARY {lo}-{hi}: {hi - lo - len(bad)} ok, failing {bad}, {time.time() - t0:.0f} s", flush=True)
