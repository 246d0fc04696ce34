timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x -m gpu -k "not fullscale" > gpurun_out/pairs_tests.log 2>&1; echo "parity+fuzz rc=$?"; tail -2 gpurun_out/pairs_tests.log
timeout 300 python -m pytest tests/test_gpu_variants.py -q -x -m gpu -k "GRES_TILED or env_variant" > gpurun_out/pairs_var.log 2>&1; echo "variants rc=$?"; tail -2 gpurun_out/pairs_var.log
WORKLOADS="C5p10k C5p20k" BENCH_ARGS="--no-cpu-baseline" bash scripts/gpu_bench_all.sh > /dev/null 2>&1
python - <<'P'
import json
for l in open('gpurun_out/bench_all.jsonl'):
    try: d=json.loads(l)
    except: continue
    if d.get('impl')=='reference': continue
    print(d['config']['workload'][:14], round(d['ms_per_step'],4), d['stage_ms'], d['roofline']['kernel'], round(d['roofline']['frac'],3))
P
