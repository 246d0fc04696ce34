# round 2 session 4: the full GPU suite (per-test timeout) on the K6 fix + replicated tables, then the K6 A/B on C5
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 2400 python -m pytest tests -m gpu -q -x --timeout 300 --timeout-method=thread --durations=12 > gpurun_out/r2s4_pytest_gpu.log 2>&1; echo "suite rc=$?"; tail -22 gpurun_out/r2s4_pytest_gpu.log
summ() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['stage_ms'].items()}, 'e2e', round(d['e2e']['ms_per_step'],3), 'roof', d['roofline']['kernel'], round(d['roofline']['frac'],3), 'other', round(d['roofline']['other']['frac'] or 0,3))"; }
for e in "SKYGPU_K6_REPL=0" "SKYGPU_K6_REPL=1" "SKYGPU_K6_REPL=0" "SKYGPU_K6_REPL=1"; do
  env $e timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/k6repl_$e.log 2>&1; echo "bench C5 [$e] rc=$?"; summ < gpurun_out/k6repl_$e.log
done
