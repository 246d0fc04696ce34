# bench every partitioning plan on one workload
W=${W:-C2}
for s in none grid angular sliced; do
  python bench.py --steps 10 --warmup 3 --workload $W --strategy $s --no-cpu-baseline > gpurun_out/plan_${W}_$s.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/plan_${W}_$s.log').read().strip().splitlines()[-1]); print('$W $s', round(d['ms_per_step'],4), d['stage_ms']['skyline'], d['tests'])"
done
