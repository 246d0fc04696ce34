# sweep an env knob over bench runs: VAR=name VALUES="a b c" W=C2
for v in $VALUES; do
  env $VAR=$v python bench.py --steps 10 --warmup 3 --workload ${W:-C2} --no-cpu-baseline > gpurun_out/sweep_${VAR}_$v.log 2>&1
  python -c "import json,sys; d=json.loads(open('gpurun_out/sweep_${VAR}_$v.log').read().strip().splitlines()[-1]); print('$VAR=$v', round(d['ms_per_step'],4), d['stage_ms'], d['tests'])"
done
