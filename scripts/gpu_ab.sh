# A/B an env knob on bench workloads: VAR=name VALUES="a b" WORKLOADS="C2 C4"
for w in ${WORKLOADS:-C2}; do for v in $VALUES; do
  env $VAR=$v timeout 300 python bench.py --steps 10 --warmup 3 --workload $w --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$w $VAR=$v', round(d['ms_per_step'],4), 'e2e', round(d['e2e']['ms_per_step'],4), 'sky_k', round(d['stage_ms']['sky_kernels'],4), d['tests']['skyline'])"
done; done
