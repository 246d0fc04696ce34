# compare the skyline engines per workload
for w in ${WORKLOADS:-C1 C2 C3 C4}; do for e in rounds grid; do
  timeout 600 python bench.py --steps 5 --warmup 3 --workload $w --sky-engine $e --no-cpu-baseline > gpurun_out/eng_${w}_$e.log 2>&1
  python -c "import json; d=json.loads(open('gpurun_out/eng_${w}_$e.log').read().strip().splitlines()[-1]); print('$w $e', round(d['ms_per_step'],3), 'e2e', round(d['e2e']['ms_per_step'],3), d['stage_ms'], d['tests']['skyline'])"
done; done
