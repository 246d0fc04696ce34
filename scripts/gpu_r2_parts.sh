# round 2 session 3: device assign_partitions + local-pruning engine (tests, C2/C4/C5 A/B),
# min-grid load-first marks A/B
timeout 1200 python -m pytest tests/test_partition.py -q -x -m gpu > gpurun_out/parts_tests.log 2>&1; echo "partition tests rc=$?"; tail -5 gpurun_out/parts_tests.log
summ() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['stage_ms'].items()}, 'e2e', round(d['e2e']['ms_per_step'],3), 'into_final', d['config'].get('tuples_into_final'), 'tests', d['tests']['skyline'])"; }
for w in C2 C4; do
  for s in none grid angular sliced; do
    for lp in "" "--local-prune"; do
      timeout 600 python bench.py --workload $w --strategy $s $lp --no-cpu-baseline --steps 10 > gpurun_out/pb.log 2>&1; echo "bench $w $s [$lp] rc=$?"; summ < gpurun_out/pb.log
    done
  done
done
for lp in "" "--local-prune"; do
  timeout 600 python bench.py --workload C5 $lp --no-cpu-baseline --steps 10 > gpurun_out/pb.log 2>&1; echo "bench C5 [$lp] rc=$?"; summ < gpurun_out/pb.log
done
for e in "SKYGPU_MG_LOADFIRST=0" "SKYGPU_MG_LOADFIRST=1"; do
  env $e timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/pb.log 2>&1; echo "bench C5 [$e] rc=$?"; summ < gpurun_out/pb.log
done
