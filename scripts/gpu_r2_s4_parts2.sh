timeout 900 python -m pytest tests/test_partition.py -q -x -m gpu -k "local_prune" > gpurun_out/parts2_tests.log 2>&1; echo "local prune tests rc=$?"; tail -3 gpurun_out/parts2_tests.log
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x -m gpu -k "cell_engine_variants" > gpurun_out/parts2_var.log 2>&1; echo "cell variants rc=$?"; tail -2 gpurun_out/parts2_var.log
summ() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['stage_ms'].items()}, 'e2e', round(d['e2e']['ms_per_step'],3), 'into_final', d['config'].get('tuples_into_final'), 'tests', d['tests']['skyline'])"; }
for w in C2 C4 C5; do
  for lp in "" "--local-prune"; do
    timeout 600 python bench.py --workload $w $lp --no-cpu-baseline --steps 10 > gpurun_out/pb.log 2>&1; echo "bench $w [$lp] rc=$?"; summ < gpurun_out/pb.log
  done
done
