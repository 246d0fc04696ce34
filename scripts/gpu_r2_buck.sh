timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "cell_engine or min_grid" > gpurun_out/b_tests.log 2>&1; echo "cell tests rc=$?"; tail -2 gpurun_out/b_tests.log
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x -k "cell_engine_variants" > gpurun_out/b_var.log 2>&1; echo "variants rc=$?"; tail -2 gpurun_out/b_var.log
for e in "" "SKYGPU_MG_NOBUCKET=1"; do
env $e timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/b_bench.log 2>&1; echo "bench [$e] rc=$?"; tail -1 gpurun_out/b_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],3), {a: round(b,3) for a,b in d['stage_ms'].items()}, d['e2e']['ms_per_step'])"
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/b_launches_C5.csv $CMD > gpurun_out/b_ncu.log 2>&1; echo "launch list rc=$?"
timeout 900 python -m pytest tests/test_gpu_fullscale.py -q -x > gpurun_out/b_full.log 2>&1; echo "fullscale rc=$?"; tail -3 gpurun_out/b_full.log
