timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "grid_engine or config_goldens" > gpurun_out/g_tests.log 2>&1; echo "grid tests rc=$?"; tail -2 gpurun_out/g_tests.log
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x > gpurun_out/g_var.log 2>&1; echo "variants rc=$?"; tail -2 gpurun_out/g_var.log
for e in "" "SKYGPU_GRID_ATOMIC=1"; do
env $e timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/g_bench.log 2>&1; echo "bench [$e] rc=$?"; tail -1 gpurun_out/g_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stage_ms'], d['e2e']['ms_per_step']); print(json.dumps(d['roofline']))"
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/g_launches_C5.csv $CMD > gpurun_out/g_ncu.log 2>&1; echo "launch list rc=$?"
ncu --set full --import-source on --clock-control none -k regex:k_grid_decide_tma -c 1 -o gpurun_out/prof_C5_k6 -f python scripts/itest_probe.py C5 > gpurun_out/ncu_full_k6.log 2>&1; echo "k6 full rc=$?"
timeout 900 python -m pytest tests/test_gpu_fullscale.py -q -x > gpurun_out/g_full.log 2>&1; echo "fullscale rc=$?"; tail -3 gpurun_out/g_full.log
