timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "grid_engine or config_goldens" > gpurun_out/g_tests.log 2>&1; echo "grid tests rc=$?"; tail -2 gpurun_out/g_tests.log
timeout 900 python -m pytest tests/test_gpu_variants.py -q -x > gpurun_out/g_var.log 2>&1; echo "variants rc=$?"; tail -2 gpurun_out/g_var.log
for cfg in "512 64" "512 32" "512 16" "64 32" "64 16" "32 16"; do set -- $cfg
SKYGPU_GRID_ROW=$1 SKYGPU_GRID_K0=$2 timeout 600 python bench.py --no-cpu-baseline --steps 5 > gpurun_out/g_bench.log 2>&1; echo "bench row=$1 k0=$2 rc=$?"; tail -1 gpurun_out/g_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); o=d['roofline'].get('other',{}); r=d['roofline']; k=r if r['kernel'].startswith('k_grid') else o; print(round(d['ms_per_step'],3), {a: round(b,3) for a,b in d['stage_ms'].items()}, 'units', k.get('units_per_step'), 'frac', round(k.get('frac',0),3))"
done
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/g_launches_C5.csv $CMD > gpurun_out/g_ncu.log 2>&1; echo "launch list rc=$?"
