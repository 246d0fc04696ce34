set -x
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "grid_engine" > gpurun_out/k6_tests.log 2>&1; echo "grid tests rc=$?"; tail -3 gpurun_out/k6_tests.log
SKYGPU_GRID_KERNEL=alu timeout 300 python scripts/c5_sky_dump.py /tmp/c5alu.npy; echo "alu rc=$?"
timeout 300 python scripts/c5_sky_dump.py cmp:/tmp/c5alu.npy; echo "tma rc=$?"
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/k6_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/k6_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stage_ms'], d['roofline']['other'])"
timeout 900 python -m pytest tests/test_gpu_fuzz.py -q -x > gpurun_out/k6_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -3 gpurun_out/k6_fuzz.log
