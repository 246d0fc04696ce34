timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/cells_tests.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/cells_tests.log
timeout 300 python scripts/c5_sky_dump.py cmp:/dev/null 2>/dev/null | head -1
timeout 900 python scripts/verify_c5_full.py 10000000 0,1 > gpurun_out/verify_c5.json 2>gpurun_out/verify_c5.err; echo "verify rc=$?"; cut -c1-600 gpurun_out/verify_c5.json
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/cells_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/cells_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stage_ms'], d['e2e']['ms_per_step'])"
bash scripts/gpu_launches.sh
