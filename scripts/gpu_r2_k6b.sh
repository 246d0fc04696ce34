timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "grid_engine" > gpurun_out/k6_tests.log 2>&1; echo "grid tests rc=$?"; tail -2 gpurun_out/k6_tests.log
SKYGPU_GRID_KERNEL=alu timeout 300 python scripts/c5_sky_dump.py /tmp/c5alu.npy; echo "alu rc=$?"
timeout 300 python scripts/c5_sky_dump.py cmp:/tmp/c5alu.npy; echo "tma rc=$?"
timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/k6_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/k6_bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['stage_ms'], d['roofline']['other'])"
ncu --set full --import-source on --clock-control none -k regex:k_grid_decide_tma -s 1 -c 1 -o gpurun_out/prof_C5_k6tma2 -f python scripts/c5_sky_dump.py /tmp/x.npy > gpurun_out/ncu_k6.log 2>&1; echo "ncu rc=$?"
