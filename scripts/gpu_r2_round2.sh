# round-2 re-entry baseline: GPU tests, default bench (C5), reference arm, C5 launch list
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -20 gpurun_out/r2_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2_bench_C5.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r2_bench_C5.log
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/r2_bench_ref.log
WORKLOADS="C2 C4" BENCH_ARGS="--no-cpu-baseline" bash scripts/gpu_bench_all.sh
CMD="python bench.py --steps 2 --warmup 3 --no-cpu-baseline"
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r2_launches_C5.csv $CMD > gpurun_out/r2_ncu_launch_C5.log 2>&1; echo "launch list rc=$?"
