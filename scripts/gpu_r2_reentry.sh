# round-2 re-entry (session 3): GPU suite + default bench (C5) + C2/C4 on HEAD
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r2s3_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/r2s3_pytest_gpu.log
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r2s3_bench_C5.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r2s3_bench_C5.log
WORKLOADS="C2 C4" BENCH_ARGS="--no-cpu-baseline" bash scripts/gpu_bench_all.sh
