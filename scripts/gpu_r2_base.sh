# round-2 baseline: GPU tests, default bench (C5), reference arm
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2_pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r2_pytest_gpu.log
timeout 900 python bench.py > gpurun_out/r2_bench_C5.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r2_bench_C5.log
timeout 900 python bench.py --impl reference > gpurun_out/r2_bench_ref.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/r2_bench_ref.log
