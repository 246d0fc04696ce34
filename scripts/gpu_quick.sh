nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -x ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
for w in ${WORKLOADS:-C2}; do timeout 600 python bench.py --steps 10 --warmup 3 --workload $w ${BENCH_ARGS:-} > gpurun_out/bench_$w.log 2>&1; echo "bench $w rc=$?"; tail -1 gpurun_out/bench_$w.log | cut -c 1-3000; done
