nvidia-smi -L
timeout 1500 python -m pytest tests -m gpu -q --timeout 600 -x ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -40 gpurun_out/pytest_gpu.log
