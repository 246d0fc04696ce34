timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_variants.py -q -x -m gpu -k "grid or decide" --timeout 300 > gpurun_out/rec_tests.log 2>&1; echo "grid parity rc=$?"; tail -2 gpurun_out/rec_tests.log
timeout 900 python -m pytest tests/test_gpu_fullscale.py tests/test_gpu_fuzz.py -q -x -m gpu > gpurun_out/rec_full.log 2>&1; echo "fullscale+fuzz rc=$?"; tail -2 gpurun_out/rec_full.log
VARIANTS="intree intree" bash scripts/gpu_k6_variants.sh
