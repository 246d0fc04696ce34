timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "grid or fuzz or random or golden or C5 or streamed" > gpurun_out/pt_grid.log 2>&1; echo "pt rc=$?"
WS="C5" bash scripts/gpu_ab2.sh
timeout 900 python scripts/verify_c5_full.py > gpurun_out/verify_c5.log 2>&1; echo "verify rc=$?"
