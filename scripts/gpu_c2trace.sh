timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > gpurun_out/pt_parity.log 2>&1; echo "pt rc=$?"
WS="C2 C4 C3" bash scripts/gpu_ab2.sh
