timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "golden or random or grid" > gpurun_out/pt_parity.log 2>&1; echo "pt rc=$?"
WS="C5 C2" bash scripts/gpu_ab2.sh
