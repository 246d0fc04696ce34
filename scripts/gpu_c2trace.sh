timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q -k "spec or cell or golden" > gpurun_out/pt_parity.log 2>&1; echo "pt rc=$?"
WS="C2 C4 C5p10k" bash scripts/gpu_ab2.sh
