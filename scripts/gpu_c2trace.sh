timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pt rc=$?"
WS="C2 C4 C1" bash scripts/gpu_ab2.sh
