timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "die_at_once" > gpurun_out/s4_die.log 2>&1; echo "die_at_once rc=$?"; tail -2 gpurun_out/s4_die.log
bash scripts/gpu_r2_parts.sh
