W=C5 bash scripts/gpu_trace.sh
