summ() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['stage_ms'].items()})"; }
for m in 0 16 64 128 256 1000 0 64; do
  SKYGPU_MG_RED_MB=$m timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/red_$m.log 2>&1; echo "bench C5 [RED_MB=$m] rc=$?"; summ < gpurun_out/red_$m.log
done
SKYGPU_MG_RED_MB=64 timeout 600 python -m pytest tests/test_gpu_fullscale.py tests/test_gpu_parity.py -q -x -m gpu -k "cells or cell_engine or min_grid or c5" > gpurun_out/red_tests.log 2>&1; echo "tests with RED_MB=64 rc=$?"; tail -2 gpurun_out/red_tests.log
