summ() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['stage_ms'].items()})"; }
for cfg in "512 64" "384 64" "768 64" "1024 64" "512 32" "512 128" "768 128" "384 128" "1024 128"; do
  set -- $cfg
  SKYGPU_GRID_ROW=$1 SKYGPU_GRID_K0=$2 timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/gs.log 2>&1; echo "bench C5 [ROW=$1 K0=$2] rc=$?"; summ < gpurun_out/gs.log
done
