summ() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['stage_ms'].items()})"; }
for e in "SKYGPU_NONE_=1" "SKYGPU_MG_NOPRIV=1" "SKYGPU_NONE_=1" "SKYGPU_MG_NOPRIV=1" "SKYGPU_MG_NOCOL=1" "SKYGPU_CELLS_SORT=1"; do
  env $e timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/kn.log 2>&1; echo "bench C5 [$e] rc=$?"; summ < gpurun_out/kn.log
done
