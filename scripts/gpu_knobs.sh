# environment-knob A/B on C5: KNOBS="A=1 B=2;C=3" (one bench per ';'-separated setting)
summ() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['stage_ms'].items()})"; }
IFS=';' read -ra SETS <<< "${KNOBS:-SKYGPU_NONE_=1}"
for e in "${SETS[@]}"; do
  env $e timeout 600 python bench.py --workload ${W:-C5} --no-cpu-baseline --steps 10 > gpurun_out/kn.log 2>&1; echo "bench ${W:-C5} [$e] rc=$?"; summ < gpurun_out/kn.log
done
