# K6 compile-time variants (scripts/build_k6_variant.sh) timed on C5 on one box
summ() { python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print(round(d['ms_per_step'],4), {k: round(v,3) for k,v in d['stage_ms'].items()})"; }
for v in ${VARIANTS:-intree}; do
  if [ $v = intree ]; then unset SKYGPU_LIB_PATH; else export SKYGPU_LIB_PATH=$PWD/paper_2412_02274_b200/_lib_v/$v/libskygpu.so; fi
  timeout 600 python bench.py --no-cpu-baseline --steps 10 > gpurun_out/k6v_$v.log 2>&1; echo "bench C5 [$v] rc=$?"; summ < gpurun_out/k6v_$v.log
done
unset SKYGPU_LIB_PATH
