run() { tag=$1; w=$2; shift; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 40 --workload $w > gpurun_out/sw5_${tag}_$w.log 2>&1; python -c "
import json;j=json.loads(open('gpurun_out/sw5_${tag}_$w.log').read().strip().splitlines()[-1]);print('$tag $w',round(j['ms_per_step'],4))"; }
for w in C2 C4 C1 C3; do
run plan $w X=1
run dir $w SKYGPU_SCAN_CELLS=d
run plan2 $w X=1
run dir2 $w SKYGPU_SCAN_CELLS=d
done
