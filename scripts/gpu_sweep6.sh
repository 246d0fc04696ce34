run() { tag=$1; w=$2; shift; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline --steps 40 --workload $w > gpurun_out/sw6_${tag}_$w.log 2>&1; python -c "
import json;j=json.loads(open('gpurun_out/sw6_${tag}_$w.log').read().strip().splitlines()[-1]);print('$tag $w',round(j['ms_per_step'],4))"; }
for w in C2 C4 C1; do
run base $w X=1
run pc32 $w SKYGPU_DIR_PER_CELL=32
run pc64 $w SKYGPU_DIR_PER_CELL=64
run pc256 $w SKYGPU_DIR_PER_CELL=256
run s24 $w SKYGPU_SOLO=24
run s12 $w SKYGPU_SOLO=12
run base2 $w X=1
done
