for sw in 2048 4096 8192 12288 16384; do
SKYGPU_SLAB_WORDS=$sw timeout 600 python bench.py --no-cpu-baseline --workload C5 --steps 5 --warmup 3 > gpurun_out/sw4_$sw.log 2>&1
python -c "
import json;j=json.loads(open('gpurun_out/sw4_$sw.log').read().strip().splitlines()[-1]);print('$sw',round(j['ms_per_step'],4), j['stage_ms']['gres_kernels'])"
done
