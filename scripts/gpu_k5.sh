# K5 scan-cell variants on C2
run() { env "$@" timeout 300 python bench.py --steps 10 --warmup 3 --workload ${W:-C2} --no-cpu-baseline 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$*', round(d['ms_per_step'],4), round(d['stage_ms']['sky_kernels'],4), d['tests']['skyline'])"; }
run X=1
run SKYGPU_SCAN_CELLS=dir
run SKYGPU_SCAN_CELLS=dir SKYGPU_DIR_PER_CELL=64
run SKYGPU_SCAN_CELLS=dir SKYGPU_DIR_PER_CELL=32
run SKYGPU_SCAN_CELLS=dir SKYGPU_DIR_PER_CELL=16
run SKYGPU_QGRID=1
