timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pt rc=$?"
for w in C2 C1 C3 C4 C5; do
timeout 600 python bench.py --no-cpu-baseline --workload $w > gpurun_out/b_pdl_$w.log 2>&1
SKYGPU_PDL=0 timeout 600 python bench.py --no-cpu-baseline --workload $w > gpurun_out/b_nopdl_$w.log 2>&1
done
