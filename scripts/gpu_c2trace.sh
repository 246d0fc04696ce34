timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pt_all.log 2>&1; echo "pt rc=$?"
for i in 1 2; do
timeout 300 python bench.py --no-cpu-baseline --workload C2 > gpurun_out/b_smem_$i.log 2>&1
SKYGPU_INTRA=2 timeout 300 python bench.py --no-cpu-baseline --workload C2 > gpurun_out/b_chunk_$i.log 2>&1
done
for w in C1 C3 C4; do timeout 300 python bench.py --no-cpu-baseline --workload $w > gpurun_out/b_$w.log 2>&1; done
SKYGPU_TRACE=1 timeout 300 python scripts/e2e_trace.py ant 1000000 3 > gpurun_out/tr_c2_plain.log 2>&1
