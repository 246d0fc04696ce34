# one bench line per workload (default K/W), appended to gpurun_out/bench_all.jsonl
: > gpurun_out/bench_all.jsonl
for w in ${WORKLOADS:-C1 C2 C3 C4 C5 C5p10k C5p20k}; do
  timeout 900 python bench.py --workload $w ${BENCH_ARGS:-} > gpurun_out/bench_$w.log 2>&1
  echo "bench $w rc=$?"
  tail -1 gpurun_out/bench_$w.log >> gpurun_out/bench_all.jsonl
done
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_C2.log 2>&1; echo "ref rc=$?"
tail -1 gpurun_out/bench_ref_C2.log >> gpurun_out/bench_all.jsonl
