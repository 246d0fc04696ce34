# seeds 200..1400 of the fuzz generator in chunks of 100 (each chunk its own process and timeout)
for lo in $(seq ${FUZZ_LO:-200} 100 ${FUZZ_HI:-1300}); do
  timeout 300 python scripts/fuzz_sweep.py $lo $((lo+100)) > gpurun_out/fuzz_$lo.log 2>&1; rc=$?
  echo "chunk $lo rc=$rc last: $(grep -c '^seed' gpurun_out/fuzz_$lo.log) seeds; $(grep 'SUMMARY\|FAIL' gpurun_out/fuzz_$lo.log | tail -3 | tr '\n' ' ')"
  if [ $rc -ne 0 ]; then echo "  stuck/failed at: $(grep '^seed' gpurun_out/fuzz_$lo.log | tail -1)"; fi
done
