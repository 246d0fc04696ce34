timeout 1500 python -m pytest tests/test_gpu_variants.py tests/test_gpu_parity.py -q -x -k "variant or kernels_agree or config_goldens" > gpurun_out/pins_tests.log 2>&1; echo "variants+configs rc=$?"; tail -3 gpurun_out/pins_tests.log
timeout 1500 python -m pytest tests/test_gpu_fullscale.py -q -x --durations=10 > gpurun_out/pins_full.log 2>&1; echo "fullscale rc=$?"; tail -15 gpurun_out/pins_full.log
cd oracle/_ref
SKYGPU_METRICS=fast timeout 900 ./acceptance_gpu --cli ./skypar_gpu --fixtures ./fixtures > ../../gpurun_out/acc_fast.txt 2>&1; echo "acc fast rc=$?"; grep "^\[" ../../gpurun_out/acc_fast.txt
for m in fast exact; do SKYGPU_METRICS=$m timeout 600 ./skypar_bench_gpu --n 1000000 --d 3 --gen ant --partitions 16 --cores 16 > ../../gpurun_out/skybench_$m.txt 2>&1; echo "bench $m rc=$?"; cat ../../gpurun_out/skybench_$m.txt; done
