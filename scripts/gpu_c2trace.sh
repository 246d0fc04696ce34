timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q > gpurun_out/pt_parity.log 2>&1; echo "pt rc=$?"
WS="C2 C1" bash scripts/gpu_ab2.sh
SKYGPU_TRACE=1 timeout 300 python scripts/e2e_trace.py ant 1000000 3 > gpurun_out/tr_c2_plain.log 2>&1
