set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "streamed" > gpurun_out/pt_stream.log 2>&1
SKYGPU_STREAM_MIN_MB=8 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_dropin_gpu.py -x -q > gpurun_out/pt_stream8.log 2>&1
SKYGPU_STREAM_MIN_MB=8 SKYGPU_TRACE=1 timeout 300 python scripts/e2e_trace.py ant 1000000 3 > gpurun_out/tr_c2_stream.log 2>&1
timeout 300 python scripts/e2e_trace.py ant 1000000 3 > gpurun_out/t_c2_plain.log 2>&1
SKYGPU_STREAM_MIN_MB=8 timeout 300 python scripts/e2e_trace.py ant 1000000 3 > gpurun_out/t_c2_stream.log 2>&1
SKYGPU_STREAM_MIN_MB=8 timeout 300 python scripts/e2e_trace.py corr 1000000 6 > gpurun_out/t_c3_stream.log 2>&1
timeout 300 python scripts/e2e_trace.py corr 1000000 6 > gpurun_out/t_c3_plain.log 2>&1
SKYGPU_STREAM_MIN_MB=1 timeout 300 python scripts/e2e_trace.py uni 100000 4 > gpurun_out/t_c1_stream.log 2>&1
timeout 300 python scripts/e2e_trace.py uni 100000 4 > gpurun_out/t_c1_plain.log 2>&1
timeout 300 python scripts/e2e_trace.py uni 10000000 5 > gpurun_out/t_c4_stream.log 2>&1
SKYGPU_OVERLAP=0 timeout 300 python scripts/e2e_trace.py uni 10000000 5 > gpurun_out/t_c4_plain.log 2>&1
