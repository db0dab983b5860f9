mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qep.py tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_macro.py -q -x --timeout 600 > gpurun_out/t_q2.log 2>&1; echo "rc=$?" >> gpurun_out/t_q2.log
timeout 600 python tools/qep_bench.py > gpurun_out/qep_bench.log 2>&1
