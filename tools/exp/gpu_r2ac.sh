mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qep.py tests/test_gpu_gemm.py tests/test_gpu_parity.py -q -x --timeout 600 -k "fp64 or qep or gemm or f64 or double" > gpurun_out/t_ac.log 2>&1; echo "rc=$?" >> gpurun_out/t_ac.log
timeout 600 python tools/qep_bench.py > gpurun_out/qep_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qep_launches.csv python tools/qep_bench.py > gpurun_out/ncu_qep.log 2>&1
