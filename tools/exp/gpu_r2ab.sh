mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_qep.py tests/test_gpu_gemm.py tests/test_gpu_parity.py tests/test_gpu_scale.py -q -x --timeout 600 > gpurun_out/t_ab.log 2>&1; echo "rc=$?" >> gpurun_out/t_ab.log
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/bench_ab_$i.log 2>&1; done
timeout 600 python tools/qep_bench.py > gpurun_out/qep_bench.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/qep_launches.csv python tools/qep_bench.py > gpurun_out/ncu_qep.log 2>&1
