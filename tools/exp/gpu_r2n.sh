mkdir -p gpurun_out
timeout 120 python tools/factor_bench.py > gpurun_out/factor_bench.log 2>&1
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_macro.py tests/test_gpu_scale.py tests/test_gpu_dropin.py -q -x > gpurun_out/t_n.log 2>&1; echo "rc=$?" >> gpurun_out/t_n.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/bench_n.log 2>&1; echo "rc=$?" >> gpurun_out/bench_n.log
bash tools/gpu_chol_trace.sh
