mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_macro.py -q -x --timeout 600 > gpurun_out/t_v.log 2>&1; echo "rc=$?" >> gpurun_out/t_v.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/bench_v.log 2>&1; echo "rc=$?" >> gpurun_out/bench_v.log
bash tools/gpu_chol_trace.sh
