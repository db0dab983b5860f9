mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_macro.py tests/test_closed_form.py -q -x > gpurun_out/chol_tests.log 2>&1; echo "rc=$?" >> gpurun_out/chol_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_o2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_o2.log
bash tools/gpu_chol_trace.sh
