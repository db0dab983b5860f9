mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py tests/test_gpu_qep.py tests/test_container.py -q -x > gpurun_out/t_k.log 2>&1; echo "rc=$?" >> gpurun_out/t_k.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_k.log 2>&1; echo "rc=$?" >> gpurun_out/bench_k.log
timeout 900 python bench.py --steps 2 --warmup 1 --mode model > gpurun_out/bench_model_k.log 2>&1; echo "rc=$?" >> gpurun_out/bench_model_k.log
