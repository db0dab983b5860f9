mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "factor or gptq or macro or golden or c1" > gpurun_out/chol_tests.log 2>&1; echo "rc=$?" >> gpurun_out/chol_tests.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_o2.log 2>&1; echo "rc=$?" >> gpurun_out/bench_o2.log
bash tools/gpu_chol_trace.sh
