mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_macro.py tests/test_gpu_qep.py -q -x --timeout 600 > gpurun_out/t_ad.log 2>&1; echo "rc=$?" >> gpurun_out/t_ad.log
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/bench_ad_$i.log 2>&1; done
bash tools/gpu_chol_trace.sh
