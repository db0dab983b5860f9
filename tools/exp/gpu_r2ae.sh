mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_macro.py tests/test_gpu_qep.py tests/test_gpu_layers.py -q -x --timeout 600 > gpurun_out/t_ae.log 2>&1; echo "rc=$?" >> gpurun_out/t_ae.log
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/bench_ae_$i.log 2>&1; done
for ib in 128 2048; do OCWG_SWEEP_TRACE_IB=$ib timeout 300 python tools/sweep_trace.py >> gpurun_out/trace_ae.log 2>&1; done
