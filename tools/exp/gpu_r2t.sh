# left-looking split-K sweep: parity subset, bench, sweep event timeline
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_macro.py tests/test_gpu_layers.py tests/test_gpu_gemm.py -q -x --timeout 600 > gpurun_out/t_t.log 2>&1; echo "rc=$?" >> gpurun_out/t_t.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/bench_t.log 2>&1; echo "rc=$?" >> gpurun_out/bench_t.log
OCWG_SWEEP_EVENTS=1 timeout 300 python tools/prof_c2.py --reps 2 > gpurun_out/sweep_ev_t.log 2>&1
