# 256-row sweep: parity subset, bench, sweep event timeline
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_macro.py -q -x --timeout 600 > gpurun_out/t_q.log 2>&1; echo "rc=$?" >> gpurun_out/t_q.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/bench_q.log 2>&1; echo "rc=$?" >> gpurun_out/bench_q.log
OCWG_SWEEP_EVENTS=1 timeout 300 python tools/prof_c2.py --reps 2 > gpurun_out/sweep_ev_q.log 2>&1
