mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_scale.py tests/test_gpu_gemm.py -q -x --timeout 600 > gpurun_out/t_pf.log 2>&1; echo "rc=$?" >> gpurun_out/t_pf.log
for i in 1 2; do timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/bench_pf_$i.log 2>&1; done
OCWG_SWEEP_EVENTS=1 timeout 300 python tools/prof_c2.py --reps 2 > gpurun_out/sweep_ev_pf.log 2>&1
