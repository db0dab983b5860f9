mkdir -p gpurun_out
for w in 16384 8192 32768; do OCWG_HESSIAN_WINDOW=$w timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bw_$w.log 2>&1; done
timeout 120 python tools/factor_bench.py > gpurun_out/factor_bench.log 2>&1
bash tools/gpu_chol_trace.sh
