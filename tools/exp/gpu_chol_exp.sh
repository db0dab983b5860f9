mkdir -p gpurun_out
for k in 1 2; do
  OCWG_CHOL_CTAS_PER_SM=$k OCWG_CHOL_TRACE=gpurun_out/chol_trace_$k.bin timeout 300 python tools/prof_c2.py --reps 1 > gpurun_out/trace_$k.log 2>&1
  OCWG_CHOL_CTAS_PER_SM=$k timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_$k.log 2>&1
done
