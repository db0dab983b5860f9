mkdir -p gpurun_out
for k in none inblock gemm; do
  OCWG_SWEEP_SKIP=$k timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_skip_$k.log 2>&1
done
timeout 300 python tools/prof_c2.py --reps 1 > gpurun_out/plain.log 2>&1 &&
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 14 -c 1 -o gpurun_out/prof_tcgemm python tools/prof_c2.py --reps 1 > gpurun_out/ncu_tcgemm.log 2>&1
