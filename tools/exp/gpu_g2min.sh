mkdir -p gpurun_out
for v in 0 1600 2100 0 1600 2100; do
  echo "min=$v" >> gpurun_out/g2min.log
  OCWG_SWEEP_GEMM2_MIN=$v timeout 300 python bench.py --steps 8 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | grep -o '"ms_per_step": [0-9.]*\|"sweep": [0-9.]*' | tr '\n' ' ' >> gpurun_out/g2min.log
  echo >> gpurun_out/g2min.log
done
