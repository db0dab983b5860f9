mkdir -p gpurun_out
for mc in 0 512 1024 2048; do
  echo "macro=$mc" >> gpurun_out/macro.log
  OCWG_CHOL_MACRO=$mc timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | grep -o '"ms_per_step": [0-9.]*' >> gpurun_out/macro.log
done
