mkdir -p gpurun_out
for sb in 128 256 384 512; do
  echo "super=$sb" >> gpurun_out/super.log
  OCWG_SWEEP_SUPER=$sb timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | grep -o '"ms_per_step": [0-9.]*' >> gpurun_out/super.log
done
