mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_macro.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for v in 1 0; do
  echo "gemm2=$v" >> gpurun_out/g2.log
  OCWG_SWEEP_GEMM2=$v timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>&1 | grep -o '"ms_per_step": [0-9.]*' >> gpurun_out/g2.log
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/launches.csv python tools/prof_c2.py --reps 2 > gpurun_out/ncu_launch.log 2>&1
