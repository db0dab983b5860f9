mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_container.py tests/test_gpu_autobit.py tests/test_gpu_layers.py tests/test_gpu_dropin.py -q -x > gpurun_out/t_j.log 2>&1; echo "rc=$?" >> gpurun_out/t_j.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_j.log 2>&1; echo "rc=$?" >> gpurun_out/bench_j.log
timeout 900 python bench.py --steps 1 --warmup 1 --mode model > gpurun_out/bench_model_j.log 2>&1; echo "rc=$?" >> gpurun_out/bench_model_j.log
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-dropin"
timeout 300 $B > gpurun_out/plain_j.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"calibrate_groups|pack_codes" -s 2 -c 2 -o gpurun_out/hbm_full $B > gpurun_out/ncu_hbm.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_hbm.log
