mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_container.py -q -x -k "pack or container or golden or c1" > gpurun_out/t_l.log 2>&1; echo "rc=$?" >> gpurun_out/t_l.log
timeout 900 python bench.py --steps 1 --warmup 1 --mode model > gpurun_out/bm_ov1.log 2>&1
OCWG_MODEL_OVERLAP=0 timeout 900 python bench.py --steps 1 --warmup 1 --mode model > gpurun_out/bm_ov0.log 2>&1
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 --no-dropin"
timeout 300 $B > gpurun_out/plain_l.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -k regex:"calibrate_groups|pack_codes" -s 2 -c 2 -o gpurun_out/hbm_full2 $B > gpurun_out/ncu_hbm2.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_hbm2.log
