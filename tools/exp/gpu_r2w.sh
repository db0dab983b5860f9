mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_scale.py -q -x --timeout 600 -k "c2" > gpurun_out/t_w.log 2>&1; echo "rc=$?" >> gpurun_out/t_w.log
timeout 300 python tools/prof_c2.py --reps 1 > gpurun_out/plain_w.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chol_tile -s 0 -c 1 -o gpurun_out/prof_chol_w python tools/prof_c2.py --reps 1 > gpurun_out/ncu_chol_w.log 2>&1
