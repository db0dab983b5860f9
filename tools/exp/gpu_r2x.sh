mkdir -p gpurun_out
timeout 300 python tools/prof_c2.py --reps 1 > gpurun_out/plain_x.log 2>&1 || exit 1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chol_tile -s 0 -c 1 -o gpurun_out/prof_chol_x python tools/prof_c2.py --reps 1 > gpurun_out/ncu_chol_x.log 2>&1
