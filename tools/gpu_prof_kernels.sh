# source-level ncu of the factor / sweep kernels on C2 (1 GPU)
mkdir -p gpurun_out
timeout 300 python tools/prof_c2.py --reps 1 > gpurun_out/plain.log 2>&1 &&
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chol_tile -c 1 \
    -o gpurun_out/prof_chol python tools/prof_c2.py --reps 1 > gpurun_out/ncu_chol.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:inblock_g -s 5 -c 1 \
    -o gpurun_out/prof_inblock python tools/prof_c2.py --reps 1 > gpurun_out/ncu_inblock.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 5 -c 1 \
    -o gpurun_out/prof_tcgemm python tools/prof_c2.py --reps 1 > gpurun_out/ncu_tcgemm.log 2>&1
echo "rc=$?" >> gpurun_out/plain.log
