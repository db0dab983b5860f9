mkdir -p gpurun_out
timeout 300 python tools/prof_c2.py --reps 1 > gpurun_out/plain_u.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm2 -s 6 -c 1 -o gpurun_out/prof_gemm2L python tools/prof_c2.py --reps 1 > gpurun_out/ncu_gemm2L.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tc_gemm2 -s 1 -c 1 -o gpurun_out/prof_gemm2S python tools/prof_c2.py --reps 1 > gpurun_out/ncu_gemm2S.log 2>&1
