mkdir -p gpurun_out
timeout 300 python tools/dmma_one.py 5 > gpurun_out/dmma_one.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_f64_dmma -s 0 -c 1 \
    -o gpurun_out/prof_dmma python tools/dmma_one.py 1 > gpurun_out/ncu_dmma.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_dmma.log
