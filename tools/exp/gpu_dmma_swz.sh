# fp64 DMMA GEMM: XOR-swizzled shared tiles (libocwg.so) against libocwg_prev.so
mkdir -p gpurun_out
L=paper_2603_28845_b200/lib
rm -f gpurun_out/dmma_swz.log
timeout 600 python -m pytest tests/test_gpu_qep.py tests/test_gpu_gemm.py tests/test_gpu_jointq.py -q -x --timeout 500 > gpurun_out/t_swz.log 2>&1; echo "rc=$?" >> gpurun_out/t_swz.log
cp $L/libocwg.so $L/libocwg_new.so
for v in new prev new prev; do
  cp $L/libocwg_$v.so $L/libocwg.so
  echo "== $v" >> gpurun_out/dmma_swz.log
  timeout 300 python tools/dmma_one.py 5 >> gpurun_out/dmma_swz.log 2>&1
  timeout 300 python tools/gemm_bench.py 2>&1 | grep fp64 >> gpurun_out/dmma_swz.log
done
cp $L/libocwg_new.so $L/libocwg.so
timeout 600 ncu --set full --clock-control none -k regex:gemm_f64_dmma -s 0 -c 1 \
    -o gpurun_out/prof_dmma_swz python tools/dmma_one.py 1 > gpurun_out/ncu_dmma_swz.log 2>&1
echo "rc=$?" >> gpurun_out/ncu_dmma_swz.log
