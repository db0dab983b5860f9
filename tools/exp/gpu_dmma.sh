# fp64 DMMA GEMM: 1024-thread (32 x 16 warp tiles) against 512-thread (32 x 32) variant
# (OCWG_DMMA_THREADS was an experiment-only switch; the library now builds the 1024-thread form only)
mkdir -p gpurun_out
rm -f gpurun_out/dmma.log
OCWG_DMMA_THREADS=1024 timeout 600 python -m pytest tests/test_gpu_qep.py tests/test_gpu_gemm.py -q -x --timeout 500 > gpurun_out/t_dmma.log 2>&1; echo "rc=$?" >> gpurun_out/t_dmma.log
for v in 1024 512 1024 512; do
  echo "== $v" >> gpurun_out/dmma.log
  OCWG_DMMA_THREADS=$v timeout 300 python tools/gemm_bench.py 2>&1 | grep fp64 >> gpurun_out/dmma.log
  OCWG_DMMA_THREADS=$v timeout 300 python tools/qep_bench.py >> gpurun_out/dmma.log 2>&1
done
