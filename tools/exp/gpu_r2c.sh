mkdir -p gpurun_out
OCWG_DEBUG_STATS=1 timeout 300 python tools/dbg_stats.py > gpurun_out/dbg_stats.log 2>&1; echo "rc=$?" >> gpurun_out/dbg_stats.log
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "gram_kernel" > gpurun_out/gramseg.log 2>&1; echo "rc=$?" >> gpurun_out/gramseg.log
