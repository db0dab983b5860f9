mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_jointq.py tests/test_gpu_dropin.py -q -s -m gpu > gpurun_out/pt_jq.log 2>&1; echo "rc=$?" >> gpurun_out/pt_jq.log
timeout 1200 python tools/jointq_bench.py > gpurun_out/jq_bench.log 2>&1; echo rc=$? >> gpurun_out/jq_bench.log
