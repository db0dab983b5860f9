# Cholesky change check: owner trace, factor-related GPU tests, C2 step
mkdir -p gpurun_out
bash tools/gpu_chol_trace.sh
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_macro.py tests/test_gpu_scale.py -x -q -m gpu > gpurun_out/pt_chol.log 2>&1; echo "rc=$?" >> gpurun_out/pt_chol.log
timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin --e2e-steps 0 > gpurun_out/b_chol.log 2>&1
