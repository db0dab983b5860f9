mkdir -p gpurun_out
free -g > gpurun_out/free.txt; nproc >> gpurun_out/free.txt
rm -f gpurun_out/r02_parity.jsonl
timeout 2400 python -m pytest tests -m gpu -q --timeout 1200 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 --mode sharded > gpurun_out/bench_sharded.log 2>&1; echo "rc=$?" >> gpurun_out/bench_sharded.log
timeout 900 python bench.py --steps 1 --warmup 1 --mode model > gpurun_out/bench_model.log 2>&1; echo "rc=$?" >> gpurun_out/bench_model.log
