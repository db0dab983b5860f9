# round 2, first GPU pass: quick gram checks, full GPU suite, bench, launch list + gram ncu
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_parity.py -q -k "hessian or accumulate or unaligned" > gpurun_out/quick.log 2>&1; echo "quick rc=$?" >> gpurun_out/quick.log
timeout 1800 python -m pytest tests -m gpu -q --timeout 900 -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
B="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0"
timeout 300 $B > gpurun_out/plain.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu_launch.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/ncu_launch.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gram_tc -s 1 -c 1 -o gpurun_out/gram_full $B > gpurun_out/ncu_gram.log 2>&1; echo "ncu gram rc=$?" >> gpurun_out/ncu_gram.log
