mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -k "hessian or accumulate or end_to_end" tests/test_gpu_scale.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:hessian_tc2 -c 1 --csv python tools/prof_c2.py --reps 1 > gpurun_out/ncu_h.log 2>&1
