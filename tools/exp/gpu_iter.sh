# parity suite + bench + C2 launch list, each bounded by its own timeout
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q --timeout 300 ${PYTEST_ARGS:-} > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python bench.py --steps 5 --warmup 3 ${BENCH_ARGS:-} > gpurun_out/bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench.log
timeout 300 python tools/prof_c2.py --reps 2 > gpurun_out/plain.log 2>&1 &&
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/launches.csv python tools/prof_c2.py --reps 2 > gpurun_out/ncu_launch.log 2>&1
echo "rc=$?" >> gpurun_out/plain.log
for ib in ${TRACE_IBS:-}; do
  OCWG_SWEEP_TRACE_IB=$ib timeout 300 python tools/sweep_trace.py >> gpurun_out/trace.log 2>&1
done
