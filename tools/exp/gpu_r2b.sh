mkdir -p gpurun_out
timeout 300 python tools/dbg_stats.py > gpurun_out/dbg_stats.log 2>&1; echo "rc=$?" >> gpurun_out/dbg_stats.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_b.log 2>&1; echo "rc=$?" >> gpurun_out/bench_b.log
