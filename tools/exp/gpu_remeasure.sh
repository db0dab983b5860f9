mkdir -p gpurun_out
timeout 900 python bench.py --mode model --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/fb_model.log 2>&1; echo "rc=$?" >> gpurun_out/fb_model.log
timeout 900 python tools/bench_configs.py --reps 2 > gpurun_out/fb_configs.log 2>&1; echo "rc=$?" >> gpurun_out/fb_configs.log
