# round-2 measurement pass: default bench (C2 with e2e, drop-in, CPU baseline), the
# C4 whole-model sweep at N=1, sharded mode at N=1, other configs, calibrate/pack ncu
mkdir -p gpurun_out
timeout 900 python bench.py > gpurun_out/fb_default.log 2>&1; echo "rc=$?" >> gpurun_out/fb_default.log
timeout 900 python bench.py --mode model --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/fb_model.log 2>&1; echo "rc=$?" >> gpurun_out/fb_model.log
timeout 300 python bench.py --mode sharded --steps 5 --warmup 3 --no-cpu-baseline --no-dropin --e2e-steps 0 > gpurun_out/fb_sharded.log 2>&1; echo "rc=$?" >> gpurun_out/fb_sharded.log
timeout 900 python tools/bench_configs.py --reps 2 > gpurun_out/fb_configs.log 2>&1; echo "rc=$?" >> gpurun_out/fb_configs.log
timeout 300 python tools/prof_c2.py --reps 1 > gpurun_out/plain_fb.log 2>&1
for k in calibrate_minmax8:calib pack_codes:pack; do
  re=${k%%:*}; nm=${k##*:}
  timeout 600 ncu --set full --clock-control none -k regex:$re -s 0 -c 1 -o gpurun_out/prof_${nm}_fb python tools/prof_c2.py --reps 1 > gpurun_out/ncu_${nm}_fb.log 2>&1
done
