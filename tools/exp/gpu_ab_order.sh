# A/B of the working-tree library (libocwg.so) against libocwg_prev.so on one box,
# with the pre-factor phase (order + damp + build) printed
mkdir -p gpurun_out
L=paper_2603_28845_b200/lib
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_layers.py tests/test_gpu_dropin.py tests/test_gpu_macro.py -q -x --timeout 600 > gpurun_out/t_ab.log 2>&1; echo "rc=$?" >> gpurun_out/t_ab.log
cp $L/libocwg.so $L/libocwg_new.so
rm -f gpurun_out/ab_lib.log
for i in 1 2 3; do
  for v in new prev; do
    cp $L/libocwg_$v.so $L/libocwg.so
    timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/ab_b.log 2>&1
    python -c "
import json
for l in open('gpurun_out/ab_b.log'):
    if l.startswith('{'): d=json.loads(l); print('$v', round(d['ms_per_step'],4), round(d['breakdown_ms']['hessian'],4), round(d['breakdown_ms']['gptq_phases']['order_damp_build'],4), d['clocks']['sm_mhz'])
" >> gpurun_out/ab_lib.log
  done
done
cp $L/libocwg_new.so $L/libocwg.so
