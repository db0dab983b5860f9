# validation of: left-looking 256-row super-blocks (4-way split-K), DMMA fp64 GEMM,
# 8-groups-per-warp min-max grids, 7-stage Hessian ring; plus QEP timing
mkdir -p gpurun_out
L=paper_2603_28845_b200/lib
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_scale.py tests/test_gpu_macro.py tests/test_gpu_gemm.py tests/test_gpu_qep.py tests/test_gpu_layers.py -q -x --timeout 600 > gpurun_out/t_aa.log 2>&1; echo "rc=$?" >> gpurun_out/t_aa.log
for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/bench_aa_s7_$i.log 2>&1
done
OCWG_SWEEP_EVENTS=1 timeout 300 python tools/prof_c2.py --reps 2 > gpurun_out/sweep_ev_aa.log 2>&1
timeout 600 python tools/qep_bench.py > gpurun_out/qep_bench.log 2>&1
cp $L/libocwg.so $L/libocwg_s7.so; cp $L/libocwg_s6.so $L/libocwg.so
for i in 1 2; do
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/bench_aa_s6_$i.log 2>&1
done
cp $L/libocwg_s7.so $L/libocwg.so
