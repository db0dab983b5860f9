# ncu --set full of the C2 step's main kernels (one launch each) + the launch list
mkdir -p gpurun_out
timeout 300 python tools/prof_c2.py --reps 1 > gpurun_out/plain.log 2>&1 || exit 1
prof() {  # name regex skip
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$2 -s $3 -c 1 \
      -o gpurun_out/prof_$1 python tools/prof_c2.py --reps 1 > gpurun_out/ncu_$1.log 2>&1
}
prof hessian hessian_tc2 0
prof chol chol_tile 0
prof inblock inblock4 5
prof tcgemm tc_gemm2 1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/launches.csv python tools/prof_c2.py --reps 2 > gpurun_out/ncu_launch.log 2>&1
echo "rc=$?" >> gpurun_out/plain.log
