# launch list + one full ncu capture of the Hessian kernel (1 GPU)
mkdir -p gpurun_out
python tools/prof_c2.py --reps 2 > gpurun_out/plain.log 2>&1 &&
ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file gpurun_out/launches.csv python tools/prof_c2.py --reps 2 > gpurun_out/ncu_launch.log 2>&1 &&
ncu --set full --clock-control none --import-source on -k regex:hessian_tc_kernel -s 1 -c 1 \
    -o gpurun_out/prof_hessian python tools/prof_c2.py --reps 2 > gpurun_out/ncu_full.log 2>&1
echo "rc=$?" >> gpurun_out/plain.log
