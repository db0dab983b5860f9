# source-level ncu of selected kernels on C2 (1 GPU); KERNELS="regex1 regex2 ..."
mkdir -p gpurun_out
timeout 300 python tools/prof_c2.py --reps 1 > gpurun_out/plain.log 2>&1 || exit 1
for k in ${KERNELS:-chol_tile inblock_g hessian_tc}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:$k -s ${SKIP:-3} -c 1 \
      -o gpurun_out/prof_$k python tools/prof_c2.py --reps 1 > gpurun_out/ncu_$k.log 2>&1
done
echo "rc=$?" >> gpurun_out/plain.log
