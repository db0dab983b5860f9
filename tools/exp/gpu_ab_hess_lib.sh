# A/B of library variants (lib_var/*.so) on the Hessian (hess_time, sustained 20 launches) and the C2 step
mkdir -p gpurun_out
rm -f gpurun_out/ab_hlib.log
for i in 1 2 3; do
for v in $VARIANTS; do
  cp paper_2603_28845_b200/lib_var/$v.so paper_2603_28845_b200/lib/libocwg.so
  timeout 120 python tools/hess_time.py > gpurun_out/nf.log 2>&1
  (echo -n "$v "; tail -1 gpurun_out/nf.log) >> gpurun_out/ab_hlib.log
done
done
cp paper_2603_28845_b200/lib_var/base.so paper_2603_28845_b200/lib/libocwg.so
