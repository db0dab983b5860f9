mkdir -p gpurun_out
rm -f gpurun_out/pf.log
for i in 1 2; do
  for f in 0 8 16 32; do
    OCWG_GRAM_PF=$f timeout 120 python tools/hess_time.py > gpurun_out/nf.log 2>&1
    (echo -n "pf=$f "; tail -1 gpurun_out/nf.log) >> gpurun_out/pf.log
  done
done
