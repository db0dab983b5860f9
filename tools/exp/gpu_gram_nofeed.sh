mkdir -p gpurun_out
rm -f gpurun_out/nofeed.log
for i in 1 2; do
  for f in 0 1; do
    OCWG_GRAM_NOFEED=$f timeout 300 python tools/hess_time.py > gpurun_out/nf.log 2>&1
    (echo -n "nofeed=$f "; tail -1 gpurun_out/nf.log) >> gpurun_out/nofeed.log
  done
done
