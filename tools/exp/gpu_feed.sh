mkdir -p gpurun_out
rm -f gpurun_out/feed.log
for i in 1 2 3; do
  for f in 0 1; do
    OCWG_GRAM_SERP=$f timeout 120 python tools/hess_time.py > gpurun_out/nf.log 2>&1
    (echo -n "serp=$f "; tail -1 gpurun_out/nf.log) >> gpurun_out/feed.log
  done
done
for f in 0 1; do
OCWG_GRAM_SERP=$f timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second -k regex:gram_tc -c 1 python tools/hess_time.py > gpurun_out/ncu_serp$f.log 2>&1
done
