mkdir -p gpurun_out
rm -f gpurun_out/trace8v.log
for v in 0 1 2; do
  echo "variant $v" >> gpurun_out/trace8v.log
  OCWG_SWEEP8_VARIANT=$v OCWG_SWEEP_TRACE_IB=256 timeout 300 python tools/sweep_trace.py >> gpurun_out/trace8v.log 2>&1
done
