mkdir -p gpurun_out
rm -f gpurun_out/trace8.log
for ib in 0 256 2048 3840; do
  OCWG_SWEEP_TRACE_IB=$ib timeout 300 python tools/sweep_trace.py >> gpurun_out/trace8.log 2>&1
done
