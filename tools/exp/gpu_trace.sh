mkdir -p gpurun_out
for ib in 0 128 256 384 2048 3968; do
  OCWG_SWEEP_TRACE_IB=$ib timeout 300 python tools/sweep_trace.py >> gpurun_out/trace.log 2>&1
done
