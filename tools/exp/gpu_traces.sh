# in-block phase traces at several positions + the Cholesky owner trace
mkdir -p gpurun_out
rm -f gpurun_out/strace.log
for ib in 0 512 640 896 3584 3968; do
  OCWG_SWEEP_TRACE_IB=$ib timeout 300 python tools/sweep_trace.py >> gpurun_out/strace.log 2>&1
done
bash tools/gpu_chol_trace.sh
