# timeline of one C2 step: sweep per-launch events (PDL off by the events), Cholesky trace, in-block phase traces
mkdir -p gpurun_out
OCWG_SWEEP_EVENTS=1 timeout 300 python tools/prof_c2.py --reps 2 > gpurun_out/sweep_ev.log 2>&1
bash tools/gpu_chol_trace.sh
rm -f gpurun_out/trace.log
for ib in 0 128 256 384 2048; do
  OCWG_SWEEP_TRACE_IB=$ib timeout 300 python tools/sweep_trace.py >> gpurun_out/trace.log 2>&1
done
