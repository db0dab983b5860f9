mkdir -p gpurun_out
rm -f /tmp/ctrace.bin
OCWG_CHOL_TRACE=/tmp/ctrace.bin timeout 300 python tools/prof_c2.py --reps 1 > gpurun_out/ctrace_run.log 2>&1
cp /tmp/ctrace.bin gpurun_out/ctrace.bin
python tools/chol_trace.py /tmp/ctrace.bin > gpurun_out/ctrace.log 2>&1
