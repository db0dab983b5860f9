# A/B of library variants in paper_2603_28845_b200/lib_var/*.so: Cholesky trace + C2 step
mkdir -p gpurun_out
rm -f gpurun_out/ab_lib.log
for i in 1 2; do
for v in $VARIANTS; do
  cp paper_2603_28845_b200/lib_var/$v.so paper_2603_28845_b200/lib/libocwg.so
  rm -f /tmp/ctrace.bin
  OCWG_CHOL_TRACE=/tmp/ctrace.bin timeout 300 python tools/prof_c2.py --reps 1 > /dev/null 2>&1
  python tools/chol_trace.py /tmp/ctrace.bin > gpurun_out/ct_$v.log 2>&1
  timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin --e2e-steps 0 > gpurun_out/ab.log 2>&1
  (echo "== $v"; head -7 gpurun_out/ct_$v.log; python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); b=d['breakdown_ms']; print('step', round(d['ms_per_step'],4), 'chol', round(b['gptq_phases']['cholesky'],4), 'hess', round(b['hessian'],4))
") >> gpurun_out/ab_lib.log
done
done
