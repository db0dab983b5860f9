mkdir -p gpurun_out
rm -f gpurun_out/ab_win.log
for i in 1 2 3; do
  for wv in 0 13798; do
    OCWG_HESSIAN_WINDOW=$wv timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin --e2e-steps 0 > gpurun_out/ab.log 2>&1
    python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); print('win=$wv', round(d['ms_per_step'],4), round(d['breakdown_ms']['hessian'],4), d['clocks']['sm_mhz'])
" >> gpurun_out/ab_win.log
  done
done
