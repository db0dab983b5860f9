mkdir -p gpurun_out
rm -f gpurun_out/ab_table.log
for i in 1 2 3; do
  for t in 1 0; do
    OCWG_SWEEP_TABLE=$t timeout 300 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/ab_t.log 2>&1
    python -c "
import json
for l in open('gpurun_out/ab_t.log'):
    if l.startswith('{'): d=json.loads(l); print('table=$t', round(d['ms_per_step'],4), round(d['breakdown_ms']['hessian'],4), d['clocks']['sm_mhz'])
" >> gpurun_out/ab_table.log
  done
done
