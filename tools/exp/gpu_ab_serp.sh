mkdir -p gpurun_out
rm -f gpurun_out/ab_serp.log
for i in 1 2 3; do
  for f in 0 1; do
    OCWG_GRAM_SERP=$f timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-dropin --e2e-steps 0 > gpurun_out/ab.log 2>&1
    python -c "
import json
for l in open('gpurun_out/ab.log'):
    if l.startswith('{'):
        d=json.loads(l); print('serp=$f', round(d['ms_per_step'],4), round(d['breakdown_ms']['hessian'],4), d['clocks'])
" >> gpurun_out/ab_serp.log
  done
done
