mkdir -p gpurun_out
OCWG_GRAM_SERP=1 timeout 600 ncu --set full --clock-control none -k regex:gram_tc -c 1 -o gpurun_out/gram_full python tools/hess_time.py > gpurun_out/ncu_gram_full.log 2>&1
