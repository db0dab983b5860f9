mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on -k regex:jq_search_rows -s 1 -c 1 -o gpurun_out/jq_full python tools/jointq_bench.py --skip-cpu --skip-c2 > gpurun_out/jq_ncu.log 2>&1
