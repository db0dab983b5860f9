mkdir -p gpurun_out
rm -f gpurun_out/stats_win.log
for w in 2048 4096 8192 16384; do
  echo "== window $w" >> gpurun_out/stats_win.log
  OCWG_STATS_WINDOW=$w OCWG_DEBUG_STATS=1 ./paper_2603_28845_b200/lib/dropin_bench >> gpurun_out/stats_win.log 2>&1
  OCWG_STATS_WINDOW=$w timeout 600 python -m pytest tests/test_gpu_parity.py -q -s -k "accumulate_stats_tensor_cores" 2>&1 | grep -E "accumulate_stats t=|passed|failed" >> gpurun_out/stats_win.log
done
