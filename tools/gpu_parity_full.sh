# BASELINE config parity at full sizes incl. C5 down (writes gpurun_out/r02_parity.jsonl)
mkdir -p gpurun_out
rm -f gpurun_out/r02_parity.jsonl
OCWG_PARITY_FULL=1 timeout 2600 python -m pytest tests/test_gpu_configs.py -q -s --timeout 2500 > gpurun_out/parity_full.log 2>&1; echo "rc=$?" >> gpurun_out/parity_full.log
