mkdir -p gpurun_out
timeout 300 python tools/gemm_bench.py > gpurun_out/gemm_bench.log 2>&1
for mc in 1024 2048; do OCWG_CHOL_MACRO=$mc timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-dropin > gpurun_out/bmac_$mc.log 2>&1; done
python - <<'PY' > gpurun_out/torch_f64.log 2>&1
import torch, time
a=torch.randn(4096,4096,dtype=torch.float64,device='cuda'); b=torch.randn(4096,4096,dtype=torch.float64,device='cuda')
for _ in range(3): c=a@b
torch.cuda.synchronize(); s=torch.cuda.Event(enable_timing=True); e=torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): c=a@b
e.record(); torch.cuda.synchronize(); ms=s.elapsed_time(e)/10
print("cublas dgemm 4096^3: %.2f ms, %.1f TFLOP/s" % (ms, 2*4096**3/ms/1e9))
PY
