"""Time the C2 Hessian kernel alone (CUDA events, 20 back-to-back launches after warm-up).
    python tools/hess_time.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_28845_b200 as g  # noqa: E402
from paper_2603_28845_b200 import dev  # noqa: E402

torch.cuda.set_device(0)
cfg = g.QuantConfig(bench.BITS, g.Scheme.asymmetric, g.Granularity.per_group, bench.GROUP)
w, x = bench.make_inputs(torch.device("cuda", 0), torch)
out = dev.LayerBuffers(bench.N_IN, bench.M_OUT, cfg, 0)
for _ in range(5):
    dev.hessian(x, out.h)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    dev.hessian(x, out.h)
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 20
f = 262144 * 4096 * 4097
print(f"hessian {ms:.4f} ms  {f / ms / 1e9:.1f} TF/s")
