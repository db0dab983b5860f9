"""Phase timing of in-block sweep launches (globaltimer trace), C2 shape.
    OCWG_SWEEP_TRACE_IB=<first row> python tools/sweep_trace.py"""
import os
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_28845_b200 as g  # noqa: E402
from paper_2603_28845_b200 import dev  # noqa: E402

torch.cuda.set_device(0)
cfg = g.QuantConfig(bench.BITS, g.Scheme.asymmetric, g.Granularity.per_group, bench.GROUP)
opts = g.GptqOptions(actorder=True, percdamp=0.01, block_cols=128)
w, x = bench.make_inputs(torch.device("cuda", 0), torch)
out = dev.LayerBuffers(bench.N_IN, bench.M_OUT, cfg, 0)
for _ in range(2):
    dev.hessian(x, out.h)
    dev.gptq(w, out.h, cfg, opts, out)
torch.cuda.synchronize()
tr = np.zeros(1024 * 8, np.uint64)
k = g.lib().ocwg_debug_sweep_trace(g.context().handle, tr.ctypes.data, tr.size)
ctas = bench.M_OUT // 16
t8 = tr[:ctas * 8].reshape(ctas, 8).astype(np.int64)
t = t8[:, :6]
t0 = t[:, 0].min()
names = ["table+acc", "lookahead", "G stage", "main loop", "epilogue"]
print(f"ib={os.environ.get('OCWG_SWEEP_TRACE_IB')}: launch span {(t[:, 5].max() - t0) / 1e3:.1f} us, "
      f"CTA start spread {(t[:, 0].max() - t0) / 1e3:.1f} us")
for nm, a, b in [("  order", 0, 6), ("  gather", 6, 7), ("  acc", 7, 1)]:
    d = (t8[:, b] - t8[:, a]) / 1e3
    print(f"  {nm:10s} mean {d.mean():6.2f} us  max {d.max():6.2f}")
for i, nm in enumerate(names):
    d = (t[:, i + 1] - t[:, i]) / 1e3
    print(f"  {nm:10s} mean {d.mean():6.2f} us  max {d.max():6.2f}")
