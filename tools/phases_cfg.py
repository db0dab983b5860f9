"""Per-phase times (order/damp, Cholesky, grids, sweep) of one layer of a
BASELINE config shape on the device API (profile mode).
    python tools/phases_cfg.py c3down"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2603_28845_b200 as g  # noqa: E402
from paper_2603_28845_b200 import dev  # noqa: E402
from tools.bench_configs import CONFIGS, inputs  # noqa: E402

name = sys.argv[1]
n, m, bits, group, frac, osc, wstd, silu = CONFIGS[name]
torch.cuda.set_device(0)
w, x = inputs(n, m, frac, osc, wstd, silu, 1234)
cfg = g.QuantConfig(bits, g.Scheme.asymmetric, g.Granularity.per_group, group)
opts = g.GptqOptions(actorder=True, percdamp=0.01, block_cols=128)
out = dev.LayerBuffers(n, m, cfg, 0)
dev.hessian(x, out.h)
del x
torch.cuda.empty_cache()
for rep in range(3):
    dev.profile(True)
    dev.gptq(w, out.h, cfg, opts, out)
    torch.cuda.synchronize()
    ph = dev.profile(False)
print(name, {k: round(v, 3) for k, v in ph.items()})
