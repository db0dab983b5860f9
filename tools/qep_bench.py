"""QEP target correction (layerwise.cpp:95-112) at C2 size through the host API
(ocwg_qep_target: fp64 gram / cross in, fp32 target out, fp64 solve on the GPU).
    python tools/qep_bench.py [n] [m]"""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import torch  # noqa: E402

import paper_2603_28845_b200 as g  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
m = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
t = 16384
gen = torch.Generator(device="cuda").manual_seed(7)
x = torch.randn(t, n, generator=gen, device="cuda", dtype=torch.float64)
xp = x + 0.05 * torch.randn(t, n, generator=gen, device="cuda", dtype=torch.float64)
gram = (xp.T @ xp).cpu().numpy()
cross = (xp.T @ (x - xp)).cpu().numpy()
w = (0.02 * torch.randn(n, m, generator=gen, device="cuda")).cpu().numpy()
del x, xp
opts = g.QepOptions(0.5, 0.01)
stats = g.CalibStats(gram, cross)
out = g.qep_target(w, stats, opts)  # warm-up
ts = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    out = g.qep_target(w, stats, opts)
    ts.append((time.perf_counter() - t0) * 1e3)
rel = float(np.max(np.abs(out - w)) / np.max(np.abs(w)))
print(f"qep_target n={n} m={m}: {min(ts):.2f} ms (host API, fp64 gram/cross in), max|corr|/max|W| {rel:.3e}")
