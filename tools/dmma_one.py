"""One fp64 DMMA GEMM (square 4096, the QEP cross.W shape) through ocwg_debug_gemm,
for an ncu capture:  python tools/dmma_one.py [reps]"""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2603_28845_b200 as g  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 1
n = 4096
a = torch.randn(n, n, dtype=torch.float64, device="cuda")
b = torch.randn(n, n, dtype=torch.float64, device="cuda")
c = torch.zeros(n, n, dtype=torch.float64, device="cuda")
ms = C.c_double()
g._check(g.lib().ocwg_debug_gemm(g.context().handle, 1, n, n, n, 1.0, a.data_ptr(), n, 0,
                                 b.data_ptr(), n, 0, 0.0, c.data_ptr(), n, 0, reps, C.byref(ms)))
ref = a @ b
err = float((c - ref).abs().max() / ref.abs().max())
print(f"dmma square {n}: {ms.value * 1e3:.1f} us/launch, {2.0 * n ** 3 / ms.value / 1e9:.2f} TF/s, "
      f"max rel err {err:.2e}")
assert err < 1e-12
