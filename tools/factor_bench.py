"""Micro-benchmark of factor_tile64 (the Cholesky's diagonal-tile kernel)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2603_28845_b200 as g  # noqa: E402

cyc = np.zeros(8, np.int64)
L = np.zeros((64, 64), np.float32)
g._check(g.lib().ocwg_debug_factor_bench(g.context().handle, 20, cyc.ctypes.data, L.ctypes.data))
r = np.arange(64)
A = np.where(r[:, None] == r[None, :], 64.0 + r[:, None], 1.0 / (1 + r[:, None] + r[None, :]))
Lref = np.linalg.cholesky(A)
print(f"factor_tile64: {cyc[1]} clk per call ({cyc[1] / 1.9e3:.2f} us at 1.9 GHz), "
      f"max |L - Lref| = {np.abs(np.tril(L) - Lref).max():.2e}, upper max {np.abs(np.triu(L, 1)).max():.1e}")
ph = cyc[2:7] - cyc[2]
print("phase clocks: chol11 %d, trsm21 %d, update22 %d, chol22 %d" % (ph[1], ph[2] - ph[1], ph[3] - ph[2], ph[4] - ph[3]))
