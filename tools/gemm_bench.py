"""Micro-benchmark of the library's SIMT GEMM on the factorisation / sweep shapes."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2603_28845_b200 as g  # noqa: E402

SHAPES = [  # (m, n, k, ta, tb, lower, label)
    (4032, 4032, 64, 0, 1, 1, "chol trailing syrk k=64 (first panel)"),
    (2048, 2048, 64, 0, 1, 1, "chol trailing syrk k=64 (mid)"),
    (4032, 64, 64, 0, 1, 0, "chol panel"),
    (64, 4096, 64, 0, 0, 0, "inverse row-block"),
    (2048, 2048, 64, 0, 0, 0, "inverse update (mid)"),
    (3968, 4096, 128, 1, 0, 0, "sweep trailing (first block)"),
    (2048, 4096, 128, 1, 0, 0, "sweep trailing (mid)"),
    (4096, 4096, 4096, 0, 0, 0, "square 4096"),
]
ctx = g.context().handle
for prec in (0, 1, 2):
    dt = torch.float64 if prec == 1 else torch.float32
    for m, n, k, ta, tb, lower, label in SHAPES:
        a = torch.randn(k if ta else m, m if ta else k, dtype=dt, device="cuda")
        b = torch.randn(n if tb else k, k if tb else n, dtype=dt, device="cuda")
        c = torch.randn(m, n, dtype=dt, device="cuda")
        ms = C.c_double()
        g._check(g.lib().ocwg_debug_gemm(ctx, prec, m, n, k, -1.0, a.data_ptr(), a.shape[1], ta,
                                         b.data_ptr(), b.shape[1], tb, 1.0, c.data_ptr(), n, lower,
                                         20, C.byref(ms)))
        fl = 2.0 * m * n * k * (0.5 if lower else 1.0)
        print(f"{["fp32", "fp64", "tc3x"][prec]} {label:40s} {ms.value * 1e3:9.1f} us "
              f"{fl / ms.value / 1e9:8.2f} TFLOP/s")
