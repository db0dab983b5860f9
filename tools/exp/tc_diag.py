"""Diagnose the tcgen05 3xTF32 GEMM: per-case max error and error pattern."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2603_28845_b200 as g  # noqa: E402

def run(impl, m, n, k, ta, tb, kind="rand"):
    rng = np.random.default_rng(0)
    if kind == "rand":
        a = rng.standard_normal((k, m) if ta else (m, k)).astype(np.float32)
        b = rng.standard_normal((n, k) if tb else (k, n)).astype(np.float32)
    else:  # structured: A = index pattern
        A = np.zeros((m, k), np.float32); B = np.zeros((k, n), np.float32)
        A[np.arange(m), np.arange(m) % k] = 1.0   # each row picks one k
        B[:, :] = (np.arange(k)[:, None] * 1000 + np.arange(n)[None, :]).astype(np.float32)
        a = A.T.copy() if ta else A
        b = B.T.copy() if tb else B
    c = np.zeros((m, n), np.float32)
    ref = (a.T if ta else a).astype(np.float64) @ (b.T if tb else b).astype(np.float64)
    ad, bd, cd = (torch.from_numpy(v).cuda() for v in (a, b, c))
    ms = C.c_double()
    g._check(g.lib().ocwg_debug_gemm(g.context().handle, impl, m, n, k, 1.0, ad.data_ptr(), a.shape[1], ta,
                                     bd.data_ptr(), b.shape[1], tb, 0.0, cd.data_ptr(), n, 0, 1, C.byref(ms)))
    out = cd.cpu().numpy().astype(np.float64)
    err = np.abs(out - ref)
    return out, ref, err

for ta in (0, 1):
    for tb in (0, 1):
        for (m, n, k) in [(128, 128, 32), (128, 128, 64), (256, 128, 32), (128, 256, 32), (200, 136, 64)]:
            out, ref, err = run(2, m, n, k, ta, tb)
            bad = err > 1e-4 * (np.abs(ref) + 1)
            print(f"ta={ta} tb={tb} {m}x{n}x{k}: maxerr {err.max():.3e} bad {bad.mean():.3f} "
                  f"bad-rows {np.unique(np.nonzero(bad)[0])[:8]} bad-cols {np.unique(np.nonzero(bad)[1])[:8]}")
        out, ref, err = run(2, 128, 128, 32, ta, tb, kind="struct")
        r = 5
        print("   struct row5 out[:8]", out[r, :8], "ref", ref[r, :8])
