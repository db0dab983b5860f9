"""Debug: which terms does the tensor-core accumulate_stats compute?"""
import sys
from pathlib import Path
import numpy as np
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import paper_2603_28845_b200 as g
from oracle import ocw_oracle as orc


def bf(a):
    return orc.bf16_round(np.ascontiguousarray(a, np.float32)).astype(np.float64)


for t, n in [(9, 4), (300, 64), (3000, 520)]:
    rng = np.random.default_rng(t)
    x = rng.standard_normal((t, n)).astype(np.float32)
    xh = (x + 0.05 * rng.standard_normal((t, n))).astype(np.float32)
    s = g.CalibStats.zeros(n)
    g.accumulate_stats(s, x, xh)
    p1 = bf(xh)
    p2 = bf(xh.astype(np.float64) - p1)
    d = x.astype(np.float64) - xh.astype(np.float64)
    d1 = bf(d)
    d2 = bf(d - d1)
    exact_g = xh.astype(np.float64).T @ xh.astype(np.float64)
    exact_c = xh.astype(np.float64).T @ d
    cands_g = {"P1P1": p1.T @ p1, "3term": p1.T @ p1 + p1.T @ p2 + p2.T @ p1, "exact": exact_g,
               "P1P1+P1P2": p1.T @ p1 + p1.T @ p2, "P1P1+P2P1": p1.T @ p1 + p2.T @ p1}
    cands_c = {"zero": np.zeros_like(exact_c), "P1D1": p1.T @ d1, "3term": p1.T @ d1 + p1.T @ d2 + p2.T @ d1,
               "exact": exact_c, "P1D1+P1D2": p1.T @ d1 + p1.T @ d2, "P1D1+P2D1": p1.T @ d1 + p2.T @ d1}
    sc = np.max(np.abs(exact_g))
    print(f"t={t} n={n}")
    for k, v in cands_g.items():
        print(f"  gram vs {k:10s} {np.max(np.abs(s.gram - v)) / sc:.3e}")
    for k, v in cands_c.items():
        print(f"  cross vs {k:10s} {np.max(np.abs(s.cross - v)) / sc:.3e}")
