"""Analyse OCWG_CHOL_TRACE output (6 u64 per item: row, col, start, k-loop
done, factor/solve done, published; globaltimer ns) along the critical path
diag(c) -> sub(c+1, c) -> diag(c+1).
    OCWG_CHOL_TRACE=/path/trace.bin python tools/prof_c2.py --reps 1
    python tools/chol_trace.py /path/trace.bin"""
import sys

import numpy as np

d = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 6).astype(np.int64)
n_items = len(d)
nt = int(round((np.sqrt(8 * n_items + 1) - 1) / 2))
d = d[-(nt * (nt + 1) // 2):]  # last factorisation in the file
t0 = d[:, 2].min()
r, c = d[:, 0], d[:, 1]
st, kd, fd, pb = (d[:, i] - t0 for i in (2, 3, 4, 5))
idx = {(int(a), int(b)): i for i, (a, b) in enumerate(zip(r, c))}
D = np.array([idx[(k, k)] for k in range(nt)])
S = np.array([idx[(k + 1, k)] for k in range(nt - 1)])
print(f"nt {nt}, items {len(d)}, span {pb.max() / 1e3:.1f} us, per column {pb.max() / nt / 1e3:.2f} us")
Dd, Ss = D[:-1], S
seg = [
    ("diag: start->kdone", kd[Dd] - st[Dd]),
    ("diag: factor", fd[Dd] - kd[Dd]),
    ("diag: store+publish", pb[Dd] - fd[Dd]),
    ("sub: kdone after diag pub", kd[Ss] - pb[Dd]),
    ("sub: solve done after max(kdone, diag pub)", fd[Ss] - np.maximum(kd[Ss], pb[Dd])),
    ("sub: store+publish", pb[Ss] - fd[Ss]),
    ("next diag kdone after sub pub", kd[D[1:]] - pb[Ss]),
    ("column interval (diag pub)", np.diff(pb[D])),
]
for name, v in seg:
    print(f"  {name:44s} mean {v.mean() / 1e3:7.2f} us  median {np.median(v) / 1e3:7.2f}")
for k in (0, 1, nt // 4, nt // 2, 3 * nt // 4, nt - 2):
    i, j = D[k], S[k] if k < nt - 1 else D[k]
    print(f"  col {k:3d}: diag st {st[i]/1e3:8.1f} kd {kd[i]/1e3:8.1f} fd {fd[i]/1e3:8.1f} pb {pb[i]/1e3:8.1f}"
          f" | sub st {st[j]/1e3:8.1f} kd {kd[j]/1e3:8.1f} fd {fd[j]/1e3:8.1f} pb {pb[j]/1e3:8.1f}")
