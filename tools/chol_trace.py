"""Analyse OCWG_CHOL_TRACE output (10 u64 per item: row, col, start, k-loop
done, diag published, sub published, diag k-step done, factor done,
sub k-step done, sub solved; globaltimer ns; pair items have row == col)."""
import sys

import numpy as np

d = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 10).astype(np.int64)
t0 = d[:, 2][d[:, 2] > 0].min()
r, c = d[:, 0], d[:, 1]
T = {k: d[:, i] - t0 for k, i in
     [("st", 2), ("kl", 3), ("dpub", 4), ("spub", 5), ("dk", 6), ("fac", 7), ("sk", 8), ("sol", 9)]}
nt = int(c.max()) + 1
pair = np.array([np.where((r == k) & (c == k))[0][0] for k in range(nt)])
print(f"items {len(d)}  span {T['spub'].max() / 1e3:.1f} us")
P = {k: v[pair] for k, v in T.items()}
seg = [("wait+diag k-step", P["dk"] - P["kl"]), ("factor", P["fac"] - P["dk"]),
       ("publish diag", P["dpub"] - P["fac"]), ("wait+sub k-step", P["sk"] - P["dpub"]),
       ("solve", P["sol"] - P["sk"]), ("publish sub", P["spub"] - P["sol"])]
for name, v in seg:
    v = v[:-1]
    print(f"  {name:18s} mean {v.mean() / 1e3:7.2f} us  median {np.median(v) / 1e3:7.2f}")
gap = (P["dk"][1:] - P["spub"][:-1]) / 1e3
print(f"  next diag k-step done - sub publish: mean {gap.mean():.2f} us; interval {np.diff(P['spub']).mean() / 1e3:.2f} us")
