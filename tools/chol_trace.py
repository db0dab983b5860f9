"""Analyse OCWG_CHOL_TRACE output (per item: r, c, start, k-loop done, solve done,
published; globaltimer ns)."""
import sys

import numpy as np

d = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 6).astype(np.int64)
t0 = d[:, 2].min()
r, c = d[:, 0], d[:, 1]
st, kl, sv, pb = (d[:, i] - t0 for i in range(2, 6))
print(f"items {len(d)}  span {pb.max() / 1e3:.1f} us")
nt = int(c.max()) + 1
print(" col   diag:start  kdone  solved  publ | sub(c+1,c): start kdone  publ | diag factor us")
for col in list(range(0, 6)) + list(range(nt // 2, nt // 2 + 3)) + list(range(nt - 4, nt)):
    i = np.where((r == col) & (c == col))[0][0]
    line = f"{col:4d} {st[i]/1e3:10.1f} {kl[i]/1e3:7.1f} {sv[i]/1e3:7.1f} {pb[i]/1e3:7.1f} |"
    s = np.where((r == col + 1) & (c == col))[0]
    if len(s):
        s = s[0]
        line += f" {st[s]/1e3:8.1f} {kl[s]/1e3:7.1f} {pb[s]/1e3:7.1f} |"
    line += f" {(sv[i]-kl[i])/1e3:6.2f}"
    print(line)
diag = np.array([np.where((r == k) & (c == k))[0][0] for k in range(nt)])
gaps = np.diff(pb[diag])
print("diag publish interval us: mean %.2f  median %.2f  max %.2f" % (gaps.mean() / 1e3, np.median(gaps) / 1e3, gaps.max() / 1e3))
fac = (sv[diag] - kl[diag]) / 1e3
print("diag factor us: mean %.2f" % fac.mean())
sub = [np.where((r == k + 1) & (c == k))[0][0] for k in range(nt - 1)]
sub = np.array(sub)
print("sub solve us (publ - kdone): mean %.2f" % ((pb[sub] - kl[sub]) / 1e3).mean())
print("diag(c+1) kdone - sub(c+1,c) publ us: mean %.2f" % ((kl[diag[1:]] - pb[sub]) / 1e3).mean())
print("sub(c+1,c) kdone - diag(c) publ us: mean %.2f" % ((kl[sub] - pb[diag[:-1]]) / 1e3).mean())
