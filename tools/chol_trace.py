"""Analyse OCWG_CHOL_TRACE output: 6 u64 per entry {r, c + 1000 kind, start,
k-loop done, factor/solve done, published} (globaltimer ns), kind 0 = worker
tile, 1 = partial S, 2 = emission, 3 = owner (critical path).
    OCWG_CHOL_TRACE=/path/trace.bin python tools/prof_c2.py --reps 1
    python tools/chol_trace.py /path/trace.bin"""
import sys

import numpy as np

d = np.fromfile(sys.argv[1], dtype=np.uint64).reshape(-1, 6).astype(np.int64)
d = d[d[:, 2] > 0]
r, ck = d[:, 0], d[:, 1]
c, kind = ck % 1000, ck // 1000
st, kd, fd, pb = (d[:, i] for i in (2, 3, 4, 5))
t0 = st.min()
st, kd, fd, pb = st - t0, kd - t0, fd - t0, pb - t0
nt = int(c.max()) + 1
own = {(int(a), int(b)): i for i, (a, b, k) in enumerate(zip(r, c, kind)) if k == 3}
par = {(int(a), int(b)): i for i, (a, b, k) in enumerate(zip(r, c, kind)) if k == 1}
print(f"nt {nt}, entries {len(d)}, span {pb.max() / 1e3:.1f} us, per column {pb.max() / nt / 1e3:.2f} us")
D = np.array([own[(k, k)] for k in range(nt)])
S = np.array([own[(k + 1, k)] for k in range(nt - 1)])
Dd = D[:-1]
seg = [
    ("diag: stage + k=c-1 update", kd[Dd] - st[Dd]),
    ("diag: factor", fd[Dd] - kd[Dd]),
    ("diag: transpose + store + publish", pb[Dd] - fd[Dd]),
    ("sub: stage + k=c-1 update", kd[S] - st[S]),
    ("sub: solve", fd[S] - kd[S]),
    ("sub: store + publish", pb[S] - fd[S]),
    ("next diag start after sub publish", st[D[1:]] - pb[S]),
    ("column interval (diag publish)", np.diff(pb[D])),
]
for name, v in seg:
    print(f"  {name:42s} mean {v.mean() / 1e3:7.2f} us  median {np.median(v) / 1e3:7.2f}")
late = [max(0, pb[par[(k, k)]] - st[D[k]]) for k in range(1, nt) if (k, k) in par]
late1 = [max(0, pb[par[(k + 1, k)]] - st[S[k]]) for k in range(1, nt - 1) if (k + 1, k) in par]
print(f"  partial diag published after owner start: mean {np.mean(late) / 1e3:.2f} us; partial sub: {np.mean(late1) / 1e3:.2f} us")
pdi = np.array([par[(k, k)] for k in range(2, nt) if (k, k) in par])
kk = c[pdi]
dur = (kd[pdi] - st[pdi]) / 1e3
print(f"  partial diag items: k-loop time mean {dur.mean():.1f} us, per k-step {np.mean(dur / np.maximum(kk - 1, 1)):.2f} us;"
      f" start before owner needs it: mean {np.mean(st[D[kk]] - st[pdi]) / 1e3:.1f} us")
fi = np.where((kind == 0) & (c >= 8))[0]
per = (kd[fi] - st[fi]) / np.maximum(c[fi], 1) / 1e3
print(f"  full items (c >= 8): k-loop per k-step min {per.min():.2f} p10 {np.percentile(per, 10):.2f} us; "
      f"dispatch-to-owner lead (column c) mean {np.mean(st[D[c[fi]]] - st[fi]) / 1e3:.1f} us")
print(f"  full items (c >= 8): k-loop per k-step mean {per.mean():.2f} us, median {np.median(per):.2f}; "
      f"solve+publish mean {np.mean(pb[fi] - kd[fi]) / 1e3:.2f} us; items {len(fi)}")
busy = np.sum(pb[kind < 3] - st[kind < 3]) / 1e3
print(f"  worker busy time {busy:.0f} us over span {pb.max() / 1e3:.0f} us -> {busy / (pb.max() / 1e3):.0f} CTAs busy on average")

# critical chain of the diagonal partials: X(c-2) published -> full item (c, c-2)
# -> partial (c, c) -> owner column c start
full = {(int(a), int(b)): i for i, (a, b, k) in enumerate(zip(r, c, kind)) if k == 0}
rows = []
for cc in range(4, nt):
    if (cc, cc - 2) not in full or (cc, cc) not in par:
        continue
    x = pb[D[cc - 2]]
    fi, pi = full[(cc, cc - 2)], par[(cc, cc)]
    rows.append((kd[fi] - x, fd[fi] - x, pb[fi] - x, st[pi] - x, kd[pi] - x, pb[pi] - x, st[D[cc]] - x))
if rows:
    a = np.array(rows) / 1e3
    names = ["full(c,c-2) k-loop done", "full solve done", "full published", "partial start",
             "partial k-loop done", "partial published", "owner column c start"]
    print("  critical chain, times after X(c-2) published (median over columns):")
    for i, nm in enumerate(names):
        print(f"    {nm:28s} {np.median(a[:, i]):7.2f} us")
