"""Per-SASS-instruction stall breakdown from an ncu report, for an address range
or the whole kernel:  python tools/ncu_stalls.py rep.ncu-rep [grep-pattern]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, data = None, []
for r in rows:
    if r and r[0] == "Address":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
tot = {c: 0 for c in cols}
for d in data:
    for c in cols:
        tot[c] += int(d[c] or 0)
allv = sum(tot.values()) or 1
print("kernel stall totals:", ", ".join(f"{c[6:]} {100 * v / allv:.1f}%" for c, v in
                                         sorted(tot.items(), key=lambda x: -x[1]) if v))
top = sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:25]
for d in top:
    br = sorted(((int(d[c] or 0), c[6:]) for c in cols), reverse=True)[:3]
    print(f'{int(d["Warp Stall Sampling (All Samples)"] or 0):6d} {d["Address"][-5:]} {d["Source"][:60]:60s} '
          + " ".join(f"{n}:{v}" for v, n in br if v))
