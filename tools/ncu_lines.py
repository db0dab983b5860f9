"""Top CUDA source lines by warp-stall samples from an ncu report.
    python tools/ncu_lines.py rep.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fname, hdr, rows = None, None, []
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr and r[0] and r[0] != "":
        try:
            s = int(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        rows.append((s, f"{fname}:{r[0]}", r[1][:110]))
tot = sum(s for s, _, _ in rows) or 1
for s, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{100 * s / tot:5.1f}% {loc:18s} {src}")
