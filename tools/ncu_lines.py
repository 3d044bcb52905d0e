"""Aggregate an .ncu-rep's SASS metrics by CUDA source line (cuda,sass view).
usage: ncu_lines.py rep [top]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
agg = defaultdict(lambda: [0.0, 0.0, ""])
line, src, fname = None, "", ""
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] in ("Function Name", "Line No"):
        continue
    if r[0] and r[0].isdigit():
        line, src = int(r[0]), r[1]
    if len(r) > 7 and r[2]:
        try:
            samp = float(r[4] or 0)
            inst = float(r[7] or 0)
        except ValueError:
            continue
        a = agg[(fname, line)]
        a[0] += samp
        a[1] += inst
        a[2] = src
tot_s = sum(v[0] for v in agg.values()) or 1
tot_i = sum(v[1] for v in agg.values()) or 1
print(f"total samples {tot_s:.0f}  total warp-inst {tot_i:.3e}")
for (f, l), (s, i, src) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{100*s/tot_s:5.1f}%s {100*i/tot_i:5.1f}%i  {f}:{l:<5} {src.strip()[:90]}")
