"""Per-source-line stall breakdown from an .ncu-rep (source page, cuda,sass view).
usage: ncu_stalls.py rep [top]"""
import csv, io, subprocess, sys
from collections import defaultdict

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 15
out = subprocess.run(["ncu", "-i", rep] + (["-k", sys.argv[3]] if len(sys.argv) > 3 else []) + ["--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr, fname, line, src = None, "", None, ""
agg = defaultdict(lambda: defaultdict(float))
srcs = {}
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if r[0] == "Function Name" or hdr is None:
        continue
    if r[0] and r[0].isdigit():
        line, src = int(r[0]), r[1]
    if len(r) > 7 and r[2]:
        for i, h in enumerate(hdr):
            if h.startswith("stall_") and "Not Issued" not in h and i < len(r):
                try:
                    agg[(fname, line)][h[6:]] += float(r[i] or 0)
                except ValueError:
                    pass
        srcs[(fname, line)] = src
tot = sum(sum(d.values()) for d in agg.values()) or 1
for k, d in sorted(agg.items(), key=lambda kv: -sum(kv[1].values()))[:top]:
    s = sum(d.values())
    reasons = ", ".join(f"{n} {100*v/s:.0f}%" for n, v in sorted(d.items(), key=lambda x: -x[1])[:3] if v)
    print(f"{100*s/tot:5.1f}% {k[0]}:{k[1]:<5} [{reasons}] {srcs[k].strip()[:60]}")
