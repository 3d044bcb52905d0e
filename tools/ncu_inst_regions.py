"""Instructions executed per source-line region of one kernel in an .ncu-rep.
usage: ncu_inst_regions.py rep file.cu name:lo-hi [name:lo-hi ...]"""
import csv, io, subprocess, sys
rep, fname = sys.argv[1], sys.argv[2]
regions = []
for a in sys.argv[3:]:
    n, r = a.split(":")
    lo, hi = r.split("-")
    regions.append((n, int(lo), int(hi)))
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
cur = ""
tot = {n: 0 for n, _, _ in regions}
tot["other"] = 0
allinst = 0
for r in csv.reader(io.StringIO(out)):
    if not r:
        continue
    if r[0] == "File Path":
        cur = r[1].split("/")[-1]
        continue
    if not r[0].isdigit() or len(r) < 8:
        continue
    try:
        inst = int(r[7])
    except ValueError:
        continue
    allinst += inst
    ln = int(r[0])
    hit = False
    if cur == fname:
        for n, lo, hi in regions:
            if lo <= ln <= hi:
                tot[n] += inst
                hit = True
                break
    if not hit:
        tot["other"] += inst
for k, v in tot.items():
    print(f"{k:12s} {v:14d}  {100.0 * v / max(allinst, 1):5.1f}%")
print(f"{'total':12s} {allinst:14d}")
