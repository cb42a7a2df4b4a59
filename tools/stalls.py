"""Top stall lines of one kernel in an ncu report (source page, SASS).
    python tools/stalls.py report.ncu-rep [min_share]"""
import csv
import subprocess
import sys

rep = sys.argv[1]
thr = float(sys.argv[2]) if len(sys.argv) > 2 else 0.015
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[1]
data = [dict(zip(hdr, r)) for r in rows[2:] if len(r) == len(hdr) and r[0] != "Address"]


def f(x):
    try:
        return float(x.replace(",", ""))
    except ValueError:
        return 0.0


key = "Warp Stall Sampling (All Samples)"
tot = sum(f(d[key]) for d in data) or 1.0
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {}
for d in data:
    for h in stalls:
        agg[h] = agg.get(h, 0.0) + f(d[h])
s = sum(agg.values()) or 1.0
print("stall mix:", ", ".join(f"{h[6:]} {v / s:.0%}" for h, v in sorted(agg.items(), key=lambda x: -x[1])[:8]))
for i, d in enumerate(data):
    v = f(d[key])
    if v / tot > thr:
        top = sorted(((f(d[h]), h) for h in stalls), reverse=True)[:2]
        print(f"{i:5d} {v / tot:6.1%} ex={f(d['Instructions Executed']):9.0f} {d['Source'][:72]:72} "
              f"{[(h[6:], int(x)) for x, h in top]}")
