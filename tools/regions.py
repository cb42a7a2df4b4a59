"""Per-region instruction counts and stall shares of one kernel in an ncu
report: consecutive SASS lines with similar execution counts are merged.
    python tools/regions.py report.ncu-rep units [min_instr]
units = the number of loop iterations to normalise by (e.g. CTA-chunks)."""
import csv
import subprocess
import sys

rep, units = sys.argv[1], float(sys.argv[2])
lim = float(sys.argv[3]) if len(sys.argv) > 3 else 10.0
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
ex = [f(d["Instructions Executed"]) / units for d in data]
sm = [f(d[key]) for d in data]
tot_s = sum(sm) or 1.0
start = 0
print(f"total instr/unit {sum(ex):.0f}")
for i in range(1, len(data) + 1):
    if i == len(data) or abs(ex[i] - ex[start]) > 0.3 * max(ex[start], 0.5):
        ins, smp = sum(ex[start:i]), sum(sm[start:i])
        if ins > lim or smp / tot_s > 0.01:
            print(f"{start:5d}-{i - 1:5d} instr/unit {ins:7.1f}  samples {smp / tot_s:5.1%}  {data[start]['Source'][:60]}")
        start = i
