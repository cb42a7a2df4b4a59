"""Summarize an `ncu --metrics gpu__time_duration.sum --csv` launch list:
per-kernel launch count, mean and total device time (cold-cache, serialized
by ncu: compare SHARES, not absolutes)."""
import csv
import sys
from collections import defaultdict


def main(path):
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(list)
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            name = d["Kernel Name"]
            name = name.replace("skan::(anonymous namespace)::", "").replace("skan::<unnamed>::", "")
            agg[(name[:70], d["Grid Size"], d["Block Size"])].append(float(d["Metric Value"].replace(",", "")))
    tot = sum(sum(v) for v in agg.values())
    print(f"{'n':>4} {'mean_us':>9} {'share':>6}  kernel [grid] [block]")
    for (k, g, b), v in sorted(agg.items(), key=lambda x: -sum(x[1])):
        print(f"{len(v):4d} {sum(v) / len(v) / 1e3:9.2f} {sum(v) / tot:6.1%}  {k} {g} {b}")


if __name__ == "__main__":
    main(sys.argv[1])
