"""Summarize an `ncu --set full` report into the JSON committed under
profiles/: per launch, duration, DRAM bytes, L2 hit rate, throughput and
the top warp-stall reasons (from the SASS source page).

    python tools/ncu_summary.py gpurun_out/<tag>/prof.ncu-rep profiles/<name>.json
"""
import csv
import io
import json
import subprocess
import sys

KEYS = {
    "gpu__time_duration.sum": "duration_us",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "lts__t_sectors_srcunit_tex_op_read.sum": "l2_read_sectors",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_throughput_pct",
    "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed": "memory_throughput_pct",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_throughput_pct",
    "smsp__inst_executed.sum": "inst_executed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_active_pct",
    "launch__registers_per_thread": "registers",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "achieved_occupancy_pct",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1, "us": 1, "nsecond": 1e-3,
         "ns": 1e-3, "msecond": 1e3, "ms": 1e3}


def ncu(*args):
    return subprocess.run(["ncu", *args], capture_output=True, text=True, check=True).stdout


def raw(rep):
    rows = list(csv.reader(io.StringIO(ncu("-i", rep, "--page", "raw", "--csv"))))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        e = {"kernel": d.get("Kernel Name", "")[:120]}
        for k, name in KEYS.items():
            v = d.get(k)
            if v in (None, ""):
                continue
            try:
                f = float(v.replace(",", ""))
            except ValueError:
                continue
            e[name] = f * SCALE.get(u.get(k, ""), 1)
        if "dram_read" in e:
            e["dram_bytes"] = e["dram_read"] + e.get("dram_write", 0.0)
        out.append(e)
    return out


def stalls(rep):
    txt = ncu("-i", rep, "--page", "source", "--csv", "--print-source", "sass")
    rows = list(csv.reader(io.StringIO(txt)))
    hdr = rows[1]
    agg, tot = {}, 0.0
    for r in rows[2:]:
        if r and r[0] == "Kernel Name":
            break
        if len(r) != len(hdr) or r[0] == "Address":
            continue
        d = dict(zip(hdr, r))
        for h in hdr:
            if h.startswith("stall_") and "Not Issued" not in h:
                try:
                    v = float(d[h] or 0)
                except ValueError:
                    continue
                agg[h[6:]] = agg.get(h[6:], 0.0) + v
                tot += v
    return {k: round(v / tot, 3) for k, v in sorted(agg.items(), key=lambda x: -x[1])[:6]} if tot else {}


def main(rep, out):
    launches = raw(rep)
    summary = {"report": rep, "launches": launches}
    try:
        summary["stall_share_first_kernel"] = stalls(rep)
    except Exception as e:  # source page needs -lineinfo; keep the rest
        summary["stall_share_first_kernel"] = f"unavailable: {e}"
    if launches:
        d = [x["dram_bytes"] for x in launches if "dram_bytes" in x]
        summary["dram_bytes_per_launch"] = sum(d) / len(d) if d else None
        t = [x["duration_us"] for x in launches if "duration_us" in x]
        summary["duration_us_mean"] = sum(t) / len(t) if t else None
    json.dump(summary, open(out, "w"), indent=1)
    print(json.dumps(summary, indent=1))


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2])
