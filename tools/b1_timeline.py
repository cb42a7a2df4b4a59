"""Phase timeline of the persistent batch-1 head kernel (skan_head_b1.cu).

Runs the cfg2 head at batch 1 with L2 flushed before each forward and prints,
per phase, the min / median / max over CTAs of the %globaltimer stamp
relative to the earliest kernel start (microseconds).

    python tools/b1_timeline.py [--reps 5]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15742_b200 as hq  # noqa: E402
from paper_2512_15742_b200 import _lib, synthetic  # noqa: E402

PHASES_V1 = {0: "start", 1: "tables", 2: "x ready", 3: "locate+hist", 4: "rowlist+tma", 5: "plane ready",
             6: "L0 partial", 7: "grid sync 1", 9: "L1 reduce+locate", 10: "L1 rows", 11: "grid sync 2",
             12: "final start", 13: "end"}
PHASES_V2 = {0: "x issued", 1: "tables issued", 11: "brackets", 2: "brackets+counts", 8: "alloc (plane TMA)",
             9: "rows ranked+TMA", 4: "plane+rec ready", 10: "L0 FMA done", 5: "L0 partials out",
             6: "grid sync", 7: "L1 done", 12: "final start", 13: "end"}
PHASES = PHASES_V1 if os.environ.get("SKAN_B1_V1") == "1" else PHASES_V2


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--flush", choices=["write", "write+read", "none"], default="write")
    args = ap.parse_args()
    cn = synthetic.synthetic_head()
    model = hq.build_model(cn)
    ws = hq.make_workspace(model, 1)
    grid = _lib.lib().skan_head_b1_grid(model.handle)
    stamps = torch.zeros(2 * grid * 16, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().skan_debug_b1_timeline(ws.handle, stamps.data_ptr()))
    x = torch.from_numpy(synthetic.synthetic_inputs(1, 2048, seed=1)).cuda()
    y = torch.zeros(20, dtype=torch.float64, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    flush_r = torch.ones(64 << 20, dtype=torch.float32, device="cuda")

    def do_flush():
        if args.flush != "none":
            flush.zero_()
        if args.flush == "write+read":
            flush_r.sum()
    import time
    for rep in range(args.reps):
        # keep the GPU busy for ~1 s first so SM clocks are at their loaded
        # value (an idle GPU starts a lone kernel at a low clock)
        t_end = time.perf_counter() + 1.0
        while time.perf_counter() < t_end:
            for _ in range(50):
                do_flush()
                hq.forward_async(model, x, 1, y, ws)
            torch.cuda.synchronize()
        stamps.zero_()
        do_flush()
        hq.forward_async(model, x, 1, y, ws)
        torch.cuda.synchronize()
        both = stamps.view(2, grid, 16).cpu().numpy().astype(np.float64)
        s, cs = both[0], both[1]
        t0 = s[:, 0].min()
        print(f"rep {rep}: kernel span {(s[:, 13].max() - t0) / 1e3:.2f} us")
        last = np.flatnonzero(s[:, 15] > 0)
        if last.size:
            r = s[last[0]]
            print(f"   last CTA {last[0]}: {(r[15] - r[14]) / max(r[13] - r[0], 1) * 1e3:.0f} MHz over its span")
        for p, name in PHASES.items():
            col = s[:, p]
            col = col[col > 0]
            if col.size == 0:
                continue
            rel = (col - t0) / 1e3
            print(f"   {p:2d} {name:18s} min {rel.min():7.2f}  med {np.median(rel):7.2f}  max {rel.max():7.2f}")
        used = [k for k in range(16) if (cs[:, k] > 0).all()]
        if len(used) > 1:
            d = np.diff(cs[:, used], axis=1)
            print("   clock64 deltas between fine stamps (cycles, median over CTAs):",
                  {f"{a}->{b}": int(np.median(d[:, q])) for q, (a, b) in enumerate(zip(used[:-1], used[1:]))})
            print("   clock64 of each fine stamp after slot", used[0], "(cycles, median over CTAs):",
                  {k: int(np.median(cs[:, k] - cs[:, used[0]])) for k in used[1:]})


if __name__ == "__main__":
    main()
