"""Is the batch-1 kernel slowed by cold instruction fetch after the L2 flush?

Times the cfg2 head A at batch 1 (CUDA events around the forward only) in
three situations:
  cold    : flush, A                       (the bench's headline situation)
  warmcode: flush, small head W, A         (same kernel code just ran on a
                                            different small head; A's tables cold)
  warm    : A, A                           (no flush: code and tables warm)
and prints the phase timeline of A in the first two.

    python tools/b1_coldcode.py [--reps 200]
"""
import argparse
import os
import statistics
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15742_b200 as hq  # noqa: E402
from paper_2512_15742_b200 import _lib, synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=200)
    args = ap.parse_args()
    A = hq.build_model(synthetic.synthetic_head())
    W = hq.build_model(synthetic.synthetic_head(dims=(2048, 128, 20), k=4096, seed=7))
    wsA, wsW = hq.make_workspace(A, 1), hq.make_workspace(W, 1)
    x = torch.from_numpy(synthetic.synthetic_inputs(1, 2048, seed=1)).cuda()
    yA = torch.zeros(20, dtype=torch.float64, device="cuda")
    yW = torch.zeros(20, dtype=torch.float64, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    t_end = time.perf_counter() + 1.0
    while time.perf_counter() < t_end:  # loaded clocks, without a deep launch backlog
        for _ in range(20):
            flush.zero_()
            hq.forward_async(A, x, 1, yA, wsA)
        torch.cuda.synchronize()

    def run(case, reps):
        ev = []
        with torch.cuda.stream(s):
            for r in range(reps + 5):
                if case in ("cold", "warmcode"):
                    flush.zero_()
                if case == "warmcode":
                    hq.forward_async(W, x, 1, yW, wsW, stream=s.cuda_stream)
                if case == "warm":
                    hq.forward_async(A, x, 1, yA, wsA, stream=s.cuda_stream)
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                hq.forward_async(A, x, 1, yA, wsA, stream=s.cuda_stream)
                b.record(s)
                if r >= 5:
                    ev.append((a, b))
        s.synchronize()
        wsA.check()
        t = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
        return statistics.median(t), t[len(t) // 10], t[9 * len(t) // 10]

    for case in ("cold", "warmcode", "warm", "cold", "warmcode", "warm"):
        m, p10, p90 = run(case, args.reps)
        print(f"{case:9s} median {m:7.2f} us  p10 {p10:7.2f}  p90 {p90:7.2f}", flush=True)

    grid = _lib.lib().skan_head_b1_grid(A.handle)
    stamps = torch.zeros(2 * grid * 16, dtype=torch.int64, device="cuda")
    for case in ("cold", "warmcode", "warm"):
        spans = []
        for rep in range(5):
            run(case, 20)
            _lib.check(_lib.lib().skan_debug_b1_timeline(wsA.handle, stamps.data_ptr()))
            stamps.zero_()
            with torch.cuda.stream(s):
                if case != "warm":
                    flush.zero_()
                if case == "warmcode":
                    hq.forward_async(W, x, 1, yW, wsW, stream=s.cuda_stream)
                if case == "warm":
                    hq.forward_async(A, x, 1, yA, wsA, stream=s.cuda_stream)
                    s.synchronize()
                    stamps.zero_()
                hq.forward_async(A, x, 1, yA, wsA, stream=s.cuda_stream)
            s.synchronize()
            _lib.check(_lib.lib().skan_debug_b1_timeline(wsA.handle, 0))
            st = stamps.view(2, grid, 16).cpu().numpy().astype(np.float64)[0]
            t0 = st[:, 0].min()
            row = {}
            for p in (1, 2, 8, 9, 4, 10, 5, 6, 7, 12, 13):
                col = st[:, p]
                col = col[col > 0]
                if col.size:
                    row[p] = round(float(np.median(col) - t0) / 1e3, 2) if p not in (12, 13) else round(
                        float(col.max() - t0) / 1e3, 2)
            spans.append(row)
        print(f"{case:9s} phase medians (us from first CTA start):")
        for r in spans:
            print("   ", r)


if __name__ == "__main__":
    main()
