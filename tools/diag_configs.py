"""CUDA-event timing of the other BASELINE.json configs on one GPU:
cfg1 (256->256, K=256, batch 1), cfg4 (dense {2048,13664,20} f32 grids,
batch 64) and cfg5 (H compressed cfg2 heads on one shared batch), L2
flushed before each call.

    python tools/diag_configs.py [--heads 4] [--reps 20]
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
from paper_2512_15742_b200 import synthetic  # noqa: E402


def timed(fn, reps, flush, stream):
    ev = []
    with torch.cuda.stream(stream):
        for r in range(reps + 3):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            if r >= 3:
                ev.append((a, b))
    stream.synchronize()
    return statistics.median(a.elapsed_time(b) * 1e3 for a, b in ev)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--heads", type=int, default=4)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--skip-dense", action="store_true")
    ap.add_argument("--only-dense", action="store_true")
    args = ap.parse_args()
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    t_end = time.perf_counter() + 1.0
    while time.perf_counter() < t_end:
        flush.zero_()

    if args.only_dense:
        args.heads = 0
    # cfg1
    cn = synthetic.synthetic_head(dims=(256, 256), k=256, grid=10, int8=True, seed=1)
    m = hq.build_model(cn)
    ws = hq.make_workspace(m, 1)
    x = torch.from_numpy(synthetic.synthetic_inputs(1, 256, seed=1)).cuda()
    y = torch.zeros(256, dtype=torch.float64, device="cuda")
    us = timed(lambda: hq.forward_async(m, x, 1, y, ws, stream=s.cuda_stream), args.reps, flush, s)
    print(f"cfg1 256->256 K=256 int8 batch 1: {us:8.2f} us  launches={ws.last_launches()}", flush=True)

    # cfg5: H cfg2 heads, one shared batch of 256
    heads = [hq.build_model(synthetic.synthetic_head(seed=2026 + 7 * h)) for h in range(args.heads)]
    if not heads:
        heads = None
    if heads:
        wss = [hq.make_workspace(h, 256) for h in heads]
        xb = torch.from_numpy(synthetic.synthetic_inputs(256, 2048, seed=5)).cuda()
        ys = [torch.zeros(256 * 20, dtype=torch.float64, device="cuda") for _ in heads]
        us = timed(lambda: hq.forward_multi(heads, wss, xb, 256, ys, stream=s.cuda_stream), max(3, args.reps // 4),
                   flush, s)
        print(f"cfg5 {args.heads} heads x batch 256: {us:10.2f} us  -> {args.heads * 256 / us * 1e6:,.0f} "
              f"head-samples/s", flush=True)
        del heads, wss

    if not args.skip_dense:
        layers = synthetic.dense_runtime_head()
        dm = hq.upload(layers)
        del layers
        dws = hq.make_workspace(dm, 64)
        xd = torch.from_numpy(synthetic.synthetic_inputs(64, 2048, seed=6)).cuda()
        yd = torch.zeros(64 * 20, dtype=torch.float64, device="cuda")
        plan = dm.plan()
        us = timed(lambda: hq.forward_async(dm, xd, 64, yd, dws, stream=s.cuda_stream), 3, flush, s)
        print(f"cfg4 dense {{2048,13664,20}} batch 64: {us:10.2f} us  -> {64 / us * 1e6:,.0f} samples/s, "
              f"{plan.payload_total / us / 1e3:,.0f} GB/s of the {plan.payload_total:,} B grid  "
              f"launches={dws.last_launches()}", flush=True)


if __name__ == "__main__":
    main()
