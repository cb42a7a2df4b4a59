"""Exact-mode (f64, bitwise equal to the reference) latency of the cfg2 head
at a few batch sizes, CUDA events, L2 flushed before each call."""
import os
import statistics
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15742_b200 as hq  # noqa: E402
from paper_2512_15742_b200 import synthetic  # noqa: E402


def main():
    model = hq.build_model(synthetic.synthetic_head())
    ws = hq.make_workspace(model, 256)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    for B in [int(b) for b in os.environ.get("EXACT_BATCHES", "1,2,4,8,16,32,64,128,256").split(",")]:
        x = torch.from_numpy(synthetic.synthetic_inputs(B, 2048, seed=1)).cuda()
        y = torch.zeros(B * 20, dtype=torch.float64, device="cuda")
        ev = []
        with torch.cuda.stream(s):
            for r in range(13):
                flush.zero_()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(s)
                hq.forward_async(model, x, B, y, ws, mode="exact", stream=s.cuda_stream)
                b.record(s)
                if r >= 3:
                    ev.append((a, b))
        s.synchronize()
        ws.check()
        t = statistics.median(a.elapsed_time(b) * 1e3 for a, b in ev)
        print(f"split<={os.environ.get('SKAN_EXACT_SPLIT_MAX', 'default')} exact B={B:4d}: {t:9.1f} us  launches={ws.last_launches()}  -> {B / t * 1e6:,.0f} samples/s", flush=True)


if __name__ == "__main__":
    main()
