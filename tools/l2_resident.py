"""Batch-1 forwards of the cfg2 head with the 256 MiB L2 flush before each,
with or without the head's persisting L2 window (skan_head_set_l2_persist):
the workload for the ncu L2 hit-rate capture of the L2-resident regime
(profiles/r2/ncu_l2_resident.json).

    ncu --cache-control none -k regex:k_head_b1 -s 20 -c 1 --metrics ... \\
        python tools/l2_resident.py [--persist]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15742_b200 as hq  # noqa: E402
from paper_2512_15742_b200 import synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--persist", action="store_true")
    ap.add_argument("--calls", type=int, default=40)
    args = ap.parse_args()
    model = hq.build_model(synthetic.synthetic_head())
    ws = hq.make_workspace(model, 1)
    s = torch.cuda.Stream()
    if args.persist:
        model.set_l2_persist(s.cuda_stream, 1.0)
    x = torch.from_numpy(synthetic.synthetic_inputs(1, 2048, seed=1)).cuda()
    y = torch.zeros(20, dtype=torch.float64, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    with torch.cuda.stream(s):
        for _ in range(args.calls):
            flush.zero_()
            hq.forward_async(model, x, 1, y, ws, stream=s.cuda_stream)
    s.synchronize()
    ws.check()
    print("ok", y[:3].tolist())


if __name__ == "__main__":
    main()
