"""Per-chunk clock64 timeline of the persistent dense-layer kernel
(k_dense_persist, cfg4 layer 0 at batch 64, CTA 0): producer thread 0, the
MMA lane and the TMA lane, cycles since the first stamp.

    python tools/dense_timeline.py [--chunks 40]
"""
import argparse
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15742_b200 as hq  # noqa: E402
from paper_2512_15742_b200 import _lib, synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--chunks", type=int, default=40)
    ap.add_argument("--batch", type=int, default=64)
    args = ap.parse_args()
    B = args.batch
    model = hq.upload(synthetic.dense_runtime_head())
    ws = hq.make_workspace(model, B)
    x = torch.from_numpy(synthetic.synthetic_inputs(B, 2048, seed=1)).cuda()
    y = torch.zeros(B * 20, dtype=torch.float64, device="cuda")
    for _ in range(3):
        hq.forward_async(model, x, B, y, ws, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    st = torch.zeros(4 * 64 * 8, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().skan_debug_gemm_timeline(st.data_ptr()))
    hq.forward_async(model, x, B, y, ws, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    _lib.check(_lib.lib().skan_debug_gemm_timeline(None))
    s = st.cpu().numpy().reshape(4, 64, 8).astype(np.int64)
    base = s[s > 0].min()
    print("chunk | A set0: top A-free arrived | A set1: top A-free arrived | lo set0: top landed arrived | mma: full issued | tma: free issued")
    for c in range(args.chunks):
        p, m, t, lw = s[0, c], s[1, c], s[2, c], s[3, c]
        if not (p.any() or m.any() or t.any() or lw.any()):
            break
        f = lambda v: f"{v - base:8d}" if v else "       -"
        print(f"{c:5d} | {f(p[0])} {f(p[1])} {f(p[2])} | {f(lw[0])} {f(lw[1])} {f(lw[2])} | {f(t[2])} {f(t[3])} {f(t[4])} | {f(m[0])} {f(m[1])} | {f(t[0])} {f(t[1])}")


if __name__ == "__main__":
    main()
