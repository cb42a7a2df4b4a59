"""Phase timeline of the tensor-core layer GEMM (CTA 0 of the first layer):
clock64 stamps of producer thread 0 and the MMA thread per chunk, printed as
cycles since the first stamp.

    python tools/gemm_timeline.py [--batch 256] [--dense]
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
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--dense", action="store_true")
    ap.add_argument("--chunks", type=int, default=24)
    args = ap.parse_args()
    B = args.batch
    if args.dense:
        model = hq.upload(synthetic.dense_runtime_head())
    else:
        model = hq.build_model(synthetic.synthetic_head())
    ws = hq.make_workspace(model, B)
    x = torch.from_numpy(synthetic.synthetic_inputs(B, 2048, seed=1)).cuda()
    y = torch.zeros(B * 20, dtype=torch.float64, device="cuda")
    for _ in range(3):
        hq.forward_async(model, x, B, y, ws, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    st = torch.zeros(2 * 64 * 8, dtype=torch.int64, device="cuda")
    _lib.check(_lib.lib().skan_debug_gemm_timeline(st.data_ptr()))
    hq.forward_async(model, x, B, y, ws, stream=torch.cuda.current_stream().cuda_stream)
    torch.cuda.synchronize()
    _lib.check(_lib.lib().skan_debug_gemm_timeline(None))
    # the last GEMM launch (layer 1) overwrote CTA 0 of layer 0: rerun layer 0 only is not
    # exposed, so read whichever launch wrote last and say which
    s = st.cpu().numpy().reshape(2, 64, 8).astype(np.int64)
    base = s[s > 0].min()
    print("chunk | producer: top  stage-free  W-done  A-free  arrived | mma: full  cp-issued  mma-issued")
    for c in range(args.chunks):
        p, m = s[0, c], s[1, c]
        if not p.any() and not m.any():
            break
        f = lambda v: f"{v - base:8d}" if v else "       -"
        print(f"{c:5d} | {f(p[0])} {f(p[1])} {f(p[2])} {f(p[3])} {f(p[4])} | {f(m[0])} {f(m[1])} {f(m[2])}")


if __name__ == "__main__":
    main()
