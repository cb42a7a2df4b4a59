"""bs256 step time of the cfg2 head architecture at several codebook sizes K
(L2 flushed before each call, CUDA events): K=16 makes every codebook-row
gather an L1 hit, so the difference to K=65536 bounds what the gathers cost
the layer GEMM.  Used for DESIGN.md §4 ("the codebook-row gathers are NOT
the limiter").  Run on a GPU box:  python tools/gemm_codebook_size.py"""
import os, sys, statistics
sys.path.insert(0, os.getcwd())
import torch
import paper_2512_15742_b200 as hq
from paper_2512_15742_b200 import synthetic
for k in (65536, 4096, 256, 16):
    model = hq.build_model(synthetic.synthetic_head(k=k))
    ws = hq.make_workspace(model, 256)
    x = torch.from_numpy(synthetic.synthetic_inputs(256, 2048, seed=1)).cuda()
    y = torch.zeros(256 * 20, dtype=torch.float64, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    ev = []
    with torch.cuda.stream(s):
        for r in range(40):
            flush.zero_()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s); hq.forward_async(model, x, 256, y, ws, stream=s.cuda_stream); b.record(s)
            if r >= 5: ev.append((a, b))
    s.synchronize()
    print(f"K={k:6d}: bs256 {statistics.median(a.elapsed_time(b)*1e3 for a,b in ev):7.1f} us", flush=True)
