"""Latency diagnostics of the cfg2 head on one GPU: CUDA-event time per
forward at several batch sizes, with L2 flushed (256 MiB write) or warm.

    python tools/diag_latency.py [--reps 200]
"""
import argparse
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15742_b200 as hq  # noqa: E402
from paper_2512_15742_b200 import synthetic  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--batches", default="1,2,4,8,16,64,256")
    ap.add_argument("--flush-with", choices=["torch", "memset", "write+read", "read"], default="torch",
                    help="L2 flush: a torch fill kernel (256 MiB write), cudaMemsetAsync, the write followed by a "
                         "256 MiB read (L2 left clean), or the read alone")
    args = ap.parse_args()
    cn = synthetic.synthetic_head()
    model = hq.build_model(cn)
    ws = hq.make_workspace(model, 256)
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    if args.flush_with == "memset":
        import ctypes
        import glob
        rt = ctypes.CDLL(sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so.12*"))[0])
        rt.cudaMemsetAsync.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p]

        class _F:
            def zero_(self):
                rt.cudaMemsetAsync(flush.data_ptr(), 0, flush.numel() * 4, torch.cuda.current_stream().cuda_stream)
        flusher = _F()
    elif args.flush_with in ("write+read", "read"):
        rd = torch.ones(64 << 20, dtype=torch.float32, device="cuda")
        acc = torch.zeros(1, dtype=torch.float32, device="cuda")
        wr = args.flush_with == "write+read"

        class _F2:
            def zero_(self):
                if wr:
                    flush.zero_()
                torch.sum(rd, dim=0, out=acc[0])
        flusher = _F2()
    else:
        flusher = flush
    s = torch.cuda.Stream()
    t_end = time.perf_counter() + 1.0
    while time.perf_counter() < t_end:
        flush.zero_()
    for B in [int(b) for b in args.batches.split(",")]:
        x = torch.from_numpy(synthetic.synthetic_inputs(B, 2048, seed=1)).cuda()
        y = torch.zeros(B * 20, dtype=torch.float64, device="cuda")
        for fl in (True, False):
            ev = []
            with torch.cuda.stream(s):
                for r in range(args.reps + 5):
                    if fl:
                        flusher.zero_()
                    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    a.record(s)
                    hq.forward_async(model, x, B, y, ws, stream=s.cuda_stream)
                    b.record(s)
                    if r >= 5:
                        ev.append((a, b))
            s.synchronize()
            ws.check()
            t = sorted(a.elapsed_time(b) * 1e3 for a, b in ev)
            print(f"B={B:4d} flush={fl!s:5} launches={ws.last_launches()} mean {statistics.mean(t):8.2f} median {statistics.median(t):8.2f} us "
                  f"p10 {t[len(t) // 10]:8.2f} p90 {t[9 * len(t) // 10]:8.2f}  -> {B / statistics.median(t) * 1e6:,.0f} samples/s",
                  flush=True)


if __name__ == "__main__":
    main()
