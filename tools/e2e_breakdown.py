"""Wall-clock breakdown of the host-buffer forward (the bench's e2e line): a
bare synchronize, the 16 KB H2D copy alone, the device-pointer forward alone
and the whole skan_forward(SKAN_PTR_HOST) call, each after an L2 flush and a
synchronize (the GPU idle when the call starts, as in the bench)."""
import os
import statistics
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15742_b200 as hq  # noqa: E402
from paper_2512_15742_b200 import _lib, synthetic  # noqa: E402


def main():
    model = hq.build_model(synthetic.synthetic_head())
    ws = hq.make_workspace(model, 1)
    x_np = synthetic.synthetic_inputs(1, 2048, seed=1)
    xh = torch.from_numpy(x_np.copy()).pin_memory()
    yh = torch.zeros(20, dtype=torch.float64).pin_memory()
    xd = torch.zeros(2048, dtype=torch.float64, device="cuda")
    yd = torch.zeros(20, dtype=torch.float64, device="cuda")
    flush = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    s = torch.cuda.Stream()
    L = _lib.lib()
    sp = s.cuda_stream

    def timed(fn, reps=300):
        t = []
        with torch.cuda.stream(s):
            for i in range(reps + 20):
                flush.zero_()
                s.synchronize()
                t0 = time.perf_counter()
                fn()
                t1 = time.perf_counter()
                if i >= 20:
                    t.append((t1 - t0) * 1e6)
        return statistics.mean(t), statistics.median(t)

    cases = {
        "sync only": lambda: s.synchronize(),
        "H2D 16 KB + sync": lambda: (xd.copy_(xh, non_blocking=True), s.synchronize()),
        "device forward + sync": lambda: (hq.forward_async(model, xd, 1, yd, ws, stream=sp), s.synchronize()),
        "host-buffer forward": lambda: _lib.check(L.skan_forward(model.handle, ws.handle, xh.data_ptr(), 2048, 1,
                                                                 yh.data_ptr(), 20, hq.MODE_FAST, _lib.SKAN_PTR_HOST,
                                                                 sp)),
    }
    for name, fn in cases.items():
        m, med = timed(fn)
        print(f"{name:24s} mean {m:7.2f} us  median {med:7.2f} us", flush=True)


if __name__ == "__main__":
    main()
