"""GPU assign_indices at scale: 2M shapes x 65,536 codebook
rows x G = 10, host-to-host wall time (the public call, buffers on the host)
and the distance work rate: shape-row pairs per second and the FP64 issue it
implies (3 G DADD/DMUL per pair)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15742_b200 as hq  # noqa: E402


def main():
    rng = np.random.default_rng(0)
    n, k, G = 2_000_000, 65_536, 10
    shapes = rng.standard_normal((n, G))
    cb = hq.Codebook(k=k, grid_size=G, entries=rng.standard_normal(k * G))
    hq.assign_indices(shapes[:1000], cb)  # warm up (module load, first launch)
    for rep in range(3):
        t0 = time.perf_counter()
        idx = hq.assign_indices(shapes, cb)
        t1 = time.perf_counter()
        pairs = n * k
        print(f"rep {rep}: {n:,} shapes x {k:,} rows, G={G}: {(t1 - t0) * 1e3:.1f} ms host-to-host, "
              f"{pairs / (t1 - t0) / 1e9:.0f} G pairs/s, {3 * G * pairs / (t1 - t0) / 1e12:.1f} TFLOP/s FP64",
              flush=True)
    # spot check against numpy on a sample
    sel = rng.choice(n, 200, replace=False)
    d = ((shapes[sel, None, :] - cb.entries.reshape(k, G)[None]) ** 2).sum(-1)
    print("sample agreement with numpy argmin:", float((d.argmin(1) == idx[sel]).mean()))


if __name__ == "__main__":
    main()
