"""Dense-layer GEMM paths (persistent k_dense_persist vs the split GEMM) against
the oracle on several dense heads at batch <= 64: worst L1-scaled error per
head (debugging aid for the fast dense path).

    python tools/dense_check.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: the checker)
import paper_2512_15742_b200 as hq  # noqa: E402
from paper_2512_15742_b200 import synthetic  # noqa: E402


def main():
    for dims, B in [((256, 1024), 64), ((512, 512, 20), 64), ((256, 1024, 20), 64), ((2048, 1408), 64),
                    ((1024, 4096), 32), ((300, 700, 20), 17), ((2048, 13664), 64)]:
        rls = synthetic.dense_runtime_head(dims=dims)
        tables = [oracle.Tables.from_runtime(rl) for rl in rls]
        model = hq.upload(rls, device=0)
        x = synthetic.synthetic_inputs(B, dims[0], seed=6)
        want, scale = oracle.port_forward_l1(tables, x, B, threads=16)
        ws = hq.make_workspace(model, max_batch=B)
        got = np.zeros(B * dims[-1])
        hq.compressed_forward(model, x, B, got, ws, mode="fast")
        err = np.abs(got - want) / np.maximum(scale, 1e-300)
        print(f"dims {dims} B={B}: worst {err.max():.3e}, bad {(err > 1e-5).sum()} / {err.size}", flush=True)


if __name__ == "__main__":
    main()
