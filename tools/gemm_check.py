"""Compressed-layer tensor-core GEMM against the oracle on single int8 layers
at several batches (debugging aid for the layer GEMM variants)."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402  (test infrastructure: the checker)
import paper_2512_15742_b200 as hq  # noqa: E402
from paper_2512_15742_b200 import synthetic  # noqa: E402
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
from helpers import l1_scale  # noqa: E402


def main():
    for dims, k, G, B in [((256, 128), 256, 10, 64), ((256, 128), 256, 10, 200), ((64, 128), 16, 10, 64),
                          ((256, 128), 256, 8, 64), ((2048, 1408, 20), 65536, 10, 256)]:
        cn = synthetic.synthetic_head(dims=dims, k=k, grid=G, int8=True, seed=5)
        tables = [oracle.Tables.from_runtime(rl) for rl in synthetic.runtime_layers(cn)]
        model = hq.build_model(cn)
        x = synthetic.synthetic_inputs(B, dims[0], seed=3, grid=G)
        want, _ = oracle.port_forward(tables, x, B)
        ws = hq.make_workspace(model, max_batch=B)
        got = np.zeros(B * dims[-1])
        hq.compressed_forward(model, x, B, got, ws, mode="fast")
        sc = l1_scale(tables, x, B)
        err = np.abs(got - want) / np.maximum(sc, 1e-300)
        o = dims[-1]
        e2 = err.reshape(B, o)
        print(f"dims {dims} K={k} G={G} B={B}: worst {err.max():.3e} bad {(err > 1e-5).sum()}/{err.size}; "
              f"ratio got/want median {np.median(got / np.where(want == 0, 1, want)):.4f}; "
              f"worst by column {np.argsort(-e2.max(0))[:6].tolist()} by sample {np.argsort(-e2.max(1))[:6].tolist()}",
              flush=True)


if __name__ == "__main__":
    main()
