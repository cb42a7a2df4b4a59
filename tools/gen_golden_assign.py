"""Generate tests/golden/assign_indices_ref.npz with the reference itself
(oracle/_ref, the unmodified holoquant sources compiled in place): shapes,
a codebook from holoquant::kmeans_codebook and the indices
holoquant::assign_indices returns for it and for the codebook with every
row duplicated (ties).  Run here (needs /root/reference); the fixture is
committed so the GPU box never needs the reference.

    python tools/gen_golden_assign.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402


def main():
    oracle.build()
    rng = np.random.default_rng(6)
    shapes = rng.uniform(-1.0, 1.0, (300, 6))          # test_gsb.cpp:104-110 shape of the case
    entries = oracle.ref_kmeans_codebook(shapes, 12, seed=2)
    idx = oracle.ref_assign_indices(shapes, entries)
    dup = np.vstack([entries, entries])
    idx_dup = oracle.ref_assign_indices(shapes, dup)
    # G = 10 shapes normalised like normalize_grid (mean 0, population std 1)
    g = rng.standard_normal((500, 10))
    g = (g - g.mean(1, keepdims=True)) / g.std(1, keepdims=True)
    entries10 = oracle.ref_kmeans_codebook(g, 64, seed=3)
    idx10 = oracle.ref_assign_indices(g, entries10)
    out = os.path.join(ROOT, "tests", "golden", "assign_indices_ref.npz")
    np.savez_compressed(out, shapes=shapes, entries=entries, idx=idx, idx_dup=idx_dup, shapes10=g,
                        entries10=entries10, idx10=idx10)
    print("wrote", out, idx[:12], idx_dup.max(), idx10[:12])


if __name__ == "__main__":
    main()
