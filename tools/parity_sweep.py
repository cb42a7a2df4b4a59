"""Randomised parity sweep over formats, grid sizes and batch sizes (fast mode
within tolerance, exact mode bitwise) against the oracle.  Run on a GPU box:
    python tools/parity_sweep.py
"""
import sys, numpy as np
import os
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, 'tests'))
import oracle, paper_2512_15742_b200 as hq
from paper_2512_15742_b200 import synthetic
from helpers import assert_close, l1_scale
seeds = [int(a) for a in sys.argv[1:]] or [2027]
cases = [
    ("int8 G10 K4096 3-layer", [oracle.Tables.from_runtime(r) for r in synthetic.runtime_layers(synthetic.synthetic_head(dims=(300, 257, 131, 7), k=4096, grid=10, int8=True, seed=11))]),
    ("int8 G7 (odd) K300", [oracle.Tables.from_runtime(r) for r in synthetic.runtime_layers(synthetic.synthetic_head(dims=(129, 200, 17), k=300, grid=7, int8=True, seed=12))]),
    ("int8 G16 K70000 wide", [oracle.Tables.from_runtime(r) for r in synthetic.runtime_layers(synthetic.synthetic_head(dims=(65, 140, 9), k=70000, grid=16, int8=True, seed=13))]),
    ("f32 G6 K1", oracle.ref_build(synthetic.CompressedNetwork([synthetic.crafted_layer(77, 133, 6, 1, 4, int8=False)])).tables()),
    ("f32 G9 K500", oracle.ref_build(synthetic.CompressedNetwork([synthetic.crafted_layer(50, 300, 9, 500, 5, int8=False)])).tables()),
    ("dense G5 odd", oracle.ref_random([33, 160, 19], 5, 0.4, 6, 0, False).tables()),
    ("dense G10", oracle.ref_random([40, 300, 21], 10, 0.4, 7, 0, False).tables()),
    ("dense G13", oracle.ref_random([20, 129, 16], 13, 0.4, 8, 0, False).tables()),
]
bad = 0
for seed in seeds:
  rng = np.random.default_rng(seed)
  for name, tables in cases:
      from test_gpu_parity import _upload
      model = _upload(tables)
      ws = hq.make_workspace(model, 256)
      for B in (1, 2, 3, 4, 5, 17, 63, 64, 65, 127, 129, 200):
          x = rng.uniform(-1.5, 1.5, B * tables[0].in_dim)
          want, _ = oracle.port_forward(tables, x, B)
          got = np.zeros(B * tables[-1].out_dim)
          hq.compressed_forward(model, x, B, got, ws, mode="fast")
          try:
              assert_close(got, want, l1_scale(tables, x, B))
          except AssertionError as e:
              bad += 1; print("FAST FAIL", name, B, str(e)[:200])
          if B in (1, 3, 64, 129):
              ex = np.zeros_like(got)
              hq.compressed_forward(model, x, B, ex, ws, mode="exact")
              if not np.array_equal(ex.view(np.uint64), want.view(np.uint64)):
                  bad += 1; print("EXACT FAIL", name, B)
      print("done", seed, name, flush=True)
print("failures", bad)
