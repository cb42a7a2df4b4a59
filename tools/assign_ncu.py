"""One assign_indices call (200k shapes x 65,536 rows, G = 10) for an ncu capture of k_assign."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2512_15742_b200 as hq  # noqa: E402

rng = np.random.default_rng(0)
cb = hq.Codebook(k=65536, grid_size=10, entries=rng.standard_normal(65536 * 10))
hq.assign_indices(rng.standard_normal((200_000, 10)), cb)
