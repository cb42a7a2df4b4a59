"""Find where tcgen05.mma (cta_group::1, M = 64) puts accumulator rows in TMEM:
for each row r of A*B, the TMEM lanes whose 32x32b readback matches it."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

from paper_2512_15742_b200 import _lib

rng = np.random.default_rng(0)
n, k = 32, 16
a = rng.standard_normal((64, k)).astype(np.float32)
b = rng.standard_normal((k, n)).astype(np.float32)
want = a.astype(np.float64) @ b.astype(np.float64)
da, db = torch.from_numpy(a).cuda(), torch.from_numpy(b).cuda()
dd = torch.zeros((128, n), dtype=torch.float32, device="cuda")
_lib.check(_lib.lib().skan_debug_gemm_tf32(da.data_ptr(), db.data_ptr(), dd.data_ptr(), n, k, 103,
                                           torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
raw = dd.cpu().numpy().astype(np.float64)
for r in range(64):
    hits = [lane for lane in range(128) if np.allclose(raw[lane], want[r], rtol=1e-5, atol=1e-5)]
    cols = None
    if not hits:  # maybe columns are split across lanes
        for lane in range(128):
            m = np.isclose(raw[lane], want[r][0], rtol=1e-5, atol=1e-5)
            if m.any():
                cols = (lane, int(np.argmax(m)))
                break
    print(r, hits, cols)
