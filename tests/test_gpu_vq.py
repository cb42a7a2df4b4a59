"""GPU assign_indices (skan_assign_indices, skan_vq.cu) against the
reference's golden assignments and the oracle restatement (gsb.cpp:275-286):
bit-identical indices, ties to the lowest row, NaN/inf rows and shapes,
K split across CTAs (merge order), the generic-dim kernel, device pointers."""
import os

import numpy as np
import pytest

import oracle
import paper_2512_15742_b200 as hq
from paper_2512_15742_b200 import _lib
from paper_2512_15742_b200.errors import ShapeError

pytestmark = pytest.mark.gpu
GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "assign_indices_ref.npz"))


def cb(entries):
    e = np.ascontiguousarray(entries, dtype=np.float64)
    return hq.Codebook(k=e.shape[0], grid_size=e.shape[1], entries=e.reshape(-1))


def test_gpu_matches_reference_golden():
    assert np.array_equal(hq.assign_indices(GOLD["shapes"], cb(GOLD["entries"])), GOLD["idx"])
    dup = np.vstack([GOLD["entries"], GOLD["entries"]])
    assert np.array_equal(hq.assign_indices(GOLD["shapes"], cb(dup)), GOLD["idx_dup"])
    assert np.array_equal(hq.assign_indices(GOLD["shapes10"], cb(GOLD["entries10"])), GOLD["idx10"])


@pytest.mark.parametrize("n,k,dim", [(20000, 4096, 10), (3, 70000, 10), (1000, 33, 17), (500, 7, 1), (700, 300, 16)])
def test_gpu_matches_oracle(n, k, dim):
    rng = np.random.default_rng(n + k + dim)
    shapes = rng.standard_normal((n, dim))
    entries = rng.standard_normal((k, dim))
    entries[k - 1] = entries[k // 3]                      # a tie across K ranges
    shapes[0] = entries[k // 3]
    shapes[1, 0] = np.nan
    entries[k - 2, 0] = np.inf                            # an infinite row never wins
    want = oracle.port_assign_indices(shapes, entries)
    assert np.array_equal(hq.assign_indices(shapes, cb(entries)), want)
    assert want[0] == k // 3


def test_gpu_edge_cases_and_device_pointers():
    import torch
    rng = np.random.default_rng(1)
    shapes = rng.standard_normal((64, 10))
    assert np.array_equal(hq.assign_indices(shapes, hq.Codebook(k=0, grid_size=10, entries=np.zeros(0))),
                          np.zeros(64, np.uint32))
    assert hq.assign_indices(np.zeros((0, 10)), cb(rng.standard_normal((5, 10)))).size == 0
    with pytest.raises(ShapeError):
        hq.assign_indices(shapes, cb(rng.standard_normal((5, 9))))
    entries = rng.standard_normal((1000, 10))
    ds, de = torch.from_numpy(shapes).cuda(), torch.from_numpy(entries).cuda()
    out = torch.zeros(64, dtype=torch.int32, device="cuda")
    _lib.check(_lib.lib().skan_assign_indices(ds.data_ptr(), 64, 10, de.data_ptr(), 1000, out.data_ptr(), 1,
                                              torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert np.array_equal(out.cpu().numpy().astype(np.uint32), oracle.port_assign_indices(shapes, entries))


def test_gpu_head_scale_subset():
    """cfg2 scale, K = 65536 rows of G = 10: a 40k-shape batch on the GPU,
    a 300-shape subset re-checked by the oracle."""
    rng = np.random.default_rng(7)
    entries = rng.standard_normal((65536, 10))
    shapes = rng.standard_normal((40000, 10))
    got = hq.assign_indices(shapes, cb(entries))
    sub = rng.choice(40000, 300, replace=False)
    assert np.array_equal(got[sub], oracle.port_assign_indices(shapes[sub], entries))
