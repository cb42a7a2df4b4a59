"""GSB-VQ nearest-row assignment (gsb.cpp:275-286), CPU side: the oracle
restatement pinned to the reference (golden fixture made by
tools/gen_golden_assign.py with the compiled reference, and live
comparisons when oracle/_ref is present), including ties and NaNs."""
import os

import numpy as np
import pytest

import oracle

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "assign_indices_ref.npz"))
needs_ref = pytest.mark.skipif(not oracle.have_ref(), reason="reference build oracle/_ref unavailable")


def test_oracle_matches_reference_golden_assignments():
    assert np.array_equal(oracle.port_assign_indices(GOLD["shapes"], GOLD["entries"]), GOLD["idx"])
    dup = np.vstack([GOLD["entries"], GOLD["entries"]])
    assert np.array_equal(oracle.port_assign_indices(GOLD["shapes"], dup), GOLD["idx_dup"])
    assert GOLD["idx_dup"].max() < GOLD["entries"].shape[0]  # ties keep the lowest row
    assert np.array_equal(oracle.port_assign_indices(GOLD["shapes10"], GOLD["entries10"]), GOLD["idx10"])


@needs_ref
@pytest.mark.parametrize("dim,k,seed", [(2, 5, 1), (10, 64, 2), (17, 9, 3), (1, 4, 4)])
def test_oracle_matches_reference_live(dim, k, seed):
    rng = np.random.default_rng(seed)
    shapes = rng.standard_normal((400, dim))
    entries = rng.standard_normal((k, dim))
    entries[k // 2] = entries[0]                    # an exact tie
    shapes[:5] = entries[[0, 1, 2, 0, k - 1]]       # zero distances
    shapes[7, 0] = np.nan                           # NaN distance never wins
    entries2 = entries.copy()
    entries2[1, -1] = np.inf
    for e in (entries, entries2):
        assert np.array_equal(oracle.port_assign_indices(shapes, e), oracle.ref_assign_indices(shapes, e))
