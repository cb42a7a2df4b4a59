"""torch.ops.share_kan: registration
and fake-tensor shapes on CPU; on the GPU, parity with the reference's
pli_lookup and with the oracle forward."""
import ctypes as C

import numpy as np
import pytest
import torch

import oracle
import paper_2512_15742_b200 as hq
import paper_2512_15742_b200.torch_ops as ops
from paper_2512_15742_b200 import synthetic

from helpers import assert_close


def test_ops_registered_with_fake_kernels():
    assert hasattr(torch.ops.share_kan, "pli_lookup") and hasattr(torch.ops.share_kan, "head_forward")
    from torch._subclasses.fake_tensor import FakeTensorMode
    with FakeTensorMode():
        x = torch.empty(7, 3, dtype=torch.float64)
        y = torch.ops.share_kan.pli_lookup(torch.empty(60, dtype=torch.float64), torch.empty(21, dtype=torch.int32),
                                           x, x, x, -1.0, 1.0, 10)
        assert y.shape == (7, 3) and y.dtype == torch.float64


def test_ops_refuse_cpu_tensors():
    with pytest.raises(hq.ContractError):
        torch.ops.share_kan.pli_lookup(torch.zeros(10, dtype=torch.float64), torch.zeros(1, dtype=torch.int32),
                                       torch.ones(1, dtype=torch.float64), torch.zeros(1, dtype=torch.float64),
                                       torch.zeros(1, dtype=torch.float64), -1.0, 1.0, 10)


@pytest.mark.gpu
def test_pli_lookup_op_matches_reference():
    rng = np.random.default_rng(3)
    k, G, lo, hi, n = 9, 10, -1.0, 1.0, 2000
    cb = rng.uniform(-1, 1, k * G)
    rows = rng.integers(0, k, n).astype(np.int32)
    g, b, x = rng.uniform(0, 2, n), rng.uniform(-1, 1, n), rng.uniform(-1.3, 1.3, n)
    dev = [torch.from_numpy(a).cuda() for a in (cb, rows, g, b, x)]
    y = torch.ops.share_kan.pli_lookup(*dev, lo, hi, G).cpu().numpy()
    for q in range(0, n, 13):
        want = C.c_double()
        assert oracle.ref().hqref_pli_lookup(cb.ctypes.data, k, G, int(rows[q]), g[q], b[q], x[q], lo, hi,
                                             C.byref(want)) == 0
        assert y[q] == want.value


@pytest.mark.gpu
def test_head_forward_op_matches_oracle():
    cn = synthetic.synthetic_head(dims=(256, 96, 12), k=1024, grid=10, int8=True, seed=21)
    model = hq.build_model(cn)
    h = ops.register_head(model, max_batch=64)
    x = synthetic.synthetic_inputs(5, 256, seed=3)
    for mode, name in ((1, "exact"), (0, "fast")):
        got = torch.ops.share_kan.head_forward(torch.from_numpy(x).cuda().view(5, 256), h, mode)
        ops.check_head(h)
        tables = [oracle.Tables.from_runtime(rl) for rl in synthetic.runtime_layers(cn)]
        want, scale = oracle.port_forward_l1(tables, x, 5)
        if name == "exact":  # bitwise the reference forward
            assert np.array_equal(got.cpu().numpy().reshape(-1), want)
        else:
            assert_close(got.cpu().numpy().reshape(-1), want, scale)
    ops.unregister_head(h)
    with pytest.raises(hq.ContractError):
        torch.ops.share_kan.head_forward(torch.zeros(1, 256, dtype=torch.float64, device="cuda"), h, 0)
