"""GPU parity at the BASELINE.json configs' own shapes, through
the C ABI, against the C oracle (pinned bitwise to the reference in
tests/test_oracle.py).  These are the shapes bench.py times.

Bars (as in tests/test_gpu_parity.py and DESIGN.md §2):
  * exact mode: bitwise equal to the reference forward
    (test_lutham.cpp:370-392);
  * fast mode: |y - y_ref| <= 1e-5 * max(|y_ref|, sum_i |term_ij|) per output,
    the scale computed by the oracle itself for EVERY output
    (oracle.port_forward_l1; acceptance.cpp:166-225 checks < 1e-5).
"""
import os

import numpy as np
import pytest

import oracle
import paper_2512_15742_b200 as hq
from paper_2512_15742_b200 import synthetic

from helpers import TOL, assert_close

pytestmark = pytest.mark.gpu

THREADS = max(1, min(16, os.cpu_count() or 1))


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _tables(cn):
    return [oracle.Tables.from_runtime(rl) for rl in synthetic.runtime_layers(cn)]


@pytest.fixture(scope="module")
def cfg2():
    cn = synthetic.synthetic_head()
    return cn, _tables(cn), hq.build_model(cn)


def test_cfg3_batch256_every_output_within_bound(torch_cuda, cfg2):
    """configs[2]: the cfg2 head at batch 256 (tensor-core layer GEMM), the
    per-output L1 bound on all 256 x 20 outputs, and bitwise reproducible."""
    _, tables, model = cfg2
    x = synthetic.synthetic_inputs(256, 2048, seed=77)
    want, scale = oracle.port_forward_l1(tables, x, 256, threads=THREADS)
    ws = hq.make_workspace(model, max_batch=256)
    got = np.zeros(256 * 20)
    hq.compressed_forward(model, x, 256, got, ws, mode="fast")
    assert ws.last_launches() > 1  # the multi-kernel GEMM route, not the batch-1 kernel
    assert_close(got, want, scale)
    again = np.zeros_like(got)
    hq.compressed_forward(model, x, 256, again, ws, mode="fast")
    assert np.array_equal(_bits(got), _bits(again))


def test_cfg2_batch1_many_inputs_within_bound(torch_cuda, cfg2):
    """configs[1]: batch 1 on the persistent kernel, 24 different feature
    vectors (each its own bracket histogram)."""
    _, tables, model = cfg2
    ws = hq.make_workspace(model, max_batch=1)
    for seed in range(24):
        x = synthetic.synthetic_inputs(1, 2048, seed=1000 + seed)
        want, scale = oracle.port_forward_l1(tables, x, 1)
        got = np.zeros(20)
        hq.compressed_forward(model, x, 1, got, ws, mode="fast")
        assert ws.last_launches() == 1
        assert_close(got, want, scale)


@pytest.fixture(scope="module")
def cfg4():
    rls = synthetic.dense_runtime_head()
    tables = [oracle.Tables.from_runtime(rl) for rl in rls]
    model = hq.upload(rls, device=0)
    return tables, model


def test_cfg4_dense_batch64_within_bound(torch_cuda, cfg4):
    """configs[3]: dense {2048,13664,20} f32 grids (1.13 GB) at batch 64."""
    tables, model = cfg4
    x = synthetic.synthetic_inputs(64, 2048, seed=6)
    want, scale = oracle.port_forward_l1(tables, x, 64, threads=THREADS)
    ws = hq.make_workspace(model, max_batch=64)
    got = np.zeros(64 * 20)
    hq.compressed_forward(model, x, 64, got, ws, mode="fast")
    assert_close(got, want, scale)


def test_cfg4_dense_exact_bitwise(torch_cuda, cfg4):
    """configs[3] in exact mode: bitwise equal to the reference forward."""
    tables, model = cfg4
    x = synthetic.synthetic_inputs(3, 2048, seed=16)
    want, ops = oracle.port_forward(tables, x, 3, threads=3)
    ws = hq.make_workspace(model, max_batch=4)
    got = np.zeros(3 * 20)
    hq.compressed_forward(model, x, 3, got, ws, mode="exact")
    assert np.array_equal(_bits(got), _bits(want))
    assert ws.interp_ops == ops


def _cfg5_heads(n):
    cns = [synthetic.synthetic_head(seed=2026 + 7 * h) if h else synthetic.synthetic_head() for h in range(n)]
    return cns, [_tables(cn) for cn in cns], [hq.build_model(cn) for cn in cns]


@pytest.fixture(scope="module")
def cfg5():
    return _cfg5_heads(4)


def test_cfg5_multi_head_batch256_against_oracle(torch_cuda, cfg5):
    """configs[4] per GPU: 4 cfg2 heads (the 8-GPU share of 32) on ONE shared
    feature batch of 256 through skan_forward_multi, each head's outputs
    against the oracle (not against the repo's single-head path)."""
    torch = torch_cuda
    _, tabs, models = cfg5
    x = synthetic.synthetic_inputs(256, 2048, seed=777)
    wss = [hq.make_workspace(m, 256) for m in models]
    xd = torch.from_numpy(x).cuda()
    ys = [torch.zeros(256 * 20, dtype=torch.float64, device="cuda") for _ in models]
    hq.forward_multi(models, wss, xd, 256, ys, mode="fast")
    torch.cuda.synchronize()
    for ws in wss:
        ws.check()
    for t, y in zip(tabs, ys):
        want, scale = oracle.port_forward_l1(t, x, 256, threads=THREADS)
        assert_close(y.cpu().numpy(), want, scale)


def test_cfg5_multi_head_exact_bitwise(torch_cuda, cfg5):
    """forward_multi in exact mode: every head bitwise equal to the oracle."""
    torch = torch_cuda
    _, tabs, models = cfg5
    x = synthetic.synthetic_inputs(4, 2048, seed=778)
    wss = [hq.make_workspace(m, 4) for m in models]
    ys = [torch.zeros(4 * 20, dtype=torch.float64, device="cuda") for _ in models]
    hq.forward_multi(models, wss, torch.from_numpy(x).cuda(), 4, ys, mode="exact")
    torch.cuda.synchronize()
    for t, y in zip(tabs, ys):
        want, _ = oracle.port_forward(t, x, 4, threads=4)
        assert np.array_equal(_bits(y.cpu().numpy()), _bits(want))


def test_many_heads_batch1_multi(torch_cuda):
    """Many small heads (north_star (5): dozens of hot-swappable heads) at
    batch 1 on one stream set, each against the oracle; then one head is
    swapped while the others keep serving."""
    torch = torch_cuda
    dims = (256, 96, 12)
    cns = [synthetic.synthetic_head(dims=dims, k=1024, grid=10, int8=True, seed=300 + h) for h in range(12)]
    tabs = [_tables(cn) for cn in cns]
    models = [hq.build_model(cn) for cn in cns]
    wss = [hq.make_workspace(m, 8) for m in models]
    x = synthetic.synthetic_inputs(8, 256, seed=5)
    xd = torch.from_numpy(x).cuda()
    for mode in ("exact", "fast"):
        ys = [torch.zeros(8 * 12, dtype=torch.float64, device="cuda") for _ in models]
        hq.forward_multi(models, wss, xd, 8, ys, mode=mode)
        torch.cuda.synchronize()
        for t, y in zip(tabs, ys):
            if mode == "exact":
                want, _ = oracle.port_forward(t, x, 8)
                assert np.array_equal(_bits(y.cpu().numpy()), _bits(want))
            else:
                want, scale = oracle.port_forward_l1(t, x, 8)
                assert_close(y.cpu().numpy(), want, scale)
    # hot swap of head 3 to new tables; every head still matches its oracle
    new = synthetic.synthetic_head(dims=dims, k=1024, grid=10, int8=True, seed=999)
    hq.swap_model(models[3], new)
    tabs[3] = _tables(new)
    ys = [torch.zeros(8 * 12, dtype=torch.float64, device="cuda") for _ in models]
    hq.forward_multi(models, wss, xd, 8, ys, mode="exact")
    torch.cuda.synchronize()
    for t, y in zip(tabs, ys):
        want, _ = oracle.port_forward(t, x, 8)
        assert np.array_equal(_bits(y.cpu().numpy()), _bits(want))
