"""GPU parity: the CUDA path through the C ABI against the oracle.

Bars (stated here and in DESIGN.md):
  * knot selection, index unpack, gain/bias/codebook decode: bit-exact;
  * SKAN_MODE_EXACT forward: bitwise equal to holoquant::compressed_forward;
  * SKAN_MODE_FAST forward: |y - y_ref| <= 1e-5 * max(|y_ref|, sum_i |term_ij|)
    per output (tests/helpers.py), and bitwise reproducible run to run.
"""
import ctypes as C

import numpy as np
import pytest

import oracle
import paper_2512_15742_b200 as hq
from paper_2512_15742_b200 import synthetic

from helpers import TOL, assert_close, l1_scale

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch_cuda():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def _bits(a):
    return np.ascontiguousarray(a, np.float64).view(np.uint64)


def _upload(tables):
    return hq.upload([t.to_runtime() for t in tables], device=0)


def _gpu_forward(model, x, batch, mode, max_batch=64):
    ws = hq.make_workspace(model, max_batch=max_batch)
    y = np.zeros(batch * model.output_dim())
    hq.compressed_forward(model, x, batch, y, ws, mode=mode)
    return y, ws


# ---------------------------------------------------------------------------
# knot selection (kan.cpp:28-58): bit-exact on >= 1e7 inputs incl. nodes

def test_locate_bitexact_1e7(torch_cuda):
    torch = torch_cuda
    rng = np.random.default_rng(7)
    total = 0
    for G, (lo, hi) in [(10, (-1.0, 1.0)), (5, (-1.0, 1.0)), (2, (0.3, 0.7)), (128, (-2.5, 3.75)),
                        (37, (-0.1, 1e-3)), (1000, (-7.0, 11.0))]:
        n = 2_000_000
        x = rng.uniform(lo - 0.5 * (hi - lo), hi + 0.5 * (hi - lo), n)
        nodes = np.array([synthetic.node_position(lo, hi, G, i) for i in range(G)])
        extra = np.concatenate([nodes, np.nextafter(nodes, -np.inf), np.nextafter(nodes, np.inf),
                                [lo, hi, -0.0, 0.0, 1e300, -1e300]])
        x = np.concatenate([x, np.tile(extra, 50)])
        idx, t, cl = hq.locate(torch.from_numpy(x).cuda(), lo, hi, G)
        wi, wt, wc, bad = oracle.port_locate_many(lo, hi, G, x)
        assert bad == 0
        assert np.array_equal(idx.cpu().numpy(), wi)
        assert np.array_equal(_bits(t.cpu().numpy()), _bits(wt))
        assert np.array_equal(cl.cpu().numpy(), wc)
        total += x.size
    assert total >= 10_000_000


def test_locate_nonfinite_raises(torch_cuda):
    torch = torch_cuda
    x = torch.tensor([0.1, float("nan"), 0.3], dtype=torch.float64, device="cuda")
    with pytest.raises(hq.ValueError):
        hq.locate(x, -1.0, 1.0, 5)
    x = torch.tensor([float("inf")], dtype=torch.float64, device="cuda")
    with pytest.raises(hq.ValueError):
        hq.locate(x, -1.0, 1.0, 5)


# ---------------------------------------------------------------------------
# forward, exact mode == reference bitwise

def _fixture_models():
    """Reference-test fixtures built by the reference itself (oracle/_ref)."""
    ms = [("random_compressed f32", oracle.ref_random([3, 5, 2], 6, 0.4, 16, 5, False)),
          ("random_compressed int8", oracle.ref_random([3, 5, 2], 6, 0.4, 16, 5, True)),
          ("dense random_net", oracle.ref_random([2, 4, 1], 7, 0.4, 2, 0, False)),
          ("zero-alloc fixture int8", oracle.ref_random([4, 24, 2], 12, 0.4, 95, 32, True)),
          ("iso G=128", oracle.ref_random([2, 16, 1], 128, 0.4, 90, 16, False))]
    for name, (i, o, G, k, s, q) in [("crafted K=65536 f32", (2, 3, 4, 65536, 5, False)),
                                     ("crafted K=1", (2, 2, 3, 1, 6, False)),
                                     ("crafted K=1 int8", (3, 2, 3, 1, 6, True)),
                                     ("crafted K=65536 int8", (5, 40, 7, 65536, 5, True)),
                                     ("crafted K=70000 int8 (u32 idx)", (7, 9, 5, 70000, 8, True)),
                                     ("crafted K=70000 f32 (u32 idx)", (7, 9, 5, 70000, 8, False)),
                                     ("cfg1 256x256 K=256 int8", (256, 256, 10, 256, 1, True)),
                                     ("cfg1 256x256 K=256 f32", (256, 256, 10, 256, 1, False))]:
        ms.append((name, oracle.ref_build(synthetic.CompressedNetwork([synthetic.crafted_layer(i, o, G, k, s,
                                                                                                int8=q)]))))
    return ms


@pytest.mark.parametrize("batch", [1, 3, 17, 64])
def test_exact_mode_bitwise_equals_reference(torch_cuda, batch):
    rng = np.random.default_rng(100 + batch)
    for name, m in _fixture_models():
        tables = m.tables()
        x = rng.uniform(-1.5, 1.5, batch * tables[0].in_dim)
        want, _ = m.forward(x, batch)
        got, _ = _gpu_forward(_upload(tables), x, batch, "exact")
        assert np.array_equal(_bits(got), _bits(want)), name


def test_exact_mode_build_model_path(torch_cuda):
    """build_model(CompressedNetwork) on the device == reference build_model + forward."""
    for q in (False, True):
        cn = synthetic.synthetic_head(dims=(40, 33, 6), k=300, grid=7, int8=q, seed=21)
        x = synthetic.synthetic_inputs(9, 40, seed=2, grid=7)
        want, _ = oracle.ref_build(cn).forward(x, 9)
        got, _ = _gpu_forward(hq.build_model(cn), x, 9, "exact")
        assert np.array_equal(_bits(got), _bits(want))


def test_exact_mode_mixed_dense_and_compressed(torch_cuda):
    dense = oracle.ref_random([6, 5], 8, 0.4, 3, 0, False).tables()[0]
    comp = oracle.ref_build(synthetic.CompressedNetwork([synthetic.crafted_layer(5, 4, 8, 12, 4, int8=True)])).tables()[0]
    tables = [dense, comp]
    x = np.random.default_rng(0).uniform(-1.5, 1.5, 11 * 6)
    want, _ = oracle.port_forward(tables, x, 11)
    got, _ = _gpu_forward(_upload(tables), x, 11, "exact")
    assert np.array_equal(_bits(got), _bits(want))


def test_exact_mode_headline_head_bitwise(torch_cuda):
    """cfg2 head {2048,1408,20}, K=65536, G=10, int8 — bitwise at batch 2."""
    cn = synthetic.synthetic_head()
    tables = [oracle.Tables.from_runtime(rl) for rl in synthetic.runtime_layers(cn)]
    x = synthetic.synthetic_inputs(2, 2048, seed=9)
    want, ops = oracle.port_forward(tables, x, 2)
    got, ws = _gpu_forward(hq.build_model(cn), x, 2, "exact")
    assert np.array_equal(_bits(got), _bits(want))
    assert ws.interp_ops == ops == 2 * 2_911_744


@pytest.mark.parametrize("batch", [1, 12, 130])
def test_exact_mode_headline_head_split_and_one_pass(torch_cuda, batch):
    """Exact mode's kernels: batch 1 the bracket-ordered terms read from the
    pair planes (k_exact_terms_planes), batch 12 the two-pass split (terms, then
    in-order sums) with layer 0 in two input blocks (12 * 1408 * 2048 doubles
    exceed the 256 MB term buffer), batch 130 the one-pass kernel
    (> kExactSplitMaxBatch).  Both bitwise equal to the reference."""
    cn = synthetic.synthetic_head()
    tables = [oracle.Tables.from_runtime(rl) for rl in synthetic.runtime_layers(cn)]
    x = synthetic.synthetic_inputs(batch, 2048, seed=batch)
    want, _ = oracle.port_forward(tables, x, batch)
    got, _ = _gpu_forward(hq.build_model(cn), x, batch, "exact")
    assert np.array_equal(_bits(got), _bits(want))


# ---------------------------------------------------------------------------
# forward, fast mode within tolerance

@pytest.mark.parametrize("batch", [1, 5, 64])
def test_fast_mode_within_tolerance(torch_cuda, batch):
    rng = np.random.default_rng(200 + batch)
    for name, m in _fixture_models():
        tables = m.tables()
        x = rng.uniform(-1.5, 1.5, batch * tables[0].in_dim)
        want, _ = m.forward(x, batch)
        got, _ = _gpu_forward(_upload(tables), x, batch, "fast")
        assert_close(got, want, l1_scale(tables, x, batch))


def test_fast_mode_headline_head(torch_cuda):
    cn = synthetic.synthetic_head()
    tables = [oracle.Tables.from_runtime(rl) for rl in synthetic.runtime_layers(cn)]
    model = hq.build_model(cn)
    # 1-2: per-sample persistent launches; 3-32: tensor-core GEMMs, layer 1
    # reducing layer 0's split partials in its prologue; 33+: separate reduction
    for batch in (1, 2, 3, 4, 17, 32, 33, 64):
        x = synthetic.synthetic_inputs(batch, 2048, seed=30 + batch)
        want, _ = oracle.port_forward(tables, x, batch)
        got, ws = _gpu_forward(model, x, batch, "fast")
        assert_close(got, want, l1_scale(tables, x, batch))
        if batch <= 2:
            assert ws.last_launches() == batch


def test_fused_small_batch_reduction_is_bitwise_the_separate_one(torch_cuda):
    """At batch <= 32 layer 1's GEMM reduces layer 0's split partials in its
    prologue; the separate k_split_reduce launch sums the same partials in
    the same f64 order, so both routes give bitwise-equal outputs.  (A last
    layer of 33-128 outputs: narrower int8 layers take k_dense_narrow.)"""
    from paper_2512_15742_b200 import _lib
    cn = synthetic.synthetic_head(dims=(1024, 512, 64), k=4096, seed=9)
    model = hq.build_model(cn)
    for batch in (3, 17, 32):
        x = synthetic.synthetic_inputs(batch, 1024, seed=40 + batch)
        prev = _lib.lib().skan_debug_set_fuse_reduce(1)
        try:
            fused, ws = _gpu_forward(model, x, batch, "fast")
            n_fused = ws.last_launches()
            _lib.lib().skan_debug_set_fuse_reduce(0)
            sep, ws = _gpu_forward(model, x, batch, "fast")
            n_sep = ws.last_launches()
        finally:
            _lib.lib().skan_debug_set_fuse_reduce(prev)
        assert n_sep == n_fused + 1
        assert np.array_equal(_bits(fused), _bits(sep))


def test_fast_mode_bitwise_reproducible(torch_cuda):
    cn = synthetic.synthetic_head(dims=(512, 300, 20), k=4096, grid=10, int8=True, seed=5)
    model = hq.build_model(cn)
    x = synthetic.synthetic_inputs(33, 512, seed=6)
    a, _ = _gpu_forward(model, x, 33, "fast")
    b, _ = _gpu_forward(model, x, 33, "fast")
    c, _ = _gpu_forward(model, x, 33, "fast")
    assert np.array_equal(_bits(a), _bits(b)) and np.array_equal(_bits(a), _bits(c))


def test_fast_mode_batch1_pair_planes(torch_cuda):
    """Batch 1 routes big int8 layers through the shared-memory pair-plane
    kernel (k_fwd_planes) and the next layer's consumer-side reduction:
    within tolerance, bitwise reproducible, several heads and seeds.  All
    heads are created before any of them runs: a head planned later with a
    smaller shared-memory footprint must not break an earlier head's launch."""
    heads = []
    for dims, k, G, seed in [((2048, 1408, 20), 65536, 10, 3), ((512, 512, 8), 4096, 10, 1),
                             ((1024, 700, 12), 8192, 6, 2), ((640, 1536, 24, 3), 1000, 16, 4),
                             ((2048, 128, 20), 4096, 10, 7)]:
        cn = synthetic.synthetic_head(dims=dims, k=k, grid=G, int8=True, seed=seed)
        tables = [oracle.Tables.from_runtime(rl) for rl in synthetic.runtime_layers(cn)]
        heads.append((dims, G, seed, tables, hq.build_model(cn)))
    for dims, G, seed, tables, model in heads:
        for xs in (1, 2):
            x = synthetic.synthetic_inputs(1, dims[0], seed=10 * seed + xs, grid=G)
            want, _ = oracle.port_forward(tables, x, 1)
            a, _ = _gpu_forward(model, x, 1, "fast")
            b, _ = _gpu_forward(model, x, 1, "fast")
            assert np.array_equal(_bits(a), _bits(b))
            assert_close(a, want, l1_scale(tables, x, 1))


def test_batch_larger_than_workspace_is_chunked(torch_cuda):
    cn = synthetic.synthetic_head(dims=(64, 48, 5), k=256, grid=10, int8=True, seed=3)
    model = hq.build_model(cn)
    x = synthetic.synthetic_inputs(50, 64, seed=8)
    a, _ = _gpu_forward(model, x, 50, "exact", max_batch=7)
    b, _ = _gpu_forward(model, x, 50, "exact", max_batch=64)
    assert np.array_equal(_bits(a), _bits(b))


# ---------------------------------------------------------------------------
# SKAN v1 files -> device heads

def test_skan_files_load_and_forward_bitwise(torch_cuda):
    rng = np.random.default_rng(42)
    for name, m in _fixture_models():
        data = m.serialize()
        model = hq.deserialize(data)
        tables = m.tables()
        x = rng.uniform(-1.5, 1.5, 5 * tables[0].in_dim)
        want, _ = m.forward(x, 5)
        got, _ = _gpu_forward(model, x, 5, "exact")
        assert np.array_equal(_bits(got), _bits(want)), name
        assert [h.k for h in model.layers] == [t.k for t in tables]


def test_load_model_from_disk(torch_cuda, tmp_path):
    m = oracle.ref_random([3, 5, 2], 6, 0.4, 21, 4, True)
    p = tmp_path / "head.skan"
    p.write_bytes(m.serialize())
    model = hq.load_model(str(p))
    x = np.linspace(-1.2, 1.2, 3 * 4)
    want, _ = m.forward(x, 4)
    got, _ = _gpu_forward(model, x, 4, "exact")
    assert np.array_equal(got, want)


# ---------------------------------------------------------------------------
# API contract (lutham.cpp:819-850, test_lutham.cpp:394-424)

def test_interp_ops_counts_edges_times_batch_independent_of_G(torch_cuda):
    for G in (5, 64):
        m = oracle.ref_random([2, 4, 1], G, 0.4, 18, 3, False)
        model = _upload(m.tables())
        ws = hq.make_workspace(model)
        x = np.full(7 * 2, 0.25)
        y = np.zeros(7)
        hq.compressed_forward(model, x, 7, y, ws)
        assert ws.interp_ops == 7 * (2 * 4 + 4 * 1)
        hq.compressed_forward(model, x, 7, y, ws, mode="exact")
        assert ws.interp_ops == 2 * 7 * 12


def test_forward_validates_spans_and_workspace(torch_cuda):
    big = _upload(oracle.ref_random([2, 9, 1], 4, 0.4, 19, 0, False).tables())
    small = _upload(oracle.ref_random([2, 3, 1], 4, 0.4, 19, 0, False).tables())
    ws = hq.make_workspace(small)
    assert ws.width() == 3
    x, y = np.zeros(2), np.zeros(1)
    with pytest.raises(hq.ContractError):
        hq.compressed_forward(big, x, 1, y, ws)
    ok = hq.make_workspace(big)
    assert ok.width() == 9
    with pytest.raises(hq.ShapeError):
        hq.compressed_forward(big, np.zeros(1), 1, y, ok)
    with pytest.raises(hq.ShapeError):
        hq.compressed_forward(big, x, 1, np.zeros(0), ok)
    with pytest.raises(hq.ShapeError):
        hq.compressed_forward(big, x, -1, y, ok)
    hq.compressed_forward(big, np.zeros(0), 0, np.zeros(0), ok)  # batch 0: no work
    assert ok.interp_ops == 0


def test_nonfinite_input_raises_value_error(torch_cuda):
    torch = torch_cuda
    model = _upload(oracle.ref_random([3, 5, 2], 6, 0.4, 16, 5, True).tables())
    ws = hq.make_workspace(model)
    for bad in (float("nan"), float("inf"), -float("inf")):
        x = np.array([0.1, bad, 0.2])
        for mode in ("fast", "exact"):
            with pytest.raises(hq.ValueError):
                hq.compressed_forward(model, x, 1, np.zeros(2), ws, mode=mode)
    xd = torch.tensor([0.1, float("nan"), 0.2], dtype=torch.float64, device="cuda")
    yd = torch.zeros(2, dtype=torch.float64, device="cuda")
    with pytest.raises(hq.ValueError):
        hq.compressed_forward(model, xd, 1, yd, ws)
    # the workspace stays usable afterwards
    y = np.zeros(2)
    hq.compressed_forward(model, np.array([0.1, 0.2, 0.3]), 1, y, ws)


def test_build_model_rejects_inconsistent_layers(torch_cuda):
    """test_lutham.cpp:277-286."""
    cl = synthetic.crafted_layer(2, 2, 3, 4, 11)
    cl.indices = cl.indices.copy(); cl.indices[0] = 4
    with pytest.raises(hq.ContractError):
        hq.build_model(synthetic.CompressedNetwork([cl]))
    cl = synthetic.crafted_layer(2, 2, 3, 4, 11)
    cl.gains = cl.gains[:-1]
    with pytest.raises(hq.ContractError):
        hq.build_model(synthetic.CompressedNetwork([cl]))
    cl = synthetic.crafted_layer(2, 2, 3, 4, 11)
    cl.gains = cl.gains.copy(); cl.gains[0] = -0.5
    with pytest.raises(hq.ContractError):
        hq.build_model(synthetic.CompressedNetwork([cl]))
    with pytest.raises(hq.ShapeError):
        hq.build_model(synthetic.CompressedNetwork([]))


def test_device_tensor_forward_matches_host_forward(torch_cuda):
    torch = torch_cuda
    cn = synthetic.synthetic_head(dims=(128, 96, 10), k=1024, grid=10, int8=True, seed=12)
    model = hq.build_model(cn)
    ws = hq.make_workspace(model, 32)
    x = synthetic.synthetic_inputs(32, 128, seed=1)
    y = np.zeros(32 * 10)
    hq.compressed_forward(model, x, 32, y, ws, mode="exact")
    xd = torch.from_numpy(x).cuda()
    yd = torch.zeros(320, dtype=torch.float64, device="cuda")
    hq.compressed_forward(model, xd, 32, yd, ws, mode="exact")
    assert np.array_equal(yd.cpu().numpy(), y)


def test_multi_head_forward_against_oracle(torch_cuda):
    torch = torch_cuda
    cns = [synthetic.synthetic_head(dims=(64, 40, 5), k=512, grid=10, int8=True, seed=s) for s in range(4)]
    heads = [hq.build_model(cn) for cn in cns]
    wss = [hq.make_workspace(h, 16) for h in heads]
    x = synthetic.synthetic_inputs(16, 64, seed=3)
    xd = torch.from_numpy(x).cuda()
    ys = [torch.zeros(16 * 5, dtype=torch.float64, device="cuda") for _ in heads]
    hq.forward_multi(heads, wss, xd, 16, ys, mode="exact")
    torch.cuda.synchronize()
    for cn, y in zip(cns, ys):
        want, _ = oracle.port_forward([oracle.Tables.from_runtime(rl) for rl in synthetic.runtime_layers(cn)], x, 16)
        assert np.array_equal(_bits(y.cpu().numpy()), _bits(want))


def test_l2_persistence_window(torch_cuda):
    torch = torch_cuda
    model = hq.build_model(synthetic.synthetic_head(dims=(64, 40, 5), k=512, grid=10, int8=True, seed=1))
    s = torch.cuda.Stream()
    model.set_l2_persist(s.cuda_stream, 1.0)
    model.set_l2_persist(s.cuda_stream, 0.0)


# ---------------------------------------------------------------------------
# primitives

def test_pli_lookup_matches_reference(torch_cuda):
    torch = torch_cuda
    rng = np.random.default_rng(14)
    k, G, lo, hi = 6, 7, -1.0, 1.0
    cb = rng.uniform(-1, 1, k * G)
    n = 5000
    rows = rng.integers(0, k, n).astype(np.int32)
    g = rng.uniform(0, 2, n)
    b = rng.uniform(-1, 1, n)
    x = rng.uniform(-1.3, 1.3, n)
    y = hq.pli_lookup(torch.from_numpy(cb).cuda(), torch.from_numpy(rows).cuda(), torch.from_numpy(g).cuda(),
                      torch.from_numpy(b).cuda(), torch.from_numpy(x).cuda(), lo, hi, G).cpu().numpy()
    for q in range(0, n, 7):
        want = C.c_double()
        assert oracle.ref().hqref_pli_lookup(cb.ctypes.data, k, G, int(rows[q]), g[q], b[q], x[q], lo, hi,
                                             C.byref(want)) == 0
        assert y[q] == want.value
    bad = torch.from_numpy(np.array([k], np.int32)).cuda()
    with pytest.raises(hq.ShapeError):
        hq.pli_lookup(torch.from_numpy(cb).cuda(), bad, torch.ones(1, dtype=torch.float64, device="cuda"),
                      torch.zeros(1, dtype=torch.float64, device="cuda"),
                      torch.zeros(1, dtype=torch.float64, device="cuda"), lo, hi, G)


def test_unpack_indices_bitexact(torch_cuda):
    torch = torch_cuda
    rng = np.random.default_rng(20)
    for bits in range(1, 33):
        for count in (1, 3, 100, 4097):
            vals = rng.integers(0, 2 ** bits, size=count, dtype=np.uint64).astype(np.uint32)
            n = oracle.ref().hqref_pack_indices(vals.ctypes.data, vals.size, bits, None, 0)
            buf = np.zeros(n, np.uint8)
            oracle.ref().hqref_pack_indices(vals.ctypes.data, vals.size, bits, buf.ctypes.data, n)
            got = hq.unpack_indices(torch.from_numpy(buf).cuda(), count, bits).cpu().numpy().view(np.uint32)
            assert np.array_equal(got, vals), (bits, count)
    # KAT test_lutham.cpp:39-40
    got = hq.unpack_indices(torch.tensor([0xff, 0x03, 0x10, 0x20], dtype=torch.uint8, device="cuda"), 3, 10)
    assert got.cpu().tolist() == [1023, 0, 513]


# ---------------------------------------------------------------------------
# tensor-core layer GEMM (skan_gemm.cu): every table format, even and odd G,
# batches that fill and do not fill a 128-sample tile

@pytest.mark.parametrize("batch", [64, 200, 300])
def test_fast_mode_tensor_core_gemm_formats(torch_cuda, batch):
    rng = np.random.default_rng(300 + batch)
    cases = [
        ("int8 u16 G=10", oracle.ref_build(synthetic.CompressedNetwork(
            [synthetic.crafted_layer(96, 150, 10, 300, 1, int8=True)])).tables()),
        ("int8 u32 K>65536 G=6", oracle.ref_build(synthetic.CompressedNetwork(
            [synthetic.crafted_layer(20, 70, 6, 70000, 2, int8=True)])).tables()),
        ("f32 G=5 (odd: 8 inputs per chunk)", oracle.ref_build(synthetic.CompressedNetwork(
            [synthetic.crafted_layer(33, 40, 5, 50, 3, int8=False)])).tables()),
        ("dense G=12", oracle.ref_random([24, 130, 17], 12, 0.4, 4, 0, False).tables()),
        ("int8 two layers", [oracle.Tables.from_runtime(rl) for rl in synthetic.runtime_layers(
            synthetic.synthetic_head(dims=(128, 96, 24), k=512, grid=10, int8=True, seed=5))]),
    ]
    for name, tables in cases:
        x = rng.uniform(-1.5, 1.5, batch * tables[0].in_dim)
        want, _ = oracle.port_forward(tables, x, batch)
        model = _upload(tables)
        got, ws = _gpu_forward(model, x, batch, "fast", max_batch=256)
        assert ws.last_launches() >= 2, name
        assert_close(got, want, l1_scale(tables, x, batch))
        again, _ = _gpu_forward(model, x, batch, "fast", max_batch=256)
        assert np.array_equal(_bits(got), _bits(again)), name  # fixed-order split reduction


@pytest.mark.parametrize("batch", [3, 16, 64, 200])
@pytest.mark.parametrize("engine", ["cuda_cores", "tensor_cores"])
def test_fast_mode_both_engines_agree_with_oracle(torch_cuda, batch, engine):
    """The fast path has two engines for batches >= 3: the tensor-core layer
    GEMM (default) and the CUDA-core kernels (k_fwd_small / k_fwd_large,
    forced here by raising the GEMM threshold).  Both meet the tolerance on
    a two-layer int8 head and a dense head."""
    from paper_2512_15742_b200 import _lib
    rng = np.random.default_rng(500 + batch)
    cases = [
        [oracle.Tables.from_runtime(rl) for rl in synthetic.runtime_layers(
            synthetic.synthetic_head(dims=(160, 136, 20), k=1024, grid=10, int8=True, seed=9))],
        oracle.ref_random([40, 144, 18], 10, 0.4, 6, 0, False).tables(),
    ]
    prev = _lib.lib().skan_debug_set_gemm_min_batch(1 << 20 if engine == "cuda_cores" else 0)
    try:
        for tables in cases:
            x = rng.uniform(-1.5, 1.5, batch * tables[0].in_dim)
            want, _ = oracle.port_forward(tables, x, batch)
            got, _ = _gpu_forward(_upload(tables), x, batch, "fast", max_batch=256)
            assert_close(got, want, l1_scale(tables, x, batch))
    finally:
        _lib.lib().skan_debug_set_gemm_min_batch(prev)


@pytest.mark.parametrize("batch", [2, 3, 5, 63, 65, 129])
def test_fast_and_exact_across_batch_routes(torch_cuda, batch):
    """Batch sizes on both sides of every routing threshold (persistent
    kernel <= 3, GEMM >= 3, stacked tiles <= 64, split-M tiles > 128) for an
    odd-G int8 head, a K > 65536 wide-index head and a dense G=13 head:
    fast within tolerance, exact bitwise (tools/parity_sweep.py runs more)."""
    rng = np.random.default_rng(900 + batch)
    cases = [
        [oracle.Tables.from_runtime(r) for r in synthetic.runtime_layers(
            synthetic.synthetic_head(dims=(129, 200, 17), k=300, grid=7, int8=True, seed=12))],
        [oracle.Tables.from_runtime(r) for r in synthetic.runtime_layers(
            synthetic.synthetic_head(dims=(65, 140, 9), k=70000, grid=16, int8=True, seed=13))],
        oracle.ref_random([20, 129, 16], 13, 0.4, 8, 0, False).tables(),
    ]
    for tables in cases:
        model = _upload(tables)
        ws = hq.make_workspace(model, 256)
        x = rng.uniform(-1.5, 1.5, batch * tables[0].in_dim)
        want, _ = oracle.port_forward(tables, x, batch)
        got = np.zeros(batch * tables[-1].out_dim)
        hq.compressed_forward(model, x, batch, got, ws, mode="fast")
        assert_close(got, want, l1_scale(tables, x, batch))
        ex = np.zeros_like(got)
        hq.compressed_forward(model, x, batch, ex, ws, mode="exact")
        assert np.array_equal(_bits(ex), _bits(want))


def test_profile_gemm_hook(torch_cuda):
    """skan_profile_gemm launches one layer's GEMM alone after a forward and
    reports the MMA work it issues; layers off the GEMM are a ContractError."""
    import ctypes as C
    from paper_2512_15742_b200 import _lib
    torch = torch_cuda
    model = hq.build_model(synthetic.synthetic_head(dims=(256, 160, 20), k=512, grid=10, int8=True, seed=8))
    ws = hq.make_workspace(model, 64)
    x = torch.from_numpy(synthetic.synthetic_inputs(64, 256, seed=1)).cuda()
    y = torch.zeros(64 * 20, dtype=torch.float64, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    hq.forward_async(model, x, 64, y, ws, stream=s)
    fl = C.c_double(0)
    _lib.check(_lib.lib().skan_profile_gemm(model.handle, ws.handle, 0, 64, s, C.byref(fl)))
    torch.cuda.synchronize()
    # stacked (batch <= 64): one M=128 x N=256 x K=8 MMA per K step, two 128-output tiles
    assert fl.value == 2.0 * 128 * 8 * 256 * (256 * 10 / 8) * 2
    hq.forward_async(model, x, 1, y, ws, stream=s)
    assert _lib.lib().skan_profile_gemm(model.handle, ws.handle, 0, 1, s, None) == 3  # SKAN_CONTRACT_ERROR


def test_zero_copy_host_forward(torch_cuda):
    """Small fast-mode batches with a page-locked output buffer take the
    low-overhead host path (one H2D copy, the persistent kernel writes y to
    host memory, mapped error flag): bitwise equal to the device-pointer
    forward; a non-finite input still raises ValueError; pageable buffers
    keep the copy path."""
    import ctypes as C
    from paper_2512_15742_b200 import _lib
    torch = torch_cuda
    cn = synthetic.synthetic_head()
    model = hq.build_model(cn)
    ws = hq.make_workspace(model, 8)
    L = _lib.lib()
    s = torch.cuda.current_stream().cuda_stream
    for batch in (1, 2):
        x = synthetic.synthetic_inputs(batch, 2048, seed=90 + batch)
        xp = torch.from_numpy(x).pin_memory()
        yp = torch.zeros(batch * 20, dtype=torch.float64).pin_memory()
        _lib.check(L.skan_forward(model.handle, ws.handle, xp.data_ptr(), xp.numel(), batch, yp.data_ptr(),
                                  yp.numel(), hq.MODE_FAST, _lib.SKAN_PTR_HOST, s))
        assert ws.last_launches() == batch
        dx = torch.from_numpy(x).cuda()
        dy = torch.zeros(batch * 20, dtype=torch.float64, device="cuda")
        hq.forward_async(model, dx, batch, dy, ws, stream=s)
        ws.check()
        assert np.array_equal(_bits(yp.numpy()), _bits(dy.cpu().numpy()))
        yn = np.zeros(batch * 20)  # pageable: copy path, same result
        hq.compressed_forward(model, x, batch, yn, ws, mode="fast")
        assert np.array_equal(_bits(yn), _bits(yp.numpy()))
    xp[2048 + 5] = float("nan")  # batch 2: per-sample persistent launches
    rc = L.skan_forward(model.handle, ws.handle, xp.data_ptr(), xp.numel(), 2, yp.data_ptr(), yp.numel(),
                        hq.MODE_FAST, _lib.SKAN_PTR_HOST, s)
    assert rc == 2  # SKAN_VALUE_ERROR
    x = synthetic.synthetic_inputs(1, 2048, seed=5)
    xp = torch.from_numpy(x).pin_memory()
    yp = torch.zeros(20, dtype=torch.float64).pin_memory()
    _lib.check(L.skan_forward(model.handle, ws.handle, xp.data_ptr(), xp.numel(), 1, yp.data_ptr(), yp.numel(),
                              hq.MODE_FAST, _lib.SKAN_PTR_HOST, s))  # the flag was reset
    xp[7] = float("inf")  # batch 1: the workspace's graph replay reports it too
    rc = L.skan_forward(model.handle, ws.handle, xp.data_ptr(), xp.numel(), 1, yp.data_ptr(), yp.numel(),
                        hq.MODE_FAST, _lib.SKAN_PTR_HOST, s)
    assert rc == 2
    # batch 1 from PAGEABLE buffers also replays the graph (x staged, y copied out): bitwise equal
    x = synthetic.synthetic_inputs(1, 2048, seed=6)
    yn = np.zeros(20)
    _lib.check(L.skan_forward(model.handle, ws.handle, x.ctypes.data, x.size, 1, yn.ctypes.data, yn.size,
                              hq.MODE_FAST, _lib.SKAN_PTR_HOST, s))
    dy = torch.zeros(20, dtype=torch.float64, device="cuda")
    hq.forward_async(model, torch.from_numpy(x).cuda(), 1, dy, ws, stream=s)
    ws.check()
    assert np.array_equal(_bits(yn), _bits(dy.cpu().numpy()))


def test_hot_swap_refills_a_resident_head(torch_cuda):
    """skan_head_swap: a head (batch-1 persistent path and the multi-kernel
    path) refilled in place serves the new tables bitwise in exact mode and
    within tolerance in fast mode; shape changes are a ContractError."""
    dims = (512, 512, 8)
    a = synthetic.synthetic_head(dims=dims, k=4096, grid=10, int8=True, seed=1)
    b = synthetic.synthetic_head(dims=dims, k=4096, grid=10, int8=True, seed=2)
    tb = [oracle.Tables.from_runtime(rl) for rl in synthetic.runtime_layers(b)]
    model = hq.build_model(a)
    ws = hq.make_workspace(model, max_batch=8)
    x = synthetic.synthetic_inputs(3, 512, seed=4)
    want, _ = oracle.port_forward(tb, x, 3)
    ta = [oracle.Tables.from_runtime(rl) for rl in synthetic.runtime_layers(a)]
    y1 = np.zeros(8)  # batch 1 from host buffers: builds the workspace's captured graph for head a
    hq.compressed_forward(model, x[:512], 1, y1, ws, mode="fast")
    wa, _ = oracle.port_forward(ta, x[:512], 1)
    assert_close(y1, wa, l1_scale(ta, x[:512], 1))
    hq.swap_model(model, b)  # ... which must be rebuilt for the new tables
    y = np.zeros(3 * 8)
    hq.compressed_forward(model, x, 3, y, ws, mode="exact")
    assert np.array_equal(_bits(y), _bits(want))
    for batch in (1, 3):
        xb = x[:batch * 512]
        wb, _ = oracle.port_forward(tb, xb, batch)
        yb = np.zeros(batch * 8)
        hq.compressed_forward(model, xb, batch, yb, ws, mode="fast")
        assert_close(yb, wb, l1_scale(tb, xb, batch))
    with pytest.raises(hq.ContractError):
        hq.swap_model(model, synthetic.synthetic_head(dims=(512, 500, 8), k=4096, grid=10, int8=True, seed=3))


# ---------------------------------------------------------------------------
# SKAN v1 direct-to-device load (§8 f1): sections unpacked on the device

def test_loaded_head_equals_uploaded_head_in_fast_mode(torch_cuda):
    """The device-built resident form of a loaded file (records, codebook
    tables, bias sums) is the host-built one: fast-mode outputs of
    deserialize(bytes) and upload(tables) are bitwise equal on every route
    (batch 1, small batches, the tensor-core GEMM)."""
    rng = np.random.default_rng(5)
    for name, m in _fixture_models():
        tables = m.tables()
        a, b = hq.deserialize(m.serialize()), _upload(tables)
        for batch in (1, 5, 64):
            x = rng.uniform(-1.5, 1.5, batch * tables[0].in_dim)
            ya, _ = _gpu_forward(a, x, batch, "fast")
            yb, _ = _gpu_forward(b, x, batch, "fast")
            assert np.array_equal(_bits(ya), _bits(yb)), (name, batch)


def test_headline_head_file_loads_on_device(torch_cuda):
    """The cfg2 head serialized by the reference (12.96 MB payload) loads
    through the device path: exact mode bitwise equal to the reference,
    fast batch 1 within the bound."""
    cn = synthetic.synthetic_head()
    ref = oracle.ref_build(cn)
    model = hq.deserialize(ref.serialize())
    tables = ref.tables()
    x = synthetic.synthetic_inputs(2, 2048, seed=61)
    want, scale = oracle.port_forward_l1(tables, x, 2, threads=2)
    got, _ = _gpu_forward(model, x, 2, "exact")
    assert np.array_equal(_bits(got), _bits(want))
    y1, ws = _gpu_forward(model, x[:2048], 1, "fast")
    assert ws.last_launches() == 1
    assert_close(y1, want[:20], scale[:20])


def test_swap_from_bytes_refills_in_place(torch_cuda):
    """skan_head_swap_bytes: the new tables serve bitwise; a corrupt file
    raises the reference's FormatError and leaves the head as it was; a file
    of other shapes is a ContractError."""
    dims = (512, 512, 8)
    a = oracle.ref_build(synthetic.synthetic_head(dims=dims, k=4096, grid=10, int8=True, seed=1))
    b = oracle.ref_build(synthetic.synthetic_head(dims=dims, k=4096, grid=10, int8=True, seed=2))
    model = hq.deserialize(a.serialize())
    ws = hq.make_workspace(model, 8)
    x = synthetic.synthetic_inputs(3, 512, seed=4)
    hq.swap_model_bytes(model, b.serialize())
    want, _ = b.forward(x, 3)
    y = np.zeros(3 * 8)
    hq.compressed_forward(model, x, 3, y, ws, mode="exact")
    assert np.array_equal(_bits(y), _bits(want))
    bad = bytearray(a.serialize())
    bad[-1:] = b""  # truncated last section: checks run, nothing is overwritten
    with pytest.raises(hq.FormatError):
        hq.swap_model_bytes(model, bytes(bad))
    hq.compressed_forward(model, x, 3, y, ws, mode="exact")
    assert np.array_equal(_bits(y), _bits(want))
    other = oracle.ref_build(synthetic.synthetic_head(dims=(512, 500, 8), k=4096, grid=10, int8=True, seed=3))
    with pytest.raises(hq.ContractError):
        hq.swap_model_bytes(model, other.serialize())


@pytest.mark.parametrize("dims,grid", [((300, 20), 10), ((97, 3), 5), ((64, 33, 32), 3), ((1000, 1), 16)])
@pytest.mark.parametrize("batch", [3, 17, 64, 200, 600])
def test_dense_narrow_layer_against_oracle(torch_cuda, dims, grid, batch):
    """Dense layers with <= 32 outputs keep the natural [in][out][G] grid and
    run k_dense_narrow at batch >= 3: row blocks staged by bulk copies when
    16-byte aligned (3 x 5 x 4 = 60-byte rows are not: the word-staging
    path), brackets likewise (batch 17: most blocks unaligned), split partials
    summed in order.  Fast mode within the bound, exact mode bitwise (the
    exact kernels read the same natural grid)."""
    rls = synthetic.dense_runtime_head(dims=dims, grid=grid, seed=11)
    tables = [oracle.Tables.from_runtime(rl) for rl in rls]
    model = hq.upload(rls, device=0)
    x = synthetic.synthetic_inputs(batch, dims[0], seed=5, grid=grid)
    ws = hq.make_workspace(model, max_batch=batch)
    got = np.zeros(batch * dims[-1])
    want, scale = oracle.port_forward_l1(tables, x, batch, threads=16)
    hq.compressed_forward(model, x, batch, got, ws, mode="fast")
    assert_close(got, want, scale)
    want_e, _ = oracle.port_forward(tables, x, batch)
    hq.compressed_forward(model, x, batch, got, ws, mode="exact")
    assert np.array_equal(_bits(got), _bits(want_e))


@pytest.mark.parametrize("dims,batch", [((256, 1024), 64), ((256, 1024, 20), 64), ((300, 700, 20), 17),
                                        ((1024, 4096), 32), ((2048, 1408), 64)])
def test_dense_persistent_schedule_against_oracle(torch_cuda, dims, batch):
    """Dense layers at batch <= 64 run the persistent tensor-core kernel
    (k_dense_persist): every SM streams an equal share of the flattened
    (output tile, chunk) schedule, so a CTA's range covers pieces of several
    tiles ("segments") and a tile several CTAs.  Short ranges (hundreds of
    segments, 1-4 chunks each) and narrow last layers exercise the segment
    drains and the reduction's plane counts.  Fast mode within the bound."""
    rls = synthetic.dense_runtime_head(dims=dims)
    tables = [oracle.Tables.from_runtime(rl) for rl in rls]
    model = hq.upload(rls, device=0)
    x = synthetic.synthetic_inputs(batch, dims[0], seed=6)
    want, scale = oracle.port_forward_l1(tables, x, batch, threads=16)
    ws = hq.make_workspace(model, max_batch=batch)
    got = np.zeros(batch * dims[-1])
    # a first call on other inputs leaves its partial planes behind: planes a
    # call does not write (CTAs without work when a layer has fewer units than
    # SMs) must not be summed
    hq.compressed_forward(model, synthetic.synthetic_inputs(batch, dims[0], seed=7), batch, got, ws, mode="fast")
    hq.compressed_forward(model, x, batch, got, ws, mode="fast")
    assert_close(got, want, scale)
