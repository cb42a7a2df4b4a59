"""Pin the oracle (CPU, no GPU): the C restatement (oracle/skan_oracle.c) must
agree bit-for-bit with the UNMODIFIED reference build (oracle/_ref) and with
the golden vectors of the reference's own test suites
(tests/golden/reference_kats.json, file:line cited per entry).
"""
import ctypes as C
import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_2512_15742_b200 import synthetic

KATS = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "reference_kats.json")))
needs_ref = pytest.mark.skipif(not oracle.have_ref(), reason="reference build oracle/_ref unavailable")


def test_node_position_kats():
    for v in KATS["node_position"]:
        assert oracle.port().oracle_node_position(v["lo"], v["hi"], v["G"], v["i"]) == v["want"], v["src"]
    # interior node of test_kan.cpp:15 (approx 0 within 1e-15)
    assert abs(oracle.port().oracle_node_position(-1.0, 1.0, 5, 2)) <= 1e-15


def _eval_spline_port(c, lo, hi, x):
    i, t, _ = oracle.port_locate(lo, hi, len(c), x)
    return c[i] * (1.0 - t) + c[i + 1] * t  # kan.cpp:60-64 (numpy float64: same IEEE ops)


def test_eval_spline_kats():
    for v in KATS["eval_spline"]:
        got = _eval_spline_port(v["c"], v["lo"], v["hi"], v["x"])
        if v["rel"] == 0.0:
            assert got == v["want"], v["src"]
        else:
            assert abs(got - v["want"]) <= v["rel"] * max(1.0, abs(v["want"])), v["src"]


def test_locate_kats():
    for v in KATS["locate"]:
        i, t, c = oracle.port_locate(v["lo"], v["hi"], v["G"], v["x"])
        assert i == v["index"] and c == v["clamped"], v["src"]
        if v["t"] is not None:
            assert t == v["t"], v["src"]
    with pytest.raises(oracle.RefError):
        oracle.port_locate(-1.0, 1.0, 5, float("nan"))


def test_nodes_reproduce_coefficients_bitwise():
    """test_kan.cpp:36-51: evaluation at every node returns the coefficient."""
    rng = np.random.default_rng(11)
    for _ in range(50):
        G = 2 + int(rng.integers(0, 40))
        lo, hi = sorted(rng.uniform(-5, 5, 2))
        if hi - lo < 1e-3:
            hi = lo + 1.0
        c = rng.uniform(-5, 5, G)
        for i in range(G):
            x = oracle.port().oracle_node_position(lo, hi, G, i)
            assert _eval_spline_port(c, lo, hi, x) == c[i]


def _adversarial_x(rng, lo, hi, G, n):
    """Random x plus every node, its float neighbours, and clamp edges."""
    xs = [rng.uniform(lo - 0.5 * (hi - lo), hi + 0.5 * (hi - lo), n)]
    nodes = np.array([synthetic.node_position(lo, hi, G, i) for i in range(G)])
    xs += [nodes, np.nextafter(nodes, -np.inf), np.nextafter(nodes, np.inf),
           np.nextafter(np.nextafter(nodes, np.inf), np.inf), np.array([lo, hi, -1e300, 1e300, -0.0, 0.0])]
    return np.concatenate(xs)


@needs_ref
def test_locate_port_equals_reference_bitwise():
    rng = np.random.default_rng(1)
    for trial in range(40):
        G = int(rng.choice([2, 3, 5, 10, 16, 20, 64, 128, 1000]))
        lo, hi = sorted(rng.uniform(-3, 3, 2))
        if trial % 4 == 0:
            lo, hi = -1.0, 1.0
        x = _adversarial_x(rng, lo, hi, G, 20000)
        a = oracle.port_locate_many(lo, hi, G, x)
        b = oracle.ref_locate_many(lo, hi, G, x)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1].view(np.uint64), b[1].view(np.uint64))
        assert np.array_equal(a[2], b[2]) and a[3] == b[3] == 0


def _dkey(a):
    """Order-preserving int64 key of a double (+0 and -0 share key 0), as the
    fast-path device locate compares them (skan_device.cuh: dkey)."""
    b = np.asarray(a, np.float64).view(np.int64).copy()
    b[b == np.int64(-0x8000000000000000)] = 0
    return b ^ ((b >> 63) & np.int64(0x7FFFFFFFFFFFFFFF))


def test_bracket_is_the_node_search_the_fast_path_uses():
    """The fast path finds locate()'s bracket without division: the unique
    i in [0, G-2] with node(i) <= x < node(i+1) over the reference's own node
    positions (kan.cpp:21-26), compared as order-preserving integer keys.
    Pinned against oracle locate on random domains, every node, +-1 ulp
    neighbours, +-0.0 and clamped inputs."""
    rng = np.random.default_rng(0)
    for trial in range(200):
        G = int(rng.choice([2, 3, 4, 5, 7, 10, 16, 33, 64, 128, 1000]))
        lo, hi = sorted(rng.uniform(-1e3, 1e3, 2)) if trial % 3 else sorted(rng.uniform(-2, 2, 2))
        if trial % 7 == 0:
            lo, hi = -1.0, 1.0
        if hi - lo < 1e-6:
            hi = lo + 1
        nodes = np.array([synthetic.node_position(lo, hi, G, i) for i in range(G)])
        x = np.concatenate([rng.uniform(lo - (hi - lo), hi + (hi - lo), 5000), nodes,
                            np.nextafter(nodes, -np.inf), np.nextafter(nodes, np.inf), [-0.0, 0.0]])
        ref_i, _, _, bad = oracle.port_locate_many(lo, hi, G, x)
        assert bad == 0
        mine = np.clip(np.searchsorted(_dkey(nodes), _dkey(np.clip(x, lo, hi)), side="right") - 1, 0, G - 2)
        assert np.array_equal(mine, ref_i)


@needs_ref
def test_gain_decode_port_equals_reference_bitwise():
    rng = np.random.default_rng(2)
    for _ in range(50):
        lmin, lstep = rng.uniform(-12, 4), rng.uniform(1e-4, 0.2)
        for code in range(-128, 128):
            a = oracle.port().oracle_dequantize_gain_code(code, lmin, lstep)
            b = oracle.ref().hqref_dequantize_gain_code(code, lmin, lstep)
            assert a == b or (math.isnan(a) and math.isnan(b))
    for v in KATS["gain_decode"]:
        got = oracle.port().oracle_dequantize_gain_code(v["code"], v["log_min"], v["log_step"])
        assert abs(got - v["want"]) <= v["rel"] * abs(v["want"]), v["src"]
        if v["rel"] == 0.0:
            assert got == v["want"]


def test_index_bits_kats():
    v = KATS["index_bits"]
    assert [oracle.port().oracle_index_bits(k) for k in v["k"]] == v["bits"]


def _pack_port(values, bits):
    a = np.asarray(values, np.uint32)
    cap = (a.size * bits + 7) // 8 + 8
    out = np.zeros(cap, np.uint8)
    n = oracle.port().oracle_pack_indices(a.ctypes.data, a.size, bits, out.ctypes.data, cap)
    return None if n == C.c_size_t(-1).value else out[:n]


def test_pack_kats_and_roundtrip():
    for v in KATS["pack_indices"]:
        assert list(_pack_port(v["values"], v["bits"])) == v["bytes"], v["src"]
    rng = np.random.default_rng(20)
    for bits in range(1, 33):
        vals = rng.integers(0, 2 ** bits, size=1 + int(rng.integers(0, 100)), dtype=np.uint64).astype(np.uint32)
        packed = _pack_port(vals, bits)
        back = np.zeros(vals.size, np.uint32)
        assert oracle.port().oracle_unpack_indices(packed.ctypes.data, packed.size, vals.size, bits,
                                                   back.ctypes.data) == 0
        assert np.array_equal(back, vals)
        if oracle.have_ref():
            n = oracle.ref().hqref_pack_indices(vals.ctypes.data, vals.size, bits, None, 0)
            buf = np.zeros(n, np.uint8)
            oracle.ref().hqref_pack_indices(vals.ctypes.data, vals.size, bits, buf.ctypes.data, n)
            assert np.array_equal(buf, packed)
    assert _pack_port([4], 2) is None  # value does not fit: ContractError (test_lutham.cpp:50)


def _plan_port(rows):
    arr = (oracle.OracleLayer * len(rows))()
    for q, r in enumerate(rows):
        arr[q].in_dim, arr[q].out_dim, arr[q].grid_size, arr[q].k = r["in"], r["out"], r["G"], r["k"]
        arr[q].flags = 1 if r.get("int8") else 0
    per = (oracle.OracleLayerPlan * len(rows))()
    sc, pay, ws = C.c_uint64(), C.c_uint64(), C.c_uint64()
    rc = oracle.port().oracle_plan_memory(arr, len(rows), per, C.byref(sc), C.byref(pay), C.byref(ws))
    return rc, per, sc.value, pay.value, ws.value


def test_plan_memory_kats():
    for v in KATS["plan_memory"]:
        rc, per, sc, pay, ws = _plan_port([v])
        assert rc == 0
        p = per[0]
        got = (p.codebook_bytes, p.index_bytes, p.unpacked_index_bytes, p.gain_bytes, p.bias_bytes, sc, pay, ws)
        want = (v["codebook"], v["index"], v["unpacked"], v["gain"], v["bias"], v["scratch"], v["payload"],
                v["working"])
        assert got == want, v["src"]
    o = KATS["plan_overflow"]
    assert _plan_port([o])[0] == 5  # PlanError


@needs_ref
def test_plan_memory_port_equals_reference():
    rng = np.random.default_rng(5)
    for _ in range(200):
        n = 1 + int(rng.integers(0, 4))
        rows = [dict(**{"in": int(rng.integers(1, 5000)), "out": int(rng.integers(1, 5000))},
                     G=int(rng.integers(2, 130)), k=int(rng.choice([0, 1, 2, 255, 256, 65536, 65537, 1 << 20])),
                     int8=bool(rng.integers(0, 2))) for _ in range(n)]
        for r in rows:
            if r["k"] == 0:
                r["int8"] = False
        rc, per, sc, pay, ws = _plan_port(rows)
        dims = np.array([[r["in"], r["out"], r["G"], r["k"]] for r in rows], np.uint32).ravel()
        flags = np.array([1 if r["int8"] else 0 for r in rows], np.uint32)
        per5 = np.zeros(5 * n, np.uint64)
        tot = np.zeros(3, np.uint64)
        assert oracle.ref().hqref_plan_memory(dims.ctypes.data, flags.ctypes.data, n, per5.ctypes.data,
                                              tot.ctypes.data) == 0
        mine = np.array([[p.codebook_bytes, p.index_bytes, p.unpacked_index_bytes, p.gain_bytes, p.bias_bytes]
                         for p in per[:n]], np.uint64).ravel()
        assert np.array_equal(mine, per5) and (sc, pay, ws) == tuple(int(t) for t in tot)


# ---------------------------------------------------------------------------
# forward: port == reference, bitwise

def _ref_fixture_models():
    """The reference tests' own fixtures: random_compressed (test_lutham.cpp:117-123),
    dense random_net, crafted K=65536 / K=1 layers (test_lutham.cpp:124-145)."""
    out = [oracle.ref_random([3, 5, 2], 6, 0.4, 16, 5, False),
           oracle.ref_random([3, 5, 2], 6, 0.4, 16, 5, True),
           oracle.ref_random([2, 4, 1], 7, 0.4, 2, 0, False),
           oracle.ref_random([4, 24, 2], 12, 0.4, 95, 32, True)]
    for (i, o, G, k, s, q) in [(2, 3, 4, 65536, 5, False), (2, 2, 3, 1, 6, False), (2, 3, 4, 65536, 5, True),
                               (7, 9, 5, 70000, 8, True), (7, 9, 5, 70000, 8, False)]:
        cn = synthetic.CompressedNetwork([synthetic.crafted_layer(i, o, G, k, s, int8=q)])
        out.append(oracle.ref_build(cn))
    return out


@needs_ref
def test_forward_port_equals_reference_bitwise():
    rng = np.random.default_rng(17)
    for m in _ref_fixture_models():
        tables = m.tables()
        batch = 32
        x = rng.uniform(-1.5, 1.5, batch * tables[0].in_dim)
        want, ops_r = m.forward(x, batch)
        got, ops_p = oracle.port_forward(tables, x, batch)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
        assert ops_p == ops_r == batch * sum(t.in_dim * t.out_dim for t in tables)
        # the reference's own oracle relation (test_lutham.cpp:370-392)
        assert np.array_equal(m.dense_oracle_forward(x, batch), want)
        # multi-stream port (one scratch per thread) is bitwise the same
        got_mt, _ = oracle.port_forward(tables, x, batch, threads=4)
        assert np.array_equal(got_mt, want)


@needs_ref
def test_forward_port_equals_reference_on_synthetic_head():
    cn = synthetic.synthetic_head(dims=(96, 64, 7), k=4096, grid=10, int8=True, seed=9)
    m = oracle.ref_build(cn)
    tables = [oracle.Tables.from_runtime(rl) for rl in synthetic.runtime_layers(cn)]
    ref_tables = m.tables()
    for a, b in zip(tables, ref_tables):  # build_model's conversion restated in synthetic.runtime_layers
        for f in oracle.Tables.FIELDS:
            va, vb = getattr(a, f), getattr(b, f)
            assert (va is None and vb is None) or np.array_equal(va, vb), f
    x = synthetic.synthetic_inputs(16, 96, seed=4)
    want, _ = m.forward(x, 16)
    got, _ = oracle.port_forward(tables, x, 16)
    assert np.array_equal(got, want)


def test_interp_ops_kat():
    v = KATS["interp_ops"]
    cn = synthetic.CompressedNetwork([synthetic.crafted_layer(2, 4, 5, 3, 18), synthetic.crafted_layer(4, 1, 5, 3, 19)])
    tables = [oracle.Tables.from_runtime(rl) for rl in synthetic.runtime_layers(cn)]
    _, ops = oracle.port_forward(tables, np.full(v["batch"] * 2, 0.25), v["batch"])
    assert ops == v["per_call"]
