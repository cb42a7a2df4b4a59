"""Seeded synthetic heads and inputs.

Tables follow the reference tests' crafted_layer (test_lutham.cpp:124-145):
codebook U(-1,1), indices uniform in [0,K), every 5th gain exactly 0 else
|U|+0.01, biases U(-1,1).  For chained layers gains are scaled by 1/sqrt(in)
and biases by 1/in so hidden activations mostly stay inside the domain.
int8 tables use the reference's encoders restated in numpy
(quant.cpp:11-86): symmetric linear int8 for codebook/biases, log2 int8 for
gains with code 127 = exact zero.  Inputs are U(-1.5,1.5) (~33% clamped)
plus a slice of exact knot positions (kan.cpp:21-26).
"""
from __future__ import annotations

from typing import Sequence, Tuple

import numpy as np

from .lutham import (Codebook, CompressedLayer, CompressedNetwork, Int8Tables, LayerHeader,
                     RuntimeLayer, kFlagInt8)

# configs named in BASELINE.json (dims per SURVEY.md §8a)
HEAD_DIMS = (2048, 1408, 20)      # cfg2/cfg3: ~12.96 MB int8 payload
HEAD_K = 65536
HEAD_G = 10
DENSE_DIMS = (2048, 13664, 20)    # cfg4: 1,130,286,080 B f32 grids
CFG1 = dict(dims=(256, 256), k=256, grid=10)


def round_half_even(x: np.ndarray) -> np.ndarray:
    """quant.cpp:11-17 (np.rint rounds half to even)."""
    return np.rint(x)


def quantize_linear_i8(values: np.ndarray) -> Tuple[np.ndarray, float]:
    """quant.cpp:25-38: scale = max|v|/127 (1 for all-zero), codes clamped to +-127."""
    v = np.asarray(values, dtype=np.float64)
    m = float(np.max(np.abs(v))) if v.size else 0.0
    scale = m / 127.0 if m > 0.0 else 1.0
    codes = np.clip(round_half_even(v / scale), -127, 127).astype(np.int8)
    return codes, scale


def quantize_gains_log_i8(gains: np.ndarray) -> Tuple[np.ndarray, float, float]:
    """quant.cpp:53-86: codes 0..126 on a log2 ladder, 127 = exact zero."""
    g = np.asarray(gains, dtype=np.float64)
    pos = g[g > 0.0]
    codes = np.full(g.shape, 127, dtype=np.int8)
    if pos.size == 0:
        return codes, 0.0, 1.0
    log_min = float(np.log2(pos.min()))
    log_max = float(np.log2(pos.max()))
    step = 1.0 if (log_max - log_min) < 1e-9 else (log_max - log_min) / 126.0
    nz = g > 0.0
    codes[nz] = np.clip(round_half_even((np.log2(g[nz]) - log_min) / step), 0, 126).astype(np.int8)
    return codes, log_min, step


def crafted_layer(in_dim: int, out_dim: int, grid: int, k: int, seed: int, int8: bool = False,
                  chained: bool = False, domain: Tuple[float, float] = (-1.0, 1.0)) -> CompressedLayer:
    rng = np.random.default_rng(seed)
    e = in_dim * out_dim
    cb = rng.uniform(-1.0, 1.0, size=k * grid)
    idx = rng.integers(0, k, size=e, dtype=np.uint32) if k > 1 else np.zeros(e, np.uint32)
    gains = np.abs(rng.uniform(-1.0, 1.0, size=e)) + 0.01
    gains[::5] = 0.0
    biases = rng.uniform(-1.0, 1.0, size=e)
    if chained:
        gains /= np.sqrt(in_dim)
        biases /= in_dim
    cl = CompressedLayer(in_dim, out_dim, grid, Codebook(k, grid, cb), idx, gains, biases,
                         domain_lo=domain[0], domain_hi=domain[1])
    if int8:
        cc, cs = quantize_linear_i8(cb)
        gc, lmin, lstep = quantize_gains_log_i8(gains)
        bc, bs = quantize_linear_i8(biases)
        cl.int8 = Int8Tables(cc, gc, bc, cs, lmin, lstep, bs)
        # like quantize_compressed_layer: double tables hold the dequantized values
        cl.codebook = Codebook(k, grid, cc.astype(np.float64) * cs)
        gq = np.exp2(lmin + gc.astype(np.float64) * lstep)
        gq[gc == 127] = 0.0
        cl.gains = gq
        cl.biases = bc.astype(np.float64) * bs
    return cl


def synthetic_head(dims: Sequence[int] = HEAD_DIMS, k: int = HEAD_K, grid: int = HEAD_G, int8: bool = True,
                   seed: int = 2026) -> CompressedNetwork:
    """The compressed detection head of cfg2/cfg3 (random tables of that architecture)."""
    layers = [crafted_layer(dims[l], dims[l + 1], grid, k, seed + 101 * l, int8=int8, chained=True)
              for l in range(len(dims) - 1)]
    return CompressedNetwork(layers)


def dense_runtime_head(dims: Sequence[int] = DENSE_DIMS, grid: int = HEAD_G, seed: int = 7):
    """cfg4 dense head as RuntimeLayer f32 grids (generated directly in float32
    to avoid a 2.3 GB float64 staging copy)."""
    rng = np.random.default_rng(seed)
    out = []
    for l in range(len(dims) - 1):
        e = dims[l] * dims[l + 1]
        t = rng.standard_normal(e * grid, dtype=np.float32)
        t *= np.float32(0.5 / np.sqrt(dims[l]))
        out.append(RuntimeLayer(LayerHeader(dims[l], dims[l + 1], grid, 0, -1.0, 1.0), table_f32=t))
    return out


def node_position(lo: float, hi: float, grid: int, i: int) -> float:
    """kan.cpp:21-26, same double ops (numpy float64 is IEEE, no contraction)."""
    if i == 0:
        return lo
    if i == grid - 1:
        return hi
    dx = (hi - lo) / float(grid - 1)
    return lo + float(i) * dx


def synthetic_inputs(batch: int, width: int, seed: int = 12345, lo: float = -1.5, hi: float = 1.5,
                     grid: int = HEAD_G, domain: Tuple[float, float] = (-1.0, 1.0),
                     node_frac: float = 0.01) -> np.ndarray:
    rng = np.random.default_rng(seed)
    x = rng.uniform(lo, hi, size=batch * width)
    nn = int(node_frac * x.size)
    if nn:
        pos = rng.choice(x.size, size=nn, replace=False)
        nodes = np.array([node_position(domain[0], domain[1], grid, i) for i in range(grid)])
        x[pos] = nodes[rng.integers(0, grid, size=nn)]
    return x


def runtime_layers(cn: CompressedNetwork):
    """build_model's resident conversion (lutham.cpp:214-271) on the host, as
    RuntimeLayer tables (used to feed identical tables to the oracle)."""
    out = []
    for cl in cn.layers:
        h = LayerHeader(cl.in_dim, cl.out_dim, cl.grid_size, cl.codebook.k, cl.domain_lo, cl.domain_hi)
        rl = RuntimeLayer(h)
        k = cl.codebook.k
        if k > 1 and k <= 65536:
            rl.idx16 = np.asarray(cl.indices, np.uint16)
        elif k > 65536:
            rl.idx32 = np.asarray(cl.indices, np.uint32)
        if cl.int8 is not None:
            t = cl.int8
            h.flags = kFlagInt8
            h.codebook_scale, h.gain_log_min = t.codebook_scale, t.gain_log_min
            h.gain_log_step, h.bias_scale = t.gain_log_step, t.bias_scale
            rl.table_i8 = np.asarray(t.codebook_codes, np.int8)
            rl.gain_codes = np.asarray(t.gain_codes, np.int8)
            rl.bias_codes = np.asarray(t.bias_codes, np.int8)
        else:
            rl.table_f32 = np.asarray(cl.codebook.entries, np.float32)
            rl.gains_f32 = np.asarray(cl.gains, np.float32)
            rl.biases_f32 = np.asarray(cl.biases, np.float32)
        out.append(rl)
    return out
