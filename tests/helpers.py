"""Test helpers: numpy evaluation of the per-output L1 scale used by the fast
mode's tolerance, |y_gpu - y_ref| <= TOL * max(|y_ref|, sum_i |term_ij|)
(SURVEY.md §7 minimum slice).  Test infrastructure only."""
import numpy as np

import oracle

TOL = 1e-5  # north_star: "within a stated fp32 relative tolerance (e.g. 1e-5)"


def _dense_grid(t: "oracle.Tables") -> np.ndarray:
    """Reconstructed per-edge grids c = g*table + b (to_dense_network, lutham.cpp:284-311)."""
    e, G = t.in_dim * t.out_dim, t.grid_size
    if t.k == 0:
        return t.table_f32.astype(np.float64).reshape(e, G)
    if t.idx16 is not None:
        idx = t.idx16.astype(np.int64)
    elif t.idx32 is not None:
        idx = t.idx32.astype(np.int64)
    else:
        idx = np.zeros(e, np.int64)
    if t.flags & 1:
        codes = np.arange(-128, 128)
        lut = np.exp2(t.gain_log_min + codes * t.gain_log_step)
        lut[codes == 127] = 0.0
        g = lut[t.gain_codes.astype(np.int64) + 128]
        b = t.bias_codes.astype(np.float64) * t.bias_scale
        cb = t.table_i8.astype(np.float64).reshape(-1, G) * t.codebook_scale
    else:
        g = t.gains_f32.astype(np.float64)
        b = t.biases_f32.astype(np.float64)
        cb = t.table_f32.astype(np.float64).reshape(-1, G)
    return g[:, None] * cb[idx] + b[:, None]


def l1_scale(tables, x: np.ndarray, batch: int, y_ref_hidden=None) -> np.ndarray:
    """Per (sample, output) max(|y|, sum_i |term_ij|) through the whole head
    (hidden activations evaluated in float64 numpy)."""
    cur = x.reshape(batch, -1).astype(np.float64)
    scale = None
    for t in tables:
        W = _dense_grid(t).reshape(t.in_dim, t.out_dim, t.grid_size)
        idx, tt, _, _ = oracle.port_locate_many(t.domain_lo, t.domain_hi, t.grid_size, cur.ravel())
        idx = idx.reshape(batch, t.in_dim)
        tt = tt.reshape(batch, t.in_dim)
        ii = np.arange(t.in_dim)[None, :, None]
        jj = np.arange(t.out_dim)[None, None, :]
        c0 = W[ii, jj, idx[:, :, None]]
        c1 = W[ii, jj, idx[:, :, None] + 1]
        terms = c0 * (1.0 - tt[:, :, None]) + c1 * tt[:, :, None]
        y = terms.sum(axis=1)
        scale = np.maximum(np.abs(y), np.abs(terms).sum(axis=1))
        cur = y
    return scale.ravel()


def assert_close(got: np.ndarray, want: np.ndarray, scale: np.ndarray, tol: float = TOL):
    err = np.abs(got - want)
    bound = tol * np.maximum(scale, 1e-300)
    bad = np.flatnonzero(err > bound)
    assert bad.size == 0, (f"{bad.size} outputs outside tolerance; worst rel err "
                           f"{np.max(err / np.maximum(scale, 1e-300)):.3e}")
    return float(np.max(err / np.maximum(scale, 1e-300))) if err.size else 0.0
