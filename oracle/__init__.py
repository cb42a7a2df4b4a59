"""TEST INFRASTRUCTURE ONLY — the parity checker, never the product.

Two CPU implementations of the reference LUTHAM path, both driven through
ctypes with the same numpy-level API:

  port()  -> liboracle.so : plain-C restatement (skan_oracle.c), each
                            function citing the reference file:line it follows
  ref()   -> _ref/libholoquant_ref.so : the UNMODIFIED reference sources
                            compiled by oracle/Makefile (+ ref_harness.cpp)

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
--impl reference legs may import this package.  The restatement is pinned
bit-for-bit to the reference build and to the reference tests' golden
vectors (tests/test_oracle.py).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import List, Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libholoquant_ref.so")

_p = C.c_void_p


class OracleLayer(C.Structure):
    """skan_oracle.h oracle_layer (= LayerHeader + RuntimeLayer views)."""
    _fields_ = [
        ("in_dim", C.c_uint32), ("out_dim", C.c_uint32), ("grid_size", C.c_uint32), ("k", C.c_uint32),
        ("domain_lo", C.c_double), ("domain_hi", C.c_double), ("flags", C.c_uint32),
        ("codebook_scale", C.c_double), ("gain_log_min", C.c_double), ("gain_log_step", C.c_double),
        ("bias_scale", C.c_double),
        ("table_f32", _p), ("table_i8", _p), ("idx16", _p), ("idx32", _p),
        ("gains_f32", _p), ("biases_f32", _p), ("gain_codes", _p), ("bias_codes", _p),
    ]


class OracleLayerPlan(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in
                ("codebook_bytes", "index_bytes", "unpacked_index_bytes", "gain_bytes", "bias_bytes")]


class RefCLayer(C.Structure):
    """ref_harness.cpp hqref_clayer (CompressedLayer + Int8Tables)."""
    _fields_ = [
        ("in_dim", C.c_int), ("out_dim", C.c_int), ("grid_size", C.c_int), ("k", C.c_int),
        ("domain_lo", C.c_double), ("domain_hi", C.c_double),
        ("codebook", _p), ("indices", _p), ("gains", _p), ("biases", _p),
        ("has_int8", C.c_int), ("codebook_codes", _p), ("gain_codes", _p), ("bias_codes", _p),
        ("codebook_scale", C.c_double), ("gain_log_min", C.c_double), ("gain_log_step", C.c_double),
        ("bias_scale", C.c_double),
    ]


def build(force: bool = False) -> None:
    """make -C oracle (the C port always; the reference build only where
    /root/reference exists — the GPU box uses the prebuilt _ref .so)."""
    if force or not os.path.exists(PORT_SO) or (os.path.isdir("/root/reference") and not os.path.exists(REF_SO)):
        subprocess.run(["make", "-s", "-C", HERE], check=True)


_port = None
_ref = None


def _load_port():
    global _port
    if _port is None:
        if not os.path.exists(PORT_SO):
            build()
        L = C.CDLL(PORT_SO)
        L.oracle_index_bits.restype = C.c_int
        L.oracle_index_bits.argtypes = [C.c_uint32]
        L.oracle_node_position.restype = C.c_double
        L.oracle_node_position.argtypes = [C.c_double, C.c_double, C.c_int, C.c_int]
        L.oracle_locate.restype = C.c_int
        L.oracle_locate.argtypes = [C.c_double, C.c_double, C.c_int, C.c_double, C.POINTER(C.c_int),
                                    C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.oracle_locate_many.restype = C.c_uint64
        L.oracle_locate_many.argtypes = [C.c_double, C.c_double, C.c_int, _p, C.c_uint64, _p, _p, _p]
        L.oracle_dequantize_gain_code.restype = C.c_double
        L.oracle_dequantize_gain_code.argtypes = [C.c_int8, C.c_double, C.c_double]
        L.oracle_dequantize_linear_code.restype = C.c_double
        L.oracle_dequantize_linear_code.argtypes = [C.c_int8, C.c_double]
        L.oracle_plan_memory.restype = C.c_int
        L.oracle_plan_memory.argtypes = [C.POINTER(OracleLayer), C.c_int, C.POINTER(OracleLayerPlan),
                                         C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(C.c_uint64)]
        L.oracle_pack_indices.restype = C.c_size_t
        L.oracle_pack_indices.argtypes = [_p, C.c_size_t, C.c_int, _p, C.c_size_t]
        L.oracle_unpack_indices.restype = C.c_int
        L.oracle_unpack_indices.argtypes = [_p, C.c_size_t, C.c_uint64, C.c_int, _p]
        L.oracle_assign_indices.restype = None
        L.oracle_assign_indices.argtypes = [_p, C.c_uint64, C.c_int, _p, C.c_int, _p]
        L.oracle_compressed_forward.restype = C.c_int
        L.oracle_compressed_forward.argtypes = [C.POINTER(OracleLayer), C.c_int, _p, C.c_int, _p, _p,
                                                C.POINTER(C.c_uint64)]
        L.oracle_compressed_forward_mt.restype = C.c_int
        L.oracle_compressed_forward_mt.argtypes = [C.POINTER(OracleLayer), C.c_int, _p, C.c_int, _p, C.c_int,
                                                   C.POINTER(C.c_uint64)]
        L.oracle_forward_l1_mt.restype = C.c_int
        L.oracle_forward_l1_mt.argtypes = [C.POINTER(OracleLayer), C.c_int, _p, C.c_int, _p, _p, C.c_int]
        _port = L
    return _port


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def _load_ref():
    global _ref
    if _ref is None:
        if not os.path.exists(REF_SO):
            build()
        if not os.path.exists(REF_SO):
            raise RuntimeError("reference build oracle/_ref/libholoquant_ref.so is unavailable")
        L = C.CDLL(REF_SO)
        sig = {
            "hqref_last_error": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]),
            "hqref_locate": (C.c_int, [C.c_double, C.c_double, C.c_int, C.c_double, C.POINTER(C.c_int),
                                       C.POINTER(C.c_double), C.POINTER(C.c_int)]),
            "hqref_locate_many": (C.c_uint64, [C.c_double, C.c_double, C.c_int, _p, C.c_uint64, _p, _p, _p]),
            "hqref_pli_lookup": (C.c_int, [_p, C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                           C.c_double, C.c_double, C.POINTER(C.c_double)]),
            "hqref_node_position": (C.c_double, [C.c_double, C.c_double, C.c_int, C.c_int]),
            "hqref_eval_spline": (C.c_double, [_p, C.c_int, C.c_double, C.c_double, C.c_double]),
            "hqref_dequantize_gain_code": (C.c_double, [C.c_int8, C.c_double, C.c_double]),
            "hqref_round_half_even": (C.c_double, [C.c_double]),
            "hqref_index_bits": (C.c_int, [C.c_uint32]),
            "hqref_pack_indices": (C.c_longlong, [_p, C.c_size_t, C.c_int, _p, C.c_size_t]),
            "hqref_unpack_indices": (C.c_int, [_p, C.c_size_t, C.c_uint64, C.c_int, _p]),
            "hqref_plan_memory": (C.c_int, [_p, _p, C.c_int, _p, _p]),
            "hqref_model_build": (C.c_int, [C.POINTER(RefCLayer), C.c_int, C.POINTER(_p)]),
            "hqref_model_build_dense": (C.c_int, [_p, C.c_int, C.c_int, C.c_double, C.c_double,
                                                  C.POINTER(_p), C.POINTER(_p)]),
            "hqref_model_random": (C.c_int, [_p, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_int, C.c_int,
                                             C.POINTER(_p)]),
            "hqref_model_deserialize": (C.c_int, [_p, C.c_size_t, C.POINTER(_p)]),
            "hqref_model_serialize": (C.c_longlong, [_p, _p, C.c_size_t]),
            "hqref_model_free": (None, [_p]),
            "hqref_assign_indices": (C.c_int, [_p, C.c_uint64, C.c_int, _p, C.c_int, _p]),
            "hqref_kmeans_codebook": (C.c_int, [_p, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_uint64, _p,
                                                C.POINTER(C.c_int)]),
            "hqref_model_nlayers": (C.c_int, [_p]),
            "hqref_model_layer": (C.c_int, [_p, C.c_int, C.POINTER(OracleLayer)]),
            "hqref_forward": (C.c_int, [_p, _p, C.c_int, _p, C.c_int, C.POINTER(C.c_uint64)]),
            "hqref_dense_oracle_forward": (C.c_int, [_p, _p, C.c_int, _p]),
            "hqref_bench": (C.c_int, [_p, C.c_int, C.c_int, C.c_int, C.c_uint64, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), C.POINTER(C.c_double)]),
            "hqref_projected_storage": (C.c_int, [C.c_uint64, C.c_uint64, C.c_uint64, C.c_int, C.c_int, _p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _ref = L
    return _ref


def port():
    return _load_port()


def ref():
    return _load_ref()


class RefError(Exception):
    def __init__(self, code, msg, offset=0, fault=-1):
        super().__init__(msg)
        self.code, self.offset, self.fault = code, offset, fault


def _ref_check(rc: int):
    if rc:
        buf = C.create_string_buffer(1024)
        off = C.c_uint64(0)
        fault = C.c_int(-1)
        ref().hqref_last_error(buf, len(buf), C.byref(off), C.byref(fault))
        raise RefError(rc, buf.value.decode(), off.value, fault.value)


# ---------------------------------------------------------------------------
# table views

class Tables:
    """RuntimeLayer-equivalent numpy tables for one layer (+ header fields)."""

    FIELDS = ("table_f32", "table_i8", "idx16", "idx32", "gains_f32", "biases_f32", "gain_codes", "bias_codes")
    DTYPES = dict(table_f32=np.float32, table_i8=np.int8, idx16=np.uint16, idx32=np.uint32,
                  gains_f32=np.float32, biases_f32=np.float32, gain_codes=np.int8, bias_codes=np.int8)

    def __init__(self, **kw):
        self.in_dim = kw["in_dim"]
        self.out_dim = kw["out_dim"]
        self.grid_size = kw["grid_size"]
        self.k = kw["k"]
        self.domain_lo = kw.get("domain_lo", -1.0)
        self.domain_hi = kw.get("domain_hi", 1.0)
        self.flags = kw.get("flags", 0)
        self.codebook_scale = kw.get("codebook_scale", 0.0)
        self.gain_log_min = kw.get("gain_log_min", 0.0)
        self.gain_log_step = kw.get("gain_log_step", 1.0)
        self.bias_scale = kw.get("bias_scale", 0.0)
        for f in self.FIELDS:
            v = kw.get(f)
            setattr(self, f, None if v is None else np.ascontiguousarray(v, dtype=self.DTYPES[f]))

    @classmethod
    def from_runtime(cls, rl) -> "Tables":
        """From a paper_2512_15742_b200.RuntimeLayer."""
        h = rl.header
        return cls(in_dim=h.in_dim, out_dim=h.out_dim, grid_size=h.grid_size, k=h.k, domain_lo=h.domain_lo,
                   domain_hi=h.domain_hi, flags=h.flags, codebook_scale=h.codebook_scale,
                   gain_log_min=h.gain_log_min, gain_log_step=h.gain_log_step, bias_scale=h.bias_scale,
                   **{f: getattr(rl, f) for f in cls.FIELDS})

    def to_c(self) -> OracleLayer:
        o = OracleLayer()
        for f in ("in_dim", "out_dim", "grid_size", "k", "domain_lo", "domain_hi", "flags", "codebook_scale",
                  "gain_log_min", "gain_log_step", "bias_scale"):
            setattr(o, f, getattr(self, f))
        for f in self.FIELDS:
            a = getattr(self, f)
            setattr(o, f, None if a is None or a.size == 0 else a.ctypes.data)
        return o

    def to_runtime(self):
        from paper_2512_15742_b200.lutham import LayerHeader, RuntimeLayer
        h = LayerHeader(self.in_dim, self.out_dim, self.grid_size, self.k, self.domain_lo, self.domain_hi,
                        self.flags, 0, self.codebook_scale, self.gain_log_min, self.gain_log_step,
                        self.bias_scale)
        return RuntimeLayer(h, **{f: getattr(self, f) for f in self.FIELDS})


def _c_layers(tables: Sequence[Tables]):
    return (OracleLayer * len(tables))(*[t.to_c() for t in tables])


# ---------------------------------------------------------------------------
# forward (port or reference)

def port_forward(tables: Sequence[Tables], inputs: np.ndarray, batch: int, threads: int = 1):
    """oracle_compressed_forward(_mt): returns (outputs, interp_ops)."""
    L = port()
    arr = _c_layers(tables)
    x = np.ascontiguousarray(inputs, dtype=np.float64)
    out = np.zeros(batch * tables[-1].out_dim, dtype=np.float64)
    ops = C.c_uint64(0)
    if threads <= 1:
        width = max(max(t.in_dim, t.out_dim) for t in tables)
        scratch = np.zeros(2 * width)
        rc = L.oracle_compressed_forward(arr, len(tables), x.ctypes.data, batch, out.ctypes.data,
                                         scratch.ctypes.data, C.byref(ops))
    else:
        rc = L.oracle_compressed_forward_mt(arr, len(tables), x.ctypes.data, batch, out.ctypes.data, threads,
                                            C.byref(ops))
    if rc:
        raise RefError(rc, "oracle forward failed")
    return out, ops.value


def port_forward_l1(tables: Sequence[Tables], inputs: np.ndarray, batch: int, threads: int = 1):
    """The port's forward plus the fast mode's per-output tolerance scale
    max(|y|, sum_i |term_ij|) of the last layer (tests/helpers.py): returns
    (outputs, scale).  Outputs are bitwise those of port_forward."""
    L = port()
    arr = _c_layers(tables)
    x = np.ascontiguousarray(inputs, dtype=np.float64)
    out = np.zeros(batch * tables[-1].out_dim, dtype=np.float64)
    scale = np.zeros_like(out)
    rc = L.oracle_forward_l1_mt(arr, len(tables), x.ctypes.data, batch, out.ctypes.data, scale.ctypes.data,
                                max(1, threads))
    if rc:
        raise RefError(rc, "oracle forward failed")
    return out, scale


class RefModel:
    """A holoquant::Model living in the reference library."""

    def __init__(self, handle):
        self.h = handle

    def __del__(self):
        try:
            if self.h:
                ref().hqref_model_free(self.h)
        except Exception:
            pass

    def nlayers(self) -> int:
        return ref().hqref_model_nlayers(self.h)

    def tables(self) -> List[Tables]:
        """Copy out the RuntimeLayer tables (lutham.hpp:91-109)."""
        out = []
        for l in range(self.nlayers()):
            o = OracleLayer()
            ref().hqref_model_layer(self.h, l, C.byref(o))
            e = o.in_dim * o.out_dim
            kg = o.k * o.grid_size if o.k else e * o.grid_size
            lens = dict(table_f32=kg, table_i8=kg, idx16=e, idx32=e, gains_f32=e, biases_f32=e, gain_codes=e,
                        bias_codes=e)
            kw = {f: getattr(o, f) for f in ("in_dim", "out_dim", "grid_size", "k", "domain_lo", "domain_hi",
                                               "flags", "codebook_scale", "gain_log_min", "gain_log_step",
                                               "bias_scale")}
            for f in Tables.FIELDS:
                p = getattr(o, f)
                if p:
                    ct = np.ctypeslib.as_ctypes_type(Tables.DTYPES[f])
                    kw[f] = np.ctypeslib.as_array(C.cast(p, C.POINTER(ct)), shape=(lens[f],)).copy()
            out.append(Tables(**kw))
        return out

    def forward(self, inputs: np.ndarray, batch: int, threads: int = 1):
        x = np.ascontiguousarray(inputs, dtype=np.float64)
        nout = self.tables_out_dim()
        out = np.zeros(batch * nout)
        ops = C.c_uint64(0)
        _ref_check(ref().hqref_forward(self.h, x.ctypes.data if x.size else None, batch,
                                       out.ctypes.data if out.size else None, threads, C.byref(ops)))
        return out, ops.value

    def dense_oracle_forward(self, inputs: np.ndarray, batch: int):
        x = np.ascontiguousarray(inputs, dtype=np.float64)
        out = np.zeros(batch * self.tables_out_dim())
        _ref_check(ref().hqref_dense_oracle_forward(self.h, x.ctypes.data, batch, out.ctypes.data))
        return out

    def tables_out_dim(self) -> int:
        o = OracleLayer()
        ref().hqref_model_layer(self.h, self.nlayers() - 1, C.byref(o))
        return o.out_dim

    def serialize(self) -> bytes:
        n = ref().hqref_model_serialize(self.h, None, 0)
        buf = (C.c_uint8 * n)()
        ref().hqref_model_serialize(self.h, buf, n)
        return bytes(buf)

    def bench(self, batch, repeats=101, warmup=10, seed=12345):
        med, p25, p75 = C.c_double(), C.c_double(), C.c_double()
        _ref_check(ref().hqref_bench(self.h, batch, repeats, warmup, seed, C.byref(med), C.byref(p25),
                                     C.byref(p75)))
        return med.value, p25.value, p75.value


def ref_build(cn) -> RefModel:
    """holoquant::build_model on a paper_2512_15742_b200.CompressedNetwork."""
    keep = []
    arr = (RefCLayer * len(cn.layers))()
    for q, cl in enumerate(cn.layers):
        d = arr[q]
        d.in_dim, d.out_dim, d.grid_size, d.k = cl.in_dim, cl.out_dim, cl.grid_size, cl.codebook.k
        d.domain_lo, d.domain_hi = cl.domain_lo, cl.domain_hi
        cb = np.ascontiguousarray(cl.codebook.entries, np.float64)
        idx = np.ascontiguousarray(cl.indices, np.uint32)
        g = np.ascontiguousarray(cl.gains, np.float64)
        b = np.ascontiguousarray(cl.biases, np.float64)
        keep += [cb, idx, g, b]
        d.codebook, d.indices, d.gains, d.biases = cb.ctypes.data, idx.ctypes.data, g.ctypes.data, b.ctypes.data
        if cl.int8 is not None:
            t = cl.int8
            cc = np.ascontiguousarray(t.codebook_codes, np.int8)
            gc = np.ascontiguousarray(t.gain_codes, np.int8)
            bc = np.ascontiguousarray(t.bias_codes, np.int8)
            keep += [cc, gc, bc]
            d.has_int8 = 1
            d.codebook_codes, d.gain_codes, d.bias_codes = cc.ctypes.data, gc.ctypes.data, bc.ctypes.data
            d.codebook_scale, d.gain_log_min = t.codebook_scale, t.gain_log_min
            d.gain_log_step, d.bias_scale = t.gain_log_step, t.bias_scale
    h = C.c_void_p()
    _ref_check(ref().hqref_model_build(arr, len(cn.layers), C.byref(h)))
    return RefModel(h)


def ref_random(dims: Sequence[int], grid: int, sigma: float, seed: int, k: int, int8: bool) -> RefModel:
    """The reference tests' fixture generator (init_network + compress_network
    [+ quantize]); k == 0 gives build_dense_model."""
    d = np.asarray(dims, dtype=np.int32)
    h = C.c_void_p()
    _ref_check(ref().hqref_model_random(d.ctypes.data, len(d), grid, sigma, seed, k, int(int8), C.byref(h)))
    return RefModel(h)


def ref_deserialize(data: bytes) -> RefModel:
    buf = np.frombuffer(data, dtype=np.uint8).copy()
    h = C.c_void_p()
    _ref_check(ref().hqref_model_deserialize(buf.ctypes.data if buf.size else None, buf.size, C.byref(h)))
    return RefModel(h)


def ref_locate(lo, hi, G, x):
    i, t, c = C.c_int(), C.c_double(), C.c_int()
    _ref_check(ref().hqref_locate(lo, hi, G, x, C.byref(i), C.byref(t), C.byref(c)))
    return i.value, t.value, bool(c.value)


def port_locate(lo, hi, G, x):
    i, t, c = C.c_int(), C.c_double(), C.c_int()
    rc = port().oracle_locate(lo, hi, G, x, C.byref(i), C.byref(t), C.byref(c))
    if rc:
        raise RefError(rc, "spline evaluated at non-finite x")
    return i.value, t.value, bool(c.value)


def _locate_many(fn, lo, hi, G, xs):
    x = np.ascontiguousarray(xs, dtype=np.float64)
    idx = np.zeros(x.size, np.int32)
    t = np.zeros(x.size, np.float64)
    cl = np.zeros(x.size, np.uint8)
    bad = fn(lo, hi, G, x.ctypes.data, x.size, idx.ctypes.data, t.ctypes.data, cl.ctypes.data)
    return idx, t, cl, int(bad)


def port_locate_many(lo, hi, G, xs):
    """oracle_locate_many: (index, t, clamped, n_nonfinite)."""
    return _locate_many(port().oracle_locate_many, lo, hi, G, xs)


def port_assign_indices(shapes: np.ndarray, entries: np.ndarray) -> np.ndarray:
    """oracle_assign_indices (gsb.cpp:275-286 restated): nearest codebook row
    per shape, f64 squared distance in dim order, ties to the lowest row."""
    s = np.ascontiguousarray(shapes, dtype=np.float64)
    e = np.ascontiguousarray(entries, dtype=np.float64)
    out = np.zeros(s.shape[0], np.uint32)
    port().oracle_assign_indices(s.ctypes.data, s.shape[0], s.shape[1], e.ctypes.data, e.shape[0], out.ctypes.data)
    return out


def ref_assign_indices(shapes: np.ndarray, entries: np.ndarray) -> np.ndarray:
    """holoquant::assign_indices (the reference, compiled) on row-major arrays."""
    s = np.ascontiguousarray(shapes, dtype=np.float64)
    e = np.ascontiguousarray(entries, dtype=np.float64)
    out = np.zeros(s.shape[0], np.uint32)
    _ref_check(ref().hqref_assign_indices(s.ctypes.data, s.shape[0], s.shape[1], e.ctypes.data, e.shape[0],
                                          out.ctypes.data))
    return out


def ref_kmeans_codebook(shapes: np.ndarray, k: int, seed: int, max_iters: int = 50) -> np.ndarray:
    """holoquant::kmeans_codebook entries (k x dim) for test codebooks."""
    s = np.ascontiguousarray(shapes, dtype=np.float64)
    e = np.zeros((k, s.shape[1]), np.float64)
    it = C.c_int(0)
    _ref_check(ref().hqref_kmeans_codebook(s.ctypes.data, s.shape[0], s.shape[1], k, max_iters, seed, e.ctypes.data,
                                           C.byref(it)))
    return e


def ref_locate_many(lo, hi, G, xs):
    """holoquant::locate over an array: (index, t, clamped, n_nonfinite)."""
    return _locate_many(ref().hqref_locate_many, lo, hi, G, xs)
