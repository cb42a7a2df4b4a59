"""Host-side mirror of the holoquant LUTHAM operator API over the C ABI.

Same names, argument meaning and error behaviour as the reference's C++ API
(/root/reference/proj/include/holoquant/{lutham,gsb,kan}.hpp), so parity
tests read like the reference's own doctest suites:

    model = build_model(compressed_network)          # lutham.hpp:121
    ws = make_workspace(model)                        # lutham.hpp:153
    compressed_forward(model, inputs, batch, outputs, ws)   # lutham.hpp:157

`Model` is a device head (resident tables on one B200); the tables live in
HBM/L2, not in host vectors.  Inputs/outputs may be numpy float64 arrays
(host pointers; copies happen inside the timed call) or CUDA float64 torch
tensors on the head's device (device pointers).
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field
from typing import List, Optional, Sequence

import numpy as np

from . import _lib
from .errors import ContractError, ShapeError

MODE_FAST = _lib.SKAN_MODE_FAST
MODE_EXACT = _lib.SKAN_MODE_EXACT
kFlagInt8 = _lib.SKAN_FLAG_INT8


def _mode(mode) -> int:
    if mode in ("fast", MODE_FAST, None):
        return MODE_FAST
    if mode in ("exact", MODE_EXACT):
        return MODE_EXACT
    raise ContractError(f"unknown mode {mode!r}")


# ---------------------------------------------------------------------------
# reference types (gsb.hpp:39-110, kan.hpp:36-96, lutham.hpp:30-80)

@dataclass
class LayerHeader:
    in_dim: int = 0
    out_dim: int = 0
    grid_size: int = 0
    k: int = 0  # 0 = dense
    domain_lo: float = -1.0
    domain_hi: float = 1.0
    flags: int = 0
    reserved: int = 0
    codebook_scale: float = 0.0
    gain_log_min: float = 0.0
    gain_log_step: float = 1.0
    bias_scale: float = 0.0

    def int8(self) -> bool:
        return bool(self.flags & kFlagInt8)

    def dense(self) -> bool:
        return self.k == 0

    def edge_count(self) -> int:
        return self.in_dim * self.out_dim

    def to_c(self) -> _lib.LayerHeaderC:
        return _lib.LayerHeaderC(self.in_dim, self.out_dim, self.grid_size, self.k, self.domain_lo,
                                 self.domain_hi, self.flags, self.reserved, self.codebook_scale,
                                 self.gain_log_min, self.gain_log_step, self.bias_scale)

    @classmethod
    def from_c(cls, h: _lib.LayerHeaderC) -> "LayerHeader":
        return cls(*(getattr(h, f) for f, _ in _lib.LayerHeaderC._fields_))


@dataclass
class ModelHeader:
    layers: List[LayerHeader] = field(default_factory=list)
    version: int = 1


@dataclass
class LayerPlan:
    codebook_bytes: int = 0
    index_bytes: int = 0
    unpacked_index_bytes: int = 0
    gain_bytes: int = 0
    bias_bytes: int = 0
    device_bytes: int = 0

    def payload_bytes(self) -> int:
        return self.codebook_bytes + self.index_bytes + self.gain_bytes + self.bias_bytes

    def working_set_bytes(self) -> int:
        return self.codebook_bytes + self.unpacked_index_bytes + self.gain_bytes + self.bias_bytes


@dataclass
class MemoryPlan:
    layers: List[LayerPlan] = field(default_factory=list)
    scratch_bytes: int = 0
    payload_total: int = 0
    working_set_total: int = 0
    device_total: int = 0


@dataclass
class Codebook:
    k: int
    grid_size: int
    entries: np.ndarray  # k*G float64, row-major

    def row(self, r: int) -> np.ndarray:
        return self.entries[r * self.grid_size:(r + 1) * self.grid_size]


@dataclass
class Int8Tables:
    codebook_codes: np.ndarray  # int8 k*G
    gain_codes: np.ndarray      # int8 E (log codes, 127 = exact zero)
    bias_codes: np.ndarray      # int8 E
    codebook_scale: float = 1.0
    gain_log_min: float = 0.0
    gain_log_step: float = 1.0
    bias_scale: float = 1.0


@dataclass
class CompressedLayer:
    in_dim: int
    out_dim: int
    grid_size: int
    codebook: Codebook
    indices: np.ndarray  # uint32 E, edge-major i*out+j
    gains: np.ndarray    # float64 E
    biases: np.ndarray   # float64 E
    domain_lo: float = -1.0
    domain_hi: float = 1.0
    int8: Optional[Int8Tables] = None

    def edge_count(self) -> int:
        return self.in_dim * self.out_dim


@dataclass
class CompressedNetwork:
    layers: List[CompressedLayer] = field(default_factory=list)


@dataclass
class KanLayer:
    in_dim: int
    out_dim: int
    grid_size: int
    coefficients: np.ndarray  # float64 E*G
    domain_lo: float = -1.0
    domain_hi: float = 1.0

    def edge_count(self) -> int:
        return self.in_dim * self.out_dim


@dataclass
class KanNetwork:
    layers: List[KanLayer] = field(default_factory=list)


@dataclass
class RuntimeLayer:
    """Resident tables of one layer (lutham.hpp:91-109)."""
    header: LayerHeader
    table_f32: Optional[np.ndarray] = None
    table_i8: Optional[np.ndarray] = None
    idx16: Optional[np.ndarray] = None
    idx32: Optional[np.ndarray] = None
    gains_f32: Optional[np.ndarray] = None
    biases_f32: Optional[np.ndarray] = None
    gain_codes: Optional[np.ndarray] = None
    bias_codes: Optional[np.ndarray] = None


# ---------------------------------------------------------------------------
# planner

def index_bits(k: int) -> int:
    """lutham.cpp:47-50."""
    return int(_lib.lib().skan_index_bits(int(k)))


def plan_memory(header: ModelHeader | Sequence[LayerHeader]) -> MemoryPlan:
    """plan_memory (lutham.cpp:52-86): byte-exact sizes from headers alone."""
    layers = header.layers if isinstance(header, ModelHeader) else list(header)
    n = len(layers)
    hs = (_lib.LayerHeaderC * max(n, 1))(*[h.to_c() for h in layers])
    per = (_lib.LayerPlanC * max(n, 1))()
    tot = _lib.MemoryPlanC()
    _lib.check(_lib.lib().skan_plan_memory(hs, n, per, C.byref(tot)))
    return _plan_from_c(per, n, tot)


def _plan_from_c(per, n, tot) -> MemoryPlan:
    return MemoryPlan(
        layers=[LayerPlan(*(getattr(per[i], f) for f, _ in _lib.LayerPlanC._fields_)) for i in range(n)],
        scratch_bytes=tot.scratch_bytes, payload_total=tot.payload_total,
        working_set_total=tot.working_set_total, device_total=tot.device_total)


# ---------------------------------------------------------------------------
# device heads

def _ptr(a: Optional[np.ndarray]) -> Optional[int]:
    return None if a is None else a.ctypes.data


class Model:
    """A resident head on one GPU (the B200 counterpart of holoquant::Model)."""

    def __init__(self, handle: C.c_void_p, keepalive=None):
        self._h = handle
        self._keep = keepalive  # host arrays only needed during creation
        self.layers: List[LayerHeader] = self._refresh_layers()
        self._keep = None

    def _refresh_layers(self) -> List[LayerHeader]:
        L = _lib.lib()
        out = []
        for l in range(L.skan_head_num_layers(self._h)):
            hc = _lib.LayerHeaderC()
            _lib.check(L.skan_head_layer_header(self._h, l, C.byref(hc)))
            out.append(LayerHeader.from_c(hc))
        return out

    @property
    def handle(self) -> C.c_void_p:
        return self._h

    def header(self) -> ModelHeader:
        return ModelHeader(layers=list(self.layers))

    def input_dim(self) -> int:
        return _lib.lib().skan_head_input_dim(self._h)

    def output_dim(self) -> int:
        return _lib.lib().skan_head_output_dim(self._h)

    def max_width(self) -> int:
        return _lib.lib().skan_head_max_width(self._h)

    def device(self) -> int:
        return _lib.lib().skan_head_device(self._h)

    def edge_count(self) -> int:
        return int(_lib.lib().skan_head_edges(self._h))

    def plan(self) -> MemoryPlan:
        n = len(self.layers)
        per = (_lib.LayerPlanC * max(n, 1))()
        tot = _lib.MemoryPlanC()
        _lib.check(_lib.lib().skan_head_plan(self._h, per, C.byref(tot)))
        return _plan_from_c(per, n, tot)

    def set_l2_persist(self, stream: int = 0, fraction: float = 1.0) -> None:
        _lib.check(_lib.lib().skan_head_set_l2_persist(self._h, stream or None, float(fraction)))

    def close(self) -> None:
        if self._h:
            _lib.lib().skan_head_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _create(descs: List[_lib.LayerDescC], device: int, keep) -> Model:
    arr = (_lib.LayerDescC * max(len(descs), 1))(*descs)
    h = C.c_void_p()
    _lib.check(_lib.lib().skan_head_create(arr, len(descs), device, C.byref(h)))
    return Model(h, keep)


def _c64(a, dtype) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a), dtype=dtype)


def build_model(cn: CompressedNetwork, device: int = 0) -> Model:
    """build_model (lutham.cpp:214-271), validated the same way, uploaded to `device`."""
    if not cn.layers:
        raise ShapeError("model has no layers")
    descs, keep = _compressed_descs(cn)
    return _create(descs, device, keep)


def _compressed_descs(cn: CompressedNetwork):
    descs, keep = [], []
    for cl in cn.layers:
        d = _lib.LayerDescC()
        d.kind = _lib.SKAN_LAYER_COMPRESSED
        d.header = LayerHeader(cl.in_dim, cl.out_dim, cl.grid_size, cl.codebook.k, cl.domain_lo,
                               cl.domain_hi).to_c()
        if cl.codebook.grid_size != cl.grid_size:
            raise ContractError("codebook does not match layer grid size")
        cb = _c64(cl.codebook.entries, np.float64)
        idx = _c64(cl.indices, np.uint32)
        g = _c64(cl.gains, np.float64)
        b = _c64(cl.biases, np.float64)
        keep += [cb, idx, g, b]
        d.codebook, d.n_codebook = _ptr(cb), cb.size
        d.indices, d.gains, d.biases = _ptr(idx), _ptr(g), _ptr(b)
        d.n_indices, d.n_gains, d.n_biases = idx.size, g.size, b.size
        if cl.int8 is not None:
            t = cl.int8
            cc, gc, bc = (_c64(t.codebook_codes, np.int8), _c64(t.gain_codes, np.int8),
                          _c64(t.bias_codes, np.int8))
            keep += [cc, gc, bc]
            d.has_int8 = 1
            d.codebook_codes, d.gain_codes, d.bias_codes = _ptr(cc), _ptr(gc), _ptr(bc)
            d.n_codebook_codes, d.n_gain_codes, d.n_bias_codes = cc.size, gc.size, bc.size
            d.codebook_scale, d.gain_log_min = t.codebook_scale, t.gain_log_min
            d.gain_log_step, d.bias_scale = t.gain_log_step, t.bias_scale
        descs.append(d)
    return descs, keep


def swap_model(model: Model, cn: CompressedNetwork, stream=None) -> None:
    """Hot swap (skan_head_swap): refill a resident head in place from a
    CompressedNetwork of the same shapes; workspaces stay valid."""
    if not cn.layers:
        raise ShapeError("model has no layers")
    descs, keep = _compressed_descs(cn)
    arr = (_lib.LayerDescC * len(descs))(*descs)
    _lib.check(_lib.lib().skan_head_swap(model.handle, arr, len(descs), stream))
    model.layers = model._refresh_layers()
    del keep


def build_dense_model(net: KanNetwork, device: int = 0) -> Model:
    """build_dense_model (lutham.cpp:177-195): coefficients cast to float32."""
    if not net.layers:
        raise ShapeError("network needs at least one layer")
    descs, keep = [], []
    for kl in net.layers:
        d = _lib.LayerDescC()
        d.kind = _lib.SKAN_LAYER_DENSE
        d.header = LayerHeader(kl.in_dim, kl.out_dim, kl.grid_size, 0, kl.domain_lo, kl.domain_hi).to_c()
        c = _c64(kl.coefficients, np.float64)
        keep.append(c)
        d.coefficients, d.n_coefficients = _ptr(c), c.size
        descs.append(d)
    return _create(descs, device, keep)


def upload(layers: Sequence[RuntimeLayer], device: int = 0) -> Model:
    """`DeviceHead upload(const Model&)`: resident tables as-is."""
    descs, keep = [], []
    for rl in layers:
        d = _lib.LayerDescC()
        d.kind = _lib.SKAN_LAYER_RUNTIME
        d.header = rl.header.to_c()
        conv = {
            "table_f32": np.float32, "table_i8": np.int8, "idx16": np.uint16, "idx32": np.uint32,
            "gains_f32": np.float32, "biases_f32": np.float32,
        }
        for name, dt in conv.items():
            a = getattr(rl, name)
            if a is not None:
                a = _c64(a, dt)
                keep.append(a)
                setattr(d, name, _ptr(a))
        for name, cname in (("gain_codes", "rt_gain_codes"), ("bias_codes", "rt_bias_codes")):
            a = getattr(rl, name)
            if a is not None:
                a = _c64(a, np.int8)
                keep.append(a)
                setattr(d, cname, _ptr(a))
        descs.append(d)
    return _create(descs, device, keep)


def deserialize(data: bytes, device: int = 0) -> Model:
    """deserialize (lutham.cpp:532-704) straight to a device head."""
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    h = C.c_void_p()
    _lib.check(_lib.lib().skan_head_load(_ptr(buf) if buf.size else None, buf.size, device, C.byref(h)))
    return Model(h)


def swap_model_bytes(model: Model, data: bytes, stream=None) -> None:
    """Hot swap from SKAN v1 bytes (skan_head_swap_bytes): the file's sections
    go to HBM, are checked and unpacked there, and refill the resident head
    in place (same shapes); deserialize's faults are raised before anything
    is overwritten."""
    buf = np.frombuffer(bytes(data), dtype=np.uint8)
    _lib.check(_lib.lib().skan_head_swap_bytes(model.handle, _ptr(buf) if buf.size else None, buf.size, stream))
    model.layers = model._refresh_layers()


def load_model(path: str, device: int = 0) -> Model:
    """load_model (lutham.cpp:715-724)."""
    h = C.c_void_p()
    _lib.check(_lib.lib().skan_head_load_file(str(path).encode(), device, C.byref(h)))
    return Model(h)


# ---------------------------------------------------------------------------
# workspaces and forward

class Workspace:
    """holoquant::Workspace: per-stream device scratch + the interp_ops counter."""

    def __init__(self, handle: C.c_void_p):
        self._h = handle

    @property
    def handle(self):
        return self._h

    @property
    def interp_ops(self) -> int:
        return int(_lib.lib().skan_workspace_interp_ops(self._h))

    def width(self) -> int:
        return _lib.lib().skan_workspace_width(self._h)

    def max_batch(self) -> int:
        return _lib.lib().skan_workspace_max_batch(self._h)

    def last_launches(self) -> int:
        return _lib.lib().skan_workspace_last_launches(self._h)

    def check(self) -> None:
        _lib.check(_lib.lib().skan_workspace_check(self._h))

    def close(self):
        if self._h:
            _lib.lib().skan_workspace_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def make_workspace(model: Model, max_batch: int = 256) -> Workspace:
    """make_workspace (lutham.cpp:757-763); all device scratch for batches up to
    max_batch (larger batches are processed in max_batch chunks)."""
    h = C.c_void_p()
    _lib.check(_lib.lib().skan_workspace_create(model.handle, int(max_batch), C.byref(h)))
    return Workspace(h)


def _is_torch(x) -> bool:
    return type(x).__module__.startswith("torch")


def compressed_forward(model: Model, inputs, batch: int, outputs, ws: Workspace, mode="fast",
                       stream=None) -> None:
    """compressed_forward (lutham.cpp:819-850).

    numpy inputs/outputs: synchronous, host copies inside the call.
    torch CUDA tensors: enqueued on `stream` (default: torch's current
    stream), then synchronized so non-finite inputs raise ValueError like
    the reference; use forward_async to skip the sync.
    """
    L = _lib.lib()
    m = _mode(mode)
    if _is_torch(inputs) or _is_torch(outputs):
        import torch
        for t in (inputs, outputs):
            if not (_is_torch(t) and t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
                raise ContractError("device forward needs contiguous float64 CUDA tensors")
        s = stream if stream is not None else torch.cuda.current_stream(inputs.device).cuda_stream
        _lib.check(L.skan_forward(model.handle, ws.handle, inputs.data_ptr(), inputs.numel(), int(batch),
                                  outputs.data_ptr(), outputs.numel(), m, _lib.SKAN_PTR_DEVICE, s))
        ws.check()
        return
    if not (isinstance(outputs, np.ndarray) and outputs.dtype == np.float64 and outputs.flags.c_contiguous):
        raise ContractError("outputs must be a contiguous float64 numpy array")
    x = np.ascontiguousarray(inputs, dtype=np.float64)
    _lib.check(L.skan_forward(model.handle, ws.handle, _ptr(x) if x.size else None, x.size, int(batch),
                              _ptr(outputs) if outputs.size else None, outputs.size, m, _lib.SKAN_PTR_HOST,
                              stream))


def forward_async(model: Model, d_inputs, batch: int, d_outputs, ws: Workspace, mode="fast",
                  stream=None) -> None:
    """Enqueue a device-pointer forward without synchronizing (ws.check() later)."""
    import torch
    s = stream if stream is not None else torch.cuda.current_stream(d_inputs.device).cuda_stream
    _lib.check(_lib.lib().skan_forward_async(model.handle, ws.handle, d_inputs.data_ptr(), int(batch),
                                             d_outputs.data_ptr(), _mode(mode), s))


def forward_multi(models: Sequence[Model], wss: Sequence[Workspace], d_inputs, batch: int, d_outputs,
                  mode="fast", stream=None) -> None:
    """H heads sharing one device feature batch (cfg5)."""
    import torch
    n = len(models)
    hs = (C.c_void_p * n)(*[m.handle for m in models])
    ws = (C.c_void_p * n)(*[w.handle for w in wss])
    ys = (C.c_void_p * n)(*[y.data_ptr() for y in d_outputs])
    s = stream if stream is not None else torch.cuda.current_stream(d_inputs.device).cuda_stream
    _lib.check(_lib.lib().skan_forward_multi(hs, ws, n, d_inputs.data_ptr(), int(batch), ys, _mode(mode), s))


# ---------------------------------------------------------------------------
# primitives on device tensors

def locate(x, lo: float, hi: float, grid_size: int):
    """Batched holoquant::locate (kan.cpp:28-58) on the GPU: (index, t, clamped)."""
    import torch
    n = x.numel()
    idx = torch.empty(n, dtype=torch.int32, device=x.device)
    t = torch.empty(n, dtype=torch.float64, device=x.device)
    cl = torch.empty(n, dtype=torch.uint8, device=x.device)
    s = torch.cuda.current_stream(x.device).cuda_stream
    _lib.check(_lib.lib().skan_locate(x.data_ptr(), n, float(lo), float(hi), int(grid_size), idx.data_ptr(),
                                      t.data_ptr(), cl.data_ptr(), s))
    return idx, t, cl


def pli_lookup(codebook, rows, g, b, x, domain_lo: float, domain_hi: float, grid_size: int):
    """Batched pli_lookup (lutham.cpp:730-739) on device tensors."""
    import torch
    n = x.numel()
    y = torch.empty(n, dtype=torch.float64, device=x.device)
    k = codebook.numel() // grid_size
    s = torch.cuda.current_stream(x.device).cuda_stream
    _lib.check(_lib.lib().skan_pli_lookup(codebook.data_ptr(), k, int(grid_size), rows.data_ptr(), g.data_ptr(),
                                          b.data_ptr(), x.data_ptr(), float(domain_lo), float(domain_hi), n,
                                          y.data_ptr(), s))
    return y


def assign_indices(shapes, codebook: Codebook) -> np.ndarray:
    """assign_indices (gsb.cpp:275-286) on the GPU: the nearest codebook row
    per shape, ties to the lowest row, bit-identical to the reference.

    shapes: a sequence of objects with a ``shape`` vector (ShapeRecord-like)
    or an (n, grid_size) float64 array.  Raises ShapeError("shape/codebook
    grid size mismatch") like the reference."""
    if isinstance(shapes, np.ndarray):
        arr = np.ascontiguousarray(shapes, dtype=np.float64)
        if arr.ndim != 2 or (arr.shape[0] and arr.shape[1] != codebook.grid_size):
            raise ShapeError("shape/codebook grid size mismatch")
    else:
        rows = [np.asarray(getattr(r, "shape", r), dtype=np.float64) for r in shapes]
        for r in rows:
            if r.size != codebook.grid_size:
                raise ShapeError("shape/codebook grid size mismatch")
        arr = np.ascontiguousarray(np.stack(rows) if rows else np.zeros((0, codebook.grid_size)))
    n = arr.shape[0]
    out = np.zeros(n, np.uint32)
    if n == 0:
        return out
    ent = np.ascontiguousarray(codebook.entries, dtype=np.float64)
    _lib.check(_lib.lib().skan_assign_indices(arr.ctypes.data, n, int(codebook.grid_size), ent.ctypes.data,
                                              int(codebook.k), out.ctypes.data, 0, None))
    return out


def unpack_indices(d_bytes, count: int, bits: int):
    """GPU unpack_indices (lutham.cpp:114-137) of a uint8 CUDA tensor."""
    import torch
    out = torch.empty(max(count, 1), dtype=torch.int32, device=d_bytes.device)
    s = torch.cuda.current_stream(d_bytes.device).cuda_stream
    _lib.check(_lib.lib().skan_unpack_indices(d_bytes.data_ptr(), d_bytes.numel(), int(count), int(bits),
                                              out.data_ptr(), s))
    return out[:count]


# ---------------------------------------------------------------------------
# benchmarking (lutham.hpp:160-183, lutham.cpp:852-951) on the device

class _MT19937_64:
    """std::mt19937_64 (the reference's bench input generator, lutham.cpp:875)."""

    def __init__(self, seed: int):
        self.mt = [0] * 312
        self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
        for i in range(1, 312):
            self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
        self.i = 312

    def _twist(self):
        mt = self.mt
        for i in range(312):
            x = (mt[i] & 0xFFFFFFFF80000000) | (mt[(i + 1) % 312] & 0x7FFFFFFF)
            xa = x >> 1
            if x & 1:
                xa ^= 0xB5026F5AA96619E9
            mt[i] = mt[(i + 156) % 312] ^ xa
        self.i = 0

    def __call__(self) -> int:
        if self.i >= 312:
            self._twist()
        y = self.mt[self.i]
        self.i += 1
        y ^= (y >> 29) & 0x5555555555555555
        y ^= (y << 17) & 0x71D67FFFEDA60000
        y ^= (y << 37) & 0xFFF7EEE000000000
        y ^= y >> 43
        return y & 0xFFFFFFFFFFFFFFFF


@dataclass
class BenchConfig:
    """lutham.hpp:160-165."""
    batch: int = 64
    repeats: int = 101
    warmup: int = 10
    seed: int = 12345


@dataclass
class BenchRow:
    """lutham.hpp:167-172 (microseconds per sample)."""
    grid_size: int = 0
    median_us: float = 0.0
    p25_us: float = 0.0
    p75_us: float = 0.0


def _percentile(sorted_v, q: float) -> float:
    """lutham.cpp:857-861: nearest-rank on the sorted samples, the index
    rounded half away from zero like std::llround (q*(n-1) >= 0)."""
    n = len(sorted_v)
    return sorted_v[int(math.floor(q * (n - 1) + 0.5))]


def bench_model(model: Model, config: BenchConfig = BenchConfig(), mode="fast") -> BenchRow:
    """bench_model (lutham.cpp:866-902) on the device: the same inputs
    (U(lo, hi) of the first layer's domain from mt19937_64(seed)), warmup,
    repeats of the synchronous host-buffer compressed_forward timed with a
    steady clock, microseconds per sample, median / p25 / p75."""
    import time
    if config.batch < 1 or config.repeats < 1 or config.warmup < 0:
        raise ShapeError("bench needs batch >= 1, repeats >= 1, warmup >= 0")
    lo, hi = model.layers[0].domain_lo, model.layers[0].domain_hi
    rng = _MT19937_64(config.seed)
    n = config.batch * model.input_dim()
    x = np.array([lo + (rng() >> 11) * 2.0 ** -53 * (hi - lo) for _ in range(n)], dtype=np.float64)
    y = np.zeros(config.batch * model.output_dim())
    ws = make_workspace(model, max_batch=config.batch)
    for _ in range(config.warmup):
        compressed_forward(model, x, config.batch, y, ws, mode=mode)
    samples = []
    for _ in range(config.repeats):
        t0 = time.perf_counter()
        compressed_forward(model, x, config.batch, y, ws, mode=mode)
        samples.append((time.perf_counter() - t0) * 1e6 / config.batch)
    samples.sort()
    return BenchRow(model.layers[0].grid_size, _percentile(samples, 0.5), _percentile(samples, 0.25),
                    _percentile(samples, 0.75))


def bench_iso_latency(models: Sequence[Model], config: BenchConfig = BenchConfig(), mode="fast") -> List[BenchRow]:
    """bench_iso_latency (lutham.cpp:904-926): models identical apart from G."""
    if not models:
        raise ShapeError("bench needs at least one model")
    ref = models[0].layers
    for m in models:
        if len(m.layers) != len(ref):
            raise ShapeError("bench models must share topology apart from grid size")
        for a, b in zip(m.layers, ref):
            if (a.in_dim, a.out_dim, a.k, a.flags, a.domain_lo, a.domain_hi) != (
                    b.in_dim, b.out_dim, b.k, b.flags, b.domain_lo, b.domain_hi):
                raise ShapeError("bench models must share topology apart from grid size")
    return [bench_model(m, config, mode) for m in models]


def bench_csv(rows: Sequence[BenchRow]) -> str:
    """bench_csv (lutham.cpp:938-951): the same header and %.17g fields."""
    out = "G,median_us,p25_us,p75_us\n"
    for r in rows:
        out += f"{r.grid_size},{r.median_us:.17g},{r.p25_us:.17g},{r.p75_us:.17g}\n"
    return out
