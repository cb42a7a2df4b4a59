"""Multi-GPU partitioning of the LUTHAM forward: one process
per GPU, torch.distributed for the plumbing (NCCL on B200s, gloo on CPU for
the tests).

The reference forward has no cross-sample state (lutham.cpp:837-848), so:

  * batch sharding (cfg3): every rank holds a replica of the head and runs a
    contiguous slice of the batch -- no collective on the hot path; outputs
    are all-gathered only when one consumer needs all of them;
  * output-column sharding (cfg4, very wide heads): rank r owns a contiguous
    block of layer 0's output columns (its slice of the edge tables,
    edge e = i*out + j, kan.hpp:40-42), the hidden activations are
    all-gathered once, and the narrow tail layers are replicated.  Each output
    column's sum over i is untouched by the split, so exact mode stays
    bitwise equal to the unsharded forward;
  * head sharding (cfg5): H heads are split into contiguous groups, the
    shared f64 feature batch is broadcast from rank 0 (f64 because the
    bit-exact layer-0 knot selection needs the caller's doubles), each rank
    runs its group on one device batch, outputs are gathered.

A "runner" is anything with ``forward_dev(x: Tensor[f64], batch) ->
Tensor[f64]`` on its rank's device; :class:`DeviceRunner` is the product's
(libskan on the rank's GPU, no host round trip).  Exchanges are
torch.distributed collectives on those tensors: NCCL moves them GPU to GPU
over NVLink/NVSwitch; under gloo (the CPU tests, or two ranks sharing one
GPU) they are staged through host memory.  The partitioning and exchange
logic here never computes edges itself.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, List, Sequence, Tuple

import numpy as np

from .lutham import (CompressedLayer, CompressedNetwork, Codebook, Int8Tables, KanLayer, LayerHeader,
                     RuntimeLayer)


def shard_ranges(n: int, world: int) -> List[Tuple[int, int]]:
    """Contiguous, balanced [lo, hi) ranges of n items over world ranks
    (the first n % world ranks get one extra)."""
    if world < 1:
        raise ValueError("world size must be >= 1")
    base, extra = divmod(n, world)
    out, lo = [], 0
    for r in range(world):
        hi = lo + base + (1 if r < extra else 0)
        out.append((lo, hi))
        lo = hi
    return out


# ---------------------------------------------------------------------------
# column slices of a layer's edge tables (edge e = i*out + j)

def _cols(a: np.ndarray, in_dim: int, out_dim: int, lo: int, hi: int, per_edge: int = 1) -> np.ndarray:
    return np.ascontiguousarray(
        np.asarray(a).reshape(in_dim, out_dim, per_edge)[:, lo:hi, :].reshape(-1))


def column_slice_compressed(cl: CompressedLayer, lo: int, hi: int) -> CompressedLayer:
    """Output columns [lo, hi) of a CompressedLayer (gsb.hpp:91-106); the
    shared codebook is kept whole."""
    if not (0 <= lo < hi <= cl.out_dim):
        raise ValueError("bad column range")
    i, o = cl.in_dim, cl.out_dim
    out = CompressedLayer(i, hi - lo, cl.grid_size, Codebook(cl.codebook.k, cl.grid_size, cl.codebook.entries),
                          _cols(cl.indices, i, o, lo, hi), _cols(cl.gains, i, o, lo, hi),
                          _cols(cl.biases, i, o, lo, hi), cl.domain_lo, cl.domain_hi)
    if cl.int8 is not None:
        t = cl.int8
        out.int8 = Int8Tables(t.codebook_codes, _cols(t.gain_codes, i, o, lo, hi), _cols(t.bias_codes, i, o, lo, hi),
                              t.codebook_scale, t.gain_log_min, t.gain_log_step, t.bias_scale)
    return out


def column_slice_runtime(rl: RuntimeLayer, lo: int, hi: int) -> RuntimeLayer:
    """Output columns [lo, hi) of a RuntimeLayer (lutham.hpp:91-109): per-edge
    tables sliced, codebook (or, for dense layers, the per-edge grids) kept."""
    h = rl.header
    if not (0 <= lo < hi <= h.out_dim):
        raise ValueError("bad column range")
    i, o, G = h.in_dim, h.out_dim, h.grid_size
    nh = LayerHeader(**{**h.__dict__, "out_dim": hi - lo})
    s = RuntimeLayer(nh)
    if h.k == 0:
        s.table_f32 = _cols(rl.table_f32, i, o, lo, hi, G)
        return s
    s.table_f32, s.table_i8 = rl.table_f32, rl.table_i8
    for name in ("idx16", "idx32", "gains_f32", "biases_f32", "gain_codes", "bias_codes"):
        a = getattr(rl, name)
        if a is not None:
            setattr(s, name, _cols(a, i, o, lo, hi))
    return s


def column_slice_dense(kl: KanLayer, lo: int, hi: int) -> KanLayer:
    i, o, G = kl.in_dim, kl.out_dim, kl.grid_size
    return KanLayer(i, hi - lo, G, _cols(kl.coefficients, i, o, lo, hi, G), kl.domain_lo, kl.domain_hi)


# ---------------------------------------------------------------------------
# runners and collectives (device-resident data path)

class DeviceRunner:
    """A resident head on this rank's GPU behind the product C ABI.
    ``forward_dev`` takes and returns f64 tensors on the head's device: the
    forward is enqueued on the current stream (skan_forward_async), nothing
    crosses to the host."""

    def __init__(self, model, max_batch: int = 256, mode: str = "fast"):
        from . import lutham
        self.model = model
        self.ws = lutham.make_workspace(model, max_batch=max_batch)
        self.mode = mode
        self._lutham = lutham

    @property
    def output_dim(self) -> int:
        return self.model.output_dim()

    def forward_dev(self, x, batch: int):
        import torch
        y = torch.empty(batch * self.model.output_dim(), dtype=torch.float64, device=x.device)
        self._lutham.forward_async(self.model, x.contiguous(), batch, y, self.ws, mode=self.mode)
        return y

    def check(self) -> None:
        """Synchronize and raise ValueError for a non-finite input (kan.cpp:29)."""
        self.ws.check()

    def forward(self, x: np.ndarray, batch: int) -> np.ndarray:
        """Host-buffer convenience (skan_forward with SKAN_PTR_HOST)."""
        y = np.zeros(batch * self.model.output_dim())
        self._lutham.compressed_forward(self.model, np.ascontiguousarray(x, np.float64), batch, y, self.ws,
                                        mode=self.mode)
        return y


def _dist():
    import torch.distributed as dist
    return dist


def _staged(t):
    """NCCL moves CUDA tensors directly (NVLink/NVSwitch); gloo (CPU tests,
    or two ranks sharing one GPU) exchanges through host memory."""
    dist = _dist()
    return t.is_cuda and dist.get_backend() != "nccl"


def all_gather_tensor(t) -> list:
    """every rank's tensor of t's shape, in rank order, on t's device"""
    import torch
    dist = _dist()
    world = dist.get_world_size()
    src = t.cpu() if _staged(t) else t.contiguous()
    parts = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(parts, src)
    return [p.to(t.device) for p in parts] if _staged(t) else parts


def broadcast_tensor(t, src: int = 0):
    dist = _dist()
    if _staged(t):
        h = t.cpu()
        dist.broadcast(h, src=src)
        t.copy_(h)
    else:
        dist.broadcast(t, src=src)
    return t


def all_gather_rows(y_local, counts: Sequence[int], width: int):
    """Concatenate every rank's [counts[r], width] block in rank order
    (uneven counts padded to the largest); device tensors in, device out."""
    import torch
    mx = max(counts)
    buf = torch.zeros((mx, width), dtype=y_local.dtype, device=y_local.device)
    n = y_local.numel() // max(width, 1)
    buf[:n] = y_local.reshape(n, width)
    parts = all_gather_tensor(buf)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)


def all_gather_columns(y_local, batch: int, widths: Sequence[int]):
    """[batch, widths[r]] column blocks of every rank -> [batch, sum(widths)]
    in rank (= column) order, contiguous on the device."""
    import torch
    mx = max(widths)
    buf = torch.zeros((batch, mx), dtype=y_local.dtype, device=y_local.device)
    w = y_local.numel() // max(batch, 1)
    buf[:, :w] = y_local.reshape(batch, w)
    parts = all_gather_tensor(buf)
    return torch.cat([p[:, :c] for p, c in zip(parts, widths)], dim=1).contiguous()


def _check(*runners):
    for r in runners:
        if hasattr(r, "check"):
            r.check()


# ---------------------------------------------------------------------------
# the three partitionings (rank-local runners, device tensors throughout)

@dataclass
class BatchSharded:
    """cfg3: replica per rank, contiguous batch slice per rank."""
    runner: object
    rank: int
    world: int

    def forward_local(self, x_global, batch: int, in_dim: int):
        lo, hi = shard_ranges(batch, self.world)[self.rank]
        return self.runner.forward_dev(x_global[lo * in_dim:hi * in_dim], hi - lo), (lo, hi)

    def forward(self, x_global, batch: int, in_dim: int):
        """Every rank returns the full [batch * out] result (one all-gather)."""
        y, _ = self.forward_local(x_global, batch, in_dim)
        counts = [hi - lo for lo, hi in shard_ranges(batch, self.world)]
        out = all_gather_rows(y, counts, self.runner.output_dim).reshape(-1)
        _check(self.runner)
        return out


@dataclass
class ColumnSharded:
    """cfg4: rank r owns layer-0 output columns shard_ranges(out0, world)[r]
    (``shard_runner``); the hidden activations are all-gathered once on the
    device, then the replicated tail (``tail_runner``, layers 1..) finishes."""
    shard_runner: object
    tail_runner: object
    out0: int
    rank: int
    world: int

    def forward(self, x, batch: int):
        h_local = self.shard_runner.forward_dev(x, batch)
        widths = [hi - lo for lo, hi in shard_ranges(self.out0, self.world)]
        hidden = all_gather_columns(h_local, batch, widths)
        y = self.tail_runner.forward_dev(hidden.reshape(-1), batch)
        _check(self.shard_runner, self.tail_runner)
        return y


def column_sharded_layers(layers: Sequence, rank: int, world: int,
                          slicer: Callable = column_slice_runtime) -> Tuple[list, list]:
    """(this rank's layer-0 column shard as a one-layer head, the tail layers)."""
    out0 = layers[0].header.out_dim if hasattr(layers[0], "header") else layers[0].out_dim
    lo, hi = shard_ranges(out0, world)[rank]
    return [slicer(layers[0], lo, hi)], list(layers[1:])


@dataclass
class HeadSharded:
    """cfg5: heads shard_ranges(H, world)[rank] on this rank, one shared f64
    feature batch broadcast from rank 0 (f64: the bit-exact layer-0 knot
    selection needs the caller's doubles).  Device runners of one GPU run
    their heads concurrently (skan_forward_multi)."""
    runners: List[object]  # this rank's heads, in global head order
    n_heads: int
    out_dim: int           # shared by all heads
    rank: int
    world: int

    def forward(self, x, batch: int, in_dim: int):
        """Returns [H, batch, out] on every rank (heads must share out_dim)."""
        import torch
        x = broadcast_tensor(x.contiguous(), src=0)
        if self.runners and all(isinstance(r, DeviceRunner) for r in self.runners):
            from . import lutham
            ys = [torch.empty(batch * self.out_dim, dtype=torch.float64, device=x.device) for _ in self.runners]
            lutham.forward_multi([r.model for r in self.runners], [r.ws for r in self.runners], x, batch, ys,
                                 mode=self.runners[0].mode)
        else:
            ys = [r.forward_dev(x, batch) for r in self.runners]
        counts = [hi - lo for lo, hi in shard_ranges(self.n_heads, self.world)]
        width = batch * self.out_dim
        local = torch.cat(ys) if ys else torch.zeros(0, dtype=torch.float64, device=x.device)
        out = all_gather_rows(local, counts, width).reshape(self.n_heads, batch, self.out_dim)
        _check(*self.runners)
        return out
