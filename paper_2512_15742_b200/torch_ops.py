"""PyTorch operator binding: the
paper's integration boundary ``torch.ops.share_kan.pli_lookup`` plus a head
forward, registered with ``torch.library.custom_op`` over the C ABI (no
extension module: the kernels are libskan.so's, the op is the dispatcher
entry).  Each op has a fake (meta) implementation so it traces under
``torch.export`` / FakeTensor with static output shapes; the real
implementation runs on CUDA only and raises on other devices (no CPU
fallback).

    import paper_2512_15742_b200.torch_ops  # registers the ops
    y = torch.ops.share_kan.pli_lookup(codebook, rows, g, b, x, lo, hi, G)
    hid = paper_2512_15742_b200.torch_ops.register_head(model, max_batch=256)
    y = torch.ops.share_kan.head_forward(x, hid, 0)    # 0 fast, 1 exact

Resident heads are registered once (``register_head``), so the op carries
only an integer handle: the codebook and tables stay resident in HBM and
the forward allocates nothing (the workspace is made at registration,
make_workspace lutham.cpp:757-763).
"""
from __future__ import annotations

import threading
from typing import Dict, Tuple

import torch

from . import _lib
from .errors import ContractError
from .lutham import Model, Workspace, make_workspace

_heads: Dict[int, Tuple[Model, Workspace]] = {}
_lock = threading.Lock()
_next = [1]


def register_head(model: Model, max_batch: int = 256) -> int:
    """Keep `model` resident for torch.ops.share_kan.head_forward; returns
    its handle (with a workspace for batches up to max_batch)."""
    ws = make_workspace(model, max_batch)
    with _lock:
        h = _next[0]
        _next[0] += 1
        _heads[h] = (model, ws)
    return h


def unregister_head(handle: int) -> None:
    """Drop the handle (the model stays alive while the caller holds it)."""
    with _lock:
        _heads.pop(int(handle), None)


def _head(handle: int) -> Tuple[Model, Workspace]:
    with _lock:
        hw = _heads.get(int(handle))
    if hw is None:
        raise ContractError(f"share_kan: unknown head handle {handle}")
    return hw


def _need_cuda(*ts: torch.Tensor) -> None:
    for t in ts:
        if t.device.type != "cuda":
            raise ContractError("share_kan ops run on CUDA tensors only (no CPU fallback)")


@torch.library.custom_op("share_kan::pli_lookup", mutates_args=())
def pli_lookup(codebook: torch.Tensor, rows: torch.Tensor, g: torch.Tensor, b: torch.Tensor, x: torch.Tensor,
               domain_lo: float, domain_hi: float, grid_size: int) -> torch.Tensor:
    """y[n] = g[n] * LinearInterp(codebook[rows[n]], x[n]) + b[n]
    (lutham.cpp:730-739), f64, the reference's operation order."""
    _need_cuda(codebook, rows, g, b, x)
    cb = codebook.contiguous().to(torch.float64)
    r = rows.contiguous().to(torch.int32)
    gg, bb, xx = (t.contiguous().to(torch.float64) for t in (g, b, x))
    n = xx.numel()
    y = torch.empty(n, dtype=torch.float64, device=xx.device)
    if n:
        k = cb.numel() // int(grid_size)
        s = torch.cuda.current_stream(xx.device).cuda_stream
        _lib.check(_lib.lib().skan_pli_lookup(cb.data_ptr(), k, int(grid_size), r.data_ptr(), gg.data_ptr(),
                                              bb.data_ptr(), xx.data_ptr(), float(domain_lo), float(domain_hi), n,
                                              y.data_ptr(), s))
    return y.view(x.shape)


@pli_lookup.register_fake
def _(codebook, rows, g, b, x, domain_lo, domain_hi, grid_size):
    return torch.empty(x.shape, dtype=torch.float64, device=x.device)


@torch.library.custom_op("share_kan::head_forward", mutates_args=())
def head_forward(x: torch.Tensor, handle: int, mode: int) -> torch.Tensor:
    """compressed_forward (lutham.cpp:819-850) of a registered resident head
    on a [batch, in_dim] f64 CUDA tensor; returns [batch, out_dim] f64.
    mode 0 = fast, 1 = exact."""
    _need_cuda(x)
    model, ws = _head(handle)
    xx = x.contiguous().to(torch.float64)
    batch = xx.shape[0] if xx.dim() > 1 else 1
    if xx.numel() != batch * model.input_dim():
        raise ContractError("share_kan.head_forward: x must be [batch, in_dim]")
    out = torch.empty((batch, model.output_dim()), dtype=torch.float64, device=xx.device)
    s = torch.cuda.current_stream(xx.device).cuda_stream
    # stream-ordered, no host sync; a non-finite input is reported by
    # check_head(handle) (skan_workspace_check), as forward_async does
    _lib.check(_lib.lib().skan_forward_async(model.handle, ws.handle, xx.data_ptr(), int(batch), out.data_ptr(),
                                             int(mode), s))
    return out


@head_forward.register_fake
def _(x, handle, mode):
    model, _ = _head(handle)
    batch = x.shape[0] if x.dim() > 1 else 1
    return torch.empty((batch, model.output_dim()), dtype=torch.float64, device=x.device)


def check_head(handle: int) -> None:
    """Synchronize the head's last forward and raise a deferred ValueError
    (non-finite input, kan.cpp:29) if there was one."""
    _head(handle)[1].check()
