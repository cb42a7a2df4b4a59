"""ctypes binding of the C ABI in include/skan.h (libskan.so, built in-tree).

There is no fallback: if the CUDA library is missing the import of any
compute entry point raises immediately (the product never routes through the
CPU oracle).
"""
from __future__ import annotations

import ctypes as C
import os

from . import errors

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libskan.so")

SKAN_OK = 0
SKAN_FLAG_INT8 = 1
SKAN_LAYER_COMPRESSED, SKAN_LAYER_DENSE, SKAN_LAYER_RUNTIME = 0, 1, 2
SKAN_MODE_FAST, SKAN_MODE_EXACT = 0, 1
SKAN_PTR_HOST, SKAN_PTR_DEVICE = 0, 1


class LayerHeaderC(C.Structure):
    _fields_ = [
        ("in_dim", C.c_uint32), ("out_dim", C.c_uint32), ("grid_size", C.c_uint32), ("k", C.c_uint32),
        ("domain_lo", C.c_double), ("domain_hi", C.c_double),
        ("flags", C.c_uint32), ("reserved", C.c_uint32),
        ("codebook_scale", C.c_double), ("gain_log_min", C.c_double),
        ("gain_log_step", C.c_double), ("bias_scale", C.c_double),
    ]


class LayerPlanC(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "codebook_bytes", "index_bytes", "unpacked_index_bytes", "gain_bytes", "bias_bytes", "device_bytes")]


class MemoryPlanC(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in ("scratch_bytes", "payload_total", "working_set_total", "device_total")]


_p = C.c_void_p


class LayerDescC(C.Structure):
    _fields_ = [
        ("kind", C.c_int),
        ("header", LayerHeaderC),
        ("codebook", _p), ("n_codebook", C.c_uint64),
        ("indices", _p), ("gains", _p), ("biases", _p),
        ("n_indices", C.c_uint64), ("n_gains", C.c_uint64), ("n_biases", C.c_uint64),
        ("has_int8", C.c_int),
        ("codebook_codes", _p), ("gain_codes", _p), ("bias_codes", _p),
        ("n_codebook_codes", C.c_uint64), ("n_gain_codes", C.c_uint64), ("n_bias_codes", C.c_uint64),
        ("codebook_scale", C.c_double), ("gain_log_min", C.c_double),
        ("gain_log_step", C.c_double), ("bias_scale", C.c_double),
        ("coefficients", _p), ("n_coefficients", C.c_uint64),
        ("table_f32", _p), ("table_i8", _p), ("idx16", _p), ("idx32", _p),
        ("gains_f32", _p), ("biases_f32", _p), ("rt_gain_codes", _p), ("rt_bias_codes", _p),
    ]


# name -> (restype, argtypes)
_SIGS = {
    "skan_last_error": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(C.c_uint64), C.POINTER(C.c_int)]),
    "skan_status_name": (C.c_char_p, [C.c_int]),
    "skan_abi_version": (C.c_int, []),
    "skan_index_bits": (C.c_int, [C.c_uint32]),
    "skan_plan_memory": (C.c_int, [C.POINTER(LayerHeaderC), C.c_int, C.POINTER(LayerPlanC), C.POINTER(MemoryPlanC)]),
    "skan_head_create": (C.c_int, [C.POINTER(LayerDescC), C.c_int, C.c_int, C.POINTER(_p)]),
    "skan_head_load": (C.c_int, [_p, C.c_size_t, C.c_int, C.POINTER(_p)]),
    "skan_head_load_file": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(_p)]),
    "skan_head_destroy": (C.c_int, [_p]),
    "skan_head_swap": (C.c_int, [_p, C.POINTER(LayerDescC), C.c_int, _p]),
    "skan_head_swap_bytes": (C.c_int, [_p, _p, C.c_size_t, _p]),
    "skan_head_num_layers": (C.c_int, [_p]),
    "skan_head_input_dim": (C.c_int, [_p]),
    "skan_head_output_dim": (C.c_int, [_p]),
    "skan_head_max_width": (C.c_int, [_p]),
    "skan_head_device": (C.c_int, [_p]),
    "skan_head_layer_header": (C.c_int, [_p, C.c_int, C.POINTER(LayerHeaderC)]),
    "skan_head_plan": (C.c_int, [_p, C.POINTER(LayerPlanC), C.POINTER(MemoryPlanC)]),
    "skan_head_edges": (C.c_uint64, [_p]),
    "skan_head_set_l2_persist": (C.c_int, [_p, _p, C.c_float]),
    "skan_workspace_create": (C.c_int, [_p, C.c_int, C.POINTER(_p)]),
    "skan_workspace_destroy": (C.c_int, [_p]),
    "skan_workspace_interp_ops": (C.c_uint64, [_p]),
    "skan_workspace_max_batch": (C.c_int, [_p]),
    "skan_workspace_width": (C.c_int, [_p]),
    "skan_workspace_last_launches": (C.c_int, [_p]),
    "skan_forward": (C.c_int, [_p, _p, _p, C.c_uint64, C.c_int, _p, C.c_uint64, C.c_int, C.c_uint, _p]),
    "skan_forward_async": (C.c_int, [_p, _p, _p, C.c_int, _p, C.c_int, _p]),
    "skan_workspace_check": (C.c_int, [_p]),
    "skan_profile_gather": (C.c_int, [_p, _p, C.c_int, C.c_int, C.c_int, _p]),
    "skan_debug_b1_timeline": (C.c_int, [_p, _p]),
    "skan_head_b1_grid": (C.c_int, [_p]),
    "skan_forward_multi": (C.c_int, [C.POINTER(_p), C.POINTER(_p), C.c_int, _p, C.c_int, C.POINTER(_p), C.c_int, _p]),
    "skan_pli_lookup": (C.c_int, [_p, C.c_int, C.c_int, _p, _p, _p, _p, C.c_double, C.c_double, C.c_int, _p, _p]),
    "skan_locate": (C.c_int, [_p, C.c_int, C.c_double, C.c_double, C.c_int, _p, _p, _p, _p]),
    "skan_unpack_indices": (C.c_int, [_p, C.c_size_t, C.c_uint64, C.c_int, _p, _p]),
    "skan_debug_gemm_tf32": (C.c_int, [_p, _p, _p, C.c_int, C.c_int, C.c_int, _p]),
    "skan_debug_gemm_timeline": (C.c_int, [_p]),
    "skan_debug_set_gemm_min_batch": (C.c_int, [C.c_int]),
    "skan_debug_set_fuse_reduce": (C.c_int, [C.c_int]),
    "skan_profile_gemm": (C.c_int, [_p, _p, C.c_int, C.c_int, _p, C.POINTER(C.c_double)]),
    "skan_assign_indices": (C.c_int, [_p, C.c_uint64, C.c_int, _p, C.c_int, _p, C.c_uint, _p]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def lib() -> C.CDLL:
    """Load libskan.so (raises if it was not built — there is no CPU path)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the LUTHAM forward has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(status: int) -> None:
    """Raise the holoquant-equivalent exception for a non-OK status."""
    if status == SKAN_OK:
        return
    buf = C.create_string_buffer(1024)
    off = C.c_uint64(0)
    fault = C.c_int(-1)
    lib().skan_last_error(buf, len(buf), C.byref(off), C.byref(fault))
    raise errors.from_status(status, buf.value.decode(errors="replace"), off.value, fault.value)
