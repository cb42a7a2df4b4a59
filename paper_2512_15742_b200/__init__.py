"""B200-native LUTHAM forward for SHARe-KAN compressed KAN heads.

A from-scratch sm_100a implementation of holoquant's compressed_forward
path behind the reference's own operator API (see lutham.py, include/skan.h).
"""
from .errors import (ContractError, CudaError, FormatError, FormatFault, HoloquantError, PlanError,
                     ShapeError, ValueError)
from .lutham import (MODE_EXACT, MODE_FAST, BenchConfig, BenchRow, Codebook, CompressedLayer, CompressedNetwork, Int8Tables,
                     KanLayer, KanNetwork, LayerHeader, LayerPlan, MemoryPlan, Model, ModelHeader,
                     RuntimeLayer, Workspace, bench_csv, bench_iso_latency, bench_model, build_dense_model,
                     build_model, compressed_forward,
                     deserialize, forward_async, forward_multi, index_bits, kFlagInt8, load_model,
                     locate, make_workspace, pli_lookup, assign_indices, plan_memory, swap_model, swap_model_bytes, unpack_indices, upload)

__all__ = [n for n in dir() if not n.startswith("_")]
