"""B200-native (sm_100a) grid-hopping location estimation.

The hot path of arXiv 2307.16550 (Grid Hopping): zero-padded range FFT,
gather-accumulate through the location->range-bin mapping operator,
interpolation-hopping combine, fused argmax, and the direct method's dense
contraction — hand-written CUDA behind the C ABI in include/gridhop_b200.h.
"""
from . import scene
from .scene import Scene, baseline, small
from .api import (Context, HopTable, InvalidArgument, GridhopRuntimeError, DomainError, CudaError,
                  precompute_hop_table, precompute_hop_table_shard, upload_hop_table,
                  synthesize, fast_time_spectra,
                  hop_decision_map, hop_argmax, hop_estimate, campaign_hop, hop_topk,
                  campaign_hop_topk, topk_local_max,
                  location_decision_map, direct_argmax, argmax_index, lib, exported_symbols,
                  scene_hash, ght1_write, ght1_read, table_save, table_load,
                  indirect_argmin, multilaterate, hop_map_mc, hop_argmax_mc, mrf1_write,
                  mrf1_read, velocity_grid, velocity, hop_estimate_topk, campaign_run, Comm,
                  comm_unique_id)

__all__ = [
    "scene", "Scene", "baseline", "small", "Context", "HopTable", "InvalidArgument",
    "GridhopRuntimeError", "DomainError", "CudaError", "precompute_hop_table",
    "upload_hop_table", "synthesize", "fast_time_spectra", "hop_decision_map", "hop_argmax",
    "hop_estimate", "campaign_hop", "location_decision_map", "direct_argmax", "argmax_index",
    "lib", "exported_symbols", "precompute_hop_table_shard", "hop_topk", "campaign_hop_topk",
    "topk_local_max", "scene_hash", "ght1_write", "ght1_read", "table_save", "table_load",
    "indirect_argmin", "multilaterate", "hop_map_mc", "hop_argmax_mc", "mrf1_write", "mrf1_read",
    "velocity_grid", "velocity", "hop_estimate_topk", "campaign_run", "Comm", "comm_unique_id",
]
