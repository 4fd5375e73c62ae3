"""paper_2604_25422_b200 -- B200-native S4ConvD depthwise conv1d (fwd / dX / dW).

The product is the C-ABI shared library ``libks_dwconv1d.so`` (sm_100a
kernels, C ABI in include/ks_dwconv1d.h, C++ drop-in in
include/kernelscope/conv_core.hpp).  This package is its Python mirror of
the reference operator interface (``conv``) plus the ctypes loader.
"""
from ._lib import (CHUNKED, FUSED, HIERARCHICAL, PAIRWISE, SEPARATE, SEQUENTIAL, KsError,
                   LIB_PATH, lib)
from .conv import (Comm, DimensionError, Peer, backward, backward_input, backward_weight, fill_pm1, forward,
                   get_option, launch_count, make_inputs, options, plan, rank_tree_sum, set_option, shard_rows,
                   step_host, variant, workspace_bytes)

__all__ = [
    "SEPARATE", "FUSED", "SEQUENTIAL", "PAIRWISE", "CHUNKED", "HIERARCHICAL", "KsError",
    "LIB_PATH", "lib", "Comm", "DimensionError", "forward", "backward", "backward_input", "backward_weight",
    "workspace_bytes", "fill_pm1", "make_inputs", "shard_rows", "step_host", "variant",
    "Peer", "plan", "rank_tree_sum", "set_option", "get_option", "options", "launch_count",
]
