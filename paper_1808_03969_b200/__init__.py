"""B200-native Rii (Reconfigurable Inverted Index, arXiv 1808.03969) hot path.

The method runs in hand-written sm_100a CUDA kernels behind the C ABI of
include/rii.h (librii_b200.so); this package is the thin Python binding.
"""
from ._lib import PATH_AUTO, PATH_IVF, PATH_LINEAR, RiiError, load  # noqa: F401
from .index import (Index, debug_counters, launch_count, read_debug_counters, merge_partials, nccl_unique_id, partial_width, shard_range,  # noqa: F401
                    torch_allgather)

__all__ = ["Index", "RiiError", "load", "launch_count", "merge_partials", "nccl_unique_id", "partial_width", "shard_range",
           "torch_allgather", "debug_counters", "read_debug_counters", "PATH_AUTO", "PATH_LINEAR", "PATH_IVF"]
