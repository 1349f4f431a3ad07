"""B200-native Rii (Reconfigurable Inverted Index, arXiv 1808.03969) hot path.

The method runs in hand-written sm_100a CUDA kernels behind the C ABI of
include/rii.h (librii_b200.so); this package is the thin Python binding.
"""
from ._lib import PATH_AUTO, PATH_IVF, PATH_LINEAR, RiiError, load  # noqa: F401
from .index import Index, launch_count, merge_partials, nccl_unique_id, partial_width, shard_range  # noqa: F401

__all__ = ["Index", "RiiError", "load", "launch_count", "merge_partials", "nccl_unique_id", "partial_width", "shard_range",
           "PATH_AUTO", "PATH_LINEAR", "PATH_IVF"]
