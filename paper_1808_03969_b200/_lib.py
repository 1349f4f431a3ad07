"""ctypes declarations of include/rii.h (argument marshalling only).

The shared library is built in-tree by ``paper_1808_03969_b200.build``.  There is
no CPU fallback: if the library cannot be loaded, or no CUDA device is usable,
every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# RII_LIB=checked selects the bounds-checked build (librii_b200_checked.so: device-side
# index / shared-memory layout assertions and a device sync after every launch; see
# common.cuh RII_DCHECK) -- the same kernels, for test runs only.
LIB_PATH = os.path.join(HERE, "librii_b200_checked.so" if os.environ.get("RII_LIB") == "checked"
                        else "librii_b200.so")

RII_OK, RII_ERR_ARG, RII_ERR_STATE, RII_ERR_OOM, RII_ERR_CUDA, RII_ERR_NCCL, RII_ERR_TRAIN = range(7)
PATH_AUTO, PATH_LINEAR, PATH_IVF = 0, 1, 2
IVF_LISTS, IVF_PAPER = 0, 1
MEM_HOST, MEM_DEVICE = 0, 1
NCCL_ID_BYTES = 128

# name -> (restype, argtypes); every symbol include/rii.h declares.
_p, _i32, _i64, _u64 = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64
SIGNATURES = {
    "rii_last_error": (C.c_char_p, [_p]),
    "rii_launch_count": (_u64, []),
    "rii_kernel_timing": (None, [_i32]),
    "rii_kernel_timing_read": (C.c_int, [_i32, C.POINTER(C.c_double), C.POINTER(_i64)]),
    "rii_debug_counters": (C.c_int, [_i32]),
    "rii_debug_counters_read": (C.c_int, [C.POINTER(_i64), _i32]),
    "rii_shard_range": (C.c_int, [_i64, _i32, _i32, C.POINTER(_i64), C.POINTER(_i64)]),
    "rii_nccl_unique_id": (C.c_int, [_p]),
    "rii_create": (C.c_int, [_i32, _i32, _i32, _i32, _i32, _i32, _p, C.POINTER(_p)]),
    "rii_create_with_transport": (C.c_int, [_i32, _i32, _i32, _i32, _i32, _i32, _p, C.POINTER(_p)]),
    "rii_destroy": (None, [_p]),
    "rii_train": (C.c_int, [_p, _p, _i64, _i32, _u64, C.c_int, _p]),
    "rii_add": (C.c_int, [_p, _p, _i64, C.c_int, _p, C.POINTER(_i64)]),
    "rii_set_rotation": (C.c_int, [_p, _p]),
    "rii_get_rotation": (C.c_int, [_p, _p, C.POINTER(_i32)]),
    "rii_rotate": (C.c_int, [_p, _p, _i64, _p, _p]),
    "rii_train_opq": (C.c_int, [_p, _p, _i64, _i32, _i32, _u64, C.c_int, _p]),
    "rii_reconfigure": (C.c_int, [_p, _i32, _i32, _u64, _p]),
    "rii_query": (C.c_int, [_p, _p, _i64, _i32, _p, _i64, _i32, C.c_int, C.c_int, _p, _p, _p, C.POINTER(_i32)]),
    "rii_partial_width": (_i32, [_i32]),
    "rii_query_partial": (C.c_int, [_p, _p, _i64, _i32, _p, _i64, _i32, C.c_int, _p, _p, C.POINTER(_i32)]),
    "rii_merge_partials": (C.c_int, [_p, _i32, _i64, _i32, _p, _p, _p]),
    "rii_get_codebook": (C.c_int, [_p, _p]),
    "rii_set_codebook": (C.c_int, [_p, _p]),
    "rii_get_codes": (C.c_int, [_p, _i64, _i64, _p]),
    "rii_get_centers": (C.c_int, [_p, _p]),
    "rii_get_postings": (C.c_int, [_p, _p, _p]),
    "rii_set_centers": (C.c_int, [_p, _p, _i32, _p]),
    "rii_save": (C.c_int, [_p, C.c_char_p]),
    "rii_load": (C.c_int, [C.c_char_p, _i32, _p, C.POINTER(_p)]),
    "rii_set_theta": (C.c_int, [_p, _i64]),
    "rii_set_ivf_mode": (C.c_int, [_p, _i32]),
    "rii_calibrate_theta": (C.c_int, [_p, _p, _i64, _i32, _p, _i32, C.c_int, _p, C.POINTER(C.c_double),
                                      C.POINTER(C.c_double), _p]),
    "rii_get_info": (C.c_int, [_p, C.POINTER(_i64), C.POINTER(_i32), C.POINTER(_i64), C.POINTER(_i64),
                               C.POINTER(_i64)]),
}

# struct rii_transport (include/rii.h): host all-gather callback for world > 1
TRANSPORT_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)


class Transport(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allgather", TRANSPORT_FN)]


_lib = None


class RiiError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"rii status {status}: {msg}")
        self.status = status


def load(path: str = LIB_PATH):
    """Load librii_b200.so (raises if it is missing: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(path):
            raise RuntimeError(f"{path} not built; run `python -m paper_1808_03969_b200.build`")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(lib, name)
            f.restype = res
            f.argtypes = args
        _lib = lib
    return _lib


def check(status: int):
    if status != RII_OK:
        raise RiiError(status, load().rii_last_error(None).decode())
