"""ctypes binding of include/sthk.h and include/sthk_sim.h (libsthk.so)."""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_char_p, c_double, c_int, c_int64, c_uint64, c_void_p

STHK_OK = 0
STHK_EINVAL = 1
STHK_ENOTLOADED = 2
STHK_ECUDA = 3
STHK_ENCCL = 4
STHK_ERANGE = 5
NCCL_ID_BYTES = 128

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


def lib_path() -> str:
    # STHK_LIB overrides the in-tree library (kernel-variant experiments only)
    return os.environ.get("STHK_LIB") or os.path.join(_HERE, "libsthk.so")


class StatsStruct(ctypes.Structure):
    _fields_ = [
        ("n", c_int64),
        ("pairs_bg", c_int64),
        ("pairs_tr", c_int64),
        ("pairs_any", c_int64),
        ("pairs_dense", c_int64),
        ("pair_kernel_ms", c_double),
        ("eval_ms", c_double),
        ("source_chunk", ctypes.c_int32),
        ("work_items", ctypes.c_int32),
        ("n_devices", ctypes.c_int32),
        ("rank", ctypes.c_int32),
        ("world", ctypes.c_int32),
        ("exec_bg", c_int64),
        ("exec_geom", c_int64),
        ("exec_sym", c_int64),
        ("kernel_mode", ctypes.c_int32),
        ("cache_hit", ctypes.c_int32),
        ("trigger_cache_hit", ctypes.c_int32),
        ("exec_far", c_int64),
        ("kernel_launches", c_int64),
        ("far_threshold", c_double),
        ("far_split_days", c_double),
        ("graph_launches", c_int64),
        ("graph_builds", c_int64),
        ("load_zero_copy", ctypes.c_int32),
        ("trigger_rows", ctypes.c_int32),
    ]


STHK_DTYPE_U64 = 0
STHK_DTYPE_F64 = 1
ALLREDUCE_FN = ctypes.CFUNCTYPE(c_int, c_void_p, c_void_p, c_int64, c_int)
EXCHANGE_FN = ctypes.CFUNCTYPE(c_int, c_void_p, c_int, POINTER(c_int), POINTER(c_void_p),
                               POINTER(c_int64), c_int, POINTER(c_int), POINTER(c_void_p),
                               POINTER(c_int64))


class HostCommStruct(ctypes.Structure):
    """sthk_host_comm (include/sthk.h)."""
    _fields_ = [("ctx", c_void_p), ("allreduce_sum", ALLREDUCE_FN), ("exchange", EXCHANGE_FN)]


# (name, restype, argtypes) for every entry point declared in include/*.h
_DPTR = POINTER(c_double)
_IPTR = POINTER(c_int)
SIGNATURES = [
    ("sthk_create", c_int, [POINTER(c_int), c_int, POINTER(c_void_p)]),
    ("sthk_nccl_unique_id", c_int, [c_void_p]),
    ("sthk_create_rank", c_int, [c_int, c_int, c_int, c_void_p, POINTER(c_void_p)]),
    ("sthk_create_rank_hosted", c_int,
     [c_int, c_int, c_int, POINTER(HostCommStruct), POINTER(c_void_p)]),
    ("sthk_destroy", c_int, [c_void_p]),
    ("sthk_load_events", c_int, [c_void_p, c_void_p, c_void_p, c_void_p, c_int64, c_double]),
    ("sthk_set_params", c_int, [c_void_p, c_void_p]),
    ("sthk_loglik", c_int, [c_void_p, _DPTR, _IPTR, c_void_p]),
    ("sthk_loglik_grad", c_int, [c_void_p, _DPTR, _IPTR, c_void_p, c_void_p]),
    ("sthk_loglik_batch", c_int, [c_void_p, _DPTR, c_int64, _DPTR, _IPTR, _DPTR]),
    ("sthk_excitation", c_int, [c_void_p, _DPTR, _DPTR, _DPTR]),
    ("sthk_excitation_batch", c_int, [c_void_p, _DPTR, c_int64, _DPTR, _DPTR, POINTER(c_int64)]),
    ("sthk_enqueue", c_int, [c_void_p, c_int, c_int]),
    ("sthk_result", c_int, [c_void_p, _DPTR, _IPTR, c_void_p, c_void_p]),
    ("sthk_set_timing", c_int, [c_void_p, c_int]),
    ("sthk_get_stats", c_int, [c_void_p, POINTER(StatsStruct)]),
    ("sthk_get_stream", c_int, [c_void_p, c_int, POINTER(c_void_p)]),
    ("sthk_set_graphs", c_int, [c_void_p, c_int]),
    ("sthk_debug_item_trace", c_int, [c_void_p, c_int, c_void_p, c_int64, POINTER(c_int64)]),
    ("sthk_set_dense", c_int, [c_void_p, c_int]),
    ("sthk_get_exchange_bytes", c_int, [c_void_p, POINTER(c_int64)]),
    ("sthk_set_kernel", c_int, [c_void_p, c_int]),
    ("sthk_set_far_tier", c_int, [c_void_p, c_int]),
    ("sthk_set_bgonly_kernel", c_int, [c_void_p, c_int]),
    ("sthk_set_far_schedule", c_int, [c_void_p, c_int, c_int, c_int]),
    ("sthk_set_background_cache", c_int, [c_void_p, c_int]),
    ("sthk_measure_fp64_peak", c_int, [c_int, c_int, _DPTR, _DPTR]),
    ("sthk_plan_partition", c_int, [_DPTR, c_int64, _DPTR, c_int, c_int, _IPTR, _IPTR]),
    ("sthk_debug_exp", c_int, [c_int, _DPTR, c_int64, _DPTR]),
    ("sthk_last_error", c_char_p, [c_void_p]),
    ("sthk_version", c_char_p, []),
    ("sthk_sim_cloud", c_int, [c_int64, _DPTR, c_uint64, _DPTR, _DPTR, _DPTR, _DPTR]),
    ("sthk_sim_cluster", c_int,
     [_DPTR, _DPTR, c_double, c_uint64, c_int64, _DPTR, _DPTR, _DPTR, _IPTR, POINTER(c_int64)]),
]


def load_library() -> ctypes.CDLL:
    """Load the in-tree libsthk.so (fails loudly if it was not built)."""
    global _LIB
    if _LIB is not None:
        return _LIB
    path = lib_path()
    if not os.path.exists(path):
        raise ImportError(
            f"{path} is missing: build the CUDA engine first "
            "(python -c 'import __graft_entry__ as g; g.build()')")
    lib = ctypes.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib
