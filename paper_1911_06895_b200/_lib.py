"""ctypes binding of libdsssp.so (include/dsssp.h).

This is the product path's only route to the device: there is no CPU
fallback.  If the library is missing, `lib()` raises ImportError.
"""

from __future__ import annotations

import ctypes
import os
import threading

from .build import LIB

DS_OK, DS_EINVAL, DS_ENOCONVERGE, DS_ECUDA, DS_ENOMEM, DS_ETIMEOUT = 0, 1, 2, 3, 4, 5
DS_EPARSE, DS_EVALID = 6, 7
DS_FMT_MTX, DS_FMT_EDGES = 0, 1
DS_IDX_I32, DS_IDX_I64 = 0, 1
DS_W_F32, DS_W_F64, DS_W_I32 = 0, 1, 2
DS_FLAG_SKIP_EMPTY, DS_FLAG_FORCE_F64, DS_FLAG_NO_LEX = 1, 2, 4
DS_MODE_FIXED32, DS_MODE_F64 = 0, 1

# Every entry point include/dsssp.h declares (checked by the CPU tests).
EXPORTS = (
    "ds_graph_create", "ds_graph_prepare", "ds_sssp", "ds_sssp_batch", "ds_result_dense",
    "ds_result_sparse",
    "ds_export_split", "ds_graph_set_stream", "ds_graph_size", "ds_graph_destroy",
    "ds_last_error", "ds_device_count", "ds_gen_rmat", "ds_graph_download", "ds_debug_trace",
    "ds_shard_create", "ds_shard_destroy", "ds_shard_probe", "ds_shard_prepare", "ds_shard_begin",
    "ds_shard_scan", "ds_shard_s_add", "ds_shard_relax", "ds_shard_result", "ds_shard_from_graph",
    "ds_shard_launches", "ds_debug_cta_times",
    "ds_release_pool", "ds_ingest_parse", "ds_ingest_info", "ds_ingest_copy",
    "ds_ingest_error_line", "ds_ingest_free",
)


class PrepInfo(ctypes.Structure):
    _fields_ = [
        ("nnz_light", ctypes.c_int64),
        ("nnz_heavy", ctypes.c_int64),
        ("min_light_weight", ctypes.c_double),
        ("phase_ceiling", ctypes.c_int64),
        ("dist_mode", ctypes.c_int32),
        ("frac_bits", ctypes.c_int32),
        ("prepare_ms", ctypes.c_double),
        ("sub_buckets", ctypes.c_int32),
        ("reserved", ctypes.c_int32),
    ]


class Stats(ctypes.Structure):
    _fields_ = [
        ("outer_iterations", ctypes.c_int64),
        ("inner_phases", ctypes.c_int64),
        ("buckets_visited", ctypes.c_int64),
        ("reached", ctypes.c_int64),
        ("edges_reached", ctypes.c_int64),
        ("edges_scanned", ctypes.c_int64),
        ("grid_barriers", ctypes.c_int64),
        ("max_distance", ctypes.c_double),
        ("kernel_ms", ctypes.c_double),
        ("dist_mode", ctypes.c_int32),
        ("fallbacks", ctypes.c_int32),
        ("pull_steps", ctypes.c_int64),
        ("launches", ctypes.c_int64),
    ]

    def as_dict(self) -> dict:
        return {name: getattr(self, name) for name, _ in self._fields_}


class DsError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


_lib = None
_lock = threading.Lock()

_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i64p = ctypes.POINTER(ctypes.c_int64)


def lib():
    """Load libdsssp.so once; raise ImportError if it was never built."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = os.environ.get("DS_LIB", LIB)
        if not os.path.exists(path):
            raise ImportError(
                f"{path} is missing: build it with `python -m paper_1911_06895_b200.build` "
                "(the solver has no CPU fallback)")
        L = ctypes.CDLL(path)
        L.ds_graph_create.argtypes = [_i64, _i64, _vp, _vp, ctypes.c_int, _vp, ctypes.c_int,
                                      ctypes.c_int, _vp, ctypes.POINTER(_vp)]
        L.ds_graph_prepare.argtypes = [_vp, ctypes.c_double, ctypes.c_uint32,
                                       ctypes.POINTER(PrepInfo)]
        L.ds_sssp.argtypes = [_vp, _i64, ctypes.c_double, ctypes.c_uint32, ctypes.POINTER(Stats)]
        L.ds_sssp_batch.argtypes = [_vp, _vp, _i64, ctypes.c_double, ctypes.c_uint32, ctypes.c_int32,
                                    _vp, _vp]
        L.ds_ingest_parse.argtypes = [ctypes.c_char_p, _i64, ctypes.c_int32, ctypes.c_int32, ctypes.c_double,
                                      ctypes.c_char_p, ctypes.POINTER(_vp)]
        L.ds_ingest_info.argtypes = [_vp, _i64p, _i64p, _i64p]
        L.ds_ingest_copy.argtypes = [_vp, _vp, _vp, _vp, _vp]
        L.ds_ingest_error_line.restype = ctypes.c_int64
        L.ds_ingest_error_line.argtypes = []
        L.ds_ingest_free.restype = None
        L.ds_ingest_free.argtypes = [_vp]
        L.ds_result_dense.argtypes = [_vp, _vp]
        L.ds_result_sparse.argtypes = [_vp, _vp, _vp]
        L.ds_export_split.argtypes = [_vp, ctypes.c_int, _vp, _vp, _vp]
        L.ds_graph_set_stream.argtypes = [_vp, _vp]
        L.ds_graph_size.argtypes = [_vp, _i64p, _i64p]
        L.ds_graph_destroy.argtypes = [_vp]
        L.ds_graph_destroy.restype = None
        L.ds_release_pool.argtypes = []
        L.ds_release_pool.restype = None
        L.ds_last_error.restype = ctypes.c_char_p
        L.ds_device_count.restype = ctypes.c_int
        L.ds_gen_rmat.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_uint64,
                                  ctypes.c_uint64, ctypes.c_int, _vp, ctypes.POINTER(_vp)]
        L.ds_graph_download.argtypes = [_vp, _vp, _vp, _vp]
        L.ds_debug_trace.argtypes = [_vp, _vp, _i64]
        L.ds_debug_trace.restype = _i64
        u64 = ctypes.c_uint64
        L.ds_shard_create.argtypes = [_i64, _i64, _i64, _i64, _vp, _vp, _vp, ctypes.c_int, _vp,
                                      ctypes.POINTER(_vp)]
        L.ds_shard_destroy.argtypes = [_vp]
        L.ds_shard_destroy.restype = None
        L.ds_shard_probe.argtypes = [_vp, ctypes.c_double, _vp]
        L.ds_shard_prepare.argtypes = [_vp, ctypes.c_double, ctypes.c_int, ctypes.c_int]
        L.ds_shard_begin.argtypes = [_vp, _i64]
        L.ds_shard_scan.argtypes = [_vp, u64, u64, _vp, _vp, ctypes.POINTER(_i64),
                                    ctypes.POINTER(u64)]
        L.ds_shard_s_add.argtypes = [_vp, _vp, _vp, _i64]
        L.ds_shard_relax.argtypes = [_vp, ctypes.c_int, _vp, _vp, _i64, u64, _vp, _vp,
                                     ctypes.POINTER(_i64), ctypes.POINTER(ctypes.c_int32)]
        L.ds_shard_result.argtypes = [_vp, _vp]
        L.ds_shard_launches.argtypes = [_vp]
        L.ds_shard_launches.restype = _i64
        L.ds_shard_from_graph.argtypes = [_vp, _i64, _i64, ctypes.POINTER(_vp)]
        L.ds_shard_from_graph.restype = ctypes.c_int
        for name in ("ds_shard_create", "ds_shard_probe", "ds_shard_prepare", "ds_shard_begin",
                     "ds_shard_scan", "ds_shard_s_add", "ds_shard_relax", "ds_shard_result"):
            getattr(L, name).restype = ctypes.c_int
        for name in ("ds_graph_create", "ds_graph_prepare", "ds_sssp", "ds_result_dense",
                     "ds_result_sparse", "ds_export_split", "ds_graph_set_stream",
                     "ds_graph_size", "ds_gen_rmat", "ds_graph_download"):
            getattr(L, name).restype = ctypes.c_int
        _lib = L
    return _lib


def check(rc: int) -> None:
    """Map a DS_* return code onto the reference's exception types."""
    if rc == DS_OK:
        return
    msg = lib().ds_last_error().decode(errors="replace")
    if rc == DS_EINVAL:
        raise ValueError(msg)
    raise DsError(rc, msg)


def device_count() -> int:
    return int(lib().ds_device_count())
