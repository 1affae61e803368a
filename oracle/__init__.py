"""CPU parity oracle -- TEST INFRASTRUCTURE ONLY.

A C restatement (``oracle.c``) of the reference's delta-stepping path
(`deltasparse.sssp.delta_stepping`, /root/reference/pkg/src/deltasparse/
sssp.py:239-313, fused backend) plus its `dijkstra_oracle` (sssp.py:316-341)
and `split_edges` (sssp.py:106-150).  Only ``tests/``, ``__graft_entry__.smoke``
and ``bench.py``'s CPU-baseline / ``--impl reference`` leg may import this
package, and only as the checker or the timed CPU baseline -- never as part of
the product path, which fails loudly without its CUDA library.

The restatement is pinned against golden vectors produced by the reference
itself (``tests/golden/make_golden.py``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liboracle.so")
_lib = None

OR_OK, OR_EINVAL, OR_ENOCONVERGE, OR_ENOMEM = 0, 1, 2, 3

_i64p = ctypes.POINTER(ctypes.c_int64)
_f64p = ctypes.POINTER(ctypes.c_double)


def build() -> str:
    """Compile liboracle.so with the committed Makefile (gcc + OpenMP)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        lib = ctypes.CDLL(_LIB_PATH)
        lib.oracle_delta_stepping.argtypes = [
            ctypes.c_int64, _i64p, _i64p, _f64p, ctypes.c_int64, ctypes.c_double,
            ctypes.c_int, ctypes.c_int, _f64p, _i64p, _i64p,
        ]
        lib.oracle_delta_stepping.restype = ctypes.c_int
        lib.oracle_dijkstra.argtypes = [ctypes.c_int64, _i64p, _i64p, _f64p, ctypes.c_int64, _f64p]
        lib.oracle_dijkstra.restype = ctypes.c_int
        lib.oracle_split.argtypes = [
            ctypes.c_int64, _i64p, _i64p, _f64p, ctypes.c_double, ctypes.c_int,
            _i64p, _i64p, _f64p, _i64p,
        ]
        lib.oracle_split.restype = ctypes.c_int
        lib.oracle_rmat_build.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_uint64, ctypes.c_uint64,
                                          ctypes.c_int]
        lib.oracle_rmat_build.restype = ctypes.c_void_p
        lib.oracle_rmat_nnz.argtypes = [ctypes.c_void_p]
        lib.oracle_rmat_nnz.restype = ctypes.c_int64
        lib.oracle_rmat_fetch.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p]
        lib.oracle_rmat_fetch.restype = None
        lib.oracle_rmat_free.argtypes = [ctypes.c_void_p]
        lib.oracle_rmat_free.restype = None
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _csr(indptr, col, val):
    indptr = np.ascontiguousarray(indptr, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int64)
    val = np.ascontiguousarray(val, dtype=np.float64)
    return indptr, col, val


def _p(a, t):
    return a.ctypes.data_as(t)


def max_threads() -> int:
    return int(_load().oracle_num_threads())


def delta_stepping(n, indptr, col, val, source, delta, skip_empty_buckets=False, threads=1):
    """Reference delta-stepping restated in C.

    Returns (dist[n] float64 with +inf for unreachable, outer_iterations,
    inner_phases).  Raises ValueError / RuntimeError like sssp.py:257-260 and
    sssp.py:297-301.
    """
    lib = _load()
    indptr, col, val = _csr(indptr, col, val)
    dist = np.empty(int(n), dtype=np.float64)
    outer = ctypes.c_int64(0)
    phases = ctypes.c_int64(0)
    rc = lib.oracle_delta_stepping(
        int(n), _p(indptr, _i64p), _p(col, _i64p), _p(val, _f64p), int(source), float(delta),
        int(bool(skip_empty_buckets)), int(threads), _p(dist, _f64p),
        ctypes.byref(outer), ctypes.byref(phases),
    )
    if rc == OR_EINVAL:
        raise ValueError("invalid source or delta")
    if rc == OR_ENOCONVERGE:
        raise RuntimeError("light phase count exceeded ceiling; relaxation is not converging")
    if rc != OR_OK:
        raise MemoryError("oracle allocation failed")
    return dist, int(outer.value), int(phases.value)


def dijkstra(n, indptr, col, val, source):
    """dijkstra_oracle (sssp.py:316-341) restated in C; dense float64 result."""
    lib = _load()
    indptr, col, val = _csr(indptr, col, val)
    dist = np.empty(int(n), dtype=np.float64)
    rc = lib.oracle_dijkstra(int(n), _p(indptr, _i64p), _p(col, _i64p), _p(val, _f64p),
                             int(source), _p(dist, _f64p))
    if rc == OR_EINVAL:
        raise ValueError(f"source {source} out of range for {n} vertices")
    if rc != OR_OK:
        raise MemoryError("oracle allocation failed")
    return dist


def split(n, indptr, col, val, delta, which):
    """split_edges (sssp.py:106-150): which=0 light, 1 heavy -> (indptr, col, val)."""
    lib = _load()
    indptr, col, val = _csr(indptr, col, val)
    nnz = ctypes.c_int64(0)
    null_i = ctypes.cast(None, _i64p)
    rc = lib.oracle_split(int(n), _p(indptr, _i64p), _p(col, _i64p), _p(val, _f64p), float(delta),
                          int(which), null_i, null_i, ctypes.cast(None, _f64p), ctypes.byref(nnz))
    if rc == OR_EINVAL:
        raise ValueError(f"delta must be a positive finite number, got {delta}")
    k = int(nnz.value)
    o_ptr = np.empty(int(n) + 1, dtype=np.int64)
    o_col = np.empty(max(k, 1), dtype=np.int64)
    o_val = np.empty(max(k, 1), dtype=np.float64)
    lib.oracle_split(int(n), _p(indptr, _i64p), _p(col, _i64p), _p(val, _f64p), float(delta),
                     int(which), _p(o_ptr, _i64p), _p(o_col, _i64p), _p(o_val, _f64p),
                     ctypes.byref(nnz))
    return o_ptr, o_col[:k], o_val[:k]


def to_sparse(dist):
    """Dense oracle distances -> (indices int64, values float64) of reached vertices,
    the shape of the reference SparseVector (core.py:46-70)."""
    idx = np.flatnonzero(np.isfinite(dist)).astype(np.int64)
    return idx, dist[idx]


def rmat(scale, edge_factor=16, seed=1, weight_seed=2, threads=0):
    """Host R-MAT CSR (indptr int64, col int32, val float32), bit-identical to
    paper_1911_06895_b200.graphs.rmat (restated in C with OpenMP in rmat.c) --
    the reference arm's input without the product's CUDA library."""
    lib = _load()
    h = lib.oracle_rmat_build(int(scale), int(edge_factor), int(seed), int(weight_seed), int(threads))
    if not h:
        raise MemoryError("oracle R-MAT generation failed")
    try:
        nnz = int(lib.oracle_rmat_nnz(h))
        n = 1 << int(scale)
        indptr = np.empty(n + 1, dtype=np.int64)
        col = np.empty(max(nnz, 1), dtype=np.int32)
        val = np.empty(max(nnz, 1), dtype=np.float32)
        lib.oracle_rmat_fetch(h, indptr.ctypes.data, col.ctypes.data, val.ctypes.data)
    finally:
        lib.oracle_rmat_free(h)
    return indptr, col[:nnz], val[:nnz]
