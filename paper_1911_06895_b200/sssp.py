"""Drop-in `delta_stepping` on the B200 (the reference's sssp.py:239-313 API).

The host side keeps the reference's Python signature, argument validation,
exception types/messages and result shape; everything between "CSR in" and
"distances out" runs in the sm_100a library behind the C-ABI
(include/dsssp.h) -- device CSR with a per-delta light/heavy split, then one
persistent cooperative kernel per source.  There is no CPU fallback: without
libdsssp.so or a CUDA device the call raises.

Reference interface mirrored (file:line under /root/reference/pkg/src/deltasparse):
  delta_stepping      sssp.py:239-313   (validation :255-260, ceiling :297-301)
  SsspResult          sssp.py:82-87
  split_edges         sssp.py:106-150   (device split, exported back to host)
  BackendChoice       fused.py:41-55    (validated, then ignored: one GPU path)
  bucket_bounds       fused.py:58-61
"""

from __future__ import annotations

import contextlib
import ctypes
import math
import os
import threading
import time
from collections import OrderedDict
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

from . import _hostio, _lib
from .containers import SparseMatrix, SparseVector

__all__ = [
    "BackendChoice",
    "SsspResult",
    "DeviceGraph",
    "bucket_bounds",
    "delta_stepping",
    "delta_stepping_batch",
    "split_edges",
    "clear_device_cache",
]


@dataclass(frozen=True)
class BackendChoice:
    """Accepted for call-site compatibility with the reference (fused.py:41-55).

    The B200 build has exactly one implementation; `kind`, `workers` and
    `chunks_per_worker` are validated like the reference and otherwise
    ignored (no multi-backend dispatch).
    """

    kind: str = "unfused"
    workers: int = 1
    chunks_per_worker: int = 1

    def __post_init__(self) -> None:
        if self.kind not in ("unfused", "fused"):
            raise ValueError(f"backend kind must be 'unfused' or 'fused', got {self.kind!r}")
        if self.workers < 1:
            raise ValueError(f"workers must be >= 1, got {self.workers}")
        if self.chunks_per_worker < 1:
            raise ValueError(f"chunks_per_worker must be >= 1, got {self.chunks_per_worker}")


@dataclass(frozen=True)
class SsspResult:
    """Same fields as the reference (sssp.py:82-87); `device_stats` carries
    the solver's counters (n_r, m_r, kernel time, ...) and is excluded from
    comparisons."""

    distances: SparseVector
    outer_iterations: int
    inner_phases: int
    elapsed: float
    device_stats: dict | None = field(default=None, compare=False, repr=False)


def bucket_bounds(index: int, delta: float) -> tuple[float, float]:
    """Half-open window of bucket `index` (fused.py:58-61)."""
    return index * delta, (index + 1) * delta


def _check_out(a, count: int, dtype, name: str) -> None:
    """Caller-provided output buffers are written through raw pointers: reject
    a wrong dtype, a non-contiguous layout or fewer than `count` elements
    instead of overrunning them."""
    dt = np.dtype(dtype)
    if hasattr(a, "data_ptr"):  # torch tensor
        if str(a.dtype).replace("torch.", "") != dt.name:
            raise ValueError(f"{name} must be {dt.name}, got {a.dtype}")
        if not a.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        if a.numel() < count:
            raise ValueError(f"{name} holds {a.numel()} elements, needs {count}")
        return
    if not isinstance(a, np.ndarray):
        raise ValueError(f"{name} must be a numpy array or a torch tensor")
    if a.dtype != dt:
        raise ValueError(f"{name} must be {dt.name}, got {a.dtype}")
    if not a.flags.c_contiguous:
        raise ValueError(f"{name} must be C-contiguous")
    if a.size < count:
        raise ValueError(f"{name} holds {a.size} elements, needs {count}")


def _ptr(a) -> int:
    if a is None:
        return 0
    if hasattr(a, "data_ptr"):  # torch tensor (host pinned or device)
        return int(a.data_ptr())
    return int(a.ctypes.data)


def _col_dtype(dt) -> int:
    if dt == np.int32:
        return _lib.DS_IDX_I32
    if dt == np.int64:
        return _lib.DS_IDX_I64
    raise ValueError(f"unsupported column dtype {dt}")


def _val_dtype(dt) -> int:
    if dt == np.float32:
        return _lib.DS_W_F32
    if dt == np.float64:
        return _lib.DS_W_F64
    if dt == np.int32:
        return _lib.DS_W_I32
    raise ValueError(f"unsupported weight dtype {dt}")


class DeviceGraph:
    """A graph resident in HBM: one `ds_graph` handle of the C-ABI library."""

    def __init__(self, handle: int, n: int, nnz: int, device: int):
        self._h = ctypes.c_void_p(handle)
        self.n = int(n)
        self.nnz = int(nnz)
        self.device = int(device)
        self.last_stats: _lib.Stats | None = None
        self.prep: _lib.PrepInfo | None = None
        # A ds_graph handle is not re-entrant (include/dsssp.h): calls that
        # touch its scratch hold this lock (ctypes releases the GIL).  The
        # reference promises that concurrent invocations on a shared
        # immutable graph are safe; they serialise here.
        self.lock = threading.RLock()
        self._users = 0        # cached handles: callers currently using it
        self._evicted = False  # dropped from the cache; closed by the last user

    # -- construction ---------------------------------------------------
    @classmethod
    def from_csr(cls, n, indptr, col, val, device: int = 0, stream: int | None = None) -> "DeviceGraph":
        """Upload a CSR.  numpy arrays (host) or torch tensors (pinned host or
        device) are accepted; dtypes int32/int64 columns, float32/float64/int32
        weights."""
        L = _lib.lib()

        def dt(a):
            return np.dtype(str(a.dtype).replace("torch.", "")) if hasattr(a, "data_ptr") else a.dtype

        if not hasattr(indptr, "data_ptr"):
            indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        if not hasattr(col, "data_ptr"):
            col = np.ascontiguousarray(col)
            if col.dtype not in (np.int32, np.int64):
                col = col.astype(np.int64)
        if not hasattr(val, "data_ptr"):
            val = np.ascontiguousarray(val)
            if val.dtype not in (np.float32, np.float64, np.int32):
                val = val.astype(np.float64)
        nnz = int(col.shape[0])
        # Large pageable host arrays (the reference's int64 / float64 layout)
        # go up through the pinned ring (_hostio): ~4x the pageable copy rate.
        staged = []
        host = [a for a in (indptr, col, val) if not hasattr(a, "data_ptr")]
        if host and sum(a.nbytes for a in host) >= _hostio.MIN_BYTES and _hostio.available():
            import torch

            free, _ = torch.cuda.mem_get_info(device)
            if 3 * sum(a.nbytes for a in host) < free:
                def up(a):
                    if hasattr(a, "data_ptr") or a.nbytes < _hostio.MIN_BYTES:
                        return a
                    t = _hostio.upload(a, device)
                    staged.append(t)
                    return t

                indptr, col, val = up(indptr), up(col), up(val)
        h = ctypes.c_void_p()
        try:
            _lib.check(L.ds_graph_create(int(n), nnz, _ptr(indptr), _ptr(col), _col_dtype(dt(col)),
                                         _ptr(val), _val_dtype(dt(val)), int(device), stream or 0,
                                         ctypes.byref(h)))
        finally:
            if staged:
                import torch

                del staged[:], indptr, col, val
                torch.cuda.empty_cache()  # the staging copies go back to the driver
        return cls(h.value, n, nnz, device)

    @classmethod
    def from_matrix(cls, matrix, device: int = 0, stream: int | None = None) -> "DeviceGraph":
        return cls.from_csr(matrix.n, matrix.indptr, matrix.col, matrix.val, device, stream)

    @classmethod
    def rmat(cls, scale: int, edge_factor: int = 16, seed: int = 1, weight_seed: int = 2,
             device: int = 0, stream: int | None = None) -> "DeviceGraph":
        """R-MAT generated on the device; identical to graphs.rmat()."""
        L = _lib.lib()
        h = ctypes.c_void_p()
        _lib.check(L.ds_gen_rmat(int(scale), int(edge_factor), int(seed), int(weight_seed),
                                 int(device), stream or 0, ctypes.byref(h)))
        n = ctypes.c_int64()
        nnz = ctypes.c_int64()
        _lib.check(L.ds_graph_size(h, ctypes.byref(n), ctypes.byref(nnz)))
        return cls(h.value, n.value, nnz.value, device)

    # -- operations -----------------------------------------------------
    def _handle(self):
        if not self._h.value:
            raise ValueError("device graph is closed")
        return self._h

    def set_stream(self, stream: int | None) -> None:
        with self.lock:
            _lib.check(_lib.lib().ds_graph_set_stream(self._handle(), stream or 0))

    def prepare(self, delta: float, force_f64: bool = False) -> _lib.PrepInfo:
        info = _lib.PrepInfo()
        flags = _lib.DS_FLAG_FORCE_F64 if force_f64 else 0
        with self.lock:
            _lib.check(_lib.lib().ds_graph_prepare(self._handle(), float(delta), flags,
                                                   ctypes.byref(info)))
            self.prep = info
        return info

    def solve(self, source: int, delta: float, skip_empty_buckets: bool = False,
              force_f64: bool = False) -> _lib.Stats:
        st = _lib.Stats()
        flags = (_lib.DS_FLAG_SKIP_EMPTY if skip_empty_buckets else 0) | (
            _lib.DS_FLAG_FORCE_F64 if force_f64 else 0)
        with self.lock:
            _lib.check(_lib.lib().ds_sssp(self._handle(), int(source), float(delta), flags,
                                          ctypes.byref(st)))
            self.last_stats = st
        return st

    def solve_batch(self, sources, delta: float, skip_empty_buckets: bool = False,
                    force_f64: bool = False, concurrency: int = 0, out=None,
                    keep: bool = True):
        """k sources through ds_sssp_batch.  Returns (stats list, dist) where
        dist is a k x n float64 array (`out` if given: host ndarray or a
        device pointer int) or None when keep=False."""
        src = np.ascontiguousarray(np.asarray(sources, dtype=np.int64).reshape(-1))
        k = int(src.size)
        stats = (_lib.Stats * max(k, 1))()
        flags = (_lib.DS_FLAG_SKIP_EMPTY if skip_empty_buckets else 0) | (
            _lib.DS_FLAG_FORCE_F64 if force_f64 else 0)
        if not keep:
            dptr, dist = None, None
        elif isinstance(out, int):
            dptr, dist = out, None
        else:
            dist = out if out is not None else np.empty((k, self.n), dtype=np.float64)
            _check_out(dist, k * self.n, np.float64, "out")
            dptr = _ptr(dist)
        with self.lock:
            _lib.check(_lib.lib().ds_sssp_batch(self._handle(), _ptr(src), k, float(delta), flags,
                                                int(concurrency), stats, dptr))
            self.last_stats = None
        return [stats[i] for i in range(k)], dist

    def result_dense(self, out=None) -> np.ndarray:
        if out is None:
            out = np.empty(self.n, dtype=np.float64)
        _check_out(out, self.n, np.float64, "out")
        with self.lock:
            _lib.check(_lib.lib().ds_result_dense(self._handle(), _ptr(out)))
        return out

    def result_sparse(self, out=None):
        """(indices int64, values float64) of reached vertices; `out` may be a
        pair of preallocated (pinned) buffers with >= reached entries."""
        with self.lock:
            r = int(self.last_stats.reached) if self.last_stats is not None else self.n
            if out is None:
                idx = np.empty(r, dtype=np.int64)
                val = np.empty(r, dtype=np.float64)
            else:
                _check_out(out[0], r, np.int64, "out[0]")
                _check_out(out[1], r, np.float64, "out[1]")
                idx, val = out[0][:r], out[1][:r]
            _lib.check(_lib.lib().ds_result_sparse(self._handle(), _ptr(idx), _ptr(val)))
        return idx, val

    def export_split(self, which: int):
        """Light (0) / heavy (1) CSR of the current prepare as host arrays."""
        with self.lock:
            if self.prep is None:
                raise ValueError("export_split needs a prepare() first")
            m = int(self.prep.nnz_heavy if which else self.prep.nnz_light)
            indptr = np.empty(self.n + 1, dtype=np.int64)
            col = np.empty(max(m, 1), dtype=np.int64)
            val = np.empty(max(m, 1), dtype=np.float64)
            _lib.check(_lib.lib().ds_export_split(self._handle(), int(which), _ptr(indptr), _ptr(col),
                                                  _ptr(val)))
        return indptr, col[:m], val[:m]

    def download_indptr(self) -> np.ndarray:
        """Row offsets only (int64, host): degrees without the edge arrays."""
        indptr = np.empty(self.n + 1, dtype=np.int64)
        with self.lock:
            _lib.check(_lib.lib().ds_graph_download(self._handle(), _ptr(indptr), None, None))
        return indptr

    def download(self, out=None):
        """Original CSR (int64 indptr, int32 col, float32 val), to host arrays
        or into `out` = (indptr, col, val) buffers (numpy, or torch tensors on
        the graph's device: no host round trip)."""
        if out is None:
            indptr = np.empty(self.n + 1, dtype=np.int64)
            col = np.empty(max(self.nnz, 1), dtype=np.int32)
            val = np.empty(max(self.nnz, 1), dtype=np.float32)
        else:
            indptr, col, val = out
            _check_out(indptr, self.n + 1, np.int64, "indptr")
            _check_out(col, self.nnz, np.int32, "col")
            _check_out(val, self.nnz, np.float32, "val")
        with self.lock:
            _lib.check(_lib.lib().ds_graph_download(self._handle(), _ptr(indptr), _ptr(col), _ptr(val)))
        return indptr, col[: self.nnz], val[: self.nnz]

    def close(self) -> None:
        with self.lock:
            if self._h.value:
                _lib.lib().ds_graph_destroy(self._h)
                self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ------------------------------------------------------------------ cache
# The reference caches derived data (transposed views) on the matrix object
# (core.py:128, 289-301).  Its SparseMatrix has __slots__ without __weakref__,
# so the device copy is cached here keyed on object identity, holding a
# strong reference to the matrix so the id cannot be recycled while cached.

_CACHE: "OrderedDict[int, tuple[object, DeviceGraph]]" = OrderedDict()
_CACHE_SIZE = 2
_CACHE_LOCK = threading.Lock()


def _retire(g: DeviceGraph) -> None:
    """Drop a cached handle: closed now if idle, else by its last user."""
    g._evicted = True
    if g._users == 0:
        g.close()


def clear_host_buffers() -> None:
    """Release the pooled pinned host buffers of the drop-in entry points
    (kept across calls: pinning 8 GB costs more than moving it)."""
    _hostio.clear()


def clear_device_cache() -> None:
    with _CACHE_LOCK:
        for _, g in _CACHE.values():
            _retire(g)
        _CACHE.clear()


@contextlib.contextmanager
def _device_graph(matrix, device: int = 0):
    """The cached device copy of `matrix`, pinned for the duration of the
    `with` block: eviction by another thread (or clear_device_cache) defers
    the close until every user has left, so no call ever runs on a freed
    handle."""
    key = id(matrix)
    with _CACHE_LOCK:
        hit = _CACHE.get(key)
        if hit is not None and hit[0] is matrix:
            _CACHE.move_to_end(key)
            g = hit[1]
        else:
            g = DeviceGraph.from_matrix(matrix, device)
            _CACHE[key] = (matrix, g)
            while len(_CACHE) > _CACHE_SIZE:
                _, (_, old) = _CACHE.popitem(last=False)
                _retire(old)
        g._users += 1
    try:
        yield g
    finally:
        with _CACHE_LOCK:
            g._users -= 1
            if g._evicted and g._users == 0:
                g.close()


# ------------------------------------------------------------------ API

def delta_stepping(
    matrix,
    source: int,
    delta: float,
    *,
    backend: BackendChoice | None = None,
    skip_empty_buckets: bool = False,
) -> SsspResult:
    """Single-source shortest paths by delta-stepping on the GPU.

    Same contract as the reference (sssp.py:239-313): `matrix` is any CSR
    object with `.n/.indptr/.col/.val` (ours or `deltasparse.SparseMatrix`);
    returns the reached vertices' float64 distances bit-identical to the
    reference, with identical `outer_iterations` / `inner_phases`.
    `elapsed` covers the device split (cached per delta) and the solve, like
    the reference's (sssp.py:263, 312).
    """
    if backend is None:
        backend = BackendChoice()
    if not 0 <= source < matrix.n:
        raise ValueError(f"source {source} out of range for {matrix.n} vertices")
    if not (delta > 0) or not math.isfinite(delta):
        raise ValueError(f"delta must be a positive finite number, got {delta}")
    start = time.perf_counter()
    with _device_graph(matrix) as g, g.lock:  # solve + fetch as one unit
        st = g.solve(int(source), float(delta), skip_empty_buckets=skip_empty_buckets)
        idx, val = g.result_sparse()
    elapsed = time.perf_counter() - start
    return SsspResult(
        distances=SparseVector(matrix.n, idx, val),
        outer_iterations=int(st.outer_iterations),
        inner_phases=int(st.inner_phases),
        elapsed=elapsed,
        device_stats=st.as_dict(),
    )


def delta_stepping_batch(
    matrix,
    sources,
    delta: float,
    *,
    backend: BackendChoice | None = None,
    skip_empty_buckets: bool = False,
    concurrency: int = 0,
) -> list[SsspResult]:
    """`delta_stepping` for several sources of one matrix -- the loop the
    reference's callers run (cli.py:119-128, the 64/16-source benchmarks) --
    with up to `concurrency` sources in flight on SM-disjoint persistent
    grids.  Each result equals `delta_stepping(matrix, s, delta, ...)`
    exactly; `elapsed` is the batch's wall time split evenly."""
    if backend is None:
        backend = BackendChoice()
    srcs = [int(s) for s in sources]
    for s in srcs:
        if not 0 <= s < matrix.n:
            raise ValueError(f"source {s} out of range for {matrix.n} vertices")
    if not (delta > 0) or not math.isfinite(delta):
        raise ValueError(f"delta must be a positive finite number, got {delta}")
    if not srcs:
        return []
    start = time.perf_counter()
    # the dense results land in a pooled pinned array (no freshly faulted
    # pages, full-rate D2H); the rows are copied out of it below
    pooled = None
    out = dist = None
    nbytes = len(srcs) * matrix.n * 8
    if _hostio.MIN_BYTES <= nbytes <= _hostio.MAX_POOLED and _hostio.available():
        try:
            pooled = _hostio.take_pinned(nbytes)
            out = pooled.numpy()[:nbytes].view(np.float64).reshape(len(srcs), matrix.n)
        except RuntimeError:  # no pinned memory to be had: the plain pageable result array
            pooled = out = None
    try:
        with _device_graph(matrix) as g:
            stats, dist = g.solve_batch(srcs, float(delta), skip_empty_buckets=skip_empty_buckets,
                                        concurrency=concurrency, out=out)
        # dense rows -> reached (index, value) pairs; numpy releases the GIL on
        # these full-row passes, so rows convert in parallel.  Sources of one
        # component reach the same set: a row with as many reached vertices as
        # the first one, all of them finite on its index set, shares that set.
        first = np.flatnonzero(dist[0] != np.inf)

        def sparse_row(i):
            row = dist[i]
            if i == 0:
                return first, row[first]
            if int(stats[i].reached) == first.size:
                vals = row[first]
                if not np.isinf(vals).any():
                    return first, vals
            idx = np.flatnonzero(row != np.inf)
            return idx, row[idx]

        if len(srcs) > 1 and matrix.n >= (1 << 16):
            with ThreadPoolExecutor(max_workers=min(len(srcs), os.cpu_count() or 1, 16)) as ex:
                rows = list(ex.map(sparse_row, range(len(srcs))))
        else:
            rows = [sparse_row(i) for i in range(len(srcs))]
    finally:
        if pooled is not None:
            out = dist = None  # views of the pooled buffer
            _hostio.give_pinned(pooled)
    elapsed = (time.perf_counter() - start) / len(srcs)
    out = []
    for (idx, val), st in zip(rows, stats):
        out.append(SsspResult(
            distances=SparseVector(matrix.n, idx, val),
            outer_iterations=int(st.outer_iterations),
            inner_phases=int(st.inner_phases),
            elapsed=elapsed,
            device_stats=st.as_dict(),
        ))
    return out


def split_edges(matrix, delta: float, workers: int = 1, chunks_per_worker: int = 1):
    """Light/heavy partition (sssp.py:106-150) computed by the device split
    kernels and returned as host `SparseMatrix` objects."""
    if not (delta > 0) or not math.isfinite(delta):
        raise ValueError(f"delta must be a positive finite number, got {delta}")
    out = []
    with _device_graph(matrix) as g, g.lock:
        g.prepare(float(delta))
        for which in (0, 1):
            indptr, col, val = g.export_split(which)
            out.append(SparseMatrix(matrix.n, indptr, col, val))
    return out[0], out[1]
