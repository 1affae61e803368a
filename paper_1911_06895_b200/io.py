"""Graph ingestion with the reference loaders' API (deltasparse/io.py), parsed
natively (csrc/ingest.cpp via ds_ingest_*).

Reference interface mirrored (file:line under /root/reference/pkg/src/deltasparse):
  GraphLoadError / ParseError / ValidationError   io.py:36-54
  GraphFile                                       io.py:57-64
  LabelMap                                        io.py:67-88
  load_matrix_market(path, default_weight)        io.py:121-193
  load_edge_list(path, directed, default_weight)  io.py:196-259
  load_graph(spec)                                io.py:262-272

Plus a binary CSR cache (`save_csr` / `load_csr`): a
parsed graph is written once and re-read at disk speed instead of re-parsing
the text and re-running matrix_build's sort.

Same grammar, line numbers, messages and exception classes; self-loops are
dropped with the same counted warning and duplicate edges keep their minimum
weight (matrix_build, core.py:247-278).  "-" reads standard input.  The
parser works on bytes: only ASCII whitespace separates tokens (the reference
also splits on Unicode spaces), which no Matrix Market or edge-list writer
emits.
"""

from __future__ import annotations

import ctypes
import logging
import sys
from dataclasses import dataclass

import numpy as np

from . import _lib
from .containers import INDEX_DTYPE, SparseMatrix

__all__ = [
    "GraphFile",
    "LabelMap",
    "GraphLoadError",
    "ParseError",
    "ValidationError",
    "load_matrix_market",
    "load_edge_list",
    "load_graph",
    "save_csr",
    "load_csr",
]

log = logging.getLogger(__name__)


# Interface types of the reference loaders (deltasparse/io.py:36-88): same
# names, attributes, message format and exception hierarchy, so callers that
# catch or construct them keep working.

class GraphLoadError(Exception):
    """Raised for any failure while loading a graph file.  The text reads
    "<path>:<line>: <message>"; the three parts stay available as
    attributes."""

    def __init__(self, path: str, lineno: int, message: str) -> None:
        self.path, self.lineno, self.message = path, lineno, message
        super().__init__("%s:%d: %s" % (path, lineno, message))


class ParseError(GraphLoadError):
    """Malformed input: a bad header, wrong token count or bad coordinate."""


class ValidationError(GraphLoadError):
    """Well-formed input with unusable values (a non-positive weight, ...)."""


@dataclass(frozen=True)
class GraphFile:
    """A graph argument of the CLI: file path (or "-"), format ("mtx" or
    "edges"), edge direction and the weight used when a line has none."""

    path: str
    format: str
    directed: bool = True
    default_weight: float = 1.0


class LabelMap:
    """Two-way map between the labels a file uses and internal ids 0..n-1
    (internal id i <-> externals[i])."""

    __slots__ = ("_externals", "_to_internal")

    def __init__(self, externals: list[int]) -> None:
        index: dict[int, int] = {}
        for internal, label in enumerate(externals):
            if index.setdefault(label, internal) != internal:
                raise ValueError("duplicate external label")
        self._externals = externals
        self._to_internal = index

    def __len__(self) -> int:
        return len(self._externals)

    def __contains__(self, label: int) -> bool:
        return label in self._to_internal

    def to_internal(self, label: int) -> int:
        return self._to_internal[label]

    def to_external(self, internal: int) -> int:
        return self._externals[internal]

    @property
    def externals(self) -> list[int]:
        return list(self._externals)


def _read(path: str) -> bytes:
    if path == "-":
        return sys.stdin.buffer.read()
    with open(path, "rb") as f:
        return f.read()


def _csr(n: int, r: np.ndarray, c: np.ndarray, w: np.ndarray) -> SparseMatrix:
    # matrix_build's CSR (core.py:266-278): sort by (row, col, weight), keep
    # the first (minimum-weight) entry of every coordinate
    if r.size:
        order = np.lexsort((w, c, r))
        r, c, w = r[order], c[order], w[order]
        first = np.concatenate([[True], (r[1:] != r[:-1]) | (c[1:] != c[:-1])])
        r, c, w = r[first], c[first], w[first]
    counts = np.bincount(r, minlength=n) if r.size else np.zeros(n, dtype=INDEX_DTYPE)
    indptr = np.zeros(n + 1, dtype=INDEX_DTYPE)
    np.cumsum(counts, out=indptr[1:])
    return SparseMatrix(n, indptr, c.astype(INDEX_DTYPE), w.astype(np.float64))


def _parse(path: str, fmt: int, directed: bool, default_weight: float):
    data = _read(path)
    L = _lib.lib()
    h = ctypes.c_void_p()
    rc = L.ds_ingest_parse(data, len(data), fmt, int(bool(directed)), float(default_weight),
                           path.encode(), ctypes.byref(h))
    if rc != _lib.DS_OK:
        full = L.ds_last_error().decode(errors="replace")
        lineno = int(L.ds_ingest_error_line())
        prefix = f"{path}:{lineno}: "
        message = full[len(prefix):] if full.startswith(prefix) else full
        if rc == _lib.DS_EPARSE:
            raise ParseError(path, lineno, message)
        if rc == _lib.DS_EVALID:
            raise ValidationError(path, lineno, message)
        _lib.check(rc)
    try:
        n, m, loops = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(L.ds_ingest_info(h, ctypes.byref(n), ctypes.byref(m), ctypes.byref(loops)))
        m_ = m.value
        r = np.empty(m_, dtype=np.int64)
        c = np.empty(m_, dtype=np.int64)
        w = np.empty(m_, dtype=np.float64)
        labels = np.empty(n.value, dtype=np.int64)
        _lib.check(L.ds_ingest_copy(h, r.ctypes.data, c.ctypes.data, w.ctypes.data,
                                    labels.ctypes.data))
    finally:
        L.ds_ingest_free(h)
    if loops.value:
        log.warning("%s: dropped %d self-loop entr%s", path, loops.value,
                    "y" if loops.value == 1 else "ies")
    return _csr(n.value, r, c, w), labels


def load_matrix_market(path: str, default_weight: float = 1.0) -> tuple[SparseMatrix, LabelMap]:
    """Read a Matrix Market coordinate file as a square graph (real, integer
    or pattern field; general or symmetric).  External labels are the file's
    1-based vertex numbers."""
    matrix, labels = _parse(path, _lib.DS_FMT_MTX, True, default_weight)
    return matrix, LabelMap(labels.tolist())


def load_edge_list(path: str, directed: bool = True,
                   default_weight: float = 1.0) -> tuple[SparseMatrix, LabelMap]:
    """Read a whitespace edge list ('u v' or 'u v w' per line); labels are
    remapped to dense ids in first-seen order (source before target)."""
    matrix, labels = _parse(path, _lib.DS_FMT_EDGES, directed, default_weight)
    return matrix, LabelMap(labels.tolist())


def load_graph(spec: GraphFile) -> tuple[SparseMatrix, LabelMap]:
    """Dispatch on the declared format (io.py:262-272); "csr" reads a binary
    cache written by `save_csr`."""
    if spec.format == "csr":
        return load_csr(spec.path)
    if spec.format == "mtx":
        return load_matrix_market(spec.path, default_weight=spec.default_weight)
    if spec.format == "edges":
        return load_edge_list(spec.path, directed=spec.directed,
                              default_weight=spec.default_weight)
    raise ValueError(f"unknown graph format {spec.format!r}")


# ------------------------------------------------------------ binary CSR cache
# Layout (little endian): 64-byte header = magic b"DSCSR\0\1\0" + int64
# n, nnz, col_bytes (4|8), w_bytes (4|8), n_labels (0|n), 2 reserved words;
# then indptr int64[n+1], col, weights, labels int64[n_labels], each array
# padded to 8 bytes.  Columns are stored as int32 when n fits, weights as
# float32 when every weight converts exactly (8 B/edge instead of 16); the
# loader widens nothing it does not have to (SparseMatrix compact=True) and the
# values are bit-identical either way.
_CSR_MAGIC = b"DSCSR\0\1\0"
_CSR_HEADER = 64


def _pad8(nbytes: int) -> int:
    return (-nbytes) % 8


def save_csr(path: str, matrix: SparseMatrix, labels: LabelMap | None = None) -> None:
    """Write `matrix` (and optionally its LabelMap) as a binary CSR cache."""
    n, nnz = matrix.n, matrix.nnz
    col = np.asarray(matrix.col)
    col = col.astype(np.int32) if n <= np.iinfo(np.int32).max else col.astype(np.int64)
    w64 = np.asarray(matrix.val, dtype=np.float64)
    w32 = w64.astype(np.float32)
    w = w32 if np.array_equal(w32.astype(np.float64), w64) else w64
    lab = (np.asarray(labels.externals, dtype=np.int64) if labels is not None
           else np.empty(0, dtype=np.int64))
    if lab.size not in (0, n):
        raise ValueError(f"label map has {lab.size} labels for {n} vertices")
    head = np.array([n, nnz, col.itemsize, w.itemsize, lab.size, 0, 0], dtype="<i8")
    with open(path, "wb") as f:
        f.write(_CSR_MAGIC)
        f.write(head.tobytes())
        for arr in (np.asarray(matrix.indptr, dtype="<i8"), col, w, lab):
            arr = arr.astype(arr.dtype.newbyteorder("<"), copy=False)
            f.write(arr.tobytes())
            f.write(b"\0" * _pad8(arr.nbytes))


def load_csr(path: str, compact: bool = True) -> tuple[SparseMatrix, LabelMap]:
    """Read a cache written by `save_csr`.  Without stored labels the map is
    the identity on 1..n, as load_matrix_market's 1-based numbering."""
    with open(path, "rb") as f:
        head = f.read(_CSR_HEADER)
        if len(head) < _CSR_HEADER or head[:8] != _CSR_MAGIC:
            raise ValueError(f"{path}: not a binary CSR cache")
        n, nnz, cb, wb, nl, _, _ = np.frombuffer(head[8:], dtype="<i8").tolist()
        if n < 1 or nnz < 0 or cb not in (4, 8) or wb not in (4, 8) or nl not in (0, n):
            raise ValueError(f"{path}: corrupt binary CSR header")
        parts = []
        for count, dt in ((n + 1, "<i8"), (nnz, "<i%d" % cb), (nnz, "<f%d" % wb), (nl, "<i8")):
            arr = np.fromfile(f, dtype=dt, count=count)
            if arr.size != count:
                raise ValueError(f"{path}: truncated binary CSR cache")
            f.seek(_pad8(arr.nbytes), 1)
            parts.append(arr)
    indptr, col, w, lab = parts
    if indptr[0] != 0 or indptr[-1] != nnz or bool(np.any(indptr[1:] < indptr[:-1])):
        raise ValueError(f"{path}: corrupt row offsets")
    if nnz and (int(col.min()) < 0 or int(col.max()) >= n):
        raise ValueError(f"{path}: column index out of range")
    matrix = SparseMatrix(n, indptr, col, w, compact=compact)
    labels = LabelMap(lab.tolist() if nl else list(range(1, n + 1)))
    return matrix, labels
