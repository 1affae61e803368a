"""Graph ingestion with the reference loaders' API (deltasparse/io.py), parsed
natively (csrc/ingest.cpp via ds_ingest_*).

Reference interface mirrored (file:line under /root/reference/pkg/src/deltasparse):
  GraphLoadError / ParseError / ValidationError   io.py:36-54
  GraphFile                                       io.py:57-64
  LabelMap                                        io.py:67-88
  load_matrix_market(path, default_weight)        io.py:121-193
  load_edge_list(path, directed, default_weight)  io.py:196-259
  load_graph(spec)                                io.py:262-272

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
]

log = logging.getLogger(__name__)


class GraphLoadError(Exception):
    """Base for anything that goes wrong while reading a graph file."""

    def __init__(self, path: str, lineno: int, message: str) -> None:
        super().__init__(f"{path}:{lineno}: {message}")
        self.path = path
        self.lineno = lineno
        self.message = message


class ParseError(GraphLoadError):
    """The file's structure is wrong: header, token counts, coordinates."""


class ValidationError(GraphLoadError):
    """The file parsed but its content is unusable, e.g. weight <= 0."""


@dataclass(frozen=True)
class GraphFile:
    """One parsed CLI graph argument: where it is and how to read it."""

    path: str
    format: str  # "mtx" | "edges"
    directed: bool = True
    default_weight: float = 1.0


class LabelMap:
    """Bijection between external vertex labels and dense internal ids."""

    __slots__ = ("_externals", "_to_internal")

    def __init__(self, externals: list[int]) -> None:
        self._externals = externals
        self._to_internal = {label: i for i, label in enumerate(externals)}
        if len(self._to_internal) != len(externals):
            raise ValueError("duplicate external label")

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
    """Dispatch on the declared format (io.py:262-272)."""
    if spec.format == "mtx":
        return load_matrix_market(spec.path, default_weight=spec.default_weight)
    if spec.format == "edges":
        return load_edge_list(spec.path, directed=spec.directed,
                              default_weight=spec.default_weight)
    raise ValueError(f"unknown graph format {spec.format!r}")
