"""CPU-only checks: the C-ABI library loads and exports every symbol the
header declares, host-side validation mirrors the reference, generators are
deterministic, and the product path refuses to run without a GPU."""

from __future__ import annotations

import math
import os
import re

import numpy as np
import pytest

from conftest import REPO
from paper_1911_06895_b200 import (
    BackendChoice,
    SparseMatrix,
    SparseVector,
    bucket_bounds,
    delta_stepping,
    graphs,
    matrix_build,
    vector_build,
)
from paper_1911_06895_b200 import _lib


def header_symbols():
    text = open(os.path.join(REPO, "include", "dsssp.h")).read()
    return sorted(set(re.findall(r"\b(ds_[a-z_]+)\s*\(", text)))


def test_library_exports_every_header_symbol():
    L = _lib.lib()
    syms = header_symbols()
    assert len(syms) >= 10
    for s in syms:
        assert hasattr(L, s), s
    assert set(syms) == set(_lib.EXPORTS)


def test_no_device_means_loud_failure():
    if _lib.device_count() > 0:
        pytest.skip("a GPU is visible")
    a = matrix_build(3, [(0, 1, 1.0)])
    with pytest.raises(RuntimeError):
        delta_stepping(a, 0, 1.0)


def test_validation_precedes_device():
    a = matrix_build(3, [(0, 1, 1.0)])
    with pytest.raises(ValueError, match="source 3 out of range for 3 vertices"):
        delta_stepping(a, 3, 1.0)
    for bad in (0.0, -2.0, math.inf, math.nan):
        with pytest.raises(ValueError, match="delta must be a positive finite number"):
            delta_stepping(a, 0, bad)


def test_backend_choice_validation():
    BackendChoice()
    BackendChoice(kind="fused", workers=4, chunks_per_worker=2)
    for kw in ({"kind": "turbo"}, {"workers": 0}, {"chunks_per_worker": 0}):
        with pytest.raises(ValueError):
            BackendChoice(**kw)


def test_bucket_bounds_values():
    assert bucket_bounds(0, 1.0) == (0.0, 1.0)
    assert bucket_bounds(3, 0.5) == (1.5, 2.0)
    assert bucket_bounds(2, 11.0) == (22.0, 33.0)


def test_containers_mirror_reference_semantics():
    a = matrix_build(3, [(0, 1, 2.0), (0, 1, 1.0), (1, 1, 5.0), (2, 0, 3.0)])
    assert a.entry_set() == {(0, 1, 1.0), (2, 0, 3.0)}
    a.check_invariants()
    with pytest.raises(ValueError):
        matrix_build(2, [(0, 1, 0.0)])
    with pytest.raises(ValueError):
        matrix_build(2, [(0, 5, 1.0)])
    v = vector_build(4, [(2, 3.0), (2, 1.0), (0, math.inf)])
    assert v.to_dict() == {2: 1.0}
    assert SparseVector(2, [0], [0.0]) != SparseVector(2, [0], [-0.0])  # bitwise
    assert SparseVector(2, [0], [1.0]) == SparseVector(2, [0], [1.0])


def test_rmat_generator_properties():
    g = graphs.rmat(10, seed=1, weight_seed=2)
    g.check_invariants()
    r = g.row_ids()
    # symmetric with one weight per undirected pair
    fwd = dict(zip(zip(r.tolist(), g.col.tolist()), g.val.tolist()))
    for (u, v), w in list(fwd.items())[:2000]:
        assert fwd[(v, u)] == w
    k = g.val.astype(np.float64) * 2**24
    assert np.all(k == np.floor(k)) and np.all(k >= 1) and np.all(k < 2**24)
    g2 = graphs.rmat(10, seed=1, weight_seed=2)
    assert g == g2


def test_grid_generator_properties():
    g = graphs.grid2d(16, seed=3)
    g.check_invariants()
    assert g.nnz == 4 * 16 * 15
    assert g.val.min() >= 1 and g.val.max() <= 100


def test_erdos_renyi_shape():
    g = graphs.erdos_renyi(1024, seed=0)
    g.check_invariants()
    assert 7000 < g.nnz < 9500
    assert g.val.min() >= 1 and g.val.max() <= 10


def test_pick_sources_nonzero_degree():
    g = graphs.rmat(10, seed=1, weight_seed=2)
    deg = np.diff(g.indptr)
    srcs = graphs.pick_sources(g.indptr, 16, seed=7)
    assert len(set(srcs)) == 16 and all(deg[s] > 0 for s in srcs)


def test_compact_matrix_keeps_exact_narrow_arrays():
    g = graphs.rmat(8, seed=1, weight_seed=2)
    assert g.col.dtype == np.int32 and g.val.dtype == np.float32
    wide = SparseMatrix(g.n, g.indptr, g.col, g.val)
    assert wide.col.dtype == np.int64 and wide.val.dtype == np.float64
    assert wide == g
