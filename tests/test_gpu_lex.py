"""Lex mode (sssp_kernel.cuh "lex mode"): the solver runs ksub internal
buckets per reference bucket and recovers the reference's counters from hop
counts carried in the distance keys.  On by default only for large graphs,
so here it is forced (DS_LEX_K) on small ones and checked bit for bit --
distances, outer_iterations in both skip modes, inner_phases -- against the
golden vectors recorded from the reference and against the oracle."""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from conftest import criterion1_graphs, graph_from_json, vec_hash
from paper_1911_06895_b200 import (
    DeviceGraph,
    SparseMatrix,
    clear_device_cache,
    delta_stepping,
    graphs,
)

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.fixture(params=[2, 4, 8])
def lex_k(request, monkeypatch):
    monkeypatch.setenv("DS_LEX_K", str(request.param))
    clear_device_cache()
    yield request.param
    clear_device_cache()


def _check(a, s, d):
    r = delta_stepping(a, s, d)
    want, outer, phases = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, d, threads=4)
    idx = np.flatnonzero(np.isfinite(want))
    assert np.array_equal(r.distances.indices, idx), (s, d)
    assert np.array_equal(_bits(r.distances.values), _bits(want[idx])), (s, d)
    assert (r.outer_iterations, r.inner_phases) == (outer, phases), (s, d)
    rs = delta_stepping(a, s, d, skip_empty_buckets=True)
    _, outer_s, phases_s = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, d,
                                                 skip_empty_buckets=True, threads=4)
    assert rs.distances == r.distances
    assert (rs.outer_iterations, rs.inner_phases) == (outer_s, phases_s), (s, d)
    return r


def test_lex_rmat_deltas(lex_k):
    a = graphs.rmat(15, seed=3, weight_seed=4)
    for d in (0.05, 0.1, 0.25, 0.7):
        for s in graphs.pick_sources(a.indptr, 3, seed=17):
            r = _check(a, int(s), d)
            assert r.device_stats["dist_mode"] == 0  # fixed point (lex needs it)


def test_lex_er_integer_weights(lex_k):
    a = graphs.erdos_renyi(1024, seed=0)  # directed: heavy steps push
    for d in (3.0, 5.0, 10.0):
        for s in (0, 17, 900):
            _check(a, s, d)


def test_lex_golden_corpus(lex_k, golden):
    # the reference's own criterion-1 corpus (float 10(1-U), int, unit
    # weights) at its recorded deltas: the golden hashes and counters
    for (a, s, kind), rec in list(zip(criterion1_graphs(), golden["criterion1"]))[::7]:
        for run in rec["runs"]:
            d = float.fromhex(run["delta"])
            r = delta_stepping(a, s, d)
            assert vec_hash(r.distances.indices, r.distances.values) == run["hash"]
            assert (r.outer_iterations, r.inner_phases) == (run["outer"], run["phases"])
            rs = delta_stepping(a, s, d, skip_empty_buckets=True)
            assert (rs.outer_iterations, rs.inner_phases) == (run["outer_skip"], run["phases_skip"])
    for rec in golden["odd_delta"]:
        n, indptr, col, val = graph_from_json(rec["graph"])
        a = SparseMatrix(n, indptr, col, val)
        for run in rec["runs"]:
            d = float.fromhex(run["delta"])
            r = delta_stepping(a, rec["source"], d)
            assert vec_hash(r.distances.indices, r.distances.values) == run["hash"]
            assert (r.outer_iterations, r.inner_phases) == (run["outer"], run["phases"])


def test_lex_batch_matches_single(lex_k):
    a = graphs.rmat(14, seed=5, weight_seed=6)
    g = DeviceGraph.from_matrix(a)
    try:
        srcs = graphs.pick_sources(a.indptr, 6, seed=3)
        stats, dist = g.solve_batch(srcs, 0.1, concurrency=3)
        for i, s in enumerate(srcs):
            st = g.solve(int(s), 0.1)
            assert np.array_equal(_bits(dist[i]), _bits(g.result_dense()))
            assert (stats[i].outer_iterations, stats[i].inner_phases) == (st.outer_iterations, st.inner_phases)
    finally:
        g.close()


# ---- wide windows: the lex-mode tail merges internal buckets into one window
# whose closure pushes every edge (sssp_kernel.cuh "wide windows"); forced from
# the second bucket on here, with growing and shrinking window sizes.
@pytest.fixture(params=["grow", "shrink", "fixed3"])
def wide_mode(request, monkeypatch):
    monkeypatch.setenv("DS_LEX_K", "2")
    monkeypatch.setenv("DS_WIDE_FORCE", "1")
    if request.param == "grow":
        monkeypatch.setenv("DS_WIDE_G0", "1")
        monkeypatch.setenv("DS_WIDE_LO", "1e18")  # every window doubles the next one
    elif request.param == "shrink":
        monkeypatch.setenv("DS_WIDE_G0", "7")
        monkeypatch.setenv("DS_WIDE_LO", "0")
        monkeypatch.setenv("DS_WIDE_HI", "100")  # halves down to the narrow schedule and re-enters
    else:
        monkeypatch.setenv("DS_WIDE_G0", "3")
        monkeypatch.setenv("DS_WIDE_LO", "0")
        monkeypatch.setenv("DS_WIDE_HI", "1e18")
    clear_device_cache()
    yield request.param
    clear_device_cache()


def test_wide_windows_rmat(wide_mode):
    a = graphs.rmat(15, seed=3, weight_seed=4)
    for d in (0.05, 0.1, 0.25):
        for s in graphs.pick_sources(a.indptr, 3, seed=23):
            _check(a, int(s), d)


def test_wide_windows_er_and_grid(wide_mode):
    a = graphs.erdos_renyi(1024, seed=0)  # directed, integer weights
    for d in (3.0, 10.0):
        for s in (0, 17):
            _check(a, s, d)
    g = graphs.grid2d(48, seed=2)  # many reference buckets per window
    _check(g, 0, 25.0)


def test_wide_windows_golden_corpus(wide_mode, golden):
    for (a, s, kind), rec in list(zip(criterion1_graphs(), golden["criterion1"]))[::11]:
        for run in rec["runs"]:
            d = float.fromhex(run["delta"])
            r = delta_stepping(a, s, d)
            assert vec_hash(r.distances.indices, r.distances.values) == run["hash"]
            assert (r.outer_iterations, r.inner_phases) == (run["outer"], run["phases"])
            rs = delta_stepping(a, s, d, skip_empty_buckets=True)
            assert (rs.outer_iterations, rs.inner_phases) == (run["outer_skip"], run["phases_skip"])


# ---- the bidirectional entry into the wide tail (heavy gather + the window's
# scan + its first round in one pass), forced at the first bucket with a heavy
# step on symmetric graphs, with whole-tail and small first windows
@pytest.fixture(params=["all", "g3", "g1"])
def bidir_mode(request, monkeypatch):
    monkeypatch.setenv("DS_LEX_K", "2")
    monkeypatch.setenv("DS_HPULL_MIN", "0")
    monkeypatch.setenv("DS_HPULL_RATIO", "0")
    monkeypatch.setenv("DS_WIDE_FRAC", "1.0")
    if request.param != "all":
        monkeypatch.setenv("DS_WIDE_ALL", "0")
        monkeypatch.setenv("DS_WIDE_G0", request.param[1:])
    clear_device_cache()
    yield request.param
    clear_device_cache()


def test_bidirectional_entry(bidir_mode):
    a = graphs.rmat(15, seed=3, weight_seed=4)
    for d in (0.05, 0.1, 0.25):
        for s in graphs.pick_sources(a.indptr, 3, seed=29):
            _check(a, int(s), d)
    _check(graphs.grid2d(48, seed=2), 0, 25.0)
    b = graphs.rmat(12, seed=9, weight_seed=1)
    for s in graphs.pick_sources(b.indptr, 4, seed=5):
        _check(b, int(s), 0.3)


def test_batch_lex_range_failure_reruns_as_a_batch():
    """fp32-lattice weights with distances beyond the key range (D >= 2^26 at 24
    fractional bits, i.e. >= 4.0): every lex solve of the batch raises the range
    flag, the handle switches to the reference's schedule and the failed sources
    run again as a batch -- same results as single solves and the oracle."""
    # a path graph with weights near 0.5: the far end lies at ~32
    n = 64
    rng = np.random.default_rng(3)
    w = (np.floor((0.5 + 0.25 * rng.random(n - 1)) * (1 << 24)) / (1 << 24))
    edges = []
    for i in range(n - 1):
        edges.append((i, i + 1, w[i]))
        edges.append((i + 1, i, w[i]))
    from paper_1911_06895_b200 import matrix_build
    a = matrix_build(n, np.array(edges))
    g = DeviceGraph.from_matrix(a)
    try:
        srcs = [0, 5, 17, 40, 63]
        stats, dist = g.solve_batch(srcs, 0.3, concurrency=3)
        for i, s in enumerate(srcs):
            want, outer, phases = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, 0.3, threads=2)
            assert np.array_equal(_bits(dist[i]), _bits(want)), s
            assert (stats[i].outer_iterations, stats[i].inner_phases) == (outer, phases), s
    finally:
        g.close()
