"""GPU parity: the sm_100a path (through the C-ABI library) against golden
vectors recorded from the reference and against the CPU oracle.

Bit-exact for distances (float64 bit patterns) and exact for the
reference's counters (outer_iterations, inner_phases, skip-mode outer).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
from conftest import criterion1_graphs, csr_hash, graph_from_json, unit_graphs, vec_hash
from paper_1911_06895_b200 import (
    BackendChoice,
    DeviceGraph,
    SparseMatrix,
    clear_device_cache,
    delta_stepping,
    delta_stepping_batch,
    graphs,
    matrix_build,
    split_edges,
)

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    a = np.ascontiguousarray(a, dtype=np.float64)
    b = np.ascontiguousarray(b, dtype=np.float64)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def check_run(matrix, source, run):
    d = float.fromhex(run["delta"])
    r = delta_stepping(matrix, source, d)
    assert vec_hash(r.distances.indices, r.distances.values) == run["hash"], (source, d)
    assert r.outer_iterations == run["outer"]
    assert r.inner_phases == run["phases"]
    rs = delta_stepping(matrix, source, d, skip_empty_buckets=True,
                        backend=BackendChoice("fused", workers=4))
    assert rs.distances == r.distances
    assert rs.outer_iterations == run["outer_skip"]
    assert rs.inner_phases == run["phases_skip"]
    if "values" in run:
        assert r.distances.indices.tolist() == run["indices"]
        assert [float(x).hex() for x in r.distances.values] == run["values"]
    return r


def test_hand_cases(golden):
    for name, case in golden["hand"].items():
        n, indptr, col, val = graph_from_json(case["graph"])
        a = SparseMatrix(n, indptr, col, val)
        for run in case["runs"]:
            check_run(a, case["source"], run)


def test_reference_hand_values():
    # test_sssp.py:161-181, 211-219: exact float bits of the traces
    a = matrix_build(3, [(0, 1, 0.4), (1, 2, 0.4), (0, 2, 0.9)])
    assert delta_stepping(a, 0, 1.0).distances.to_dict() == {0: 0.0, 1: 0.4, 2: 0.4 + 0.4}
    b = matrix_build(4, [(0, 1, 0.4), (0, 3, 5.0), (1, 3, 4.2)])
    assert delta_stepping(b, 0, 1.0).distances.get(3) == 0.4 + 4.2
    c = matrix_build(4, [(0, 1, 1.0), (1, 2, 1.0), (2, 3, 1.0)])
    r = delta_stepping(c, 0, 1.0)
    assert r.distances.to_dict() == {0: 0.0, 1: 1.0, 2: 2.0, 3: 3.0}
    assert (r.outer_iterations, r.inner_phases) == (4, 4)
    one = matrix_build(1, [])
    r = delta_stepping(one, 0, 1.0)
    assert r.distances.to_dict() == {0: 0.0} and r.outer_iterations == 1


def test_trusting_constructor_weights(golden):
    # zero / negative / inf / nan weights vanish in the split (sssp.py:96-97)
    for case in golden["trusting"]:
        n, indptr, col, val = graph_from_json(case["graph"])
        a = SparseMatrix(n, indptr, col, val)
        for run in case["runs"]:
            check_run(a, case["source"], run)


def test_criterion1_corpus(golden, corpus_dist):
    offs = corpus_dist["offsets"]
    for (a, s, kind), rec in zip(criterion1_graphs(), golden["criterion1"]):
        assert csr_hash(a.indptr, a.col, a.val) == rec["graph_hash"]
        for run in rec["runs"]:
            check_run(a, s, run)
        if rec["case"] < 100:
            c = rec["case"]
            r = delta_stepping(a, s, 1.0)
            assert np.array_equal(r.distances.indices, corpus_dist["indices"][offs[c]:offs[c + 1]])
            assert bits_equal(r.distances.values, corpus_dist["values"][offs[c]:offs[c + 1]])
    clear_device_cache()


def test_odd_delta_rounding_corpus(golden):
    for rec in golden["odd_delta"]:
        n, indptr, col, val = graph_from_json(rec["graph"])
        a = SparseMatrix(n, indptr, col, val)
        for run in rec["runs"]:
            check_run(a, rec["source"], run)


def test_unit_corpus(golden):
    for a, rec in zip(unit_graphs(), golden["unit"]):
        r = check_run(a, 0, rec["runs"][0])
        assert r.distances.nnz == a.n
        assert r.inner_phases == r.outer_iterations


def test_baseline_shaped_small(golden):
    bs = golden["baseline_shaped"]
    er = graphs.erdos_renyi(1024, seed=0)
    check_run(er, 0, bs["er1024"]["runs"][0])
    for scale in (10, 12):
        g = graphs.rmat(scale, seed=1, weight_seed=2)
        for run in bs[f"rmat{scale}"]["runs"]:
            check_run(g, run["source"], run)
    for side in (32, 64):
        g = graphs.grid2d(side, seed=3)
        check_run(g, 0, bs[f"grid{side}"]["runs"][0])


def test_split_edges_parity(golden):
    for rec in golden["split"]:
        n, indptr, col, val = graph_from_json(rec["graph"])
        a = SparseMatrix(n, indptr, col, val)
        light, heavy = split_edges(a, float.fromhex(rec["delta"]))
        assert csr_hash(light.indptr, light.col, light.val) == rec["light"]
        assert csr_hash(heavy.indptr, heavy.col, heavy.val) == rec["heavy"]


def test_argument_errors_match_reference():
    a = matrix_build(3, [(0, 1, 1.0)])
    with pytest.raises(ValueError, match="out of range"):
        delta_stepping(a, 3, 1.0)
    with pytest.raises(ValueError):
        delta_stepping(a, -1, 1.0)
    for bad in (0.0, -2.0, math.inf, math.nan):
        with pytest.raises(ValueError, match="delta must be a positive finite number"):
            delta_stepping(a, 0, bad)
    with pytest.raises(ValueError):
        split_edges(a, 0.0)


def test_invalid_csr_rejected_by_device_library():
    with pytest.raises(ValueError, match="column index out of range"):
        DeviceGraph.from_csr(3, np.array([0, 1, 1, 1]), np.array([7]), np.array([1.0]))
    with pytest.raises(ValueError, match="indptr"):
        DeviceGraph.from_csr(3, np.array([0, 2, 1, 1]), np.array([1]), np.array([1.0]))


def test_fixed_point_overflow_falls_back_to_f64():
    # integer weights fit 32 bits but path sums do not -> exact f64 rerun
    w = float(2**31)
    a = matrix_build(4, [(0, 1, w), (1, 2, w), (2, 3, w)])
    r = delta_stepping(a, 0, 1e9)
    assert r.distances.to_dict() == {0: 0.0, 1: w, 2: 2 * w, 3: 3 * w}
    assert r.device_stats["fallbacks"] == 1
    want, outer, phases = oracle.delta_stepping(4, a.indptr, a.col, a.val, 0, 1e9)
    assert bits_equal(r.distances.to_dense(), want)
    assert (r.outer_iterations, r.inner_phases) == (outer, phases)


def _dense_check(g: DeviceGraph, a, source, delta, threads, force_f64=False):
    st = g.solve(source, delta, force_f64=force_f64)
    got = g.result_dense()
    want, outer, phases = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, source, delta,
                                                threads=threads)
    assert bits_equal(got, want), (source, delta)
    assert st.inner_phases == phases
    assert st.outer_iterations == outer
    return st


def test_rmat18_sources_vs_oracle():
    a = graphs.rmat(18, seed=1, weight_seed=2)
    g = DeviceGraph.from_matrix(a)
    threads = max(1, oracle.max_threads())
    for s in graphs.pick_sources(a.indptr, 16, seed=7):
        st = _dense_check(g, a, s, 0.1, threads)
        assert st.dist_mode == 0  # exact fixed-point path
    s0 = graphs.pick_sources(a.indptr, 1, seed=11)[0]
    for d in (0.05, 0.25):
        _dense_check(g, a, s0, d, threads)
    # binary64 path gives the same bits
    st = _dense_check(g, a, s0, 0.1, threads, force_f64=True)
    assert st.dist_mode == 1
    g.close()


def test_er1024_config():
    a = graphs.erdos_renyi(1024, seed=0)
    g = DeviceGraph.from_matrix(a)
    for s in range(0, 1024, 97):
        _dense_check(g, a, s, 3.0, 1)
    g.close()


def test_grid_256_vs_oracle():
    a = graphs.grid2d(256, seed=3)
    g = DeviceGraph.from_matrix(a)
    _dense_check(g, a, 0, 25.0, max(1, oracle.max_threads()))
    g.close()


def test_device_rmat_generator_matches_host():
    for scale in (8, 12):
        host = graphs.rmat(scale, seed=1, weight_seed=2)
        dev = DeviceGraph.rmat(scale, 16, 1, 2)
        indptr, col, val = dev.download()
        assert np.array_equal(indptr, host.indptr)
        assert np.array_equal(col, host.col)
        assert np.array_equal(val, host.val)
        dev.close()


def test_grid_4096_vs_dijkstra():
    a = graphs.grid2d(4096, seed=3)
    g = DeviceGraph.from_matrix(a)
    st = g.solve(0, 25.0)
    got = g.result_dense()
    want = oracle.dijkstra(a.n, a.indptr, a.col, a.val, 0)
    assert bits_equal(got, want)
    assert st.reached == a.n
    # skip-mode outer counts non-empty buckets; non-skip is max(d)//delta + 1
    assert st.outer_iterations == math.floor(want.max() / 25.0) + 1
    g.close()


def test_rmat20_fixed_vs_f64_and_dijkstra():
    g = DeviceGraph.rmat(20, 16, 1, 2)
    indptr, col, val = g.download()
    s = graphs.pick_sources(indptr, 1, seed=7)[0]
    st = g.solve(s, 0.1)
    fixed = g.result_dense()
    st64 = g.solve(s, 0.1, force_f64=True)
    f64 = g.result_dense()
    assert bits_equal(fixed, f64)
    assert (st.inner_phases, st.outer_iterations) == (st64.inner_phases, st64.outer_iterations)
    want = oracle.dijkstra(g.n, indptr, col, val, s)
    assert bits_equal(fixed, want)
    g.close()


_PULL_SCRIPT = r"""
import os, sys, numpy as np
sys.path.insert(0, os.environ["REPO"])
import oracle
from paper_1911_06895_b200 import DeviceGraph, graphs
a = graphs.rmat(16, seed=3, weight_seed=4)
g = DeviceGraph.from_matrix(a)
for s in graphs.pick_sources(a.indptr, 3, seed=5):
    st = g.solve(s, 0.1)
    got = g.result_dense()
    want, outer, phases = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, 0.1, threads=4)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))
    assert (st.inner_phases, st.outer_iterations) == (phases, outer)
    assert st.pull_steps > 0, st.pull_steps
d = graphs.erdos_renyi(1024, seed=0)
h = DeviceGraph.from_matrix(d)
st = h.solve(0, 3.0)
assert st.pull_steps == 0  # directed: A^T != A, push only
print("pull ok")
"""


def test_pull_variant_exact_on_symmetric_graphs():
    """The opt-in pull (vxm) build: light and heavy pulls forced on, bit-exact."""
    import os
    import subprocess
    import sys

    from paper_1911_06895_b200.build import LIB_PULL, REPO

    if not os.path.exists(LIB_PULL):
        pytest.skip("pull variant not built")
    env = dict(os.environ, DS_LIB=LIB_PULL, DS_PULL_L="0.2", DS_PULL_H="0.2", REPO=REPO)
    r = subprocess.run([sys.executable, "-c", _PULL_SCRIPT], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "pull ok" in r.stdout


_HANDOFF_SCRIPT = r"""
import os, sys, numpy as np
sys.path.insert(0, os.environ["REPO"])
import oracle
from paper_1911_06895_b200 import DeviceGraph, graphs
cases = [(graphs.rmat(16, seed=3, weight_seed=4), 0.1), (graphs.grid2d(64, seed=3), 25.0),
         (graphs.erdos_renyi(1024, seed=0), 3.0)]
for a, d in cases:
    g = DeviceGraph.from_matrix(a)
    for s in graphs.pick_sources(a.indptr, 2, seed=5):
        st = g.solve(s, d)
        got = g.result_dense()
        want, outer, phases = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, d, threads=4)
        assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (a.n, s)
        assert (st.inner_phases, st.outer_iterations) == (phases, outer)
        st64 = g.solve(s, d, force_f64=True)
        assert np.array_equal(g.result_dense().view(np.uint64), want.view(np.uint64))
    g.close()
print("handoff ok")
"""


def test_giant_push_handoff_is_exact():
    """Every push handed to a standalone launch (thresholds forced down): the
    light ones to k_big_relax, the heavy ones to the gathered heavy step
    (k_big_pull + k_big_commit) on symmetric graphs or to k_big_relax
    (DS_HEAVY_PULL=0, and always for the directed ER graph); the resumed
    persistent kernel stays bit-exact."""
    import os
    import subprocess
    import sys

    from paper_1911_06895_b200.build import REPO

    for pull in ("1", "0"):
        env = dict(os.environ, DS_BIG_L="64", DS_BIG_H="64", DS_HEAVY_PULL=pull, REPO=REPO)
        r = subprocess.run([sys.executable, "-c", _HANDOFF_SCRIPT], env=env, capture_output=True,
                           text=True, timeout=900)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "handoff ok" in r.stdout


def test_block_local_kernel_is_exact():
    """The small-frontier kernel (CTA-0-only phases) forced on for every graph
    shape, with tiny and large local thresholds."""
    import os
    import subprocess
    import sys

    from paper_1911_06895_b200.build import REPO

    for le in ("64", "100000"):
        env = dict(os.environ, DS_SMALL="1", DS_LOCAL_E=le, REPO=REPO)
        r = subprocess.run([sys.executable, "-c", _HANDOFF_SCRIPT], env=env, capture_output=True,
                           text=True, timeout=900)
        assert r.returncode == 0, r.stdout + r.stderr
        assert "handoff ok" in r.stdout


def test_batch_matches_single_solves():
    """ds_sssp_batch (concurrent contexts on SM-disjoint grids) gives every
    source exactly the single-source result and counters."""
    cases = [(graphs.rmat(16, seed=1, weight_seed=2), 0.1, 7),
             (graphs.grid2d(64, seed=3), 25.0, 3),
             (graphs.erdos_renyi(1024, seed=0), 3.0, 5)]
    for a, d, k in cases:
        g = DeviceGraph.from_matrix(a)
        srcs = list(graphs.pick_sources(a.indptr, k, seed=3))
        for skip, f64 in ((False, False), (True, True)):
            want = []
            for s in srcs:
                st = g.solve(s, d, skip_empty_buckets=skip, force_f64=f64)
                want.append((st.inner_phases, st.outer_iterations, st.reached, st.edges_reached,
                             g.result_dense()))
            for conc in (1, 2, 3):
                stats, dist = g.solve_batch(srcs, d, skip_empty_buckets=skip, force_f64=f64,
                                            concurrency=conc)
                assert dist.shape == (k, a.n)
                for i, st in enumerate(stats):
                    assert (st.inner_phases, st.outer_iterations, st.reached,
                            st.edges_reached) == want[i][:4], (conc, i)
                    assert bits_equal(dist[i], want[i][4]), (conc, i)
                    assert st.dist_mode == (1 if f64 else 0)
        # the handle keeps working for single solves after a batch
        st = g.solve(srcs[0], d)
        assert bits_equal(g.result_dense(), want[0][4])
        g.close()


def test_batch_public_api_vs_oracle_and_overflow():
    a = graphs.erdos_renyi(1024, seed=0)
    srcs = list(range(0, 1024, 101))
    res = delta_stepping_batch(a, srcs, 3.0, concurrency=3)
    for s, r in zip(srcs, res):
        want, outer, phases = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, 3.0)
        assert bits_equal(r.distances.to_dense(), want), s
        assert (r.outer_iterations, r.inner_phases) == (outer, phases)
        assert r.distances == delta_stepping(a, s, 3.0).distances
    # sources whose fixed-point distances overflow are rerun in binary64
    w = float(2**31)
    b = matrix_build(4, [(0, 1, w), (1, 2, w), (2, 3, w)])
    res = delta_stepping_batch(b, [0, 1, 2, 3], 1e9, concurrency=2)
    for s, r in zip([0, 1, 2, 3], res):
        want, outer, phases = oracle.delta_stepping(4, b.indptr, b.col, b.val, s, 1e9)
        assert bits_equal(r.distances.to_dense(), want), s
        assert (r.outer_iterations, r.inner_phases) == (outer, phases)
    assert res[0].device_stats["fallbacks"] == 1
    assert delta_stepping_batch(a, [], 3.0) == []
    with pytest.raises(ValueError, match="out of range"):
        delta_stepping_batch(a, [0, 5000], 3.0)


def test_reference_property_suites():
    """The reference's own property tests for this path, on the GPU:
    distances invariant across delta, skip mode never counts more outer
    iterations (test_sssp.py:361-386), unit-weight connected graphs settle
    bucket i at distance i (test_sssp.py:389-401)."""
    from refgen import random_connected_unit_graph, random_graph

    deltas = (0.5, 1.0, 3.0, 11.0)
    rng = np.random.default_rng(103)
    for _ in range(15):
        n = int(rng.integers(2, 50))
        a = random_graph(n, int(rng.integers(1, 4 * n)), rng, weights="int")
        source = int(rng.integers(0, n))
        results = [delta_stepping(a, source, d) for d in deltas]
        for r in results[1:]:
            assert r.distances == results[0].distances
        for d, r in zip(deltas, results):
            sk = delta_stepping(a, source, d, skip_empty_buckets=True)
            assert sk.distances == r.distances and sk.outer_iterations <= r.outer_iterations
    rng = np.random.default_rng(107)
    for _ in range(10):
        n = int(rng.integers(2, 60))
        a = random_connected_unit_graph(n, int(rng.integers(0, n)), rng)
        r = delta_stepping(a, 0, 1.0)
        want, _, _ = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, 0, 1.0)
        assert bits_equal(r.distances.to_dense(), want)
        assert r.distances.nnz == n
        assert r.outer_iterations == int(want.max()) + 1
    # the same invariance at scale: R-MAT 16, four deltas, fixed-point mode
    g = DeviceGraph.from_matrix(graphs.rmat(16, seed=5, weight_seed=6))
    s = int(graphs.pick_sources(g.download()[0], 1, seed=1)[0])
    base = None
    for d in (0.05, 0.1, 0.25, 1.0):
        st = g.solve(s, d)
        assert st.dist_mode == 0
        dd = g.result_dense()
        base = dd if base is None else base
        assert bits_equal(dd, base), d
    g.close()


def test_device_resident_inputs_and_dtypes():
    """ds_graph_create from device pointers (torch CUDA tensors) and from
    pinned host tensors, with int32/int64 columns and f32/f64/i32 weights,
    gives the host-numpy graph's results bit for bit."""
    import torch

    def T(x):  # the containers' arrays are read-only; torch wants writable memory
        return torch.from_numpy(np.array(x))

    a = graphs.rmat(14, seed=3, weight_seed=4)
    s = int(graphs.pick_sources(a.indptr, 1, seed=2)[0])
    want, outer, phases = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, 0.1)
    variants = [
        (T(a.indptr).cuda(), T(a.col.astype(np.int32)).cuda(),
         T(a.val.astype(np.float32)).cuda()),
        (T(a.indptr).cuda(), T(a.col).cuda(),
         T(a.val).cuda()),
        (T(a.indptr).pin_memory(), T(a.col.astype(np.int32)).pin_memory(),
         T(a.val.astype(np.float32)).pin_memory()),
    ]
    for ip, c, v in variants:
        g = DeviceGraph.from_csr(a.n, ip, c, v)
        st = g.solve(s, 0.1)
        assert bits_equal(g.result_dense(), want)
        assert (st.outer_iterations, st.inner_phases) == (outer, phases)
        g.close()
    # integer weights (i32) against the oracle
    b = graphs.erdos_renyi(1024, seed=0)
    g = DeviceGraph.from_csr(b.n, T(b.indptr).cuda(),
                             T(b.col.astype(np.int32)).cuda(),
                             T(b.val.astype(np.int32)).cuda())
    st = g.solve(5, 3.0)
    want, outer, phases = oracle.delta_stepping(b.n, b.indptr, b.col, b.val, 5, 3.0)
    assert bits_equal(g.result_dense(), want)
    assert (st.outer_iterations, st.inner_phases) == (outer, phases)
    g.close()


def test_batch_into_device_buffer():
    """ds_sssp_batch writing its k x n results straight into device memory."""
    import torch

    a = graphs.rmat(15, seed=8, weight_seed=9)
    g = DeviceGraph.from_matrix(a)
    srcs = list(graphs.pick_sources(a.indptr, 5, seed=4))
    out = torch.empty((len(srcs), a.n), dtype=torch.float64, device="cuda")
    stats, none = g.solve_batch(srcs, 0.1, concurrency=2, out=int(out.data_ptr()))
    assert none is None
    torch.cuda.synchronize()
    host = out.cpu().numpy()
    for i, s in enumerate(srcs):
        st = g.solve(s, 0.1)
        assert bits_equal(host[i], g.result_dense())
        assert stats[i].inner_phases == st.inner_phases
    g.close()


def _fixpoint_certificate(indptr, col, val, d_h, s):
    """Size-independent exactness check (tools/rmat27_cert.py): over every
    kept edge (w > 0, sssp.py:106-150) with finite d[u], min_u fl(d[u] + w)
    is >= d[v] everywhere and == d[v] for every reached v != s."""
    import torch

    dev = torch.device("cuda:0")
    n = len(indptr) - 1
    d = torch.from_numpy(d_h).to(dev)
    ip = torch.from_numpy(indptr).to(dev)
    rows = torch.repeat_interleave(torch.arange(n, device=dev), ip[1:] - ip[:-1])
    c = torch.from_numpy(col).to(dev).long()
    w = torch.from_numpy(val).to(dev).double()
    du = d[rows]
    keep = (w > 0) & torch.isfinite(du)
    best = torch.full((n,), float("inf"), dtype=torch.float64, device=dev)
    best.scatter_reduce_(0, c[keep], (du + w)[keep], reduce="amin")
    reached = torch.isfinite(d)
    others = reached.clone()
    others[s] = False
    assert d_h[s] == 0.0
    assert bool((best >= d).all()), "an edge still improves a distance"
    assert bool((best[others] == d[others]).all()), "a distance is not achieved by any edge"
    assert bool(torch.isinf(best[~reached]).all())


@pytest.mark.parametrize("delta", [0.05, 0.25])
def test_rmat22_fixpoint_certificate(delta):
    g = DeviceGraph.rmat(22, 16, 1, 2)
    try:
        indptr, col, val = g.download()
        g.prepare(delta)
        for s in graphs.pick_sources(indptr, 2, seed=5):
            g.solve(int(s), delta)
            _fixpoint_certificate(indptr, col, val, g.result_dense(), int(s))
    finally:
        g.close()
