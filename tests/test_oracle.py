"""Pin the CPU oracle (oracle/oracle.c) against golden vectors recorded from
the unmodified reference (tests/golden/make_golden.py).  CPU only."""

from __future__ import annotations

import math

import numpy as np
import pytest

import oracle
from conftest import criterion1_graphs, csr_hash, graph_from_json, unit_graphs, vec_hash
from paper_1911_06895_b200 import graphs


def check_run(n, indptr, col, val, source, run, threads=1):
    d = float.fromhex(run["delta"])
    dist, outer, phases = oracle.delta_stepping(n, indptr, col, val, source, d, threads=threads)
    idx, v = oracle.to_sparse(dist)
    assert vec_hash(idx, v) == run["hash"]
    assert outer == run["outer"]
    assert phases == run["phases"]
    dist2, outer_s, phases_s = oracle.delta_stepping(n, indptr, col, val, source, d,
                                                     skip_empty_buckets=True, threads=threads)
    assert np.array_equal(dist.view(np.uint64), dist2.view(np.uint64))
    assert outer_s == run["outer_skip"]
    assert phases_s == run["phases_skip"]
    if "values" in run:
        assert idx.tolist() == run["indices"]
        assert [float(x).hex() for x in v] == run["values"]


def test_hand_cases(golden):
    for name, case in golden["hand"].items():
        n, indptr, col, val = graph_from_json(case["graph"])
        for run in case["runs"]:
            check_run(n, indptr, col, val, case["source"], run)


def test_reintroduction_and_heavy_min_values(golden):
    # exact float bits from the reference's hand traces (test_sssp.py:161-219)
    r = golden["hand"]["reintroduction"]["runs"][0]
    assert [float.fromhex(x) for x in r["values"]] == [0.0, 0.4, 0.4 + 0.4]
    h = golden["hand"]["heavy_min"]["runs"][0]
    assert float.fromhex(h["values"][-1]) == 0.4 + 4.2


def test_trusting_constructor_weights(golden):
    for case in golden["trusting"]:
        n, indptr, col, val = graph_from_json(case["graph"])
        for run in case["runs"]:
            check_run(n, indptr, col, val, case["source"], run)


def test_criterion1_corpus(golden, corpus_dist):
    recs = golden["criterion1"]
    offs = corpus_dist["offsets"]
    for (a, s, kind), rec in zip(criterion1_graphs(), recs):
        assert csr_hash(a.indptr, a.col, a.val) == rec["graph_hash"]
        assert s == rec["source"]
        for run in rec["runs"]:
            check_run(a.n, a.indptr, a.col, a.val, s, run)
        if rec["case"] < 100:
            c = rec["case"]
            dist, _, _ = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, 1.0)
            idx, v = oracle.to_sparse(dist)
            assert np.array_equal(idx, corpus_dist["indices"][offs[c]:offs[c + 1]])
            assert np.array_equal(v.view(np.uint64),
                                  corpus_dist["values"][offs[c]:offs[c + 1]].view(np.uint64))


def test_odd_delta_rounding_corpus(golden):
    for rec in golden["odd_delta"]:
        n, indptr, col, val = graph_from_json(rec["graph"])
        for run in rec["runs"]:
            check_run(n, indptr, col, val, rec["source"], run)


def test_unit_corpus_bfs_counters(golden):
    for a, rec in zip(unit_graphs(), golden["unit"]):
        assert csr_hash(a.indptr, a.col, a.val) == rec["graph_hash"]
        check_run(a.n, a.indptr, a.col, a.val, 0, rec["runs"][0])
        run = rec["runs"][0]
        assert run["nnz"] == a.n
        assert run["phases"] == run["outer"]


def test_baseline_shaped(golden):
    bs = golden["baseline_shaped"]
    er = graphs.erdos_renyi(1024, seed=0)
    assert csr_hash(er.indptr, er.col, er.val) == bs["er1024"]["graph_hash"]
    check_run(er.n, er.indptr, er.col, er.val, 0, bs["er1024"]["runs"][0], threads=2)
    for scale in (10, 12):
        g = graphs.rmat(scale, seed=1, weight_seed=2)
        assert csr_hash(g.indptr, g.col, g.val) == bs[f"rmat{scale}"]["graph_hash"]
        for run in bs[f"rmat{scale}"]["runs"]:
            check_run(g.n, g.indptr, g.col, g.val, run["source"], run, threads=4)
    for side in (32, 64):
        g = graphs.grid2d(side, seed=3)
        assert csr_hash(g.indptr, g.col, g.val) == bs[f"grid{side}"]["graph_hash"]
        check_run(g.n, g.indptr, g.col, g.val, 0, bs[f"grid{side}"]["runs"][0])


def test_split_edges(golden):
    for rec in golden["split"]:
        n, indptr, col, val = graph_from_json(rec["graph"])
        d = float.fromhex(rec["delta"])
        assert csr_hash(*oracle.split(n, indptr, col, val, d, 0)) == rec["light"]
        assert csr_hash(*oracle.split(n, indptr, col, val, d, 1)) == rec["heavy"]


def test_dijkstra_matches_delta_stepping_on_int_corpus(golden):
    for (a, s, kind), rec in zip(criterion1_graphs()[:200], golden["criterion1"][:200]):
        dist = oracle.dijkstra(a.n, a.indptr, a.col, a.val, s)
        idx, v = oracle.to_sparse(dist)
        assert vec_hash(idx, v) == rec["dijkstra_hash"]


def test_oracle_rejects_bad_arguments():
    indptr = np.array([0, 1, 1, 1]); col = np.array([1]); val = np.array([1.0])
    for bad in (0.0, -2.0, math.inf, math.nan):
        with pytest.raises(ValueError):
            oracle.delta_stepping(3, indptr, col, val, 0, bad)
    with pytest.raises(ValueError):
        oracle.delta_stepping(3, indptr, col, val, 3, 1.0)


def test_threads_do_not_change_results():
    g = graphs.rmat(11, seed=5, weight_seed=6)
    base = oracle.delta_stepping(g.n, g.indptr, g.col, g.val, 3, 0.1, threads=1)
    for t in (2, 4):
        got = oracle.delta_stepping(g.n, g.indptr, g.col, g.val, 3, 0.1, threads=t)
        assert np.array_equal(got[0].view(np.uint64), base[0].view(np.uint64))
        assert got[1:] == base[1:]


def test_host_rmat_generator_matches_graphs_rmat():
    # the reference arm's input generator (oracle/rmat.c) must build exactly
    # the CSR of graphs.rmat, which the device generator is pinned to as well
    import oracle
    from paper_1911_06895_b200 import graphs

    for scale, ef, seed, wseed in [(6, 16, 1, 2), (11, 16, 1, 2), (14, 16, 1, 2), (12, 8, 5, 9)]:
        ip, col, val = oracle.rmat(scale, ef, seed, wseed)
        a = graphs.rmat(scale, ef, seed, wseed)
        assert np.array_equal(ip, a.indptr)
        assert np.array_equal(col, a.col)
        assert np.array_equal(val.view(np.uint32), np.asarray(a.val, dtype=np.float32).view(np.uint32))
