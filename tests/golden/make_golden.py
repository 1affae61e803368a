"""Generate golden vectors from the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `deltasparse` read-only from /root/reference/pkg/src and records
its outputs for:

* the reference's own hand cases (tests/test_sssp.py:151-219, 287-299,
  349-362; tests/test_acceptance.py:351-380) -- full distance dicts;
* the criterion-1 corpus (700 graphs, CORPUS_SEED=20260816,
  tests/test_acceptance.py:48-66) x delta in {0.5, 1, 3, 11}, plus skip mode;
* the criterion-6 unit-graph corpus (tests/test_acceptance.py:222-244);
* a rounding corpus with non-dyadic deltas (0.1, 0.3, 1/3, 0.7, 2.2);
* graphs with weights the trusting constructor lets through (0, <0, inf, nan);
* this repo's BASELINE-shaped generators at small sizes (ER n=1024, R-MAT
  scale 10/12, grid 32x32 / 64x64);
* split_edges (sssp.py:106-150) light/heavy CSRs.

Outputs: tests/golden/golden.json (counters + hashes + small full vectors)
and tests/golden/corpus_dist.npz (full distances of the first 100 corpus
graphs).  The GPU box never needs /root/reference: tests read only these.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, REPO)
sys.dont_write_bytecode = True

import deltasparse as ref  # noqa: E402

from paper_1911_06895_b200 import graphs  # noqa: E402

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import refgen  # noqa: E402

CORPUS_SEED = 20260816
DELTAS = (0.5, 1.0, 3.0, 11.0)
ODD_DELTAS = (0.1, 0.3, 1.0 / 3.0, 0.7, 2.2)


def vec_hash(idx, val) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(idx, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(val, dtype="<f8").tobytes())
    return h.hexdigest()


def csr_hash(indptr, col, val) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(indptr, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(col, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(val, dtype="<f8").tobytes())
    return h.hexdigest()


def csr_json(a):
    return {"n": a.n, "indptr": a.indptr.tolist(), "col": a.col.tolist(),
            "val": [float(x).hex() for x in a.val]}


def run(a, s, d, skip=False, fused=False):
    be = ref.BackendChoice("fused") if fused else None
    r = ref.delta_stepping(a, s, d, backend=be, skip_empty_buckets=skip)
    return r


def solve_record(a, s, d, fused=False, full=False):
    r = run(a, s, d, fused=fused)
    rs = run(a, s, d, skip=True, fused=fused)
    assert rs.distances == r.distances
    rec = {"delta": float(d).hex(), "outer": r.outer_iterations, "phases": r.inner_phases,
           "outer_skip": rs.outer_iterations, "phases_skip": rs.inner_phases,
           "hash": vec_hash(r.distances.indices, r.distances.values), "nnz": r.distances.nnz}
    if full:
        rec["indices"] = r.distances.indices.tolist()
        rec["values"] = [float(x).hex() for x in r.distances.values]
    return rec


def hand_cases():
    b = ref.matrix_build
    cases = {
        "unit_path": (b(4, [(0, 1, 1.0), (1, 2, 1.0), (2, 3, 1.0)]), 0, [1.0, 0.5, 3.0]),
        "reintroduction": (b(3, [(0, 1, 0.4), (1, 2, 0.4), (0, 2, 0.9)]), 0, [1.0, 0.3]),
        "heavy_min": (b(4, [(0, 1, 0.4), (0, 3, 5.0), (1, 3, 4.2)]), 0, [1.0]),
        "single_vertex": (b(1, []), 0, [1.0]),
        "isolated_source": (b(3, [(1, 2, 1.0)]), 0, [1.0]),
        "disconnected": (b(6, [(0, 1, 2.0), (1, 2, 2.0), (4, 5, 1.0)]), 0, list(DELTAS)),
        "star_long_spoke": (b(7, [(0, k, 1.0) for k in range(1, 6)] + [(0, 6, 100.0)]), 0,
                            list(DELTAS)),
        "triangle": (b(3, [(0, 1, 1.0), (1, 2, 1.0), (0, 2, 3.0)]), 0, [1.0, 0.5]),
    }
    out = {}
    for name, (a, s, ds) in cases.items():
        out[name] = {"graph": csr_json(a), "source": s,
                     "runs": [solve_record(a, s, d, full=True) for d in ds]}
    return out


def trusting_cases():
    """Weights the validating builder rejects but the trusting constructor
    accepts: the split silently drops them (sssp.py:96-97)."""
    rng = np.random.default_rng(4242)
    out = []
    for k in range(20):
        n = int(rng.integers(3, 40))
        a = ref.random_graph(n, int(rng.integers(n, 5 * n)), rng, weights="float")
        val = a.val.copy()
        if val.size:
            pick = rng.choice(val.size, size=max(1, val.size // 5), replace=False)
            bad = np.array([0.0, -1.5, np.inf, np.nan, -0.0])
            val[pick] = bad[rng.integers(0, bad.size, size=pick.size)]
        t = ref.SparseMatrix(n, a.indptr, a.col, val)
        s = int(rng.integers(0, n))
        runs = [solve_record(t, s, d, full=True) for d in (0.5, 3.0)]
        out.append({"graph": csr_json(t), "source": s, "runs": runs})
    return out


def criterion1_corpus():
    rng = np.random.default_rng(CORPUS_SEED)
    recs, full_idx, full_val, offs = [], [], [], [0]
    mine_rng = np.random.default_rng(CORPUS_SEED)
    for case in range(700):
        kind = "int" if case < 500 else "float"
        n = int(rng.integers(1, 201))
        m = int(rng.integers(0, 2001))
        a = ref.random_graph(n, m, rng, weights=kind)
        s = int(rng.integers(0, n))
        # the restated generator must reproduce the reference's matrices
        n2 = int(mine_rng.integers(1, 201))
        m2 = int(mine_rng.integers(0, 2001))
        b = refgen.random_graph(n2, m2, mine_rng, weights=kind)
        s2 = int(mine_rng.integers(0, n2))
        assert (n, m, s) == (n2, m2, s2)
        assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.col, b.col)
        assert np.array_equal(a.val.view(np.uint64), b.val.view(np.uint64))
        want = ref.dijkstra_oracle(a, s)
        runs = [solve_record(a, s, d) for d in DELTAS]
        for r in runs:
            if kind == "int":
                assert r["hash"] == vec_hash(want.indices, want.values)
        recs.append({"case": case, "n": n, "m": m, "source": s, "kind": kind,
                     "nnz": a.nnz, "graph_hash": csr_hash(a.indptr, a.col, a.val),
                     "dijkstra_hash": vec_hash(want.indices, want.values), "runs": runs})
        if case < 100:
            r = run(a, s, 1.0)
            full_idx.append(r.distances.indices)
            full_val.append(r.distances.values)
            offs.append(offs[-1] + r.distances.nnz)
    np.savez_compressed(os.path.join(HERE, "corpus_dist.npz"),
                        indices=np.concatenate(full_idx), values=np.concatenate(full_val),
                        offsets=np.array(offs, dtype=np.int64))
    return recs


def odd_delta_corpus():
    rng = np.random.default_rng(CORPUS_SEED + 100)
    recs = []
    for case in range(150):
        n = int(rng.integers(2, 120))
        m = int(rng.integers(0, 8 * n))
        kind = "float" if case % 3 else "int"
        a = ref.random_graph(n, m, rng, weights=kind)
        # shrink float weights toward the delta range so light edges exist
        if kind == "float":
            a = ref.SparseMatrix(a.n, a.indptr, a.col, a.val / 10.0)
        s = int(rng.integers(0, n))
        runs = [solve_record(a, s, d) for d in ODD_DELTAS]
        recs.append({"case": case, "graph": csr_json(a), "source": s, "runs": runs})
    return recs


def unit_corpus():
    rng = np.random.default_rng(CORPUS_SEED + 6)
    recs = []
    mine = np.random.default_rng(CORPUS_SEED + 6)
    for case in range(50):
        n = int(rng.integers(2, 121))
        a = ref.random_connected_unit_graph(n, int(rng.integers(0, 2 * n)), rng)
        n2 = int(mine.integers(2, 121))
        b = refgen.random_connected_unit_graph(n2, int(mine.integers(0, 2 * n2)), mine)
        assert np.array_equal(a.indptr, b.indptr) and np.array_equal(a.col, b.col)
        runs = [solve_record(a, 0, 1.0)]
        recs.append({"case": case, "n": n, "graph_hash": csr_hash(a.indptr, a.col, a.val),
                     "runs": runs})
    return recs


def baseline_shaped():
    out = {}
    er = graphs.erdos_renyi(1024, seed=0)
    a = ref.SparseMatrix(er.n, er.indptr, er.col, er.val)
    a.check_invariants()
    out["er1024"] = {"graph_hash": csr_hash(a.indptr, a.col, a.val), "source": 0,
                     "runs": [solve_record(a, 0, 3.0, full=True)]}
    for scale in (10, 12):
        g = graphs.rmat(scale, seed=1, weight_seed=2)
        a = ref.SparseMatrix(g.n, g.indptr, g.col.astype(np.int64), g.val.astype(np.float64))
        a.check_invariants()
        srcs = graphs.pick_sources(g.indptr, 4, seed=7)
        runs = []
        for s in srcs:
            for d in (0.05, 0.1, 0.25):
                rec = solve_record(a, s, d, fused=True)
                rec["source"] = s
                runs.append(rec)
        out[f"rmat{scale}"] = {"graph_hash": csr_hash(a.indptr, a.col, a.val), "runs": runs}
    for side in (32, 64):
        g = graphs.grid2d(side, seed=3)
        a = ref.SparseMatrix(g.n, g.indptr, g.col.astype(np.int64), g.val.astype(np.float64))
        a.check_invariants()
        out[f"grid{side}"] = {"graph_hash": csr_hash(a.indptr, a.col, a.val), "source": 0,
                              "runs": [solve_record(a, 0, 25.0, fused=True)]}
    return out


def split_cases():
    rng = np.random.default_rng(CORPUS_SEED + 3)
    recs = []
    for _ in range(40):
        n = int(rng.integers(2, 80))
        a = ref.random_graph(n, int(rng.integers(0, 6 * n)), rng, weights="float")
        d = float(10.0 * rng.random() + 0.05)
        light, heavy = ref.split_edges(a, d)
        recs.append({"graph": csr_json(a), "delta": d.hex(),
                     "light": csr_hash(light.indptr, light.col, light.val),
                     "heavy": csr_hash(heavy.indptr, heavy.col, heavy.val)})
    return recs


def main():
    gold = {
        "generator": "tests/golden/make_golden.py",
        "reference": "/root/reference/pkg/src/deltasparse (unmodified)",
        "hand": hand_cases(),
        "trusting": trusting_cases(),
        "criterion1": criterion1_corpus(),
        "odd_delta": odd_delta_corpus(),
        "unit": unit_corpus(),
        "baseline_shaped": baseline_shaped(),
        "split": split_cases(),
    }
    with open(os.path.join(HERE, "golden.json"), "w") as f:
        json.dump(gold, f, separators=(",", ":"))
    print("wrote golden.json and corpus_dist.npz")


if __name__ == "__main__":
    main()
