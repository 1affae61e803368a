"""Small solves for compute-sanitizer runs (memcheck / racecheck / synccheck /
initcheck): R-MAT 10 (push + heavy gather), grid 32^2 (block-local kernel),
ER 1024 (directed: push only), a batch at concurrency 2, forced binary64.
Each result is checked against the oracle so a sanitizer-perturbed schedule
that changed a result would also fail here.

    compute-sanitizer --tool racecheck python tools/sanitize_probe.py
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import oracle
from paper_1911_06895_b200 import DeviceGraph, graphs


def check(g, a, s, delta, **kw):
    st = g.solve(s, delta, **kw)
    got = g.result_dense()
    want, outer, phases = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, delta)
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64)), (s, delta, kw)
    assert (st.outer_iterations, st.inner_phases) == (outer, phases), (s, delta, kw)
    return st


cases = [(graphs.rmat(10, seed=1, weight_seed=2), 0.1), (graphs.grid2d(32, seed=3), 25.0),
         (graphs.erdos_renyi(1024, seed=0), 3.0)]
for a, delta in cases:
    g = DeviceGraph.from_matrix(a)
    srcs = graphs.pick_sources(a.indptr, 2, seed=5)
    for s in srcs:
        check(g, a, int(s), delta)
    check(g, a, int(srcs[0]), delta, force_f64=True)
    stats, dist = g.solve_batch(srcs, delta, concurrency=2)
    for i, s in enumerate(srcs):
        want, _, _ = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, int(s), delta)
        assert np.array_equal(dist[i].view(np.uint64), want.view(np.uint64))
    g.close()
print("sanitize probe ok")
