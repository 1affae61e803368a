"""Parity at the headline sizes (BASELINE.json configs[3] and configs[4]).

* R-MAT 24, delta in {0.05, 0.1, 0.25} (configs[3], the bench's workload):
  one bench-pool source per delta (graphs.pick_sources(..., 64, seed=7), the
  pool bench.py draws from) against the C restatement of the reference
  (oracle/, all host threads): distances bit for bit and both counters
  (sssp.py:239-313, counters :296 and :304); the forced-binary64 mode (the
  path every non-lattice weight takes) must reproduce the same result.
R-MAT 27 (configs[4]) is in test_gpu_rmat27.py (its own module, so this
module's R-MAT 24 graph is freed first).
"""

from __future__ import annotations

import numpy as np
import pytest

import oracle
from paper_1911_06895_b200 import DeviceGraph, graphs

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


@pytest.fixture(scope="module")
def rmat24():
    g = DeviceGraph.rmat(24, 16, 1, 2)
    indptr, col, val = g.download()
    # the oracle's layout (int64 columns, float64 weights), converted once
    col = col.astype(np.int64)
    val = val.astype(np.float64)
    yield g, indptr, col, val
    g.close()


@pytest.mark.parametrize("delta,k", [(0.05, 1), (0.1, 0), (0.25, 2)])
def test_rmat24_headline_vs_oracle(rmat24, delta, k):
    g, indptr, col, val = rmat24
    s = int(graphs.pick_sources(indptr, 64, seed=7)[k])
    st = g.solve(s, delta)
    got = g.result_dense()
    want, outer, phases = oracle.delta_stepping(g.n, indptr, col, val, s, delta,
                                                threads=max(1, oracle.max_threads()))
    assert np.array_equal(_bits(got), _bits(want)), f"distances differ (source {s}, delta {delta})"
    assert (st.outer_iterations, st.inner_phases) == (outer, phases)
    assert st.edges_reached == int(np.diff(indptr)[np.isfinite(want)].sum())
    # skip_empty_buckets=True: same distances and phases; outer = visited buckets
    sk = g.solve(s, delta, skip_empty_buckets=True)
    assert np.array_equal(_bits(g.result_dense()), _bits(want))
    assert sk.inner_phases == phases and sk.outer_iterations == sk.buckets_visited
    # forced binary64 distances (u64 atomicMin on the bit patterns)
    f = g.solve(s, delta, force_f64=True)
    assert f.dist_mode == 1
    assert np.array_equal(_bits(g.result_dense()), _bits(want))
    assert (f.outer_iterations, f.inner_phases) == (outer, phases)
    g.prepare(delta)  # back to the fixed-point split for the next case
