"""Drop-in contract beyond the numbers: concurrent callers on one shared
matrix, the phase-ceiling error path (sssp.py:268-274,
296-301) and caller-buffer validation.  Through the C-ABI library."""

from __future__ import annotations

import math
import threading

import numpy as np
import pytest

import oracle
from paper_1911_06895_b200 import (
    DeviceGraph,
    SparseMatrix,
    clear_device_cache,
    delta_stepping,
    delta_stepping_batch,
    graphs,
    matrix_build,
)

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.ascontiguousarray(a, dtype=np.float64).view(np.uint64)


def test_concurrent_threads_share_one_matrix():
    # four threads solve different sources of ONE matrix object while a fifth
    # keeps evicting the device cache: every result must equal the oracle
    a = graphs.rmat(14, seed=3, weight_seed=4)
    b = graphs.rmat(12, seed=5, weight_seed=6)  # a second matrix: cache churn
    srcs = [int(s) for s in graphs.pick_sources(a.indptr, 8, seed=21)]
    want = {}
    for s in srcs:
        d, outer, phases = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, 0.1, threads=4)
        want[s] = (oracle.to_sparse(d), outer, phases)
    errors = []
    stop = threading.Event()

    def worker(k):
        try:
            for rep in range(3):
                for s in srcs[k::4]:
                    r = delta_stepping(a, s, 0.1)
                    (idx, val), outer, phases = want[s]
                    assert np.array_equal(r.distances.indices, idx), s
                    assert np.array_equal(_bits(r.distances.values), _bits(val)), s
                    assert (r.outer_iterations, r.inner_phases) == (outer, phases), s
                    if rep == 1:
                        rs = delta_stepping_batch(a, [s, srcs[0]], 0.1)
                        assert rs[0].distances == r.distances
        except Exception as e:  # noqa: BLE001 - reported below
            errors.append(e)

    def churn():
        while not stop.is_set():
            delta_stepping(b, 0, 0.1)
            clear_device_cache()

    ts = [threading.Thread(target=worker, args=(k,)) for k in range(4)]
    c = threading.Thread(target=churn)
    c.start()
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    stop.set()
    c.join()
    clear_device_cache()
    assert not errors, errors[0]


def test_phase_ceiling_error_path(monkeypatch):
    # the ceiling formula (sssp.py:268-274) ...
    a = graphs.rmat(10, seed=1, weight_seed=2)
    g = DeviceGraph.from_matrix(a)
    try:
        info = g.prepare(0.1)
        light = a.val[(a.val > 0) & (a.val <= 0.1)]
        assert info.phase_ceiling == a.n * (int(math.ceil(0.1 / float(light.min()))) + 2)
    finally:
        g.close()
    # ... and its RuntimeError (sssp.py:296-301), reached with a test ceiling
    monkeypatch.setenv("DS_CEILING_OVERRIDE", "3")
    clear_device_cache()
    m = matrix_build(6, [(0, 1, 0.25), (1, 2, 0.25), (2, 3, 0.25), (3, 4, 0.25), (4, 5, 0.25)])
    with pytest.raises(RuntimeError, match=r"light phase count exceeded ceiling 3; "
                                           r"relaxation is not converging"):
        delta_stepping(m, 0, 1.0)
    with pytest.raises(RuntimeError, match="exceeded ceiling 3"):
        delta_stepping_batch(m, [0], 1.0)
    monkeypatch.delenv("DS_CEILING_OVERRIDE")
    clear_device_cache()
    r = delta_stepping(m, 0, 1.0)  # 4 + 2 phases: fine with the real ceiling
    want, outer, phases = oracle.delta_stepping(m.n, m.indptr, m.col, m.val, 0, 1.0)
    assert (r.outer_iterations, r.inner_phases) == (outer, phases) == (2, 6)
    assert r.distances.to_dict()[5] == 1.25
    clear_device_cache()


def test_caller_buffers_are_validated():
    a = graphs.rmat(10, seed=1, weight_seed=2)
    g = DeviceGraph.from_matrix(a)
    try:
        st = g.solve(0, 0.1)
        with pytest.raises(ValueError, match="float64"):
            g.result_dense(out=np.empty(a.n, dtype=np.float32))
        with pytest.raises(ValueError, match="needs"):
            g.result_dense(out=np.empty(a.n - 1, dtype=np.float64))
        with pytest.raises(ValueError, match="contiguous"):
            g.result_dense(out=np.empty(2 * a.n, dtype=np.float64)[::2])
        r = int(st.reached)
        with pytest.raises(ValueError, match="int64"):
            g.result_sparse(out=(np.empty(r, dtype=np.int32), np.empty(r)))
        with pytest.raises(ValueError, match="needs"):
            g.solve_batch([0, 1], 0.1, out=np.empty((1, a.n)))
        good = g.result_dense(out=np.empty(a.n, dtype=np.float64))
        assert good[0] == 0.0 or np.isfinite(good).any()
    finally:
        g.close()
