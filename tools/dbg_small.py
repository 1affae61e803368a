import os, sys, time
sys.path.insert(0, "/root/repo")
import numpy as np
import oracle
from paper_1911_06895_b200 import DeviceGraph, graphs
cases = [("rmat16", graphs.rmat(16, seed=3, weight_seed=4), 0.1), ("grid64", graphs.grid2d(64, seed=3), 25.0),
         ("er", graphs.erdos_renyi(1024, seed=0), 3.0)]
for name, a, d in cases:
    g = DeviceGraph.from_matrix(a)
    for s in graphs.pick_sources(a.indptr, 2, seed=5):
        for f64 in (False, True):
            t = time.time()
            try:
                st = g.solve(s, d, force_f64=f64)
                got = g.result_dense()
                want, outer, phases = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, d, threads=4)
                ok = np.array_equal(got.view(np.uint64), want.view(np.uint64)) and (st.inner_phases, st.outer_iterations) == (phases, outer)
                print(name, s, f64, "ok" if ok else "MISMATCH", round(time.time() - t, 2), st.inner_phases, phases, flush=True)
            except Exception as e:
                print(name, s, f64, "ERR", e, round(time.time() - t, 2), flush=True)
    g.close()
