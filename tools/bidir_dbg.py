import os, sys, itertools
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_1911_06895_b200 import DeviceGraph, graphs
a = graphs.rmat(15, seed=3, weight_seed=4)
s, d = 19651, 0.05
want, outer, phases = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, d, threads=8)
print("oracle", outer, phases)
base = dict(os.environ)
for k, g0, bid, allin in itertools.product((1, 2, 4), (1, 2, 3, 4, 8), (0, 1), (0, 1)):
    env = dict(base, DS_LEX_K=str(k), DS_HPULL_MIN="0", DS_HPULL_RATIO="0", DS_WIDE_FRAC="1.0", DS_WIDE_G0=str(g0), DS_BIDIR=str(bid), DS_DEBUG_PREP="0")
    if not allin: env["DS_WIDE_ALL"] = "0"
    elif g0 != 1: continue
    os.environ.clear(); os.environ.update(env)
    g = DeviceGraph.from_matrix(a)
    st = g.solve(s, d)
    got = g.result_dense()
    okd = np.array_equal(got.view(np.uint64), want.view(np.uint64))
    print(f"k={k} g0={g0} bidir={bid} all={allin}: dist_ok={okd} outer={st.outer_iterations} phases={st.inner_phases} steps={st.grid_barriers}", "OK" if (okd and st.inner_phases == phases) else "MISMATCH")
    g.close()
