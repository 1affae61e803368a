"""Per-source kernel time, single solves vs ds_sssp_batch, lex vs classic, on
the bench pool (R-MAT SCALE, delta 0.1); results must agree bit for bit."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1911_06895_b200 import DeviceGraph, graphs
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
k = int(sys.argv[2]) if len(sys.argv) > 2 else 16
g = DeviceGraph.rmat(scale, 16, 1, 2)
ip = g.download_indptr()
pool = graphs.pick_sources(ip, 64, seed=7)[:k]
out = {}
ref = {}
for name, env in (("classic", "0"), ("lex", None)):
    if env is None:
        os.environ.pop("DS_LEX", None)
    else:
        os.environ["DS_LEX"] = env
    g.prepare(0.1)
    g.solve(pool[0], 0.1)
    single = []
    for s in pool:
        st = g.solve(s, 0.1)
        single.append(st.kernel_ms)
        d = g.result_dense().view(np.uint64).copy()
        if s in ref:
            assert np.array_equal(ref[s][0], d) and ref[s][1] == (st.outer_iterations, st.inner_phases), s
        else:
            ref[s] = (d, (st.outer_iterations, st.inner_phases))
    stats, dist = g.solve_batch(pool, 0.1, concurrency=1)
    for i, s in enumerate(pool):
        assert np.array_equal(ref[s][0], dist[i].view(np.uint64)), ("batch", s)
    out[name] = {"single_mean": float(np.mean(single)), "batch_mean": float(np.mean([st.kernel_ms for st in stats])),
                 "single": [round(x, 2) for x in single], "batch": [round(st.kernel_ms, 2) for st in stats]}
print(json.dumps(out))
