"""Same-process A/B of lex / pile settings on the bench pool: mean kernel ms,
work and barriers per config; every config must match the classic result
bit for bit (distances and counters)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1911_06895_b200 import DeviceGraph, graphs
scale = int(sys.argv[1]); delta = float(sys.argv[2]); nsrc = int(sys.argv[3])
confs = [("classic", {"DS_LEX": "0"})]
for spec in sys.argv[4:]:
    parts = spec.split()
    confs.append((parts[0], dict(kv.split("=", 1) for kv in parts[1:])))
g = DeviceGraph.rmat(scale, 16, 1, 2)
ip = g.download_indptr()
pool = graphs.pick_sources(ip, 64, seed=7)[:nsrc]
base = dict(os.environ)
ref, out, bad = {}, {}, []
for name, env in confs:
    os.environ.clear(); os.environ.update(base); os.environ.update(env)
    info = g.prepare(delta)
    g.solve(pool[0], delta)
    ms, sc, br = [], [], []
    for s in pool:
        st = g.solve(s, delta)
        ms.append(st.kernel_ms); sc.append(st.edges_scanned); br.append(st.grid_barriers)
        d = g.result_dense().view(np.uint64).copy()
        key = (st.outer_iterations, st.inner_phases, st.dist_mode)
        if s not in ref:
            ref[s] = (d, key)
        elif not (np.array_equal(ref[s][0], d) and ref[s][1] == key):
            bad.append((name, s, key, ref[s][1]))
    out[name] = {"ms": round(float(np.mean(ms)), 3), "scanned": int(np.mean(sc)), "barriers": int(np.mean(br)),
                 "ksub": info.sub_buckets}
print(json.dumps({"scale": scale, "delta": delta, "res": out, "mismatch": bad[:5]}))
