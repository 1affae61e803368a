"""Same-process A/B of runtime knobs (env vars read at every solve).

    python tools/env_probe.py SCALE DELTA NSRC "NAME VAR=VAL ..." "NAME2 ..."

Each configuration solves the same sources (R-MAT, device-generated); the
first configuration is the reference: every other one must match its
distances bit for bit and its counters exactly.  Prints mean kernel ms per
configuration (interleaved per source, so clock drift hits all alike).
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

from paper_1911_06895_b200 import DeviceGraph, graphs

scale = int(sys.argv[1])
delta = float(sys.argv[2])
nsrc = int(sys.argv[3])
confs = []
for spec in sys.argv[4:]:
    parts = spec.split()
    confs.append((parts[0], dict(kv.split("=", 1) for kv in parts[1:])))
if not confs:
    confs = [("default", {})]
g = DeviceGraph.rmat(scale, 16, 1, 2)
indptr = g.download()[0]
srcs = graphs.pick_sources(indptr, nsrc, seed=7)
base_env = dict(os.environ)


def run(env, s):
    os.environ.clear()
    os.environ.update(base_env)
    os.environ.update(env)
    st = g.solve(int(s), delta)
    return st, g.result_dense()


run(confs[0][1], srcs[0])  # warm-up
times = {name: [] for name, _ in confs}
bad = []
for s in srcs:
    ref = None
    for name, env in confs:
        st, d = run(env, s)
        times[name].append(st.kernel_ms)
        key = (st.outer_iterations, st.inner_phases)
        if ref is None:
            ref = (d.view(np.uint64).copy(), key)
        elif not (np.array_equal(ref[0], d.view(np.uint64)) and ref[1] == key):
            bad.append((name, int(s)))
out = {"scale": scale, "delta": delta, "sources": len(srcs),
       "mean_ms": {k: float(np.mean(v)) for k, v in times.items()}, "mismatches": bad}
print(json.dumps(out))
