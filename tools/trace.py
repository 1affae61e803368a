"""Per-step timeline of one solve (DS_TRACE=1): time per step kind."""
import os, sys, ctypes, collections
os.environ["DS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1911_06895_b200 import DeviceGraph, graphs, _lib

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
delta = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
g = DeviceGraph.rmat(scale, 16, 1, 2)
indptr, _, _ = g.download()
srcs = graphs.pick_sources(indptr, 3, seed=7)
names = ["scan", "light_relax", "light_capture", "heavy_capture", "heavy_relax", "light_pull", "light_commit", "heavy_pull", "heavy_commit", "light_local", "heavy_local", "unsettled_capture", "heavy_gather", "hop_pass", "bidir"]
for s in srcs:
    st = g.solve(s, delta)
    cap = 1 << 16
    buf = np.zeros(1 + 2 * cap, dtype=np.uint64)
    m = _lib.lib().ds_debug_trace(g._handle(), buf.ctypes.data, cap)
    t0 = int(buf[0]); ts = buf[1::2][:m].astype(np.int64); info = buf[2::2][:m]
    kinds = (info >> np.uint64(56)).astype(int); work = (info & np.uint64((1 << 56) - 1)).astype(np.int64)
    dt = np.diff(np.concatenate([[t0], ts]))
    agg = collections.defaultdict(lambda: [0, 0, 0])
    for k, d, w in zip(kinds, dt, work):
        agg[names[k]][0] += 1; agg[names[k]][1] += int(d); agg[names[k]][2] += int(w)
    print(f"source {s}: kernel {st.kernel_ms:.3f} ms, steps {m}, traced {dt.sum()/1e6:.3f} ms")
    for k, (c, d, w) in sorted(agg.items(), key=lambda x: -x[1][1]):
        print(f"   {k:14s} n={c:4d} time={d/1e6:8.3f} ms  avg={d/c/1e3:8.1f} us  work={w}")
    if s == srcs[0]:
        big = np.argsort(-dt)[:12]
        for i in sorted(big):
            print(f"      step {i:4d} {names[kinds[i]]:14s} {dt[i]/1e3:9.1f} us work={work[i]}")
