"""Dump every step (kind, work, time) of one solve (DS_TRACE=1)."""
import os, sys
os.environ["DS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1911_06895_b200 import DeviceGraph, graphs, _lib
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
delta = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
g = DeviceGraph.rmat(scale, 16, 1, 2)
indptr, _, _ = g.download()
s = graphs.pick_sources(indptr, 1, seed=7)[0]
g.solve(s, delta)
st = g.solve(s, delta)
names = ["scan", "l_relax", "l_capt", "h_capt", "h_relax", "l_pull", "l_commit", "h_pull", "h_commit", "l_local", "h_local", "u_capt", "h_gather"]
cap = 1 << 16
buf = np.zeros(1 + 2 * cap, dtype=np.uint64)
m = _lib.lib().ds_debug_trace(g._handle(), buf.ctypes.data, cap)
t0 = int(buf[0]); ts = buf[1::2][:m].astype(np.int64); info = buf[2::2][:m]
kinds = (info >> np.uint64(56)).astype(int); work = (info & np.uint64((1 << 56) - 1)).astype(np.int64)
dt = np.diff(np.concatenate([[t0], ts]))
print(f"kernel {st.kernel_ms:.3f} ms steps {m}")
for i in range(m):
    print(f"{i:4d} {names[kinds[i]]:9s} work={work[i]:11d} t={dt[i]/1e3:8.1f}us")
