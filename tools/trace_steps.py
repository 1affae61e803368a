import os, sys, collections
os.environ["DS_TRACE"] = "1"
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1911_06895_b200 import DeviceGraph, graphs, _lib
g = DeviceGraph.rmat(24, 16, 1, 2)
indptr, _, _ = g.download()
s = graphs.pick_sources(indptr, 3, seed=7)[0]
names = ["scan", "light_relax", "light_capture", "heavy_capture", "heavy_relax", "light_pull", "light_commit", "heavy_pull", "heavy_commit", "light_local", "heavy_local", "unsettled_capture", "heavy_gather", "hop_pass", "bidir"]
st = g.solve(s, 0.1)
st = g.solve(s, 0.1)
cap = 1 << 16
buf = np.zeros(1 + 2 * cap, dtype=np.uint64)
m = _lib.lib().ds_debug_trace(g._handle(), buf.ctypes.data, cap)
t0 = int(buf[0]); ts = buf[1::2][:m].astype(np.int64); info = buf[2::2][:m]
kinds = (info >> np.uint64(56)).astype(int); work = (info & np.uint64((1 << 56) - 1)).astype(np.int64)
dt = np.diff(np.concatenate([[t0], ts]))
for i in range(m):
    print(i, names[kinds[i]], round(dt[i]/1e3,1), work[i])
