"""Per-step-kind timeline of one grid 4096^2 solve (DS_TRACE=1)."""
import os, sys, collections
os.environ["DS_TRACE"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1911_06895_b200 import DeviceGraph, graphs, _lib
side = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
a = graphs.grid2d(side, seed=3)
g = DeviceGraph.from_matrix(a)
names = ["scan", "light_relax", "light_capture", "heavy_capture", "heavy_relax", "light_pull",
         "light_commit", "heavy_pull", "heavy_commit", "light_local", "heavy_local", "unsettled_capture",
         "heavy_gather", "hop_pass", "bidir"]
g.solve(0, 25.0)
st = g.solve(0, 25.0)
cap = 1 << 20
buf = np.zeros(1 + 2 * cap, dtype=np.uint64)
m = _lib.lib().ds_debug_trace(g._handle(), buf.ctypes.data, cap)
t0 = int(buf[0]); ts = buf[1::2][:m].astype(np.int64); info = buf[2::2][:m]
kinds = (info >> np.uint64(56)).astype(int); work = (info & np.uint64((1 << 56) - 1)).astype(np.int64)
dt = np.diff(np.concatenate([[t0], ts]))
agg = collections.defaultdict(lambda: [0, 0, 0])
for k, d, w in zip(kinds, dt, work):
    agg[names[k]][0] += 1; agg[names[k]][1] += int(d); agg[names[k]][2] += int(w)
print(f"grid{side}: kernel {st.kernel_ms:.1f} ms, steps {m}, traced {dt.sum()/1e6:.1f} ms, "
      f"buckets {st.buckets_visited}, phases {st.inner_phases}, barriers {st.grid_barriers}")
for k, (c, d, w) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"   {k:14s} n={c:6d} time={d/1e6:9.3f} ms  avg={d/c/1e3:8.1f} us  work={w}")
