"""One grid 4096^2 solve from the corner (BASELINE configs[2]; for ncu --set full captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_06895_b200 import DeviceGraph, graphs
g = DeviceGraph.from_matrix(graphs.grid2d(4096, seed=3))
g.prepare(25.0)
st = g.solve(0, 25.0)
print("grid4096 source 0 kernel_ms", st.kernel_ms, "launches", st.launches, "buckets", st.buckets_visited,
      "phases", st.inner_phases, "barriers", st.grid_barriers)
