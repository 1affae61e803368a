"""One R-MAT 24 source solve (for ncu --set full captures of the solver launches)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_06895_b200 import DeviceGraph, graphs
g = DeviceGraph.rmat(24, 16, 1, 2)
ip, _, _ = g.download()
s = int(graphs.pick_sources(ip, 64, seed=7)[0])  # the bench pool's first source
g.prepare(0.1)
st = g.solve(s, 0.1)
print("source", s, "kernel_ms", st.kernel_ms, "launches", st.launches, "edges", st.edges_reached)
