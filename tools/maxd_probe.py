import sys; sys.path.insert(0, '/root/repo')
from paper_1911_06895_b200 import DeviceGraph, graphs
import numpy as np
g = DeviceGraph.rmat(27, 16, 1, 2)
ip = g.download_indptr()
for s in graphs.pick_sources(ip, 4, seed=7):
    st = g.solve(int(s), 0.1)
    print("rmat27 source", s, "max_d", st.max_distance, "phases", st.inner_phases, "buckets", st.buckets_visited, "ms", st.kernel_ms)
