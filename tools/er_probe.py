"""ER-1024 (BASELINE configs[0]) solve latency, one source at a time."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1911_06895_b200 import DeviceGraph, graphs
a = graphs.erdos_renyi(1024, seed=0)
g = DeviceGraph.from_matrix(a)
g.solve(0, 3.0)
ms = [g.solve(s, 3.0).kernel_ms for s in range(0, 1024, 16)]
t = time.perf_counter()
for s in range(0, 1024, 16):
    g.solve(s, 3.0)
wall = (time.perf_counter() - t) / 64 * 1e3
st = g.solve(0, 3.0)
print(f"ER1024 small={os.environ.get('DS_SMALL')}: kernel {np.mean(ms):.3f} ms, wall {wall:.3f} ms/solve, "
      f"barriers {st.grid_barriers}, phases {st.inner_phases}")
