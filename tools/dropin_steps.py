"""delta_stepping_batch on a reference-layout SparseMatrix (R-MAT 24, 64 sources), step by step
with the device cache cleared in between (each step uploads and splits again)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1911_06895_b200 import DeviceGraph, SparseMatrix, graphs, clear_device_cache, delta_stepping_batch
g = DeviceGraph.rmat(24, 16, 1, 2)
ip, col, val = g.download(); g.close()
a = SparseMatrix(len(ip) - 1, ip, col.astype(np.int64), val.astype(np.float64))
src = [int(s) for s in graphs.pick_sources(ip, 64, seed=7)]
for rep in range(4):
    clear_device_cache()
    t = time.perf_counter()
    rs = delta_stepping_batch(a, src, 0.1, concurrency=4)
    dt = time.perf_counter() - t
    m = sum(r.device_stats["edges_reached"] for r in rs)
    print(f"step {rep}: {dt*1e3:.0f} ms, {m/dt/1e9:.1f} GTEPS")
