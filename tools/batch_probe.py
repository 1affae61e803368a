"""Batch throughput (ds_sssp_batch) vs concurrency on one graph."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1911_06895_b200 import DeviceGraph, graphs
arg = sys.argv[1] if len(sys.argv) > 1 else "18"
delta = 0.1
if arg.startswith("grid"):  # gridSIDE: 4-neighbour grid, delta 25
    g = DeviceGraph.from_matrix(graphs.grid2d(int(arg[4:]), seed=3))
    delta = 25.0
    scale = arg
else:
    scale = int(arg)
    g = DeviceGraph.rmat(scale, 16, 1, 2)
ip, _, _ = g.download()
src = graphs.pick_sources(ip, 16, seed=7)
g.prepare(delta)
for conc in (1, 2, 3, 4, 6, 8):
    g.solve_batch(src, delta, concurrency=conc, keep=False)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(3):
        st, _ = g.solve_batch(src, delta, concurrency=conc, keep=False)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t) / 3
    m = sum(s.edges_reached for s in st)
    print(f"{'' if arg.startswith('grid') else 'rmat'}{scale} conc={conc}: {dt / len(src) * 1e3:.3f} ms/source, {m / dt / 1e9:.2f} GTEPS")
