"""Latency of the first and later solves in a fresh process (R-MAT scale argv[1], default 20)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1911_06895_b200 import DeviceGraph, graphs
g = DeviceGraph.rmat(int(sys.argv[1]) if len(sys.argv) > 1 else 20, 16, 1, 2)
ip, _, _ = g.download()
s = int(graphs.pick_sources(ip, 1, seed=7)[0])
g.prepare(0.1)
print([round(g.solve(s, 0.1).kernel_ms, 2) for _ in range(4)])
