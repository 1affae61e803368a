"""Prepare (split) time at R-MAT 24, with and without DS_SORT_ROWS."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1911_06895_b200 import DeviceGraph
g = DeviceGraph.rmat(24, 16, 1, 2)
for d in (0.1, 0.2, 0.1, 0.2):
    torch.cuda.synchronize(); t = time.perf_counter(); info = g.prepare(d); torch.cuda.synchronize()
    print(f"sort={os.environ.get('DS_SORT_ROWS','0')} delta={d} prepare {(time.perf_counter()-t)*1e3:.1f} ms (device {info.prepare_ms:.1f} ms)")
