"""Per-source solve time of RMAT-24 at reduced persistent-grid sizes
(DS_GRID_SMS), to size concurrent multi-source teams."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1911_06895_b200 import DeviceGraph, graphs
g = DeviceGraph.rmat(24, 16, 1, 2)
indptr = g.download()[0]
srcs = graphs.pick_sources(indptr, 8, seed=7)
g.solve(int(srcs[0]), 0.1)
ms = []
for s in srcs:
    r = g.solve(int(s), 0.1)
    ms.append(r.kernel_ms)
print(json.dumps({"sms": os.environ.get("DS_GRID_SMS"), "big_h": os.environ.get("DS_BIG_H"), "mean_ms": float(np.mean(ms))}))
