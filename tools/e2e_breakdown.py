"""Where the e2e step's time goes (host timers around each public-API call)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1911_06895_b200 import DeviceGraph, graphs
g = DeviceGraph.rmat(24, 16, 1, 2)
ip, col, val = g.download(); g.close()
pi, pc, pv = (torch.from_numpy(x).pin_memory() for x in (ip, col, val))
src = graphs.pick_sources(ip, 8, seed=7)
idx = torch.empty(len(ip), dtype=torch.int64).pin_memory(); vb = torch.empty(len(ip), dtype=torch.float64).pin_memory()
def T(f):
    torch.cuda.synchronize(); t = time.perf_counter(); r = f(); torch.cuda.synchronize(); return r, (time.perf_counter() - t) * 1e3
for rep in range(3):
    h, t_create = T(lambda: DeviceGraph.from_csr(len(ip) - 1, pi, pc, pv))
    _, t_prep = T(lambda: h.prepare(0.1))
    ts, tr = [], []
    for s in src:
        _, a = T(lambda: h.solve(s, 0.1)); ts.append(a)
        _, b = T(lambda: h.result_sparse(out=(idx.numpy(), vb.numpy()))); tr.append(b)
    _, t_close = T(lambda: h.close())
    print(f"create {t_create:.1f} ms, prepare {t_prep:.1f} ms, solves {sum(ts):.1f} ms ({[round(x,1) for x in ts]}), "
          f"results {sum(tr):.1f} ms, close {t_close:.1f} ms")
