"""Where the bench's e2e step goes: host timers (device-synchronised) around from_csr (pinned H2D +
validation + relabeling), prepare (split), solve_batch with a pinned host output, close."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1911_06895_b200 import DeviceGraph, graphs
g = DeviceGraph.rmat(24, 16, 1, 2)
ip, col, val = g.download(); g.close()
pi, pc, pv = (torch.from_numpy(x).pin_memory() for x in (ip, col, val))
n = len(ip) - 1
src = graphs.pick_sources(ip, 64, seed=7)
out = torch.empty((64, n), dtype=torch.float64).pin_memory()
def T(f):
    torch.cuda.synchronize(); t = time.perf_counter(); r = f(); torch.cuda.synchronize(); return r, (time.perf_counter() - t) * 1e3
for rep in range(3):
    h, t_create = T(lambda: DeviceGraph.from_csr(n, pi, pc, pv))
    _, t_prep = T(lambda: h.prepare(0.1))
    (st, _), t_batch = T(lambda: h.solve_batch(src, 0.1, concurrency=4, out=out.numpy()))
    (st2, _), t_dev = T(lambda: h.solve_batch(src, 0.1, concurrency=4, keep=False))
    _, t_close = T(lambda: h.close())
    print(f"create {t_create:.1f} ms, prepare {t_prep:.1f} ms, batch->host {t_batch:.1f} ms (device-only {t_dev:.1f}), "
          f"close {t_close:.1f} ms; H2D {(pi.numel()*8+pc.numel()*4+pv.numel()*4)/1e9:.2f} GB, D2H {out.numel()*8/1e9:.2f} GB")
