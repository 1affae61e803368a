"""Where delta_stepping_batch's time goes on a reference-layout SparseMatrix (int64 columns, f64 values,
pageable numpy arrays): upload, split, solves + dense D2H, dense -> sparse rows, result objects."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from concurrent.futures import ThreadPoolExecutor
from paper_1911_06895_b200 import DeviceGraph, SparseMatrix, graphs, clear_device_cache
g = DeviceGraph.rmat(24, 16, 1, 2)
ip, col, val = g.download(); g.close()
a = SparseMatrix(len(ip) - 1, ip, col.astype(np.int64), val.astype(np.float64))
src = [int(s) for s in graphs.pick_sources(ip, 64, seed=7)]
def T(f):
    torch.cuda.synchronize(); t = time.perf_counter(); r = f(); torch.cuda.synchronize(); return r, (time.perf_counter() - t) * 1e3
for rep in range(2):
    h, t_up = T(lambda: DeviceGraph.from_matrix(a))
    _, t_prep = T(lambda: h.prepare(0.1))
    (st, dist), t_solve = T(lambda: h.solve_batch(src, 0.1, concurrency=4))
    def row(i):
        r = dist[i]; idx = np.flatnonzero(r != np.inf); return idx, r[idx]
    t = time.perf_counter()
    with ThreadPoolExecutor(16) as ex: rows = list(ex.map(row, range(64)))
    t_rows = (time.perf_counter() - t) * 1e3
    _, t_close = T(lambda: h.close())
    print(f"upload {t_up:.0f} ms, prepare {t_prep:.0f} ms, solve_batch->numpy {t_solve:.0f} ms, dense->sparse rows {t_rows:.0f} ms, close {t_close:.0f} ms")
