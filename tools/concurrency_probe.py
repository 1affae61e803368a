"""Do independent solves on SM-partitioned grids overlap?  T graph handles on
T streams, each solving 8 sources from its own host thread (DS_GRID_SMS sets
every handle's persistent grid).  Prints the aggregate per-source time."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1911_06895_b200 import DeviceGraph, graphs
T = int(sys.argv[1])
g0 = DeviceGraph.rmat(24, 16, 1, 2)
ip, col, val = g0.download(); g0.close()
src = graphs.pick_sources(ip, 8 * T, seed=7)
streams = [torch.cuda.Stream() for _ in range(T)]
hs = [DeviceGraph.from_csr(len(ip) - 1, ip, col, val, stream=streams[i].cuda_stream) for i in range(T)]
for h in hs:
    h.prepare(0.1)
    h.solve(int(src[0]), 0.1)
torch.cuda.synchronize()
ms = [[] for _ in range(T)]
def work(i):
    for s in src[i::T]:
        ms[i].append(hs[i].solve(int(s), 0.1).kernel_ms)
th = [threading.Thread(target=work, args=(i,)) for i in range(T)]
t0 = time.perf_counter()
for t in th: t.start()
for t in th: t.join()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) * 1e3
print(f"T={T} sms={os.environ.get('DS_GRID_SMS')} wall/source {wall / len(src):.2f} ms, "
      f"mean kernel {np.mean([x for m in ms for x in m]):.2f} ms")
