"""Does the solver slow the copy engine (or the reverse)?  Device-only batches on one thread while
another streams 134 MB pinned D2H copies of an unrelated buffer."""
import os, sys, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1911_06895_b200 import DeviceGraph, graphs
g = DeviceGraph.rmat(24, 16, 1, 2)
ip = g.download_indptr()
src = graphs.pick_sources(ip, 64, seed=7)
g.prepare(0.1)
n = g.n
dev = torch.empty((4, n), dtype=torch.float64, device="cuda")
host = torch.empty((16, n), dtype=torch.float64).pin_memory()
stop = False; copied = [0]
NS = int(sys.argv[1]) if len(sys.argv) > 1 else 1   # concurrent copy streams
PARTS = int(sys.argv[2]) if len(sys.argv) > 2 else 1  # pieces per 134 MB vector
def copier():
    ss = [torch.cuda.Stream() for _ in range(NS)]
    i = 0
    step = n // PARTS
    while not stop:
        for k, s in enumerate(ss):
            with torch.cuda.stream(s):
                for q in range(PARTS):
                    if q % NS == k or NS >= PARTS:
                        host[(i + k) % 16, q * step:(q + 1) * step].copy_(dev[(i + k) % 4, q * step:(q + 1) * step], non_blocking=True)
        for s in ss: s.synchronize()
        copied[0] += NS if NS >= PARTS else 1; i += NS
def batch():
    torch.cuda.synchronize(); t = time.perf_counter()
    st, _ = g.solve_batch(src, 0.1, concurrency=4, keep=False)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    return sum(s.edges_reached for s in st) / dt / 1e9, dt
batch()
print("batch alone: %.1f GTEPS" % batch()[0])
th = threading.Thread(target=copier); th.start()
time.sleep(0.2); c0 = copied[0]; t0 = time.perf_counter()
gt, dt = batch()
c1 = copied[0]; t1 = time.perf_counter()
stop = True; th.join()
print(f"streams {NS} parts {PARTS}: " "batch with concurrent D2H: %.1f GTEPS; D2H %.1f GB/s meanwhile" % (gt, (c1 - c0) * n * 8 / (t1 - t0) / 1e9))
