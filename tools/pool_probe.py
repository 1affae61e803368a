"""Mean single-solve kernel time over the bench pool (R-MAT SCALE, DELTA) and
the ds_sssp_batch throughput at concurrency CONC -- one JSON line, for A/B
runs of library builds (DS_LIB) and knobs (env)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1911_06895_b200 import DeviceGraph, graphs
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
delta = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
nsrc = int(sys.argv[3]) if len(sys.argv) > 3 else 16
conc = int(sys.argv[4]) if len(sys.argv) > 4 else 4
g = DeviceGraph.rmat(scale, 16, 1, 2)
ip = g.download_indptr()
pool = graphs.pick_sources(ip, 64, seed=7)
info = g.prepare(delta)
g.solve(pool[0], delta)
ms = [g.solve(s, delta).kernel_ms for s in pool[:nsrc]]
g.solve_batch(pool[:conc], delta, concurrency=conc, keep=False)
import torch
torch.cuda.synchronize()
t0 = time.perf_counter()
stats, _ = g.solve_batch(pool, delta, concurrency=conc, keep=False)
torch.cuda.synchronize()
t = time.perf_counter() - t0
print(json.dumps({"lib": os.path.basename(os.environ.get("DS_LIB", "libdsssp.so")), "lex": os.environ.get("DS_LEX"),
                  "ksub": info.sub_buckets, "single_ms": round(float(np.mean(ms)), 3),
                  "batch_gteps": round(sum(s.edges_reached for s in stats) / t / 1e9, 1)}))
