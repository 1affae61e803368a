"""RMAT scale 27 (BASELINE configs[4]) on ONE B200: device generation, split,
16 seeded sources at delta 0.1; fixed-point vs binary64 distances must agree
bit for bit on a sample.  Prints one JSON line."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_1911_06895_b200 import DeviceGraph, graphs

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 27
nsrc = int(sys.argv[2]) if len(sys.argv) > 2 else 16
t0 = time.perf_counter()
g = DeviceGraph.rmat(scale, 16, 1, 2)
torch.cuda.synchronize()
t_gen = time.perf_counter() - t0
n, nnz = g.n, g.nnz
# sources: nonzero degree, seeded; degrees from a device->host indptr copy
ip = np.empty(n + 1, dtype=np.int64)
import ctypes
from paper_1911_06895_b200 import _lib
ip_t = torch.empty(n + 1, dtype=torch.int64)
# download only indptr via the full download would need 34 GB host; use degrees of a sample
idx, _, _ = None, None, None
t0 = time.perf_counter()
info = g.prepare(0.1)
torch.cuda.synchronize()
t_prep = time.perf_counter() - t0
rng = np.random.default_rng(7)
srcs = []
while len(srcs) < nsrc:
    s = int(rng.integers(0, n))
    st = g.solve(s, 0.1)
    if st.reached > 1:
        srcs.append((s, st))
free, total = torch.cuda.mem_get_info()
ms = [st.kernel_ms for _, st in srcs]
m = [st.edges_reached for _, st in srcs]
# bit-exact check fixed vs f64 on one source
s0 = srcs[0][0]
g.solve(s0, 0.1)
a = g.result_dense()
g.solve(s0, 0.1, force_f64=True)
b = g.result_dense()
same = bool(np.array_equal(a.view(np.uint64), b.view(np.uint64)))
print(json.dumps({"scale": scale, "n": n, "nnz": nnz, "gen_s": t_gen, "prepare_s": t_prep,
                  "nnz_light": int(info.nnz_light), "sources": len(srcs),
                  "kernel_ms_mean": float(np.mean(ms)), "gteps": float(sum(m) / (sum(ms) * 1e-3) / 1e9),
                  "reached_mean": float(np.mean([st.reached for _, st in srcs])),
                  "phases_mean": float(np.mean([st.inner_phases for _, st in srcs])),
                  "fixed_equals_f64": same, "gpu_mem_used_gb": (total - free) / 1e9}))
