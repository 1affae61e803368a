"""Micro-benchmark of the push kernels on the real R-MAT giant steps, through
the partitioned path at world 1 (standalone k_shard_relax launches, so each
library variant's register/occupancy choice shows)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
os.environ.setdefault("MASTER_ADDR", "127.0.0.1"); os.environ.setdefault("MASTER_PORT", "29611")
dist.init_process_group("gloo", rank=0, world_size=1)
from paper_1911_06895_b200 import DeviceGraph, graphs
from paper_1911_06895_b200.distributed import DeviceShard, PartitionedDeltaStepping
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
g = DeviceGraph.rmat(scale, 16, 1, 2)
indptr = g.download()[0]
sh = DeviceShard.from_graph(g, 0, g.n)
g.close()
times = {"light": [], "heavy": []}
orig_l, orig_h = sh.relax_light, sh.relax_heavy
def tl(*a):
    torch.cuda.synchronize(); t = time.perf_counter(); r = orig_l(*a); torch.cuda.synchronize()
    times["light"].append((time.perf_counter() - t, a[2])); return r
def th():
    torch.cuda.synchronize(); t = time.perf_counter(); r = orig_h(); torch.cuda.synchronize()
    times["heavy"].append(time.perf_counter() - t); return r
sh.relax_light, sh.relax_heavy = tl, th
solver = PartitionedDeltaStepping(sh, sh.n, dist, "cpu")
s = graphs.pick_sources(indptr, 1, seed=7)[0]
solver.solve(s, 0.1, on_device=True)
for rep in range(2):
    times = {"light": [], "heavy": []}
    solver.solve(s, 0.1, on_device=True)
hv = sorted(times["heavy"], reverse=True)
big_l = sorted(times["light"], key=lambda x: -x[0])[:3]
print(f"{os.environ.get('DS_LIB','default')}: heavy max {hv[0]*1e3:.3f} ms, heavy sum {sum(hv)*1e3:.3f} ms, "
      f"light sum {sum(t for t,_ in times['light'])*1e3:.3f} ms, top light {[round(t*1e3,3) for t,_ in big_l]}")
dist.destroy_process_group()
