"""Push statistics of one R-MAT solve from its final distances (analysis only).

For every reached vertex u, its heavy row is pushed once, in the heavy step of
bucket b(u) = floor(d(u)/delta).  A push u->v is useless when v is already
settled then (d(v) < hi of b(u)).  Reports, per bucket and in total, how many
heavy pushes are useless, split by the target's degree rank (hubs first, the
solver's relabeling order), to size settled-bitmap pre-checks.

    python tools/heavy_stats.py [SCALE] [DELTA]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

from paper_1911_06895_b200 import DeviceGraph, graphs

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
delta = float(sys.argv[2]) if len(sys.argv) > 2 else 0.1
g = DeviceGraph.rmat(scale, 16, 1, 2)
indptr, col, val = g.download()
s = int(graphs.pick_sources(indptr, 64, seed=7)[0])
g.solve(s, delta)
d = torch.from_numpy(g.result_dense()).cuda()
n = g.n
ip = torch.from_numpy(indptr).cuda()
deg = ip[1:] - ip[:-1]
# degree rank (descending, stable) ~ the solver's relabeling
order = torch.argsort(-deg, stable=True)
rank = torch.empty_like(order)
rank[order] = torch.arange(n, device="cuda")
b = torch.where(torch.isfinite(d), torch.floor(d / delta), torch.full_like(d, -1)).long()
nb = int(b.max()) + 1
tot = torch.zeros(nb, dtype=torch.long, device="cuda")
useless = torch.zeros(nb, dtype=torch.long, device="cuda")
ltot = torch.zeros(nb, dtype=torch.long, device="cuda")
kcuts = [14, 16, 18, 20, 22]
hub = torch.zeros(len(kcuts), dtype=torch.long, device="cuda")
hub_useless = torch.zeros(len(kcuts), dtype=torch.long, device="cuda")
tight = torch.zeros(nb, dtype=torch.long, device="cuda")
lset = torch.zeros(nb, dtype=torch.long, device="cuda")   # light pushes to targets settled before the bucket
hdeg = torch.zeros(n, dtype=torch.long, device="cuda")    # heavy degree per vertex
CH = 1 << 26
m = len(col)
row_of = None
for e0 in range(0, m, CH):
    e1 = min(m, e0 + CH)
    c = torch.from_numpy(col[e0:e1]).cuda().long()
    w = torch.from_numpy(val[e0:e1]).cuda()
    u = torch.searchsorted(ip, torch.arange(e0, e1, device="cuda"), right=True) - 1
    bu = b[u]
    ok = bu >= 0
    heavy = ok & (w > delta)
    light = ok & (w > 0) & (w <= delta)
    hi = (bu + 1).double() * delta
    us = heavy & (d[c] < hi)
    tot += torch.bincount(bu[heavy], minlength=nb)
    ltot += torch.bincount(bu[light], minlength=nb)
    useless += torch.bincount(bu[us], minlength=nb)
    lo = bu.double() * delta
    lset += torch.bincount(bu[light & (d[c] < lo)], minlength=nb)
    hdeg += torch.bincount(u[ok & (w > delta)], minlength=n)
    tt = heavy & (d[u] + w == d[c])
    tight += torch.bincount(bu[tt], minlength=nb)
    rc = rank[c]
    for i, k in enumerate(kcuts):
        h = heavy & (rc < (1 << k))
        hub[i] += h.sum()
        hub_useless[i] += (h & us).sum()
print(f"rmat{scale} delta={delta} source={s} n={n} nnz={m}")
print(f"heavy pushes {int(tot.sum())}  useless (target settled) {int(useless.sum())} "
      f"({float(useless.sum())/max(1,float(tot.sum())):.3f})  tight {int(tight.sum())}")
for i in range(nb):
    if int(tot[i]) or int(ltot[i]):
        print(f"  bucket {i:3d}: S-light-edges {int(ltot[i]):11d} heavy {int(tot[i]):11d} "
              f"useless {int(useless[i]):11d} ({float(useless[i])/max(1,float(tot[i])):.3f}) tight {int(tight[i])}")
for i, k in enumerate(kcuts):
    print(f"  targets rank < 2^{k}: {int(hub[i])} pushes ({float(hub[i])/float(tot.sum()):.3f}), "
          f"useless {int(hub_useless[i])} ({float(hub_useless[i])/float(tot.sum()):.3f} of all)")

# pull volume: heavy edges of the rows still unsettled after bucket i's light closure
bv = b.clone()
bv[bv < 0] = 1 << 30
for i in range(nb):
    if int(tot[i]) or int(ltot[i]):
        U = int(hdeg[bv > i].sum())
        print(f"  bucket {i:3d}: push {int(tot[i]):11d}  pull(unsettled rows) {U:11d}  light {int(ltot[i])} "
              f"light-to-settled {int(lset[i])}")
