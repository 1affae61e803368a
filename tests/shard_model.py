"""TEST INFRASTRUCTURE ONLY: a numpy model of one partitioned-solver shard.

Implements the same interface as `paper_1911_06895_b200.distributed.DeviceShard`
(probe / prepare / begin / scan / s_add / relax_light / relax_heavy / result)
in binary64 with sequential relaxations -- a valid linearisation of the
device's atomics -- so the CPU (gloo, world_size 2) tests can exercise the
partitioning, the per-phase frontier exchange and the all-reduced control
decisions of `PartitionedDeltaStepping` without a GPU.  Never imported by the
product package.
"""

from __future__ import annotations

import math

import numpy as np

NONE = (1 << 64) - 1


def _bits(x: float) -> int:
    return int(np.array([x], dtype=np.float64).view(np.uint64)[0])


def _val(b: int) -> float:
    return float(np.array([b & ((1 << 64) - 1)], dtype=np.uint64).view(np.float64)[0])


class NumpyShard:
    device = "cpu"

    def __init__(self, n, v0, v1, indptr, col_local, val):
        import torch

        self.torch = torch
        self.n, self.v0, self.nl = int(n), int(v0), int(v1 - v0)
        self.indptr = np.asarray(indptr, dtype=np.int64)
        self.col = np.asarray(col_local, dtype=np.int64)
        self.val = np.asarray(val, dtype=np.float64)

    def probe(self, delta):
        w = self.val
        light = (w > 0) & (w <= delta)
        heavy = (w > delta) & (w < math.inf)
        return {"min_light": float(w[light].min()) if light.any() else math.inf,
                "max_w": float(w[light | heavy].max()) if (light | heavy).any() else 0.0,
                "frac": 99,  # the model computes in binary64 only
                "nL": int(light.sum()), "nH": int(heavy.sum())}

    def prepare(self, delta, mode, frac):
        assert mode == 1, "numpy shard model runs in f64 mode"
        self.delta = delta

    def begin(self, source):
        self.dist = np.full(self.nl, np.inf)
        if self.v0 <= source < self.v0 + self.nl:
            self.dist[source - self.v0] = 0.0
        self.S = {}

    def _t(self, ids, vals):
        torch = self.torch
        return (torch.tensor(np.asarray(ids, dtype=np.int32)),
                torch.tensor(np.asarray(vals, dtype=np.float64).view(np.int64)))

    def scan(self, L, H):
        lo, hi = _val(L), _val(H)
        d = self.dist
        sel = np.flatnonzero((d >= lo) & (d < hi))
        beyond = d[(d >= hi) & np.isfinite(d)]
        nm = _bits(float(beyond.min())) if beyond.size else NONE
        ids, vals = self._t(sel + self.v0, d[sel])
        return ids, vals, int(sel.size), nm

    def s_add(self, ids, vals, count):
        v = vals.numpy().view(np.float64)
        for u, x in zip(ids.numpy().tolist(), v.tolist()):
            self.S[u] = x

    def _relax(self, pairs, light, hi):
        nxt = []
        seen = set()
        d = self.dist
        for u, du in pairs:
            for e in range(self.indptr[u], self.indptr[u + 1]):
                w = self.val[e]
                if light and not (w > 0 and w <= self.delta):
                    continue
                if not light and not (w > self.delta and w < math.inf):
                    continue
                v = self.col[e]
                nd = du + w
                if nd < d[v]:
                    d[v] = nd
                    if light and nd < hi and v not in seen:
                        seen.add(v)
                        nxt.append(v)
        return nxt

    def relax_light(self, ids, vals, count, H):
        pairs = list(zip(ids.numpy().tolist(), vals.numpy().view(np.float64).tolist()))
        nxt = self._relax(pairs, True, _val(H))
        out_ids, out_vals = self._t(np.asarray(nxt, dtype=np.int64) + self.v0, self.dist[nxt])
        return out_ids, out_vals, len(nxt), False

    def relax_heavy(self):
        self._relax(list(self.S.items()), False, math.inf)
        self.S = {}
        return False

    def result(self):
        return self.dist.copy()
