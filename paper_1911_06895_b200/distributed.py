"""1-D vertex-partitioned delta-stepping across ranks.

One process per GPU (torch.distributed; NCCL over NVLink on GPUs, gloo for the
CPU test harness).  Rank r owns input ids [bounds[r], bounds[r+1]) and holds
the edges whose *target* it owns ("owner computes", `ds_shard_*` in
include/dsssp.h).  Per light phase every rank relaxes the *global* frontier
into its own targets with local atomics, then the new frontier (ids + captured
values) is all-gathered: that single exchange per phase is the only data-path
collective.  Heavy steps need none -- every rank accumulated the same S from
the exchanged frontiers.  Bucket selection and termination are decided
identically on every rank from all-reduced scalars, so distances,
`outer_iterations` and `inner_phases` equal the single-GPU solver's (and the
reference's, sssp.py:239-313).

The per-rank compute is a *shard* object; `DeviceShard` runs the sm_100a
kernels through the C-ABI.  (The CPU test harness plugs a numpy model of the
same interface in from tests/, never from here.)
"""

from __future__ import annotations

import ctypes
import math
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib
from .sssp import _ptr

NONE = (1 << 64) - 1          # "no value" for u64 minima coming out of a shard
I64_NONE = (1 << 63) - 1      # the same sentinel carried in int64 tensors
MODE_FIXED32, MODE_F64 = _lib.DS_MODE_FIXED32, _lib.DS_MODE_F64

__all__ = ["partition_bounds", "shard_csr", "DeviceShard", "PartitionedDeltaStepping",
           "ShardedResult", "bucket_index_of"]


def partition_bounds(n: int, world: int) -> list[int]:
    """Contiguous, balanced vertex ranges (the R-MAT ids are already scrambled)."""
    return [r * n // world for r in range(world + 1)]


def shard_csr(indptr, col, val, v0: int, v1: int):
    """Edges whose target lies in [v0, v1) as a CSR over ALL sources, with
    local target ids -- the shard layout `ds_shard_create` expects."""
    indptr = np.asarray(indptr, dtype=np.int64)
    col = np.asarray(col)
    keep = (col >= v0) & (col < v1)
    cs = np.zeros(col.shape[0] + 1, dtype=np.int64)
    np.cumsum(keep, out=cs[1:])
    counts = cs[indptr[1:]] - cs[indptr[:-1]]
    out_ptr = np.zeros(indptr.shape[0], dtype=np.int64)
    np.cumsum(counts, out=out_ptr[1:])
    return out_ptr, (col[keep] - v0).astype(np.int32), np.asarray(val)[keep].astype(np.float64)


def bucket_index_of(value: float, delta: float) -> int:
    """sssp.py:230-236."""
    index = int(value // delta)
    while index * delta > value:
        index -= 1
    while (index + 1) * delta <= value:
        index += 1
    return index


def _f64_bits(x: float) -> int:
    return struct.unpack("<Q", struct.pack("<d", x))[0]


def _bits_f64(b: int) -> float:
    return struct.unpack("<d", struct.pack("<Q", b & ((1 << 64) - 1)))[0]


def _ceil_u32(x: float) -> int:
    if not (x < 4294967295.0):
        return 0xFFFFFFFF
    c = math.ceil(x)
    return 0xFFFFFFFF if c >= 4294967295 else int(c)


class DeviceShard:
    """One rank's shard on its GPU (C-ABI `ds_shard_*`).  Frontier buffers are
    torch tensors on the shard's device: ids int32, values int64 (u64 bits)."""

    def __init__(self, n: int, v0: int, v1: int, indptr, col_local, val, device: int = 0,
                 stream: int | None = None):
        import torch

        self.torch = torch
        self.n, self.v0, self.nl = int(n), int(v0), int(v1 - v0)
        self.device = torch.device("cuda", device)
        L = _lib.lib()
        h = ctypes.c_void_p()
        indptr = np.ascontiguousarray(indptr, dtype=np.int64)
        col_local = np.ascontiguousarray(col_local, dtype=np.int32)
        val = np.ascontiguousarray(val, dtype=np.float64)
        _lib.check(L.ds_shard_create(self.n, self.v0, self.nl, int(col_local.shape[0]),
                                     _ptr(indptr), _ptr(col_local), _ptr(val), int(device),
                                     stream or 0, ctypes.byref(h)))
        self._h = h
        m = max(self.nl, 1)
        self.out_ids = torch.empty(m, dtype=torch.int32, device=self.device)
        self.out_vals = torch.empty(m, dtype=torch.int64, device=self.device)

    @classmethod
    def from_graph(cls, graph, v0: int, v1: int) -> "DeviceShard":
        """Cut the shard [v0, v1) on the device from a resident `DeviceGraph`."""
        import torch

        self = cls.__new__(cls)
        self.torch = torch
        self.n, self.v0, self.nl = int(graph.n), int(v0), int(v1 - v0)
        self.device = torch.device("cuda", graph.device)
        h = ctypes.c_void_p()
        _lib.check(_lib.lib().ds_shard_from_graph(graph._handle(), int(v0), int(v1), ctypes.byref(h)))
        self._h = h
        m = max(self.nl, 1)
        self.out_ids = torch.empty(m, dtype=torch.int32, device=self.device)
        self.out_vals = torch.empty(m, dtype=torch.int64, device=self.device)
        return self

    def close(self):
        if self._h.value:
            _lib.lib().ds_shard_destroy(self._h)
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def probe(self, delta: float) -> dict:
        out = (ctypes.c_uint64 * 5)()
        _lib.check(_lib.lib().ds_shard_probe(self._h, float(delta), out))
        min_l = _bits_f64(out[0]) if out[0] != NONE else math.inf
        return {"min_light": min_l, "max_w": _bits_f64(out[1]), "frac": int(out[2]),
                "nL": int(out[3]), "nH": int(out[4])}

    def prepare(self, delta: float, mode: int, frac: int) -> None:
        key = (float(delta), int(mode), int(frac))
        if getattr(self, "_prepared", None) == key:
            return  # split cached per (delta, mode), like the single-GPU handle
        _lib.check(_lib.lib().ds_shard_prepare(self._h, float(delta), int(mode), int(frac)))
        self._prepared = key

    def begin(self, source: int) -> None:
        _lib.check(_lib.lib().ds_shard_begin(self._h, int(source)))

    def scan(self, L: int, H: int):
        cnt = ctypes.c_int64()
        nm = ctypes.c_uint64()
        _lib.check(_lib.lib().ds_shard_scan(self._h, L, H, _ptr(self.out_ids), _ptr(self.out_vals),
                                            ctypes.byref(cnt), ctypes.byref(nm)))
        c = int(cnt.value)
        return self.out_ids[:c].clone(), self.out_vals[:c].clone(), c, int(nm.value)

    def s_add(self, ids, vals, count: int) -> None:
        _lib.check(_lib.lib().ds_shard_s_add(self._h, _ptr(ids), _ptr(vals), int(count)))

    def relax_light(self, ids, vals, count: int, H: int):
        oc = ctypes.c_int64()
        ov = ctypes.c_int32()
        _lib.check(_lib.lib().ds_shard_relax(self._h, 0, _ptr(ids), _ptr(vals), int(count), H,
                                             _ptr(self.out_ids), _ptr(self.out_vals),
                                             ctypes.byref(oc), ctypes.byref(ov)))
        c = int(oc.value)
        return self.out_ids[:c].clone(), self.out_vals[:c].clone(), c, bool(ov.value)

    def relax_heavy(self) -> bool:
        oc = ctypes.c_int64()
        ov = ctypes.c_int32()
        _lib.check(_lib.lib().ds_shard_relax(self._h, 1, None, None, 0, 0, None, None,
                                             ctypes.byref(oc), ctypes.byref(ov)))
        return bool(ov.value)

    def launches(self) -> int:
        """Solver kernels this shard has launched so far."""
        return int(_lib.lib().ds_shard_launches(self._h))

    def result(self, on_device: bool = False):
        """Owned float64 distances: numpy (host) or a torch tensor left on the GPU."""
        if on_device:
            out = self.torch.empty(max(self.nl, 1), dtype=self.torch.float64, device=self.device)
        else:
            out = np.empty(max(self.nl, 1), dtype=np.float64)
        _lib.check(_lib.lib().ds_shard_result(self._h, _ptr(out)))
        return out[: self.nl]


@dataclass
class ShardedResult:
    local: np.ndarray      # float64 distances of the owned range (+inf = unreachable)
    v0: int
    outer_iterations: int
    inner_phases: int
    buckets_visited: int
    exchanged: int         # frontier entries all-gathered over the run
    mode: int


class PartitionedDeltaStepping:
    """Host driver of the partitioned solver for one rank.

    `shard` implements probe/prepare/begin/scan/s_add/relax_light/relax_heavy/
    result; `pg` is torch.distributed (already initialised).  Exchanges run on
    `xdev` ("cuda" for NCCL, "cpu" for gloo)."""

    def __init__(self, shard, n: int, pg, xdev):
        import torch

        self.torch = torch
        self.shard = shard
        self.n = int(n)
        self.pg = pg
        self.xdev = torch.device(xdev)
        self.world = pg.get_world_size()

    # -- collectives ---------------------------------------------------
    # Per light phase the protocol needs exactly two collectives and one host
    # read: a tiny all-gather of every rank's (count, flag) pair -- the counts
    # size the frontier exchange, the flag carries a fixed-point overflow --
    # and one all-gather of the packed (id, value) frontier entries.
    def _allreduce(self, value, op, dtype):
        t = self.torch.tensor([value], dtype=dtype, device=self.xdev)
        self.pg.all_reduce(t, op=op)
        return t.item()

    def _exchange_meta(self, *vals) -> np.ndarray:
        """All-gather a few int64 scalars per rank -> (world, k) host array."""
        torch = self.torch
        t = torch.tensor([int(v) for v in vals], dtype=torch.int64, device=self.xdev)
        parts = [torch.empty_like(t) for _ in range(self.world)]
        self.pg.all_gather(parts, t)
        return torch.stack(parts).cpu().numpy()

    def _gather_entries(self, ids, vals, counts, packed32: bool = False):
        """All-gather every rank's frontier (ids int32, u64 values as int64)
        as ONE padded int64 tensor per rank: 8-byte (id << 32 | value) words
        when every value fits 32 bits (fixed-point mode), else (2, max count)
        rows of ids and values."""
        torch = self.torch
        counts = [int(c) for c in counts]
        total = sum(counts)
        dev = ids.device if counts[self.pg.get_rank()] else getattr(self.shard, "device", self.xdev)
        if total == 0:
            return (torch.empty(0, dtype=torch.int32, device=dev),
                    torch.empty(0, dtype=torch.int64, device=dev), 0)
        m = max(counts)
        mine = counts[self.pg.get_rank()]
        rows = 1 if packed32 else 2
        buf = torch.zeros((rows, m), dtype=torch.int64, device=self.xdev)
        if mine:
            i64 = ids.to(self.xdev).to(torch.int64)
            v64 = vals.to(self.xdev)
            if packed32:
                buf[0, :mine] = (i64 << 32) | v64
            else:
                buf[0, :mine] = i64
                buf[1, :mine] = v64
        outs = [torch.empty_like(buf) for _ in range(self.world)]
        self.pg.all_gather(outs, buf)
        if packed32:
            words = torch.cat([o[0, :k] for o, k in zip(outs, counts)])
            out_i = (words >> 32).to(torch.int32).to(dev)
            out_v = (words & 0xFFFFFFFF).to(dev)
        else:
            out_i = torch.cat([o[0, :k] for o, k in zip(outs, counts)]).to(torch.int32).to(dev)
            out_v = torch.cat([o[1, :k] for o, k in zip(outs, counts)]).to(dev)
        return out_i, out_v, total

    # -- solve ---------------------------------------------------------
    def _decide_mode(self, delta: float, force_f64: bool):
        R = self.pg.ReduceOp
        torch = self.torch
        info = self.shard.probe(delta)
        min_l = self._allreduce(info["min_light"], R.MIN, torch.float64)
        max_w = self._allreduce(info["max_w"], R.MAX, torch.float64)
        frac = int(self._allreduce(info["frac"], R.MAX, torch.int64))
        n_l = int(self._allreduce(info["nL"], R.SUM, torch.int64))
        mode, fb = MODE_F64, 0
        if not force_f64 and frac <= 60 and math.ldexp(max_w, frac) < 4294967295.0:
            mode, fb = MODE_FIXED32, frac
        per = 2 if n_l == 0 else int(math.ceil(delta / min_l)) + 2
        return mode, fb, self.n * per

    def solve(self, source: int, delta: float, skip_empty_buckets: bool = False,
              force_f64: bool = False, on_device: bool = False) -> ShardedResult:
        """Joint solve of one source.  `local` is numpy, or a device tensor
        when on_device=True (no host copy of the distances)."""
        if not 0 <= source < self.n:
            raise ValueError(f"source {source} out of range for {self.n} vertices")
        if not (delta > 0) or not math.isfinite(delta):
            raise ValueError(f"delta must be a positive finite number, got {delta}")
        key = (float(delta), bool(force_f64))
        if getattr(self, "_mode_key", None) != key:
            self._mode = self._decide_mode(delta, force_f64)
            self._mode_key = key
        mode, frac, ceiling = self._mode
        res = self._run(source, delta, mode, frac, ceiling, on_device)
        if res is None:  # a fixed-point sum overflowed on some rank: exact f64 rerun
            mode, frac, ceiling = self._decide_mode(delta, True)
            self._mode, self._mode_key = (mode, frac, ceiling), (float(delta), False)
            res = self._run(source, delta, mode, frac, ceiling, on_device)
        local, phases, visited, exchanged = res
        R = self.pg.ReduceOp
        if on_device:
            fin = local[self.torch.isfinite(local)]
            mx = float(fin.max().item()) if fin.numel() else -math.inf
        else:
            fin = local[np.isfinite(local)]
            mx = float(fin.max()) if fin.size else -math.inf
        mx = self._allreduce(mx, R.MAX, self.torch.float64)
        outer = visited if skip_empty_buckets else bucket_index_of(mx, delta) + 1
        return ShardedResult(local, self.shard.v0, outer, phases, visited, exchanged, mode)

    def _window(self, idx: int, delta: float, mode: int, frac: int):
        lo, hi = idx * delta, (idx + 1) * delta
        if mode == MODE_FIXED32:
            return _ceil_u32(math.ldexp(lo, frac)), _ceil_u32(math.ldexp(hi, frac))
        return _f64_bits(lo), _f64_bits(hi)

    def _value(self, v: int, mode: int, frac: int) -> float:
        return math.ldexp(float(v), -frac) if mode == MODE_FIXED32 else _bits_f64(v)

    def _run(self, source, delta, mode, frac, ceiling, on_device=False):
        sh = self.shard
        sh.prepare(delta, mode, frac)
        sh.begin(source)
        idx, phases, visited, exchanged = 0, 0, 0, 0
        heavy_ovf = 0  # the previous bucket's heavy-step overflow, carried in the next scan's meta
        while True:
            L, H = self._window(idx, delta, mode, frac)
            ids, vals, cnt, nmin = sh.scan(L, H)
            meta = self._exchange_meta(cnt, I64_NONE if nmin == NONE else nmin, heavy_ovf)
            if meta[:, 2].max():
                return None  # a fixed-point sum overflowed on some rank: exact f64 rerun
            fc = int(meta[:, 0].sum())
            nm = int(meta[:, 1].min())
            if fc == 0:
                if nm == I64_NONE:
                    break  # nothing stored beyond the window: done
                idx = bucket_index_of(self._value(nm, mode, frac), delta)
                continue
            visited += 1
            F, Fv, nf = self._gather_entries(ids, vals, meta[:, 0], packed32=mode == MODE_FIXED32)
            exchanged += nf
            sh.s_add(F, Fv, nf)
            while True:  # light phases (sssp.py:292-301)
                phases += 1
                if phases > ceiling:
                    raise RuntimeError(f"light phase count exceeded ceiling {ceiling}; "
                                       "relaxation is not converging")
                nids, nvals, ncnt, ovf = sh.relax_light(F, Fv, nf, H)
                meta = self._exchange_meta(ncnt, int(ovf))
                if meta[:, 1].max():
                    return None
                F, Fv, nf = self._gather_entries(nids, nvals, meta[:, 0], packed32=mode == MODE_FIXED32)
                exchanged += nf
                if nf == 0:
                    break
                sh.s_add(F, Fv, nf)
            heavy_ovf = int(sh.relax_heavy())  # S values are final; no exchange needed
            idx += 1
        local = sh.result(on_device=True) if on_device else sh.result()
        return local, phases, visited, exchanged
