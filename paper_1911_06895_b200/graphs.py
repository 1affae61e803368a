"""Seeded synthetic graph generators for the BASELINE configs.

There is no public dataset on this path: every config is a
seeded synthetic graph.  Generators here are *counter-based* (splitmix64 of
the edge / pair index), so the host numpy version and the on-device CUDA
generator (`ds_gen_rmat` in the C-ABI library) produce identical CSRs.

Conventions:
* symmetrised graphs carry one weight per undirected pair, shared by both
  directions (mirrors the undirected loader, io.py:253-257);
* fp32-uniform weights are k * 2^-24 with k in [1, 2^24) (k = 0 remapped to
  1 -- a zero weight would silently vanish in the reference's split,
  sssp.py:96-97);
* self-loops dropped, duplicates collapsed (matrix_build, core.py:268-275).

(The restatements of the reference's small test generators, used to
regenerate its corpora, live with the tests: tests/refgen.py.)
"""

from __future__ import annotations

import numpy as np

from .containers import SparseMatrix, matrix_build

__all__ = [
    "splitmix64",
    "rmat",
    "grid2d",
    "erdos_renyi",
    "pick_sources",
    "RMAT_A", "RMAT_B", "RMAT_C",
]

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
GOLDEN = np.uint64(0x9E3779B97F4A7C15)

# Graph500 R-MAT quadrant probabilities (BASELINE.json configs 2,4,5) as
# 32-bit integer thresholds so host and device agree exactly.
RMAT_A = int(0.57 * 2**32)
RMAT_B = int(0.19 * 2**32)
RMAT_C = int(0.19 * 2**32)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 finaliser over uint64 (wrapping arithmetic)."""
    with np.errstate(over="ignore"):
        z = (np.asarray(x, dtype=np.uint64) + GOLDEN)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def _scramble(v: np.ndarray, scale: int, seed: int) -> np.ndarray:
    """Bijective vertex relabelling on [0, 2^scale) (Graph500-style scramble;
    spreads R-MAT hubs across the id space)."""
    mask = np.uint64((1 << scale) - 1)
    half = np.uint64(max(1, (scale + 1) // 2))
    with np.errstate(over="ignore"):
        x = v.astype(np.uint64)
        x = (x * np.uint64(0x9E3779B97F4A7C15 | 1)) & mask
        x ^= x >> half
        x = (x * np.uint64(0xD6E8FEB86659FD93)) & mask
        x ^= x >> half
        x = (x + np.uint64(seed) * np.uint64(0x632BE59BD9B4E019)) & mask
    return x


def _pair_hash(a: np.ndarray, b: np.ndarray, seed: int) -> np.ndarray:
    lo = np.minimum(a, b).astype(np.uint64)
    hi = np.maximum(a, b).astype(np.uint64)
    with np.errstate(over="ignore"):
        key = (lo << np.uint64(32)) | hi
        return splitmix64(key ^ (np.uint64(seed) * np.uint64(0xD1B54A32D192ED03)))


def lattice_weight(a: np.ndarray, b: np.ndarray, seed: int) -> np.ndarray:
    """fp32-uniform [0,1) weight of the undirected pair {a,b}: k * 2^-24,
    k = top 24 hash bits, 0 -> 1."""
    k = (_pair_hash(a, b, seed) >> np.uint64(40)).astype(np.int64)
    k[k == 0] = 1
    return (k.astype(np.float64) * 2.0**-24).astype(np.float32)


def int_weight(a: np.ndarray, b: np.ndarray, seed: int, wmax: int) -> np.ndarray:
    """Integer weight U{1..wmax} of the undirected pair {a,b}."""
    return ((_pair_hash(a, b, seed) >> np.uint64(16)) % np.uint64(wmax)).astype(np.int64) + 1


def _csr_from_keys(n: int, keys: np.ndarray):
    keys = np.unique(keys)  # sorted (row, col) with duplicates collapsed
    u = (keys >> np.uint64(32)).astype(np.int64)
    v = (keys & np.uint64(0xFFFFFFFF)).astype(np.int64)
    counts = np.bincount(u, minlength=n)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    return indptr, u, v


def rmat_edges(scale: int, edge_factor: int = 16, seed: int = 1):
    """Directed R-MAT edge list before symmetrisation: (src, dst) uint64."""
    m = edge_factor << scale
    k = np.arange(m, dtype=np.uint64)
    src = np.zeros(m, dtype=np.uint64)
    dst = np.zeros(m, dtype=np.uint64)
    with np.errstate(over="ignore"):
        seed_mix = np.uint64(seed) * GOLDEN
        for level in range(scale):
            h = splitmix64((k * np.uint64(64) + np.uint64(level)) ^ seed_mix)
            r = (h >> np.uint64(32)).astype(np.int64)
            bit = np.uint64(1 << (scale - 1 - level))
            row = r >= RMAT_A + RMAT_B           # quadrants c, d
            col = ((r >= RMAT_A) & (r < RMAT_A + RMAT_B)) | (r >= RMAT_A + RMAT_B + RMAT_C)
            src |= np.where(row, bit, np.uint64(0))
            dst |= np.where(col, bit, np.uint64(0))
    return _scramble(src, scale, seed), _scramble(dst, scale, seed)


def rmat(scale: int, edge_factor: int = 16, seed: int = 1, weight_seed: int = 2,
         compact: bool = True) -> SparseMatrix:
    """R-MAT (a,b,c,d = .57,.19,.19,.05), self-loops dropped, symmetrised,
    deduplicated, fp32-lattice weights per undirected pair.  Host version for
    scales the CPU handles in seconds (<= 20); `ds_gen_rmat` builds the same
    CSR on the device for scale 24/27."""
    n = 1 << scale
    s, d = rmat_edges(scale, edge_factor, seed)
    keep = s != d
    s, d = s[keep], d[keep]
    keys = np.concatenate([(s << np.uint64(32)) | d, (d << np.uint64(32)) | s])
    indptr, u, v = _csr_from_keys(n, keys)
    w = lattice_weight(u, v, weight_seed)
    return SparseMatrix(n, indptr, v.astype(np.int32), w, compact=compact)


def grid2d(side: int, wmax: int = 100, seed: int = 3, compact: bool = True) -> SparseMatrix:
    """side x side 4-neighbour grid, both directions, integer weights
    U{1..wmax} per undirected edge; vertex id = r*side + c."""
    n = side * side
    v = np.arange(n, dtype=np.int64)
    r, c = v // side, v % side
    nbr = np.stack([v - side, v - 1, v + 1, v + side], axis=1)  # ascending ids
    ok = np.stack([r > 0, c > 0, c < side - 1, r < side - 1], axis=1)
    counts = ok.sum(axis=1)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    col = nbr[ok]
    src = np.repeat(v, counts)
    w = int_weight(src, col, seed, wmax).astype(np.float32)
    return SparseMatrix(n, indptr, col.astype(np.int32), w, compact=compact)


def erdos_renyi(n: int = 1024, p: float | None = None, wmin: int = 1, wmax: int = 10,
                seed: int = 0) -> SparseMatrix:
    """Directed G(n, p): each ordered pair i != j present with probability p
    (default 8/(n-1)), integer weights U{wmin..wmax}; numpy PCG64 seeded."""
    if p is None:
        p = 8.0 / (n - 1)
    rng = np.random.default_rng(seed)
    present = rng.random((n, n)) < p
    np.fill_diagonal(present, False)
    w = rng.integers(wmin, wmax + 1, size=(n, n))
    counts = present.sum(axis=1)
    indptr = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=indptr[1:])
    rows, cols = np.nonzero(present)
    return SparseMatrix(n, indptr, cols, w[rows, cols].astype(np.float64))


def pick_sources(indptr: np.ndarray, count: int, seed: int = 7) -> list[int]:
    """`count` distinct seeded random sources with nonzero out-degree."""
    deg = np.diff(np.asarray(indptr))
    cand = np.flatnonzero(deg > 0)
    rng = np.random.default_rng(seed)
    pick = rng.choice(cand.shape[0], size=min(count, cand.shape[0]), replace=False)
    return [int(x) for x in cand[pick]]
