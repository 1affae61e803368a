"""Randomised parity sweep against the CPU oracle: graph shapes (R-MAT,
ER directed, grids, random sparse), weight kinds (fp32 lattice -> fixed
point, integers, non-dyadic floats -> binary64), deltas, both skip modes,
single and batched solves, forced kernels.  Prints one line per failure and a
summary; exit status 1 on any mismatch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
from paper_1911_06895_b200 import DeviceGraph, graphs, matrix_build

budget = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2024)
t_end = time.time() + budget
runs = fails = 0


def make():
    kind = rng.integers(0, 4)
    if kind == 0:
        a = graphs.rmat(int(rng.integers(8, 15)), seed=int(rng.integers(1, 1000)),
                        weight_seed=int(rng.integers(1, 1000)))
    elif kind == 1:
        a = graphs.erdos_renyi(int(rng.integers(64, 4096)), seed=int(rng.integers(0, 1000)))
    elif kind == 2:
        a = graphs.grid2d(int(rng.integers(8, 96)), seed=int(rng.integers(0, 1000)))
    else:
        n = int(rng.integers(2, 3000))
        m = int(rng.integers(1, 8 * n))
        u = rng.integers(0, n, m); v = rng.integers(0, n, m)
        wk = rng.integers(0, 3)
        w = (rng.integers(1, 50, m).astype(np.float64) if wk == 0 else
             rng.random(m) * 10 + 1e-3 if wk == 1 else
             rng.integers(1, 1 << 20, m) / float(1 << 20))
        a = matrix_build(n, np.column_stack([u, v, w]))
    return a


base_env = dict(os.environ)


def knobs():
    """Random solver knobs: lex mode forced with ksub 1..8 (and there wide
    windows off / forced with random growth), the heavy gather forced on small
    graphs (any ratio) or off."""
    env = dict(base_env)
    lk = int(rng.integers(0, 5))
    if lk:
        env["DS_LEX"] = "1"
        env["DS_LEX_K"] = str(1 << (lk - 1))
    wd = int(rng.integers(0, 4)) if lk else 0
    for k in ("DS_WIDE", "DS_WIDE_FORCE", "DS_WIDE_G0", "DS_WIDE_LO", "DS_WIDE_HI"):
        env.pop(k, None)
    if wd == 1:
        env["DS_WIDE"] = "0"
    elif wd >= 2:
        # wide windows from the second bucket on: growing (LO huge), shrinking
        # back to the narrow schedule (HI tiny), or at the default thresholds
        env["DS_WIDE_FORCE"] = "1"
        env["DS_WIDE_G0"] = str(int(rng.choice([1, 2, 3, 7])))
        gr = int(rng.integers(0, 3))
        if gr == 0:
            env["DS_WIDE_LO"] = "1e18"
        elif gr == 1:
            env["DS_WIDE_LO"] = "0"; env["DS_WIDE_HI"] = str(int(rng.choice([0, 50, 2000])))
    for k in ("DS_WIDE_FRAC", "DS_WIDE_ALL", "DS_BIDIR"):
        env.pop(k, None)
    if lk and wd == 0 and rng.integers(0, 2):
        # bidirectional entry reachable at the first heavy step (symmetric graphs, gather chosen)
        env["DS_WIDE_FRAC"] = "1.0"
        if rng.integers(0, 2):
            env["DS_WIDE_ALL"] = "0"; env["DS_WIDE_G0"] = str(int(rng.choice([1, 2, 5])))
    hp = int(rng.integers(0, 3))
    if hp == 1:
        env["DS_HPULL_MIN"] = "0"
        env["DS_HPULL_RATIO"] = str(float(rng.choice([0.0, 0.3, 1.0, 3.0])))
    elif hp == 2:
        env["DS_HPULL"] = "0"
    os.environ.clear()
    os.environ.update(env)
    return (f"lex={env.get('DS_LEX_K', '-')} hpull={hp} wide={wd} g0={env.get('DS_WIDE_G0', '-')} "
            f"lo={env.get('DS_WIDE_LO', '-')} hi={env.get('DS_WIDE_HI', '-')} frac={env.get('DS_WIDE_FRAC', '-')} "
            f"all={env.get('DS_WIDE_ALL', '-')}")


while time.time() < t_end:
    a = make()
    tag = knobs()
    g = DeviceGraph.from_matrix(a)
    deg = np.diff(a.indptr)
    cands = np.flatnonzero(deg > 0)
    if cands.size == 0:
        g.close(); continue
    srcs = [int(x) for x in rng.choice(cands, size=min(3, cands.size), replace=False)]
    wmax = float(a.val.max()) if a.val.size else 1.0
    delta = float(rng.choice([wmax / 10, wmax / 3, wmax, wmax * 2, 0.05 + rng.random()]))
    skip = bool(rng.integers(0, 2))
    f64 = bool(rng.integers(0, 4) == 0)
    for s in srcs:
        want, outer, phases = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, delta, skip_empty_buckets=skip, threads=8)
        st = g.solve(s, delta, skip_empty_buckets=skip, force_f64=f64)
        got = g.result_dense()
        ok = np.array_equal(got.view(np.uint64), want.view(np.uint64)) and \
            (st.outer_iterations, st.inner_phases) == (outer, phases)
        runs += 1
        if not ok:
            fails += 1
            print(f"FAIL single n={a.n} nnz={a.nnz} s={s} delta={delta!r} skip={skip} f64={f64} {tag}", flush=True)
    stats, dist = g.solve_batch(srcs, delta, skip_empty_buckets=skip, force_f64=f64,
                                concurrency=int(rng.integers(1, 4)))
    for i, s in enumerate(srcs):
        want, outer, phases = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, delta, skip_empty_buckets=skip, threads=8)
        ok = np.array_equal(dist[i].view(np.uint64), want.view(np.uint64)) and \
            (stats[i].outer_iterations, stats[i].inner_phases) == (outer, phases)
        runs += 1
        if not ok:
            fails += 1
            print(f"FAIL batch n={a.n} nnz={a.nnz} s={s} delta={delta!r} skip={skip} f64={f64} {tag}", flush=True)
    g.close()
print(f"fuzz: {runs} solves, {fails} mismatches", flush=True)
sys.exit(1 if fails else 0)
