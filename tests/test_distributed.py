"""Partitioned solver with world_size 2.

CPU: gloo + the numpy shard model (tests/shard_model.py) -- checks the
partitioning, the per-phase frontier all-gather and the all-reduced control
against the oracle, bit-exact with identical counters.
GPU: the same protocol with two ranks sharing cuda:0 (gloo exchange; the ranks
only meet in host-side collectives, never inside kernels) running the sm_100a
shard kernels.
"""

from __future__ import annotations

import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cases(small: bool):
    from paper_1911_06895_b200 import graphs
    from conftest import criterion1_graphs

    out = []
    corpus = criterion1_graphs()
    for k in (3, 17, 42, 101, 250, 499, 500, 511, 600, 699):
        a, s, _ = corpus[k]
        for d in (0.5, 3.0):
            out.append((f"corpus{k}", a, s, d))
    g = graphs.rmat(9 if small else 12, seed=1, weight_seed=2)
    for s in graphs.pick_sources(g.indptr, 2, seed=7):
        out.append(("rmat", g, s, 0.1))
    out.append(("grid", graphs.grid2d(16 if small else 48, seed=3), 0, 25.0))
    return out


def _worker(rank, world, port, use_gpu, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        sys.path.insert(0, REPO)
        sys.path.insert(0, os.path.join(REPO, "tests"))
        import torch.distributed as dist

        import oracle
        from paper_1911_06895_b200.distributed import (PartitionedDeltaStepping, partition_bounds,
                                                       shard_csr)

        dist.init_process_group("gloo", rank=rank, world_size=world)
        fails = []
        for name, a, s, d in _cases(small=not use_gpu):
            b = partition_bounds(a.n, world)
            ptr, col, val = shard_csr(a.indptr, a.col, a.val, b[rank], b[rank + 1])
            if use_gpu:
                from paper_1911_06895_b200.distributed import DeviceShard

                sh = DeviceShard(a.n, b[rank], b[rank + 1], ptr, col, val, device=0)
            else:
                from shard_model import NumpyShard

                sh = NumpyShard(a.n, b[rank], b[rank + 1], ptr, col, val)
            solver = PartitionedDeltaStepping(sh, a.n, dist, "cpu")
            r = solver.solve(s, d)
            rs = solver.solve(s, d, skip_empty_buckets=True)
            parts = [None] * world
            dist.all_gather_object(parts, r.local)
            if rank == 0:
                got = np.concatenate(parts)
                want, outer, phases = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, d)
                _, outer_s, _ = oracle.delta_stepping(a.n, a.indptr, a.col, a.val, s, d,
                                                      skip_empty_buckets=True)
                ok = (np.array_equal(got.view(np.uint64), want.view(np.uint64))
                      and r.outer_iterations == outer and r.inner_phases == phases
                      and rs.outer_iterations == outer_s and rs.inner_phases == phases)
                if not ok:
                    fails.append((name, s, d, r.outer_iterations, outer, r.inner_phases, phases))
            if use_gpu:
                sh.close()
        dist.barrier()
        dist.destroy_process_group()
        if rank == 0:
            q.put(fails)
    except Exception as e:  # surface worker errors in the parent
        q.put(f"rank {rank}: {type(e).__name__}: {e}")
        raise


def _run(use_gpu: bool):
    ctx = mp.get_context("spawn")
    q = ctx.SimpleQueue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, use_gpu, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=900)
    res = q.get() if not q.empty() else "no result"
    for p in procs:
        assert p.exitcode == 0, res
    assert res == [], res


def test_partitioned_protocol_world2_cpu_gloo():
    _run(use_gpu=False)


@pytest.mark.gpu
def test_partitioned_device_shards_world2_gloo():
    _run(use_gpu=True)


def test_bench_self_spawns_ranks_on_cpu():
    # `python bench.py --gpus 2` outside torchrun re-launches itself under
    # torch.distributed.run with two ranks; the reference arm runs on rank 0
    # only (the CPU-only arm: no GPU needed here)
    import json
    import subprocess

    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py"), "--gpus", "2", "--impl", "reference",
                        "--steps", "1", "--warmup", "0", "--scale", "10", "--scale", "10",
                        "--no-python-ref"], capture_output=True, text=True, timeout=600, cwd=REPO)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["n_gpus"] == 2 and d["value"] > 0
    assert d["config"]["workload"] == "rmat10_ef16_delta0.1"
