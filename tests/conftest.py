"""Shared test setup: the `gpu` marker and golden-fixture helpers."""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(REPO, "tests", "golden")
if REPO not in sys.path:
    sys.path.insert(0, REPO)
TESTS = os.path.dirname(os.path.abspath(__file__))
if TESTS not in sys.path:
    sys.path.insert(0, TESTS)
import refgen  # noqa: E402  (reference test-graph generators, test infrastructure)
# arm the device watchdog (opt-in in the library): a broken build fails a
# test with DS_ETIMEOUT instead of hanging the GPU
os.environ.setdefault("DS_TIMEOUT_S", "300")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def vec_hash(idx, val) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(idx, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(val, dtype="<f8").tobytes())
    return h.hexdigest()


def csr_hash(indptr, col, val) -> str:
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(indptr, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(col, dtype="<i8").tobytes())
    h.update(np.ascontiguousarray(val, dtype="<f8").tobytes())
    return h.hexdigest()


def graph_from_json(g):
    indptr = np.array(g["indptr"], dtype=np.int64)
    col = np.array(g["col"], dtype=np.int64)
    val = np.array([float.fromhex(x) for x in g["val"]], dtype=np.float64)
    return g["n"], indptr, col, val


@pytest.fixture(scope="session")
def golden():
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)


@pytest.fixture(scope="session")
def corpus_dist():
    return np.load(os.path.join(GOLDEN, "corpus_dist.npz"))


def criterion1_graphs():
    """Regenerate the reference's criterion-1 corpus (test_acceptance.py:55-66)
    with the restated generator (graphs.random_graph)."""
    from paper_1911_06895_b200 import graphs

    rng = np.random.default_rng(20260816)
    out = []
    for case in range(700):
        kind = "int" if case < 500 else "float"
        n = int(rng.integers(1, 201))
        m = int(rng.integers(0, 2001))
        a = refgen.random_graph(n, m, rng, weights=kind)
        s = int(rng.integers(0, n))
        out.append((a, s, kind))
    return out


def unit_graphs():
    from paper_1911_06895_b200 import graphs

    rng = np.random.default_rng(20260816 + 6)
    out = []
    for _ in range(50):
        n = int(rng.integers(2, 121))
        out.append(refgen.random_connected_unit_graph(n, int(rng.integers(0, 2 * n)), rng))
    return out
