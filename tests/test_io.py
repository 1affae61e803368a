"""Native graph-file ingestion (csrc/ingest.cpp) against the reference
loaders' recorded outputs (tests/golden/io_golden.json, written by
tests/golden/make_io_golden.py from deltasparse/io.py).  Host only."""

from __future__ import annotations

import json
import logging
import os

import numpy as np
import pytest

import refgen
from paper_1911_06895_b200 import io as dio

HERE = os.path.dirname(os.path.abspath(__file__))
IO_DIR = os.path.join(HERE, "golden", "io")
GOLD = json.load(open(os.path.join(HERE, "golden", "io_golden.json")))


def _check(got_fn, want, path, caplog):
    if want["ok"]:
        caplog.clear()
        with caplog.at_level(logging.WARNING, logger=dio.log.name):
            m, labels = got_fn()
        assert m.n == want["n"]
        assert m.indptr.tolist() == want["indptr"]
        assert m.col.tolist() == want["col"]
        assert [float(x).hex() for x in m.val] == want["val"]
        assert labels.externals == want["labels"]
        warns = [r.getMessage() for r in caplog.records if r.name == dio.log.name]
        norm = [w.split(": ", 1)[1] for w in want["warnings"]]
        assert [w.split(": ", 1)[1] for w in warns] == norm
        assert all(w.startswith(path + ": ") for w in warns)
    else:
        cls = getattr(dio, want["cls"])
        with pytest.raises(cls) as ei:
            got_fn()
        assert ei.value.lineno == want["lineno"]
        assert ei.value.message == want["message"]
        assert ei.value.path == path
        assert str(ei.value) == f"{path}:{want['lineno']}: {want['message']}"
        assert isinstance(ei.value, dio.GraphLoadError)


@pytest.mark.parametrize("key", sorted(GOLD["mtx"]))
def test_matrix_market_matches_reference(key, caplog):
    name, dw = key.split("|")
    path = os.path.join(IO_DIR, name + ".mtx")
    _check(lambda: dio.load_matrix_market(path, float(dw)), GOLD["mtx"][key], path, caplog)


@pytest.mark.parametrize("name", sorted(GOLD["edges"]))
def test_edge_list_matches_reference(name, caplog):
    want = GOLD["edges"][name]
    path = os.path.join(IO_DIR, name + ".txt")
    _check(lambda: dio.load_edge_list(path, want["directed"], 1.0), want, path, caplog)


def test_load_graph_dispatch_and_label_map():
    m, lab = dio.load_graph(dio.GraphFile(os.path.join(IO_DIR, "label_order.txt"), "edges"))
    assert lab.externals == [100, 7, 3, 42]
    assert lab.to_internal(7) == 1 and lab.to_external(3) == 42 and 3 in lab and len(lab) == 4
    m2, lab2 = dio.load_graph(dio.GraphFile(os.path.join(IO_DIR, "general_real.mtx"), "mtx"))
    assert lab2.externals == [1, 2, 3, 4]
    with pytest.raises(ValueError, match="unknown graph format"):
        dio.load_graph(dio.GraphFile("x", "csv"))
    with pytest.raises(ValueError, match="duplicate external label"):
        dio.LabelMap([1, 1])


def test_large_generated_edge_list_roundtrip(tmp_path):
    # a bigger file through the native parser vs a numpy restatement
    rng = np.random.default_rng(5)
    u = rng.integers(0, 5000, 200_000)
    v = rng.integers(0, 5000, 200_000)
    w = rng.integers(1, 100, 200_000) / 8.0
    p = tmp_path / "g.txt"
    p.write_text("".join(f"{a} {b} {float(c)!r}\n" for a, b, c in zip(u, v, w)))
    m, lab = dio.load_edge_list(str(p), directed=False)
    ext = lab.externals
    # first-seen order of labels, source before target
    seen = {}
    for a, b in zip(u.tolist(), v.tolist()):
        seen.setdefault(a, len(seen))
        seen.setdefault(b, len(seen))
    assert ext == list(seen)
    r = np.array([seen[a] for a in u.tolist()])
    c = np.array([seen[b] for b in v.tolist()])
    keep = r != c
    rr = np.concatenate([r[keep], c[keep]])
    cc = np.concatenate([c[keep], r[keep]])
    ww = np.concatenate([w[keep], w[keep]])
    dense = {}
    for a, b, x in zip(rr.tolist(), cc.tolist(), ww.tolist()):
        dense[(a, b)] = min(x, dense.get((a, b), np.inf))
    got = {}
    for a in range(m.n):
        for k in range(m.indptr[a], m.indptr[a + 1]):
            got[(a, int(m.col[k]))] = float(m.val[k])
    assert got == dense


def test_binary_csr_cache_roundtrip(tmp_path):
    from paper_1911_06895_b200 import graphs

    rng = np.random.default_rng(5)
    cases = [
        graphs.erdos_renyi(256, seed=1),                        # int weights -> f32 storage
        refgen.random_graph(300, 2000, rng, weights="float"),   # arbitrary f64 weights
        graphs.rmat(10, seed=3),                                # fp32-lattice weights
    ]
    for k, m in enumerate(cases):
        labels = dio.LabelMap([int(x) for x in rng.permutation(10 * m.n)[: m.n] + 1])
        for lab in (None, labels):
            p = str(tmp_path / f"g{k}.csr")
            dio.save_csr(p, m, lab)
            got, glab = dio.load_csr(p)
            assert got == m
            got.check_invariants()
            want = lab.externals if lab is not None else list(range(1, m.n + 1))
            assert glab.externals == want
            spec = dio.GraphFile(path=p, format="csr")
            assert dio.load_graph(spec)[0] == m


def test_binary_csr_cache_rejects_bad_files(tmp_path):
    from paper_1911_06895_b200 import graphs

    m = graphs.erdos_renyi(64, seed=2)
    p = tmp_path / "g.csr"
    dio.save_csr(str(p), m)
    raw = p.read_bytes()
    bad = tmp_path / "bad.csr"
    for blob, msg in ((b"not a cache at all" * 8, "not a binary CSR cache"),
                      (raw[: len(raw) - 16], "truncated"),
                      (raw[:8] + (0).to_bytes(8, "little") + raw[16:], "corrupt binary CSR header")):
        bad.write_bytes(blob)
        with pytest.raises(ValueError, match=msg):
            dio.load_csr(str(bad))
    # row offsets that do not end at nnz
    head = 64
    broken = bytearray(raw)
    broken[head + 8 * m.n: head + 8 * (m.n + 1)] = (m.nnz + 1).to_bytes(8, "little")
    bad.write_bytes(bytes(broken))
    with pytest.raises(ValueError, match="corrupt row offsets"):
        dio.load_csr(str(bad))
