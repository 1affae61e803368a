"""Golden outputs of the reference graph loaders (deltasparse/io.py).

Run in the build container (where /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_io_golden.py

Writes a set of small synthetic graph files (Matrix Market and edge lists,
well-formed and malformed) under tests/golden/io/, loads each with the
UNMODIFIED reference `load_matrix_market` / `load_edge_list`, and records
the resulting CSR, label map and self-loop count -- or the exception class,
line number and message -- in tests/golden/io_golden.json.
"""

from __future__ import annotations

import json
import logging
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
IO_DIR = os.path.join(HERE, "io")
sys.path.insert(0, "/root/reference/pkg/src")

from deltasparse import io as ref_io  # noqa: E402

MTX = {
    "general_real": "%%MatrixMarket matrix coordinate real general\n% comment\n4 4 5\n1 2 0.5\n2 3 1.25\n3 4 2\n4 1 3e-1\n1 3 7\n",
    "symmetric_integer": "%%MatrixMarket matrix coordinate integer symmetric\n3 3 3\n1 2 4\n2 3 5\n3 1 6\n",
    "pattern_general": "%%MatrixMarket matrix coordinate pattern general\n3 3 3\n1 2\n2 3\n3 1\n",
    "pattern_symmetric": "%%MatrixMarket matrix coordinate pattern symmetric\n3 3 2\n2 1\n3 2\n",
    "duplicates_and_loops": "%%MatrixMarket matrix coordinate real general\n3 3 6\n1 2 5\n1 2 2\n2 2 1\n1 2 9\n3 1 1\n3 3 4\n",
    "crlf_blank_comments": "%%MatrixMarket Matrix Coordinate REAL General\r\n%c1\r\n\r\n  3 3 2  \r\n% mid\r\n1 3 1.5\r\n\r\n3 2 2.5\r\n",
    "cr_only": "%%MatrixMarket matrix coordinate real general\r2 2 1\r1 2 0.25\r",
    "no_final_newline": "%%MatrixMarket matrix coordinate real general\n2 2 1\n2 1 8",
    "underscores_and_forms": "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 2 1_0.5\n2 3 .5\n3 1 1E1\n",
    "empty_graph": "%%MatrixMarket matrix coordinate real general\n5 5 0\n",
    # errors
    "err_empty": "",
    "err_header": "%%MatrixMarket matrix array real general\n2 2\n",
    "err_header_tokens": "%%MatrixMarket matrix coordinate real\n",
    "err_field": "%%MatrixMarket matrix coordinate complex general\n",
    "err_symmetry": "%%MatrixMarket matrix coordinate real hermitian\n",
    "err_size_tokens": "%%MatrixMarket matrix coordinate real general\n3 3\n",
    "err_size_ints": "%%MatrixMarket matrix coordinate real general\n3 x 1\n",
    "err_not_square": "%%MatrixMarket matrix coordinate real general\n3 4 1\n1 2 1\n",
    "err_dim": "%%MatrixMarket matrix coordinate real general\n0 0 0\n",
    "err_too_many": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 1\n2 1 1\n",
    "err_tokens": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2\n",
    "err_coord_int": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1.0 2 1\n",
    "err_coord_range": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 3 1\n",
    "err_weight": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 abc\n",
    "err_weight_hex": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 0x1p3\n",
    "err_weight_zero": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 0\n",
    "err_weight_neg": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 -1.5\n",
    "err_weight_inf": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 inf\n",
    "err_weight_nan": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 2 nan\n",
    "err_missing_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "err_short": "%%MatrixMarket matrix coordinate real general\n3 3 3\n1 2 1\n% end\n",
}

EDGES = {
    "basic_weighted": ("10 20 1.5\n20 30 2\n30 10 0.25\n", True),
    "unweighted_default": ("5 6\n6 7\n7 5\n", True),
    "undirected": ("1 2 3\n2 3 4\n", False),
    "comments_loops_dups": ("# hdr\n% also comment\n4 4 1\n4 9 2\n4 9 1\n\n9 4 5\n", True),
    "label_order": ("100 7\n7 3\n3 100\n42 42\n", True),
    "crlf": ("1 2 1\r\n2 3 1\r\n", False),
    "plus_and_underscore": ("+1 1_0 2\n10 +3 1e0\n", True),
    # errors
    "err_tokens": ("1 2 3 4\n", True),
    "err_single": ("1\n", True),
    "err_label": ("a b\n", True),
    "err_negative": ("1 -2\n", True),
    "err_weight": ("1 2 x\n", True),
    "err_weight_zero": ("1 2 0.0\n", True),
    "err_empty": ("", True),
    "err_only_comments": ("# a\n# b\n", True),
}


def record(fn, *args):
    loops = []

    class H(logging.Handler):
        def emit(self, rec):
            loops.append(rec.getMessage())

    h = H()
    ref_io.log.addHandler(h)
    try:
        m, labels = fn(*args)
        return {"ok": True, "n": m.n, "indptr": m.indptr.tolist(), "col": m.col.tolist(),
                "val": [float(x).hex() for x in m.val], "labels": labels.externals,
                "warnings": loops}
    except ref_io.GraphLoadError as e:
        return {"ok": False, "cls": type(e).__name__, "lineno": e.lineno, "message": e.message}
    finally:
        ref_io.log.removeHandler(h)


def main():
    os.makedirs(IO_DIR, exist_ok=True)
    out = {"mtx": {}, "edges": {}}
    for name, text in MTX.items():
        path = os.path.join(IO_DIR, name + ".mtx")
        with open(path, "w", newline="") as f:
            f.write(text)
        for dw in (1.0, 2.5):
            out["mtx"][f"{name}|{dw}"] = record(ref_io.load_matrix_market, path, dw)
    for name, (text, directed) in EDGES.items():
        path = os.path.join(IO_DIR, name + ".txt")
        with open(path, "w", newline="") as f:
            f.write(text)
        out["edges"][name] = record(ref_io.load_edge_list, path, directed, 1.0)
        out["edges"][name]["directed"] = directed
    with open(os.path.join(HERE, "io_golden.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print(f"{len(out['mtx'])} mtx + {len(out['edges'])} edge-list cases")


if __name__ == "__main__":
    main()
