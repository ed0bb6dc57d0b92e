"""Golden fixtures for the formats and metrics either side of the path, from the LIVE
reference (dev container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_graphio.py

For a set of small seeded graphs: the text the reference's writers produce (fileio.py:
199-216, :240-243, :271-278), the arrays its readers return (fileio.py:70-263), its
error class and message for every malformed input below, and its metrics report
(metrics.py:253-281) for several partitions.  Output: tests/golden/graphio.json.
"""

from __future__ import annotations

import io
import json
import os
import sys
import warnings

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from geopart import fileio as F  # noqa: E402
from geopart import metrics as M  # noqa: E402
from geopart.baselines import sfc_labels  # noqa: E402
from geopart.graph import GeometricGraph, Partition  # noqa: E402


def rgg(n, d, radius, seed):
    rng = np.random.default_rng(seed)
    pts = rng.random((n, d))
    diff = pts[:, None, :] - pts[None, :, :]
    close = (diff ** 2).sum(-1) < radius ** 2
    u, v = np.nonzero(np.triu(close, 1))
    return pts, np.stack([u, v], 1)


def grid(w, h):
    idx = np.arange(w * h).reshape(h, w)
    e = np.concatenate([np.stack([idx[:, :-1].ravel(), idx[:, 1:].ravel()], 1),
                        np.stack([idx[:-1, :].ravel(), idx[1:, :].ravel()], 1)])
    ys, xs = np.divmod(np.arange(w * h), w)
    return np.stack([xs, ys], 1).astype(float), e


def graphs():
    out = {}
    pts, e = grid(12, 9)
    out["grid12x9"] = GeometricGraph.from_edges(len(pts), e, pts)
    pts, e = rgg(300, 2, 0.09, 1)
    rng = np.random.default_rng(2)
    out["rgg300_w"] = GeometricGraph.from_edges(
        300, e, pts, rng.integers(1, 6, 300).astype(float),
        np.round(rng.random(len(e)) * 4 + 0.25, 2))
    pts, e = rgg(200, 3, 0.22, 3)
    rng = np.random.default_rng(4)
    out["rgg200_3d_real"] = GeometricGraph.from_edges(
        200, e, pts, rng.random(200) + 0.1, rng.random(len(e)) + 1e-5)
    out["path3"] = GeometricGraph.from_edges(3, [(0, 1), (1, 2)], [[0, 0], [1, 0], [2, 0.5]])
    out["single"] = GeometricGraph.from_edges(1, np.empty((0, 2), int), [[0.5, 0.25]])
    out["isolated"] = GeometricGraph.from_edges(
        6, [(0, 2), (2, 5)], np.random.default_rng(5).random((6, 2)), [1, 2, 3, 1, 2, 3])
    pts, e = rgg(120, 2, 0.16, 6)
    out["rgg120_ew"] = GeometricGraph.from_edges(
        120, e, pts, None, np.random.default_rng(7).integers(1, 9, len(e)).astype(float))
    return out


def text_of(fn, *a):
    s = io.StringIO()
    fn(*a, s)
    return s.getvalue()


def partitions(name, g):
    rng = np.random.default_rng(sum(map(ord, name)))
    n = g.n
    out = {}
    if n >= 10:
        out["rand5"] = (rng.integers(0, 5, n), 5)
        out["sfc7"] = (sfc_labels(g.coords, g.vertex_weights, 7), 7)
        lab = rng.integers(0, 8, n)
        out["empty_block"] = (lab, 10)
        # two far-apart halves share block 0: disconnected
        order = np.argsort(g.coords[:, 0], kind="stable")
        lab = np.empty(n, dtype=np.int64)
        lab[order] = np.arange(n) * 4 // n
        lab[lab == 3] = 0
        out["split_block"] = (lab, 3)
    out["one"] = (np.zeros(n, dtype=np.int64), 1)
    out["each"] = (np.arange(n) % max(1, min(n, 4)), max(1, min(n, 4)))
    return out


BAD_GRAPHS = {
    # name: (graph text, coords text or None)
    "missing_header": ("% only a comment\n", None),
    "empty": ("", None),
    "header_one_field": ("3\n2\n1 3\n2\n", None),
    "header_five_fields": ("3 2 0 1 7\n2\n1 3\n2\n", None),
    "header_nonnumeric": ("x 2\n2\n1 3\n2\n", None),
    "header_bad_sizes": ("0 0\n", None),
    "header_fmt_alpha": ("3 2 ab\n2\n1 3\n2\n", None),
    "header_vsize": ("3 2 100\n2\n1 3\n2\n", None),
    "header_ncon2": ("3 2 10 2\n1 2\n1 1 3\n1 2\n", None),
    "header_ncon_alpha": ("3 2 10 z\n1 2\n1 1 3\n1 2\n", None),
    "too_few_lines": ("3 2\n2\n1 3\n", None),
    "too_many_lines": ("3 2\n2\n1 3\n2\n1\n\n", None),
    "missing_vweight": ("3 2 10\n1 2\n\n1 2\n", None),
    "bad_vweight": ("3 2 10\n1 2\nq 1 3\n1 2\n", None),
    "zero_vweight": ("3 2 10\n1 2\n0 1 3\n1 2\n", None),
    "inf_vweight": ("3 2 10\n1 2\ninf 1 3\n1 2\n", None),
    "dangling": ("3 2 1\n2 1.5\n1 1.5 3\n2 2\n", None),
    "nonnumeric_id": ("3 2\n2\n1 x3\n2\n", None),
    "float_id": ("3 2\n2\n1 3.0\n2\n", None),
    "out_of_range": ("3 2\n2\n1 4\n2\n", None),
    "negative_id": ("3 2\n2\n1 -3\n2\n", None),
    "self_loop": ("3 2\n2\n2 3\n2\n", None),
    "duplicate": ("3 2\n2 2\n1 3\n2\n", None),
    "bad_eweight": ("3 2 1\n2 1\n1 1 3 w\n2 2\n", None),
    "neg_eweight": ("3 2 1\n2 1\n1 1 3 -2\n2 -2\n", None),
    "edge_count": ("3 3\n2\n1 3\n2\n", None),
    "asymmetric": ("3 2\n2 3\n1\n2\n", None),
    "asymmetric_later": ("4 3\n2\n1 3\n2\n3\n", None),
    "eweight_asym": ("3 2 1\n2 1\n1 2 3 5\n2 5\n", None),
    "first_error_wins": ("4 3\n2\n1 9\n3 3\n3 q\n", None),
    "dup_before_selfloop": ("4 3\n2 2\n1\n3\n4\n", None),
    "coords_short": ("3 2\n2\n1 3\n2\n", "0 0\n1 1\n"),
    "coords_4cols": ("3 2\n2\n1 3\n2\n", "0 0 0 0\n1 1 1 1\n2 2 2 2\n"),
    "coords_nan": ("3 2\n2\n1 3\n2\n", "0 0\n1 nan\n2 2\n"),
    "coords_bad_token": ("3 2\n2\n1 3\n2\n", "0 0\n1 1x\n2 2\n"),
    "coords_ragged": ("3 2\n2\n1 3\n2\n", "0 0\n1\n2 2\n"),
    "coords_empty": ("3 2\n2\n1 3\n2\n", "# nothing\n\n"),
}

GOOD_GRAPHS = {
    # reader corner cases that must parse (text, coords)
    "comments_everywhere": ("% c\n  % indented\n3 2\n% mid\n2\n1 3\n%x\n2\n% tail\n", None),
    "crlf": ("3 2\r\n2\r\n1 3\r\n2\r\n", "0 0\r\n1 1\r\n2 2\r\n"),
    "no_final_newline": ("3 2\n2\n1 3\n2", "0 0\n1 1\n2 2"),
    "trailing_blank_lines": ("3 2\n2\n1 3\n2\n\n  \n\t\n", None),
    "blank_is_isolated": ("4 1\n2\n1\n\n\n", None),
    "tabs_and_spaces": ("3 2  011 \n 1\t2 1.5 \n2  1 1.5\t3 2e0\n  3 2 2.0\n", None),
    "fmt_variants": ("3 2 001\n2 7\n1 7 3 0.5\n2 0.5\n", None),
    "python_tokens": ("3 2 10\n+1 2\n1_0 1 3\n1e0 +2\n", None),
    "leading_zero_ids": ("3 2\n02\n001 3\n2\n", None),
    "coords_sci_comments": ("3 2\n2\n1 3\n2\n",
                            "# x y\n1e-3 -2.5E+2 # first\n\n.5 5.\n+1.25 0.1\n"),
    "coords_17g": ("2 1\n2\n1\n", "0.10000000000000001 2.2250738585072014e-308\n"
                                   "1.7976931348623157e+308 4.9406564584124654e-324\n"),
}

TABLES = {
    # name: (text, "coords" | "labels", kwargs)
    "labels_plain": ("0\n3\n2\n1\n", "labels", {}),
    "labels_k": ("0\n1\n", "labels", {"k": 5}),
    "labels_expect_bad": ("0\n1\n", "labels", {"expect_n": 3}),
    "labels_negative": ("0\n-1\n", "labels", {}),
    "labels_float": ("0\n1.0\n", "labels", {}),
    "labels_two_cols": ("0 1\n1 0\n", "labels", {}),
    "labels_one_row": ("0 1 2\n", "labels", {}),
    "labels_empty": ("", "labels", {}),
    "labels_comment": ("# ids\n2\n\n0 # zero\n", "labels", {}),
    "labels_big": ("1\n9223372036854775807\n", "labels", {}),
    "labels_overflow": ("1\n9223372036854775808\n", "labels", {}),
    "labels_plus": ("+3\n007\n", "labels", {}),
    "coords_ok": ("0 1\n2 3\n", "coords", {"expect_n": 2}),
    "coords_inf": ("0 1\n2 inf\n", "coords", {}),
    "coords_one_col": ("0\n1\n", "coords", {}),
    "coords_ragged_late": ("0 1\n2 3\n\n4 5 6\n", "coords", {}),
    "coords_bad_before_ragged": ("0 1\n2 x\n4\n", "coords", {}),
    "coords_ragged_before_bad": ("0 1\n2\n4 x\n", "coords", {}),
    "coords_ragged_and_bad_same_row": ("0 1\n2 x 3\n", "coords", {}),
    "coords_underscore": ("0 1\n2 1_0\n", "coords", {}),
    "coords_20_digits": ("0.12345678901234567890 1\n2 123456789012345678901234567890\n",
                         "coords", {}),
}


def arr(a):
    a = np.asarray(a)
    if a.dtype.kind == "f":
        return {"f64_hex": [float(x).hex() for x in a.ravel()], "shape": list(a.shape)}
    return {"i64": [int(x) for x in a.ravel()], "shape": list(a.shape)}


def graph_arrays(g):
    return {"offsets": arr(g.offsets), "neighbors": arr(g.neighbors),
            "vertex_weights": arr(g.vertex_weights), "coords": arr(g.coords),
            "edge_weights": None if g.edge_weights is None else arr(g.edge_weights)}


def attempt(fn):
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        try:
            return {"ok": fn()}
        except Exception as e:
            return {"error": type(e).__name__, "message": str(e)}


def main():
    out = {"graphs": {}, "bad_graphs": {}, "good_graphs": {}, "tables": {}}
    for name, g in graphs().items():
        gt, ct = text_of(F.write_metis_graph, g), text_of(F.write_coords, g.coords)
        back = F.load_metis_graph(io.StringIO(gt), io.StringIO(ct))
        rec = {"graph_text": gt, "coords_text": ct, "arrays": graph_arrays(back), "partitions": {}}
        for pname, (lab, k) in partitions(name, g).items():
            part = Partition(assignment=lab, k=k)
            rep = json.loads(M.evaluate(g, part).to_json())
            rec["partitions"][pname] = {
                "labels": [int(x) for x in lab], "k": int(k), "report": rep,
                "text": text_of(F.write_partition, part)}
        out["graphs"][name] = rec
    for name, (gt, ct) in BAD_GRAPHS.items():
        res = attempt(lambda: F.load_metis_graph(io.StringIO(gt),
                                                 None if ct is None else io.StringIO(ct)))
        assert "error" in res, name
        out["bad_graphs"][name] = {"graph_text": gt, "coords_text": ct, **res}
    for name, (gt, ct) in GOOD_GRAPHS.items():
        g = F.load_metis_graph(io.StringIO(gt), None if ct is None else io.StringIO(ct))
        out["good_graphs"][name] = {"graph_text": gt, "coords_text": ct,
                                    "arrays": graph_arrays(g)}
    for name, (text, kind, kw) in TABLES.items():
        if kind == "coords":
            res = attempt(lambda: arr(F.load_coords(io.StringIO(text), **kw)))
        else:
            def run():
                p = F.read_partition(io.StringIO(text), **kw)
                return {"labels": arr(p.assignment), "k": int(p.k)}
            res = attempt(run)
        out["tables"][name] = {"text": text, "kind": kind, "kwargs": kw, **res}
    with open(os.path.join(HERE, "graphio.json"), "w") as f:
        json.dump(out, f, indent=0, sort_keys=True)
    print({k: len(v) for k, v in out.items()})


if __name__ == "__main__":
    main()
