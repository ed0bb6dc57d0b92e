"""GPU parity tests of the formats / metrics row, through the
package's reference-shaped API (fileio.py, metrics.py, graph.py, cli.py -> C ABI):
bit-exact against the golden vectors made from the live reference, against the CPU
oracle on larger seeded graphs, and through size-independent properties at sizes the
oracle cannot reach."""
import io
import json
import math

import numpy as np
import pytest

import graphio_cases as G
from oracle import graphio_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gold():
    return G.golden()


@pytest.fixture(scope="module")
def api():
    from paper_1805_01208_b200 import fileio, graph, metrics

    class A:
        pass

    a = A()
    a.fileio, a.graph, a.metrics = fileio, graph, metrics
    return a


def _src(text):
    return None if text is None else io.StringIO(text)


def _check_graph(g, want):
    assert G.same_bits(g.offsets, G.arr(want["offsets"]))
    assert G.same_bits(g.neighbors, G.arr(want["neighbors"]))
    assert G.same_bits(g.vertex_weights, G.arr(want["vertex_weights"]))
    assert G.same_bits(g.coords, G.arr(want["coords"]))
    w = G.arr(want["edge_weights"])
    assert (g.edge_weights is None) == (w is None)
    if w is not None:
        assert G.same_bits(g.edge_weights, w)


def test_reads_reference_written_files(api, gold):
    for name, rec in {**gold["graphs"], **gold["good_graphs"]}.items():
        g = api.fileio.load_metis_graph(_src(rec["graph_text"]), _src(rec["coords_text"]))
        _check_graph(g, rec["arrays"])


def test_byte_stream_and_path_sources(api, gold, tmp_path):
    rec = gold["graphs"]["rgg300_w"]
    (tmp_path / "g.graph").write_text(rec["graph_text"])
    (tmp_path / "g.xyz").write_text(rec["coords_text"])
    _check_graph(api.fileio.load_metis_graph(str(tmp_path / "g.graph"), tmp_path / "g.xyz"),
                 rec["arrays"])
    _check_graph(api.fileio.load_metis_graph(io.BytesIO(rec["graph_text"].encode()),
                                             io.BytesIO(rec["coords_text"].encode())),
                 rec["arrays"])


def test_error_messages_equal_the_reference(api, gold):
    for name, rec in gold["bad_graphs"].items():
        with pytest.raises(api.fileio.MetisParseError) as ei:
            api.fileio.load_metis_graph(_src(rec["graph_text"]), _src(rec["coords_text"]))
        assert str(ei.value) == rec["message"], name


def test_tables(api, gold):
    for name, rec in gold["tables"].items():
        coords = rec["kind"] == "coords"
        fn = api.fileio.load_coords if coords else api.fileio.read_partition
        if "error" in rec:
            with pytest.raises(api.fileio.MetisParseError) as ei:
                fn(io.StringIO(rec["text"]), **rec["kwargs"])
            assert str(ei.value) == rec["message"], name
        elif coords:
            assert G.same_bits(fn(io.StringIO(rec["text"]), **rec["kwargs"]), G.arr(rec["ok"])), name
        else:
            p = fn(io.StringIO(rec["text"]), **rec["kwargs"])
            assert G.same_bits(p.assignment, G.arr(rec["ok"]["labels"])), name
            assert p.k == rec["ok"]["k"], name


def test_rejects_non_ascii_and_control_bytes(api):
    with pytest.raises(ValueError):
        api.fileio.load_metis_graph(io.BytesIO(b"2 1\n2\n1 \xc3\xa9\n"))
    with pytest.raises(ValueError):
        api.fileio.load_coords(io.BytesIO(b"0 1\x0b2\n"))


def test_metrics_and_partition_writer_equal_the_reference(api, gold):
    from paper_1805_01208_b200.types import Partition

    un = lambda x: math.inf if x == "unbounded" else float(x)  # noqa: E731
    for name, rec in gold["graphs"].items():
        g = api.fileio.load_metis_graph(_src(rec["graph_text"]), _src(rec["coords_text"]))
        for pname, p in rec["partitions"].items():
            part = Partition(assignment=np.array(p["labels"], dtype=np.int64), k=p["k"])
            rep = api.metrics.evaluate(g, part)
            want = p["report"]
            tag = (name, pname)
            assert (rep.n, rep.m, rep.k) == (want["n"], want["m"], want["k"]), tag
            for key in ("edge_cut", "comm_max", "comm_total", "imbalance"):
                assert getattr(rep, key) == want[key], tag + (key,)
            assert rep.harmonic_diameter == un(want["harmonic_diameter"]), tag
            assert rep.block_weights == want["block_weights"], tag
            assert rep.block_comm == want["block_comm"], tag
            assert rep.block_diameters == [un(x) for x in want["block_diameters"]], tag
            assert json.loads(rep.to_json()) == want, tag
            # the stand-alone functions
            assert api.metrics.edge_cut(g, part) == want["edge_cut"]
            assert api.metrics.comm_volumes(g, part)[0] == want["comm_max"]
            s = io.StringIO()
            api.fileio.write_partition(part, s)
            assert s.getvalue() == p["text"], tag
            back = api.fileio.read_partition(io.StringIO(p["text"]), expect_n=g.n, k=p["k"])
            assert G.same_bits(back.assignment, part.assignment)


def test_writers_equal_the_reference(api, gold):
    for name, rec in gold["graphs"].items():
        g = api.fileio.load_metis_graph(_src(rec["graph_text"]), _src(rec["coords_text"]))
        s, c = io.StringIO(), io.StringIO()
        api.fileio.write_metis_graph(g, s)
        api.fileio.write_coords(g.coords, c)
        assert s.getvalue() == rec["graph_text"], name
        assert c.getvalue() == rec["coords_text"], name


def test_partition_writer_edge_cases(api, tmp_path):
    for vals in ([0], [7, 0, 12345678901, 3], [-5, 10 ** 18, 0]):
        s = io.StringIO()
        api.fileio.write_partition(np.array(vals, dtype=np.int64), s)
        assert s.getvalue() == O.format_labels(vals)
    s = io.BytesIO()
    api.fileio.write_partition(np.array([], dtype=np.int64), s)
    assert s.getvalue() == b"\n"
    api.fileio.write_partition(np.array([2.0, 1.9, 0.0]), str(tmp_path / "p"))
    assert (tmp_path / "p").read_text() == "2\n1\n0\n"


@pytest.mark.parametrize("n,weights", [(20000, "none"), (20000, "int"), (6000, "real")])
def test_larger_graphs_against_the_oracle(api, n, weights):
    from paper_1805_01208_b200.types import Partition

    n, off, nb, pts = G.random_geometric(n, seed=n + len(weights))
    rng = np.random.default_rng(3)
    vw = ew = None
    if weights == "int":
        vw = rng.integers(1, 9, n).astype(np.float64)
        half = rng.integers(1, 5, len(nb)).astype(np.float64)
    elif weights == "real":
        vw = rng.random(n) + 0.01
        half = rng.random(len(nb)) * 3 + 1e-7
    if weights != "none":  # symmetric edge weights: weight of (u, v) from min/max id
        src = np.repeat(np.arange(n), np.diff(off))
        lo, hi = np.minimum(src, nb), np.maximum(src, nb)
        key = lo * n + hi
        _, inv = np.unique(key, return_inverse=True)
        ew = half[:inv.max() + 1][inv]
    text = G.metis_text(n, off, nb, vw, ew)
    ctext = "".join("%.17g %.17g\n" % (x, y) for x, y in pts)
    g = api.fileio.load_metis_graph(io.StringIO(text), io.StringIO(ctext))
    assert G.same_bits(g.offsets, off) and G.same_bits(g.neighbors, nb)
    assert G.same_bits(g.coords, pts)
    assert G.same_bits(g.vertex_weights, np.ones(n) if vw is None else vw)
    if ew is not None:
        assert G.same_bits(g.edge_weights, ew)
    o_off, o_nb, o_vw, o_ew = O.parse_metis(text)
    assert G.same_bits(o_off, off) and G.same_bits(o_nb, nb)
    # metrics: stripes by x (connected blocks) and random labels (many components)
    k = 12
    stripes = np.minimum((pts[:, 0] * k).astype(np.int64), k - 1)
    for lab, kk in ((stripes, k), (rng.integers(0, 5, n), 6)):
        want = O.report(off, nb, o_vw, o_ew, lab, kk)
        rep = api.metrics.evaluate(g, Partition(assignment=lab, k=kk))
        for key in ("edge_cut", "comm_max", "comm_total", "imbalance", "harmonic_diameter"):
            assert getattr(rep, key) == want[key], (weights, kk, key)
        assert rep.block_weights == want["block_weights"]
        assert rep.block_comm == want["block_comm"]
        assert rep.block_diameters == want["block_diameters"]


def test_tokenizer_carries_across_chunk_and_tile_boundaries(api):
    """Comments, CRLF pairs and tokens placed across the tokenizer's 32-byte thread chunks
    and 8 KiB tiles (the comment carry, the '\\r' look-ahead and the token scan all cross
    them), against np.loadtxt on the same text."""
    import warnings

    rng = np.random.default_rng(13)
    TILE = 8192
    for trial in range(6):
        parts, size, rows = [], 0, 0
        while size < 5 * TILE + 1000:
            kind = rng.integers(0, 6)
            if kind == 0:      # a long comment, likely to straddle a boundary
                line = "#" + "c # 1 2 3 " * int(rng.integers(1, 200))
            elif kind == 1:    # blank line with blanks and tabs
                line = " \t" * int(rng.integers(0, 40))
            else:              # a data row, values of very different lengths
                a = rng.standard_normal() * 10.0 ** int(rng.integers(-30, 30))
                b = int(rng.integers(-10 ** 9, 10 ** 9))
                line = (" " * int(rng.integers(0, 30))) + ("%.17g" % a) + \
                    ("\t" * int(rng.integers(1, 4))) + str(b) + \
                    ("  # trailing " + "x" * int(rng.integers(0, 120)) if kind == 2 else "")
                rows += 1
            # pad so that interesting bytes land on tile / chunk boundaries now and then
            if rng.integers(0, 4) == 0 and kind != 1:
                room = (-(size + len(line)) - int(rng.integers(0, 3))) % 32
                line += " " * room
            eol = ("\r\n", "\n", "\r\n", "\n")[trial % 4] if trial < 4 else \
                ("\r\n" if rng.integers(0, 2) else "\n")
            parts.append(line + eol)
            size += len(parts[-1])
        text = "".join(parts)
        if trial % 2:
            text = text.rstrip("\r\n")   # no final newline
        with warnings.catch_warnings():
            warnings.simplefilter("ignore")
            # universal newlines, as a file opened by path
            want = np.loadtxt(io.StringIO(text.replace("\r\n", "\n")), dtype=np.float64, ndmin=2)
        got = api.fileio.load_coords(io.BytesIO(text.encode()))
        assert want.shape == (rows, 2) and G.same_bits(got, want), trial
    # a '\\r' as the last byte of a tile, its '\\n' the first byte of the next one
    body = "".join("%d %d\r\n" % (i, i * i) for i in range(3000))
    for shift in range(0, 12):
        text = " " * shift + body
        got = api.fileio.load_coords(io.BytesIO(text.encode()))
        assert got.shape == (3000, 2) and got[-1, 1] == 2999.0 ** 2 and got[17, 0] == 17.0
    g = api.fileio.load_metis_graph(io.BytesIO(("%% c\r\n3 2\r\n2\r\n1 3\r\n2" ).encode()))
    assert g.neighbors.tolist() == [1, 0, 2, 1]


def test_many_tokens_outside_the_plain_grammar(api):
    """Thousands of tokens the device leaves to Python / numpy (the batched host path) and
    long mantissas decided on the device: the arrays equal the oracle's."""
    n, off, nb, pts = G.random_geometric(5000, seed=4)
    rng = np.random.default_rng(9)
    vw = rng.integers(1, 9, n).astype(np.float64)
    lines = G.metis_text(n, off, nb, vw).split("\n")
    for u in range(n):   # every vertex weight as +d, d_0 or 1e0-style: all valid for float()
        t = lines[u + 1].split()
        w = int(vw[u])
        t[0] = (f"+{w}", f"{w}_0", f"{w}e0", f"{w}.000000000000000000000")[u % 4]
        if u % 7 == 0 and len(t) > 1:
            t[1] = "+" + t[1]     # int() accepts a sign
        lines[u + 1] = " ".join(t)
    text = "\n".join(lines)
    want = O.parse_metis(text)
    g = api.fileio.load_metis_graph(io.StringIO(text))
    assert G.same_bits(g.offsets, want[0]) and G.same_bits(g.neighbors, want[1])
    assert G.same_bits(g.vertex_weights, want[2])
    ctext = "".join("%.25g %.30e\n" % (x, y) if i % 3 else "%.17g nan\n" % x
                    for i, (x, y) in enumerate(pts))
    with pytest.raises(api.fileio.MetisParseError, match="non-finite coordinate"):
        api.fileio.load_coords(io.StringIO(ctext))
    ctext = ctext.replace("nan", "1e400").replace("1e400", "0x", 1)
    with pytest.raises(api.fileio.MetisParseError) as ei:
        api.fileio.load_coords(io.StringIO(ctext))
    with pytest.raises(O.ParseError) as eo:
        O.coords_of(ctext)
    assert str(ei.value) == str(eo.value)
    ctext = "".join("%.25g %.30e\n" % (x, y) for x, y in pts)
    assert G.same_bits(api.fileio.load_coords(io.StringIO(ctext)), O.coords_of(ctext))


def test_high_degree_vertices(api):
    """Hubs above the per-thread neighbor limit take the warp-per-vertex volume path."""
    from paper_1805_01208_b200.types import Partition

    n = 4000
    rng = np.random.default_rng(21)
    ring = np.stack([np.arange(n), (np.arange(n) + 1) % n], 1)
    hubs = []
    for h, deg in ((0, 3000), (7, 49), (8, 48), (1234, 700)):
        others = rng.choice(np.setdiff1d(np.arange(n), [h, (h - 1) % n, (h + 1) % n]), deg,
                            replace=False)
        hubs.append(np.stack([np.full(deg, h), others], 1))
    e = np.concatenate([ring] + hubs)
    e = np.unique(np.sort(e, axis=1), axis=0)
    _, off, nb = G.csr_from_edges(n, e)
    g = api.graph.GeometricGraph(off, nb, rng.random((n, 2)), np.ones(n))
    g.validate()
    for k in (3, 40, 500):
        lab = rng.integers(0, k, n)
        part = Partition(assignment=lab, k=k)
        cmax, ctot, per = api.metrics.comm_volumes(g, part)
        wmax, wtot, wper = O.comm_volumes(off, nb, lab, k)
        assert (cmax, ctot) == (wmax, wtot) and np.array_equal(per, wper), k
        assert api.metrics.edge_cut(g, part) == O.edge_cut(off, nb, None, lab)
        assert np.array_equal(api.metrics.block_diameter_lower_bounds(g, part),
                              O.diameters(off, nb, lab, k)), k
    text = G.metis_text(n, off, nb)
    back = api.fileio.load_metis_graph(io.StringIO(text))
    assert G.same_bits(back.neighbors, nb) and G.same_bits(back.offsets, off)


def test_injected_errors_match_the_oracle(api):
    n, off, nb, pts = G.random_geometric(30000, seed=11)
    base = G.metis_text(n, off, nb).split("\n")
    rng = np.random.default_rng(8)
    edits = {
        "junk token": lambda t: t + " 12x",
        "out of range": lambda t: t + f" {n + 5}",
        "self loop": None,
        "duplicate": lambda t: t + " " + t.split()[0] if t.split() else t + " 1 1",
        "float id": lambda t: t + " 7.5",
        "python int": lambda t: t.replace(t.split()[0], "+" + t.split()[0], 1) if t.split() else t,
    }
    for what, fn in edits.items():
        lines = list(base)
        for ln in sorted(rng.choice(np.arange(2, n), size=3, replace=False).tolist()):
            lines[ln] = (lines[ln] + f" {ln}") if fn is None else fn(lines[ln])
        text = "\n".join(lines)
        try:
            O.parse_metis(text)
            want = None
        except O.ParseError as e:
            want = str(e)
        if want is None:
            api.fileio.load_metis_graph(io.StringIO(text))
        else:
            with pytest.raises(api.fileio.MetisParseError) as ei:
                api.fileio.load_metis_graph(io.StringIO(text))
            assert str(ei.value) == want, what


def test_million_vertex_grid_properties(api):
    """3M vertices / 6M edges: parsed arrays equal the generator's; stripe partition has
    the analytic cut, volumes and diameters; written labels read back."""
    from paper_1805_01208_b200.types import Partition

    w, h, k = 2000, 1500, 8
    n, off, nb, pts = G.grid_graph(w, h)
    # vectorised METIS text (the test's own writer): every row is its sorted neighbors
    ids = (nb + 1).astype(str)
    deg = np.diff(off)
    sep = np.full(len(nb), " ", dtype="<U1")
    sep[off[1:] - 1] = "\n"
    body = "".join(np.char.add(ids, sep).tolist())
    text = f"% grid {w}x{h}\n{n} {len(nb) // 2}\n" + body
    g = api.fileio.load_metis_graph(io.BytesIO(text.encode()))
    assert G.same_bits(g.offsets, off) and G.same_bits(g.neighbors, nb)
    assert deg.min() == 2
    lab = (np.arange(n) % w) * k // w      # vertical stripes of width w/k
    part = Partition(assignment=lab, k=k)
    rep = api.metrics.evaluate(g, part)
    assert rep.edge_cut == (k - 1) * h
    assert rep.comm_total == 2 * (k - 1) * h and rep.comm_max == 2 * h
    assert rep.block_weights == [float(h * (w // k))] * k
    assert rep.block_diameters == [float(w // k - 1 + h - 1)] * k
    assert rep.imbalance == 0.0
    s = io.BytesIO()
    api.fileio.write_partition(part, s)
    back = api.fileio.read_partition(io.BytesIO(s.getvalue()), expect_n=n)
    assert G.same_bits(back.assignment, lab) and back.k == k


def test_graph_validate_messages(api):
    GG, GE = api.graph.GeometricGraph, api.graph.GraphError
    pts = np.zeros((3, 2))
    ok = GG([0, 1, 3, 4], [1, 0, 2, 1], pts, np.ones(3))
    ok.validate()
    cases = [
        (GG([0, 1, 3, 4], [1, 0, 3, 1], pts, np.ones(3)), "neighbor id out of range"),
        (GG([0, 1, 3, 4], [0, 0, 2, 1], pts, np.ones(3)), "self loop"),
        (GG([0, 2, 4, 4], [1, 1, 0, 0], pts, np.ones(3)), "parallel edge"),
        (GG([0, 1, 2, 3], [1, 2, 0], pts, np.ones(3)), "adjacency is not symmetric"),
        (GG([0, 3, 2, 4], [1, 0, 2, 1], pts, np.ones(3)), "CSR offsets not nondecreasing"),
        (GG([0, 1, 3, 4], [1, 0, 2, 1], pts, np.ones(3), [1, 1, 2, 3]),
         "edge weight differs between the two directions"),
        (GG([0, 1, 3, 4], [1, 0, 2, 1], pts, np.ones(3), [1, 1, -2, -2]),
         "edge weights must be strictly positive"),
        (GG([0, 1, 3, 4], [1, 0, 2, 1], pts, [1, 0, 1]), "vertex weights must be strictly positive"),
    ]
    for g, msg in cases:
        with pytest.raises(GE, match=msg):
            g.validate()
    g = GG.from_edges(4, [(0, 1), (2, 1), (3, 0)], np.zeros((4, 2)), edge_weights=[1, 2, 3])
    assert g.neighbors.tolist() == [1, 3, 0, 2, 1, 0] and g.edge_weights.tolist() == [1, 3, 1, 2, 2, 3]


def test_cli_partition_evaluate_compare(api, gold, tmp_path, capsys):
    from paper_1805_01208_b200 import cli
    from paper_1805_01208_b200.kmeans import KMeansSettings, balanced_kmeans

    rec = gold["graphs"]["rgg300_w"]
    gp, cp = tmp_path / "g.graph", tmp_path / "g.xyz"
    gp.write_text(rec["graph_text"])
    cp.write_text(rec["coords_text"])
    out, rp = tmp_path / "g.part", tmp_path / "r.json"
    rc = cli.main(["partition", "--graph", str(gp), "--coords", str(cp), "--k", "6", "--out",
                   str(out), "--report", str(rp), "--seed", "3"])
    line = capsys.readouterr().out
    g = api.fileio.load_metis_graph(str(gp), str(cp))
    want = balanced_kmeans(g, KMeansSettings(k=6, seed=3))
    got = api.fileio.read_partition(str(out), expect_n=g.n)
    assert np.array_equal(got.assignment, want.assignment)
    assert rc == (3 if want.balance_failed else 0)
    assert "algo=geographer k=6 n=300" in line
    rep = api.metrics.MetricsReport.from_json(rp.read_text())
    assert rep.edge_cut == api.metrics.edge_cut(g, want)
    assert cli.main(["evaluate", "--graph", str(gp), "--partition", str(out)]) == 0
    text = capsys.readouterr().out
    assert text.splitlines()[0] == "vertices: 300" and f"edge_cut: {int(rep.edge_cut)}" in text
    assert cli.main(["compare", "--graph", str(gp), "--coords", str(cp), "--k", "6",
                     "--report", str(tmp_path / "c.json")]) == 0
    table = json.loads((tmp_path / "c.json").read_text())
    assert table["ratios"]["geographer"]["edge_cut"] == pytest.approx(1.0)
    assert cli.main(["partition", "--graph", str(tmp_path / "nope"), "--coords", str(cp),
                     "--k", "2", "--out", str(out)]) == 2
    bad = tmp_path / "bad.graph"
    bad.write_text("3 2\n2\n1 4\n2\n")
    assert cli.main(["evaluate", "--graph", str(bad), "--partition", str(out)]) == 2
    assert "line 3: neighbor id 4 out of range 1..3" in capsys.readouterr().err
