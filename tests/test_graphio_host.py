"""Host-side logic of the formats / metrics modules (no GPU): header and vertex-line
arbitration (fileio._header, _vertex_line) against the golden messages, the report
type's text / JSON round trip, the CLI parser, and the shim's name swapping."""
import math
import os
import sys

import pytest

import graphio_cases as G
from paper_1805_01208_b200 import cli, fileio, metrics

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_header_messages_equal_the_reference():
    gold = G.golden()["bad_graphs"]
    for name in ("header_one_field", "header_five_fields", "header_nonnumeric",
                 "header_bad_sizes", "header_fmt_alpha", "header_vsize", "header_ncon2",
                 "header_ncon_alpha"):
        head = gold[name]["graph_text"].splitlines()[0]
        with pytest.raises(fileio.MetisParseError) as ei:
            fileio._header(head, 1)
        assert str(ei.value) == gold[name]["message"], name
    assert fileio._header("7 9 011 1", 3) == (7, 9, True, True)
    assert fileio._header("7 9 1", 3) == (7, 9, False, True)
    assert fileio._header("7 9", 3) == (7, 9, False, False)


def test_vertex_line_messages_equal_the_reference():
    gold = G.golden()["bad_graphs"]
    for name in ("missing_vweight", "bad_vweight", "zero_vweight", "inf_vweight", "dangling",
                 "nonnumeric_id", "float_id", "out_of_range", "negative_id", "self_loop",
                 "duplicate", "bad_eweight", "neg_eweight"):
        msg = gold[name]["message"]
        lines = gold[name]["graph_text"].splitlines()
        n, m, vw, ew = fileio._header(lines[0], 1)
        no = int(msg.split(":")[0].split()[1])
        with pytest.raises(fileio.MetisParseError) as ei:
            fileio._vertex_line(lines[no - 1], no, no - 2, n, vw, ew)
        assert str(ei.value) == msg, name
    # tokens only Python accepts are values, not errors
    assert fileio._vertex_line("1_0 +1 3", 5, 1, 12, True, False) == (10.0, [0, 2], None)
    assert fileio._vertex_line("2 1e0 3 .5", 2, 0, 3, False, True) == (1.0, [1, 2], [1.0, 0.5])


def test_report_round_trip_and_text():
    r = metrics.MetricsReport(n=4, m=3, k=2, edge_cut=1.0, comm_max=1.0, comm_total=2.0,
                              imbalance=0.5, harmonic_diameter=math.inf,
                              block_weights=[3.0, 1.5], block_comm=[1.0, 1.0],
                              block_diameters=[math.inf, 2.0])
    back = metrics.MetricsReport.from_json(r.to_json())
    assert back == r
    text = r.to_text().splitlines()
    assert text[:4] == ["vertices: 4", "edges: 3", "blocks: 2", "edge_cut: 1"]
    assert text[6] == "imbalance: 0.5" and text[7] == "harmonic_diameter: unbounded"
    assert text[8] == "block 0: weight 3 comm 1 diameter unbounded"
    assert text[9] == "block 1: weight 1.5 comm 1 diameter 2"
    assert metrics.harmonic_mean_diameters([2.0, math.inf]) == 4.0
    assert metrics.harmonic_mean_diameters([math.inf]) == math.inf
    assert metrics.geometric_mean([1.0, 4.0]) == pytest.approx(2.0)
    with pytest.raises(ValueError):
        metrics.geometric_mean([1.0, 0.0])


def test_cli_parser_and_argument_errors(capsys):
    p = cli.build_parser()
    a = p.parse_args(["partition", "--graph", "g", "--coords", "c", "--k", "4", "--out", "o"])
    assert (a.algo, a.epsilon, a.seed, a.p, a.max_iter, a.max_balance_iter, a.init_sample) == \
        ("geographer", 0.03, 0, 1, 50, 20, 100)
    assert not a.no_erosion and a.sfc_depth is None and a.report is None
    with pytest.raises(SystemExit):
        p.parse_args(["partition", "--graph", "g", "--coords", "c", "--k", "4", "--out", "o",
                      "--algo", "rcb"])
    # argument errors of compare are reported like the reference's (exit code 2)
    assert cli.main(["compare", "--graph", "a", "--graph", "b", "--coords", "c", "--k", "2"]) == 2
    assert "each --graph needs a matching --coords" in capsys.readouterr().err
    assert cli.main(["compare", "--graph", "a", "--coords", "c", "--k", "2", "--algos", "sfc"]) == 2
    assert "geographer" in capsys.readouterr().err


def test_install_formats_swaps_the_reference_names():
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "geopart")):
        pytest.skip("baseline/_ref missing (made by build())")
    sys.path.insert(0, ref)
    try:
        import geopart.cli as rc
        import geopart.fileio as rf
        import geopart.graph as rg
        import geopart.metrics as rm

        from paper_1805_01208_b200 import integration

        keep = {m: dict(vars(m)) for m in (rc, rf, rm)}
        keep_validate = rg.GeometricGraph.validate
        calls = {}
        old = integration.install_formats(counter=calls)
        try:
            assert rf.load_metis_graph.__wrapped__ is fileio.load_metis_graph
            assert rc.load_metis_graph is rf.load_metis_graph      # names bound at import
            assert rm.evaluate.__wrapped__ is metrics.evaluate and rc.evaluate is rm.evaluate
            assert old["fileio.read_partition"] is keep[rf]["read_partition"]
            assert rg.GeometricGraph.validate is not keep_validate
            # this package's errors surface as the reference's classes
            import io

            with pytest.raises(rf.MetisParseError, match="line 1: missing header"):
                rf.load_metis_graph(io.StringIO(""))
            assert calls["load_metis_graph"] == 1
        finally:
            for m, d in keep.items():
                for k, v in d.items():
                    setattr(m, k, v)
            rg.GeometricGraph.validate = keep_validate
    finally:
        sys.path.remove(ref)
        for name in [m for m in sys.modules if m.split(".")[0] == "geopart"]:
            del sys.modules[name]
