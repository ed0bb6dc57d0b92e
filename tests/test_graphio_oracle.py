"""CPU tests of the formats / metrics row: the oracle
(oracle/graphio_oracle.py) against the golden vectors made from the live reference, and
the tokenizer's decimal -> binary64 conversion (host build of the kernel's code) against
Python's float()."""
import ctypes
import random
import struct

import numpy as np
import pytest

import graphio_cases as G
from oracle import graphio_oracle as O


@pytest.fixture(scope="module")
def gold():
    return G.golden()


def _check_graph_arrays(got, want):
    off, nb, vw, ew = got
    assert G.same_bits(off, G.arr(want["offsets"]))
    assert G.same_bits(nb, G.arr(want["neighbors"]))
    assert G.same_bits(vw, G.arr(want["vertex_weights"]))
    w = G.arr(want["edge_weights"])
    assert (ew is None) == (w is None)
    if w is not None:
        assert G.same_bits(ew, w)


def test_oracle_parses_reference_written_graphs(gold):
    for name, rec in gold["graphs"].items():
        _check_graph_arrays(O.parse_metis(rec["graph_text"]), rec["arrays"])
        c = O.coords_of(rec["coords_text"], expect_n=len(G.arr(rec["arrays"]["offsets"])) - 1)
        assert G.same_bits(c, G.arr(rec["arrays"]["coords"])), name


def test_oracle_reader_corner_cases(gold):
    for name, rec in gold["good_graphs"].items():
        _check_graph_arrays(O.parse_metis(rec["graph_text"]), rec["arrays"])
        if rec["coords_text"] is not None:
            assert G.same_bits(O.coords_of(rec["coords_text"]), G.arr(rec["arrays"]["coords"]))


def test_oracle_error_messages(gold):
    for name, rec in gold["bad_graphs"].items():
        with pytest.raises(O.ParseError) as ei:
            off, *_ = O.parse_metis(rec["graph_text"])
            if rec["coords_text"] is not None:
                O.coords_of(rec["coords_text"], expect_n=len(off) - 1)
        assert str(ei.value) == rec["message"], name


def test_oracle_tables(gold):
    for name, rec in gold["tables"].items():
        fn = O.coords_of if rec["kind"] == "coords" else O.labels_of
        if "error" in rec:
            with pytest.raises(O.ParseError) as ei:
                fn(rec["text"], **rec["kwargs"])
            assert str(ei.value) == rec["message"], name
        elif rec["kind"] == "coords":
            assert G.same_bits(fn(rec["text"], **rec["kwargs"]), G.arr(rec["ok"])), name
        else:
            a, k = fn(rec["text"], **rec["kwargs"])
            assert G.same_bits(a, G.arr(rec["ok"]["labels"])) and k == rec["ok"]["k"], name


def test_oracle_metrics_and_writer(gold):
    for name, rec in gold["graphs"].items():
        off, nb, vw, ew = O.parse_metis(rec["graph_text"])
        for pname, p in rec["partitions"].items():
            lab = np.array(p["labels"], dtype=np.int64)
            got = O.report(off, nb, vw, ew, lab, p["k"])
            want = p["report"]
            un = lambda x: float("inf") if x == "unbounded" else float(x)  # noqa: E731
            for key in ("edge_cut", "comm_max", "comm_total", "imbalance"):
                assert got[key] == want[key], (name, pname, key)
            assert got["harmonic_diameter"] == un(want["harmonic_diameter"]), (name, pname)
            assert got["block_weights"] == want["block_weights"], (name, pname)
            assert got["block_comm"] == want["block_comm"], (name, pname)
            assert got["block_diameters"] == [un(x) for x in want["block_diameters"]], (name, pname)
            assert O.format_labels(lab) == p["text"]


@pytest.fixture(scope="module")
def parse_number():
    from paper_1805_01208_b200 import build

    build.build()
    from paper_1805_01208_b200 import _native as N

    def parse(s):
        v = ctypes.c_int64(0)
        b = s.encode()
        return N.lib.gp_parse_number_host(b, len(b), ctypes.byref(v)), v.value

    return parse


def test_decimal_conversion_matches_python_float(parse_number):
    """The kernel's Eisel-Lemire conversion (compiled for the host): every token it
    accepts as REAL has exactly float()'s bits; INT tokens equal int()."""
    rng = random.Random(5)
    checked = suspects = 0

    def check(s):
        nonlocal checked, suspects
        kind, v = parse_number(s)
        checked += 1
        if kind == 3:
            suspects += 1
        elif kind == 0:
            assert int(s) == v, s
        else:
            assert kind == 1 and struct.pack("<d", float(s)) == struct.pack("<q", v), s

    for i in range(60000):
        x = struct.unpack("<d", struct.pack("<Q", rng.getrandbits(64)))[0]
        if x != x or x in (float("inf"), float("-inf")):
            continue
        for s in (repr(x), "%.17g" % x, "%.15g" % x, "%.10e" % x, "%.25g" % x, "%.40e" % x):
            check(s)
    for i in range(60000):
        nd = rng.randint(1, 19)
        m = rng.randint(0, 10 ** nd - 1)
        check(f"{m}e{rng.randint(-345, 310)}")
        sm, pos = str(m).zfill(nd), rng.randint(0, nd)
        check(sm[:pos] + "." + sm[pos:] + (f"E{rng.randint(-30, 30):+d}" if i % 2 else ""))
    for e in range(40):  # ties: odd multiples of a half ulp
        for m in (2 ** 53 + 1, 2 ** 53 + 3, 2 ** 54 + 2, 2 ** 54 + 6):
            check(f"{m}e{e - 20}")
            check(f"{m}.0")
    for s in ("4.9e-324", "2.4703282292062327e-324", "2.4703282292062328e-324",
              "2.2250738585072011e-308", "2.2250738585072014e-308", "1.7976931348623157e308",
              "1.7976931348623159e308", "1e-400", "1e400", "-0.0", ".5", "5.", "+.5e+1", "00012"):
        check(s)
    for s in ("12345678901234567890", "1234567890123456789", "0.10000000000000000555",
              "9007199254740993.00000000000000000001", "123456789012345678901234567890",
              "9007199254740992.99999999999999999999"):
        check(s)
        assert parse_number(s)[0] in (1, 3), s    # never an int64 beyond 18 digits
    assert parse_number("123456789012345678901234567890")[0] == 1
    assert suspects < checked // 50   # long mantissas are decided by bracketing (w, w + 1)
    for s in ("nan", "inf", "1_0", ".", "-", "1e", "1e+", "e5", "1.2.3", "0x10", "1,2"):
        assert parse_number(s)[0] == 3, s
    assert parse_number("%abc")[0] == 2
