"""Pin the CPU oracle against golden vectors produced by the live reference.

Fixtures: tests/golden/make_golden.py (reference run in the dev container).
"""
import numpy as np
import pytest

import cases
import golden_io
from oracle import geographer_oracle as O


def test_keys_match_reference_golden():
    gold = golden_io.load("keys")
    for name, (pts, lo, hi, depth) in cases.key_inputs().items():
        got = O.hilbert_keys(pts, lo, hi, depth)
        assert got.dtype == np.uint64
        assert np.array_equal(got, gold[name]), name


@pytest.mark.parametrize("name", ["C1", "C2", "C3"])
def test_sfc_stage_matches_reference_golden(name):
    spec = next(s for s in cases.SFC_CASES if s["name"] == name)
    gold = golden_io.load("sfc_" + name)
    pts, _ = cases.partition_inputs(spec)
    d = pts.shape[1]
    keys = O.hilbert_keys(pts, pts.min(axis=0), pts.max(axis=0), O.DEFAULT_DEPTH[d])
    order = O.sfc_order(keys)
    assert np.array_equal(golden_io.sha(keys, "<u8"), gold["keys_sha256"])
    assert np.array_equal(golden_io.sha(order, "<i4"), gold["order_sha256"])
    pos = O.center_positions(pts.shape[0], spec["settings"]["k"])
    assert np.array_equal(pts[order][pos], gold["init_centers"])


def _cases(skip_big=True):
    return [c["name"] for c in cases.PARTITION_CASES if not (skip_big and c["name"] == "C1")]


@pytest.mark.parametrize("name", _cases(skip_big=False))
def test_partition_matches_reference_golden(name):
    if not golden_io.host_matches_golden_numerics():
        pytest.skip("host numpy pow/exp/einsum bits differ from the fixture host")
    spec = next(c for c in cases.PARTITION_CASES if c["name"] == name)
    pts, w = cases.partition_inputs(spec)
    s = dict(spec["settings"])
    s.pop("audit_bounds", None)
    res = O.run(pts, w, O.Knobs(**s))
    gold = golden_io.load("part_" + name)
    meta = golden_io.index()["partitions"][name]
    assert np.array_equal(res.assignment, gold["assignment"])
    assert np.array_equal(res.centers, gold["centers"])
    assert np.array_equal(res.influence, gold["influence"])
    assert np.array_equal(res.block_weights, gold["block_weights"])
    assert np.array_equal(res.empty_blocks, gold["empty_blocks"])
    assert res.balance_failed == meta["balance_failed"]
    assert res.converged == meta["converged"]
    assert res.records == meta["records"]


@pytest.mark.parametrize("dim,depth", [(2, d) for d in range(1, 9)] + [(3, d) for d in range(1, 5)])
def test_oracle_hilbert_bijective_adjacent(dim, depth):
    side = 1 << depth
    axes = np.meshgrid(*([np.arange(side, dtype=np.uint64)] * dim), indexing="ij")
    cells = np.stack([a.ravel() for a in axes], axis=1)
    keys = O.hilbert_from_cells(cells, depth)
    order = np.argsort(keys, kind="stable")
    assert np.array_equal(keys[order], np.arange(len(cells), dtype=np.uint64))
    steps = np.abs(np.diff(cells[order].astype(np.int64), axis=0)).sum(axis=1)
    assert np.all(steps == 1)


def test_sample_ranks_is_inverse_permutation():
    r = O.sample_ranks(1000, 3)
    perm = np.random.default_rng(3).permutation(1000)
    assert np.array_equal(r[perm], np.arange(1000))
