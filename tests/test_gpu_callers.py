"""Parity of the path's callers on the device: the SFC baseline
(gp_sfc_cut after the K1/K2/K3 bootstrap kernels) and GeographerPartitioner
(fit through the partition path, predict through gp_predict).  Bit-exact
against golden vectors from the live reference, against the oracle on this
host, and through size-independent properties at full sizes.  Mirrors the
reference's tests/test_estimators.py and tests/test_baselines.py::TestSfc."""
import numpy as np
import pytest

import cases
import golden_io
from conftest import has_cuda

pytestmark = pytest.mark.gpu

if has_cuda():
    import torch

    from paper_1805_01208_b200 import hilbert_keys, BoundingBox
    from paper_1805_01208_b200.baselines import sfc_labels, sfc_labels_device, sfc_partition
    from paper_1805_01208_b200.estimators import (
        GeographerPartitioner, SFCPartitioner, predict_blocks,
    )


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_cuda():
        pytest.fail("CUDA device required for -m gpu tests")


@pytest.fixture(scope="module")
def gold():
    return golden_io.load("callers")


def _oracle():
    from oracle import geographer_oracle as O

    return O


# ------------------------------------------------------------------ SFC cut
def test_sfc_labels_match_reference_golden(gold):
    for name, (X, w, k, depth) in cases.sfc_cut_inputs().items():
        assert np.array_equal(sfc_labels(X, w, k, depth), gold[f"sfc/{name}"]), name


@pytest.mark.parametrize("wkind", ["unit", "int", "f32", "f64", "tiny"])
@pytest.mark.parametrize("d", [2, 3])
def test_sfc_labels_match_oracle(wkind, d):
    O = _oracle()
    rng = np.random.default_rng(["unit", "int", "f32", "f64", "tiny"].index(wkind) * 10 + d)
    n = 150_000
    X = rng.random((n, d))
    w = {"unit": np.ones(n), "int": rng.integers(1, 1000, n).astype(float),
         "f32": rng.uniform(1, 4, n).astype(np.float32).astype(float),
         "f64": rng.random(n) + 0.5, "tiny": rng.random(n) * 1e-30}[wkind]
    for k in (1, 3, 97, 4096):
        assert np.array_equal(sfc_labels(X, w, k), O.sfc_labels(X, w, k)), (wkind, d, k)


def test_sfc_blocks_are_contiguous_ranges_of_curve_order():
    rng = np.random.default_rng(4)
    X, w = rng.random((5000, 2)), rng.integers(1, 9, 5000).astype(float)
    labels = sfc_labels(X, w, 5)
    keys = hilbert_keys(X, BoundingBox.of_points(X))
    along = labels[np.lexsort((np.arange(5000), keys))]
    assert (np.diff(along) >= 0).all()


def test_sfc_unit_weights_divisible_gives_equal_runs():
    pts = np.random.default_rng(5).random((120, 2))
    assert np.array_equal(np.bincount(sfc_labels(pts, np.ones(120), 6), minlength=6),
                          np.full(6, 20))


def test_sfc_k_equals_n_and_rejects_bad_k():
    pts = np.random.default_rng(6).random((7, 2))
    assert sorted(sfc_labels(pts, np.ones(7), 7)) == list(range(7))
    with pytest.raises(ValueError):
        sfc_labels(pts, np.ones(7), 8)
    with pytest.raises(ValueError):
        sfc_labels(pts, np.ones(7), 0)


def test_sfc_partition_wrapper_flags_imbalance():
    class G:
        pass

    g = G()
    g.coords = np.random.default_rng(7).random((1000, 3))
    g.vertex_weights = np.ones(1000)
    p = sfc_partition(g, 3, epsilon=0.03)
    assert np.bincount(p.assignment, minlength=3).sum() == 1000
    assert not p.balance_failed and p.empty_blocks.size == 0


def test_sfc_full_size_properties():
    # 2^24 3D points, unit weights: equal runs along the curve when k | n
    n, k = 1 << 24, 1024
    g = torch.Generator(device="cuda").manual_seed(0)
    X = torch.rand((n, 3), dtype=torch.float64, device="cuda", generator=g)
    lab = sfc_labels_device(X, None, k)
    counts = torch.bincount(lab, minlength=k)
    assert int(counts.min()) == n // k and int(counts.max()) == n // k
    # integer weights: every cut is where the exact prefix crosses j*total/k
    w = torch.randint(1, 61, (n,), device="cuda", dtype=torch.int64).to(torch.float64)
    lab = sfc_labels_device(X, w, k)
    bw = torch.zeros(k, dtype=torch.float64, device="cuda").index_add_(0, lab, w)
    total = float(w.sum())
    assert abs(float(bw.sum()) - total) == 0.0
    assert float(bw.max()) <= total / k + 60.0


# ------------------------------------------------------------------ predict
def test_predict_matches_reference_golden(gold):
    for name, (X, C, f) in cases.predict_inputs().items():
        assert np.array_equal(predict_blocks(X, C, f), gold[f"predict/{name}"]), name


@pytest.mark.parametrize("d,k", [(2, 16), (2, 1024), (3, 256), (3, 4096)])
def test_predict_matches_oracle(d, k):
    O = _oracle()
    rng = np.random.default_rng(d * 10007 + k)
    X = rng.random((20_000, d))
    C = rng.random((k, d))
    f = rng.uniform(0.8, 1.25, k)
    assert np.array_equal(predict_blocks(X, C, f), O.predict_labels(X, C, f))


def test_predict_non_finite_and_extreme_influence():
    O = _oracle()
    rng = np.random.default_rng(9)
    X, C = rng.random((2000, 2)), rng.random((7, 2))
    for f in (np.array([1, np.nan, 1, 1, np.nan, 1, 1.0]), np.array([1e-200, 1, 1, 1, 1, 1, 1e200]),
              np.array([np.inf, 1, 1, 1, 1, 1, 1.0]), np.array([0.0, 1, 1, 1, 1, 1, 1.0])):
        with np.errstate(all="ignore"):
            ref = np.argmin(np.linalg.norm(X[:, None, :] - C, axis=2) / f, axis=1)
        assert np.array_equal(predict_blocks(X, C, f), ref)
        assert np.array_equal(O.predict_labels(X, C, f), ref)


# ---------------------------------------------------------------- estimators
@pytest.fixture(scope="module")
def cloud():
    return np.random.default_rng(0).random((400, 2))


def test_estimator_matches_reference_golden(gold, cloud):
    est = GeographerPartitioner(k=6).fit(cloud)
    assert np.array_equal(est.labels_, gold["est/labels"])
    assert np.array_equal(est.cluster_centers_, gold["est/centers"])
    assert np.array_equal(est.influence_, gold["est/influence"])
    assert est.n_iter_ == int(gold["est/n_iter"][0])
    new = np.random.default_rng(2).random((300, 2))
    assert np.array_equal(est.predict(new), gold["est/predict_new"])


def test_fit_sets_attributes(cloud):
    est = GeographerPartitioner(k=5).fit(cloud)
    assert est.labels_.shape == (400,)
    assert est.cluster_centers_.shape == (5, 2) and est.influence_.shape == (5,)
    assert est.imbalance_ <= 0.03 and not est.balance_failed_ and est.n_iter_ >= 1


def test_fit_predict_and_predict_reproduce_labels(cloud):
    est = GeographerPartitioner(k=4, random_state=1)
    assert np.array_equal(est.fit_predict(cloud), est.labels_)
    est = GeographerPartitioner(k=6).fit(cloud)
    assert np.array_equal(est.predict(cloud), est.labels_)
    out = GeographerPartitioner(k=3).fit(cloud).predict(np.random.default_rng(2).random((50, 2)))
    assert out.min() >= 0 and out.max() < 3


def test_predict_dimension_mismatch(cloud):
    est = GeographerPartitioner(k=3).fit(cloud)
    with pytest.raises(ValueError, match="dimension"):
        est.predict(np.random.default_rng(3).random((5, 3)))


def test_sample_weight_and_ranks(cloud):
    w = np.random.default_rng(4).integers(1, 4, size=400).astype(float)
    est = GeographerPartitioner(k=4, epsilon=0.05).fit(cloud, sample_weight=w)
    bw = np.bincount(est.labels_, weights=w, minlength=4)
    assert bw.max() / np.ceil(bw.sum() / 4) - 1 <= 0.05 + 1e-12
    a = GeographerPartitioner(k=5, ranks=1).fit(cloud)
    b = GeographerPartitioner(k=5, ranks=4).fit(cloud)
    assert np.array_equal(a.labels_, b.labels_)


def test_3d_points():
    pts = np.random.default_rng(5).random((200, 3))
    est = GeographerPartitioner(k=4).fit(pts)
    assert est.cluster_centers_.shape == (4, 3)
    O = _oracle()
    assert np.array_equal(est.predict(pts), O.predict_labels(pts, est.cluster_centers_,
                                                             est.influence_))


def test_sfc_partitioner(cloud):
    est = SFCPartitioner(k=8).fit(cloud)
    assert est.labels_.shape == (400,) and est.imbalance_ <= 0.03
    assert SFCPartitioner(k=4, sfc_depth=10).fit(cloud).labels_.max() < 4
