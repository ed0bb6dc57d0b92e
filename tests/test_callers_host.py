"""CPU side of the path's callers: the oracle restatements of
sfc_labels and predict against golden vectors from the live reference, and the
estimators' host logic (parameters, input checks) — no device calls."""
import numpy as np
import pytest

import cases
import golden_io
from oracle import geographer_oracle as O


@pytest.fixture(scope="module")
def gold():
    return golden_io.load("callers")


def test_oracle_sfc_labels_match_reference_golden(gold):
    for name, (X, w, k, depth) in cases.sfc_cut_inputs().items():
        assert np.array_equal(O.sfc_labels(X, w, k, depth), gold[f"sfc/{name}"]), name


def test_oracle_predict_matches_reference_golden(gold):
    for name, (X, C, f) in cases.predict_inputs().items():
        assert np.array_equal(O.predict_labels(X, C, f), gold[f"predict/{name}"]), name


def test_oracle_predict_nan_semantics():
    rng = np.random.default_rng(1)
    X, C = rng.random((30, 2)), rng.random((5, 2))
    f = np.array([1.0, 1.0, np.nan, 1.0, np.nan])
    ref = np.argmin(np.linalg.norm(X[:, None, :] - C, axis=2) / f, axis=1)
    assert np.array_equal(O.predict_labels(X, C, f), ref)


def test_oracle_estimator_fixture_consistent(gold):
    # the fitted estimator's predict on its training data reproduces its labels (2D)
    rng = np.random.default_rng(0)
    cloud = rng.random((400, 2))
    got = O.predict_labels(cloud, gold["est/centers"], gold["est/influence"])
    assert np.array_equal(got, gold["est/labels"])


# ------------------------------------------------------- estimator host logic
@pytest.fixture(scope="module")
def est_mod():
    pytest.importorskip("sklearn")
    from paper_1805_01208_b200 import build

    build.build()
    from paper_1805_01208_b200 import estimators

    return estimators


def test_get_set_params_round_trip(est_mod):
    est = est_mod.GeographerPartitioner(k=7, epsilon=0.1, ranks=4)
    params = est.get_params()
    assert params["k"] == 7 and params["epsilon"] == 0.1 and params["ranks"] == 4
    assert est_mod.GeographerPartitioner().set_params(**params).get_params() == params


def test_clone_preserves_params(est_mod):
    from sklearn.base import clone

    est = est_mod.GeographerPartitioner(k=9, erosion=False, init_sample=0)
    assert clone(est).get_params() == est.get_params()
    assert clone(est_mod.SFCPartitioner(k=5)).get_params()["k"] == 5


def test_predict_before_fit_raises(est_mod):
    from sklearn.exceptions import NotFittedError

    with pytest.raises(NotFittedError):
        est_mod.GeographerPartitioner(k=3).predict(np.zeros((4, 2)))


@pytest.mark.parametrize("X,w,k,match", [
    (np.zeros((3,)), None, 2, "2-d coordinate"),
    (np.zeros((3, 5)), None, 2, "2- or 3-dimensional"),
    (np.array([[np.nan, 0.0], [0.0, 0.0]]), None, 2, "finite"),
    (np.zeros((4, 2)), np.array([1.0, -1.0, 1.0, 1.0]), 2, "strictly positive"),
    (np.zeros((4, 2)), np.ones(3), 2, "shape"),
    (np.zeros((4, 2)), None, 10, "1 <= k <= 4"),
    (np.zeros((0, 2)), None, 1, "at least one point"),
])
def test_rejects_bad_inputs_before_any_device_work(est_mod, X, w, k, match):
    for cls in (est_mod.GeographerPartitioner, est_mod.SFCPartitioner):
        with pytest.raises(ValueError, match=match):
            cls(k=k).fit(X, sample_weight=w)
