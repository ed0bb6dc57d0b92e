"""Golden fixtures for the path's callers from the LIVE reference (dev container):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden_callers.py

sfc_labels (baselines.py:62-89) and GeographerPartitioner.predict's arithmetic
(estimators.py:107-114) on the seeded inputs of cases.sfc_cut_inputs /
cases.predict_inputs, plus one fitted estimator (labels, centers, influence and
predict on new points).  Outputs: tests/golden/callers.npz.
"""

from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, HERE)
sys.path.insert(0, "/root/reference/pkg/src")

import cases  # noqa: E402
from geopart.baselines import sfc_labels  # noqa: E402
from geopart.estimators import GeographerPartitioner  # noqa: E402


def main():
    out = {}
    for name, (X, w, k, depth) in cases.sfc_cut_inputs().items():
        out[f"sfc/{name}"] = sfc_labels(X, w, k, depth)
    for name, (X, C, f) in cases.predict_inputs().items():
        dist = np.linalg.norm(X[:, None, :] - C, axis=2)
        out[f"predict/{name}"] = np.argmin(dist / f, axis=1)
    rng = np.random.default_rng(0)
    cloud = rng.random((400, 2))
    est = GeographerPartitioner(k=6).fit(cloud)
    new = np.random.default_rng(2).random((300, 2))
    out["est/labels"] = est.labels_
    out["est/centers"] = est.cluster_centers_
    out["est/influence"] = est.influence_
    out["est/predict_new"] = est.predict(new)
    out["est/n_iter"] = np.array([est.n_iter_])
    np.savez_compressed(os.path.join(HERE, "callers.npz"), **out)
    print(len(out), "arrays")


if __name__ == "__main__":
    main()
