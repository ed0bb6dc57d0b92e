"""scikit-learn estimators over the B200 partition path (reference
estimators.py:23-142).

* GeographerPartitioner.fit runs balanced_kmeans_points on the device;
  predict is the brute-force n x k argmin kernel gp_predict, bit-identical to
  argmin(linalg.norm(X[:, None] - centers, axis=2) / influence, axis=1).
* SFCPartitioner.fit runs the device SFC cut (baselines.sfc_labels).

Parameters, fitted attributes, input checks (reference validation.py:10-41)
and error types/messages are the reference's.  RCBPartitioner is not part of
this build.
"""

from __future__ import annotations

import numpy as np
import torch
from sklearn.base import BaseEstimator, ClusterMixin
from sklearn.utils.validation import check_is_fitted

from . import _native as N
from .baselines import sfc_labels
from .control import imbalance
from .kmeans import balanced_kmeans_points
from .types import KMeansSettings

__all__ = ["GeographerPartitioner", "SFCPartitioner", "predict_blocks"]


# ------------------------------------------------ input checks (validation.py)
def _coords(X) -> np.ndarray:
    X = np.asarray(X, dtype=np.float64)
    if X.ndim != 2:
        raise ValueError(f"expected a 2-d coordinate array, got shape {X.shape}")
    n, d = X.shape
    problem = ("need at least one point" if n < 1 else
               f"only 2- or 3-dimensional points are supported, got d={d}" if d not in (2, 3)
               else "coordinates must be finite" if not np.isfinite(X).all() else None)
    if problem:
        raise ValueError(problem)
    return X


def _sample_weight(sample_weight, n: int) -> np.ndarray:
    if sample_weight is None:
        return np.ones(n, dtype=np.float64)
    w = np.asarray(sample_weight, dtype=np.float64)
    if w.shape != (n,):
        raise ValueError(f"sample_weight must have shape ({n},), got {w.shape}")
    if not (np.isfinite(w).all() and (w > 0).all()):
        raise ValueError("sample weights must be finite and strictly positive")
    return w


def _block_count(k, n: int) -> int:
    k = int(k)
    if k < 1 or k > n:
        raise ValueError(f"k must satisfy 1 <= k <= {n}, got {k}")
    return k


# ------------------------------------------------ predict kernel wrapper
def predict_blocks(X, centers, influence, device=None) -> np.ndarray:
    """argmin_c norm(X - centers[c]) / influence[c] per row, on the device
    (gp_predict); int64 like numpy's argmin."""
    dev = torch.device(device if device is not None else "cuda")
    X = np.ascontiguousarray(X, dtype=np.float64)
    C = np.ascontiguousarray(centers, dtype=np.float64)
    f = np.ascontiguousarray(influence, dtype=np.float64)
    n, d = X.shape
    k = C.shape[0]
    with np.errstate(all="ignore"):
        safe = bool(np.isfinite(f).all() and (f >= 1e-150).all() and (f <= 1e150).all())
    Xd = torch.from_numpy(X).to(dev)
    Cd = torch.from_numpy(C).to(dev)
    fd = torch.from_numpy(f).to(dev)
    out = torch.empty(n, dtype=torch.int64, device=dev)
    N.call("gp_predict", Xd.data_ptr(), n, d, Cd.data_ptr(), fd.data_ptr(), k, int(safe),
           out.data_ptr(), torch.cuda.current_stream(dev).cuda_stream)
    return out.cpu().numpy()


class GeographerPartitioner(ClusterMixin, BaseEstimator):
    """Balanced k-means with influence weights, bootstrapped from a Hilbert
    curve (estimators.py:23-114).  See the reference for the parameters;
    ``ranks`` is accepted and, as in the reference, does not change results."""

    def __init__(self, k=8, epsilon=0.03, max_iter=50, max_balance_iter=20,
                 influence_step_cap=0.05, delta_threshold=None, erosion=True, init_sample=100,
                 ranks=1, random_state=0, sfc_depth=None, audit_bounds=False):
        self.k = k
        self.epsilon = epsilon
        self.max_iter = max_iter
        self.max_balance_iter = max_balance_iter
        self.influence_step_cap = influence_step_cap
        self.delta_threshold = delta_threshold
        self.erosion = erosion
        self.init_sample = init_sample
        self.ranks = ranks
        self.random_state = random_state
        self.sfc_depth = sfc_depth
        self.audit_bounds = audit_bounds

    def _settings(self, k: int) -> KMeansSettings:
        return KMeansSettings(
            k=k, epsilon=self.epsilon, max_iter=self.max_iter,
            max_balance_iter=self.max_balance_iter,
            influence_step_cap=self.influence_step_cap, delta_threshold=self.delta_threshold,
            erosion=self.erosion, init_sample=self.init_sample, seed=self.random_state,
            sfc_depth=self.sfc_depth, audit_bounds=self.audit_bounds)

    def fit(self, X, y=None, sample_weight=None):
        X = _coords(X)
        w = _sample_weight(sample_weight, X.shape[0])
        settings = self._settings(_block_count(self.k, X.shape[0]))
        part, stats = balanced_kmeans_points(X, w, settings, p=self.ranks, return_stats=True)
        fs = stats.final_state
        self.labels_ = part.assignment
        self.cluster_centers_ = fs.centers
        self.influence_ = fs.influence
        self.imbalance_ = imbalance(fs.block_weights)
        self.balance_failed_ = part.balance_failed
        self.n_iter_ = len(stats.iterations)
        self.stats_ = stats
        return self

    def predict(self, X):
        """Blocks of new points under the fitted centers and influences."""
        check_is_fitted(self, "cluster_centers_")
        X = _coords(X)
        if X.shape[1] != self.cluster_centers_.shape[1]:
            raise ValueError("dimension differs from the fitted data")
        return predict_blocks(X, self.cluster_centers_, self.influence_)


class SFCPartitioner(ClusterMixin, BaseEstimator):
    """Greedy cuts along the Hilbert curve order (estimators.py:129-142)."""

    def __init__(self, k=8, sfc_depth=None):
        self.k = k
        self.sfc_depth = sfc_depth

    def fit(self, X, y=None, sample_weight=None):
        X = _coords(X)
        w = _sample_weight(sample_weight, X.shape[0])
        k = _block_count(self.k, X.shape[0])
        self.labels_ = sfc_labels(X, w, k, self.sfc_depth)
        self.imbalance_ = imbalance(np.bincount(self.labels_, weights=w, minlength=k))
        return self
