"""Public value types of the drop-in boundary.

Same names, fields, defaults and validation as the reference so that callers
(and the reference's own tests) can switch packages without edits:
  KMeansSettings  kmeans.py:65-101     ClusterState   kmeans.py:104-129
  PointBounds     kmeans.py:132-147    BalanceInfo    kmeans.py:242-252
  IterationRecord kmeans.py:255-265    KMeansStats    kmeans.py:268-285
  Partition       graph.py:131-166     BoundingBox    geometry.py:51-86
  GeometryError   geometry.py:35-36    GraphError     graph.py
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


class GeometryError(ValueError):
    """Malformed geometric input (unsupported dimension, depth, non-finite box)."""


class GraphError(ValueError):
    """Malformed graph or partition."""


@dataclass(frozen=True)
class BoundingBox:
    lo: np.ndarray
    hi: np.ndarray

    def __post_init__(self):
        lo = np.asarray(self.lo, dtype=np.float64)
        hi = np.asarray(self.hi, dtype=np.float64)
        object.__setattr__(self, "lo", lo)
        object.__setattr__(self, "hi", hi)
        if lo.ndim != 1 or lo.shape != hi.shape:
            raise GeometryError("box corners must be 1-d arrays of equal length")
        if not (np.isfinite(lo).all() and np.isfinite(hi).all()):
            raise GeometryError("non-finite box corner")
        if (lo > hi).any():
            raise GeometryError("box lower corner exceeds upper corner")

    @property
    def dim(self) -> int:
        return int(self.lo.shape[0])

    @classmethod
    def of_points(cls, points) -> "BoundingBox":
        pts = np.asarray(points, dtype=np.float64)
        if pts.ndim != 2 or pts.shape[0] == 0:
            raise GeometryError("need a nonempty (n, d) point array")
        return cls(pts.min(axis=0), pts.max(axis=0))

    def diagonal(self) -> float:
        return float(np.linalg.norm(self.hi - self.lo))

    def contains(self, p) -> bool:
        p = np.asarray(p, dtype=np.float64)
        return bool((p >= self.lo).all() and (p <= self.hi).all())


@dataclass(frozen=True)
class KMeansSettings:
    k: int
    epsilon: float = 0.03
    max_iter: int = 50
    max_balance_iter: int = 20
    influence_step_cap: float = 0.05
    delta_threshold: float | None = None
    erosion: bool = True
    init_sample: int = 100
    seed: int = 0
    sfc_depth: int | None = None
    audit_bounds: bool = False

    def __post_init__(self):
        checks = (
            (self.k < 1, "k must be >= 1"),
            (self.epsilon < 0, "epsilon must be >= 0"),
            (self.max_iter < 1 or self.max_balance_iter < 1, "iteration budgets must be >= 1"),
            (not 0 < self.influence_step_cap < 1, "influence_step_cap must lie in (0, 1)"),
            (self.delta_threshold is not None and self.delta_threshold < 0,
             "delta_threshold must be >= 0"),
            (self.init_sample < 0, "init_sample must be >= 0"),
            (self.sfc_depth is not None and self.sfc_depth < 1, "sfc_depth must be >= 1"),
        )
        for bad, msg in checks:
            if bad:
                raise ValueError(msg)


@dataclass
class ClusterState:
    centers: np.ndarray
    influence: np.ndarray
    block_weights: np.ndarray
    last_move: np.ndarray

    @property
    def k(self) -> int:
        return self.centers.shape[0]

    @property
    def dim(self) -> int:
        return self.centers.shape[1]

    @classmethod
    def initial(cls, centers) -> "ClusterState":
        c = np.array(centers, dtype=np.float64)
        k = c.shape[0]
        return cls(c, np.ones(k), np.zeros(k), np.zeros(k))


@dataclass
class PointBounds:
    upper: np.ndarray
    lower: np.ndarray

    @classmethod
    def fresh(cls, m: int) -> "PointBounds":
        return cls(np.full(m, np.inf), np.zeros(m))


@dataclass
class BalanceInfo:
    rounds: int
    imbalance: float
    block_weights: np.ndarray
    skip_decisions: int
    total_decisions: int
    distance_evals: int
    imbalance_history: list = field(default_factory=list)


@dataclass
class IterationRecord:
    phase: str
    active_points: int
    balance_rounds: int
    imbalance: float
    skip_decisions: int
    total_decisions: int
    distance_evals: int
    objective: float
    max_move: float


@dataclass
class KMeansStats:
    iterations: list = field(default_factory=list)
    converged: bool = False
    balance_failed: bool = False
    audited_point_iterations: int = 0
    bound_violations: int = 0
    skip_check_failures: int = 0
    final_state: ClusterState | None = None

    def skip_fraction(self, last: int | None = None) -> float:
        recs = [r for r in self.iterations if r.phase == "full"]
        if last is not None:
            recs = recs[-last:]
        total = sum(r.total_decisions for r in recs)
        return 0.0 if total == 0 else sum(r.skip_decisions for r in recs) / total


@dataclass
class Partition:
    assignment: np.ndarray
    k: int
    balance_failed: bool = False
    empty_blocks: np.ndarray = field(default_factory=lambda: np.array([], dtype=np.int64))

    def __post_init__(self):
        self.assignment = np.asarray(self.assignment, dtype=np.int64)
        self.empty_blocks = np.asarray(self.empty_blocks, dtype=np.int64)

    @property
    def n(self) -> int:
        return int(self.assignment.shape[0])

    def validate(self, n: int | None = None):
        if self.k < 1:
            raise GraphError("k must be >= 1")
        if n is not None and self.assignment.shape[0] != n:
            raise GraphError("partition length does not match vertex count")
        if self.assignment.size == 0:
            raise GraphError("empty partition")
        if self.assignment.min() < 0 or self.assignment.max() >= self.k:
            raise GraphError("block id out of range")

    def block_weights(self, vertex_weights=None) -> np.ndarray:
        if vertex_weights is None:
            vertex_weights = np.ones(self.n)
        return np.bincount(self.assignment, weights=vertex_weights, minlength=self.k)
