"""Host-side k-sized control math of the balance / movement loops.

All of it is O(k) numpy run between kernel launches.  It must produce the
reference's bits: the reference computes these quantities with numpy on the
host (kmeans.py:170-239, metrics.py:26-40), so this module applies the very
same numpy operations in the same order.  Nothing here touches per-point data.
"""

from __future__ import annotations

import functools
import math
from dataclasses import replace

import numpy as np

from .types import ClusterState, GraphError, PointBounds

UB_SLACK = 1.0 + 1e-12  # kmeans.py:61
LB_SLACK = 1.0 - 1e-12  # kmeans.py:62


def balance_target(total_weight: float, k: int) -> float:
    """metrics.py:26-30: ceil(total / k), integer ceil when the total is integral."""
    if float(total_weight).is_integer():
        return float(-(-int(total_weight) // k))
    return float(math.ceil(total_weight / k))


def imbalance(block_weights) -> float:
    """metrics.py:33-40: max / ceil(total/k) - 1."""
    bw = np.asarray(block_weights, dtype=np.float64)
    total = float(bw.sum())
    if total <= 0:
        raise GraphError("total weight must be positive")
    return float(bw.max() / balance_target(total, bw.shape[0]) - 1.0)


def initial_center_positions(n: int, k: int) -> np.ndarray:
    """kmeans.py:170-173: floor(i*n/k + n/(2k)) as ((2i+1) n) // (2k)."""
    i = np.arange(k, dtype=np.int64)
    return ((2 * i + 1) * n) // (2 * k)


def influence_factor(block_w: np.ndarray, target: float, cap: float, dim: int) -> np.ndarray:
    """Multiplicative influence step of kmeans.py:187-190."""
    with np.errstate(divide="ignore"):
        gamma = np.where(block_w > 0, target / np.where(block_w > 0, block_w, 1.0), np.inf)
    return np.clip(gamma ** (1.0 / dim), 1.0 - cap, 1.0 + cap)


def adapt_influence(state: ClusterState, target_weight: float, cap: float) -> ClusterState:
    if not 0 < cap < 1:
        raise ValueError("cap must lie in (0, 1)")
    if not target_weight > 0:
        raise ValueError("target weight must be positive")
    step = influence_factor(state.block_weights, target_weight, cap, state.dim)
    return replace(state, influence=state.influence * step)


@functools.lru_cache(maxsize=None)
def _norm_order_is_sequential() -> bool:
    """Does this host's np.linalg.norm(axis=1) sum a row's squares left to right?
    (numpy's iterator / SIMD paths decide it; probed once per process.)"""
    rng = np.random.default_rng(4321)
    out = True
    for d in (2, 3):
        x = (rng.random((20000, d)) - 0.5) * rng.uniform(1e-3, 1e3, (20000, 1))
        out = out and np.array_equal(np.linalg.norm(x, axis=1), _row_norms_seq(x))
    return bool(out)


def _row_norms_seq(diff: np.ndarray) -> np.ndarray:
    sq = diff * diff
    s = sq[:, 0]
    for j in range(1, diff.shape[1]):
        s = s + sq[:, j]
    return np.sqrt(s)


def row_norms(diff: np.ndarray) -> np.ndarray:
    """np.linalg.norm(diff, axis=1) (kmeans.py:588), bit for bit: numpy reduces the
    squared components of a row in order, sqrt((x^2 + y^2) + z^2); the explicit sum
    avoids the slow short-axis reduction (~0.4 ms at k = 16384).  Where a probe finds
    this host's numpy summing in another order, np.linalg.norm itself is used."""
    if not _norm_order_is_sequential():
        return np.linalg.norm(diff, axis=1)
    return _row_norms_seq(diff)


def eroded(influence: np.ndarray, moves: np.ndarray, beta: float) -> np.ndarray:
    """kmeans.py:204-205: influence ** (1 - alpha), alpha = 2/(1+exp(-delta/beta)) - 1."""
    alpha = 2.0 / (1.0 + np.exp(-moves / beta)) - 1.0
    return influence ** (1.0 - alpha)


def erode_influence(state: ClusterState, beta: float) -> ClusterState:
    if not beta > 0:
        raise ValueError("beta must be strictly positive")
    return replace(state, influence=eroded(state.influence, state.last_move, beta))


def effective_distance(p, center, influence: float) -> float:
    """kmeans.py:150-154."""
    if not influence > 0:
        raise ValueError("influence must be strictly positive")
    d = np.asarray(p, dtype=np.float64) - np.asarray(center, dtype=np.float64)
    return math.sqrt(float(np.dot(d, d))) / influence


def relax_is_identity(old_infl, new_infl, moves) -> bool:
    """The early return of kmeans.py:223-228."""
    return moves.shape == old_infl.shape and not moves.any() and np.array_equal(old_infl, new_infl)


def relax_bounds(bounds: PointBounds, assignment, old_influence, new_influence,
                 center_moves) -> PointBounds:
    """Eager array form of the bound relaxation (kmeans.py:208-239), for API parity.

    The device path never materialises this per point; it composes the same
    affine maps lazily (:class:`BoundMaps`).
    """
    if relax_is_identity(old_influence, new_influence, center_moves):
        return bounds
    ratio = old_influence / new_influence
    shift = center_moves / new_influence
    assignment = np.asarray(assignment)
    has = assignment >= 0
    c = np.where(has, assignment, 0)
    upper = np.where(has, (bounds.upper * ratio[c] + shift[c]) * UB_SLACK, bounds.upper)
    lower = np.maximum((bounds.lower * ratio.min() - shift.max()) * LB_SLACK, 0.0)
    return PointBounds(upper=upper, lower=lower)


def sample_schedule(n: int, init_sample: int) -> list[int]:
    """kmeans.py:456-460."""
    if init_sample <= 0 or n <= init_sample:
        return []
    rounds = math.ceil(math.log2(n / init_sample))
    return [init_sample * 2**j for j in range(rounds)]


def _f32_up(x):
    x = np.asarray(x, dtype=np.float64)
    f = x.astype(np.float32)
    return np.where(f.astype(np.float64) < x, np.nextafter(f, np.float32(np.inf)), f)


def _f32_down(x):
    x = np.asarray(x, dtype=np.float64)
    f = x.astype(np.float32)
    return np.where(f.astype(np.float64) > x, np.nextafter(f, np.float32(-np.inf)), f)


class BoundMaps:
    """Cumulative affine maps standing in for per-point eager relaxation.

    A point scanned when the maps were (S_c, T_c) / (A, B) stores
    ub~ = (best - T_c)/S_c and lb~ = (second + B)/A.  Each relaxation of
    kmeans.py:229-238 is affine in the bound (ub' = (ub*r_c + s_c)*UB_SLACK and
    lb' = max((lb*min r - max s)*LB_SLACK, 0)), so composing the maps instead
    of rewriting n bounds gives the same sound bounds.  Host rounding in the
    composition is at most ~3 ulps per step relative to each of scale and
    shift; the device widens every evaluated bound by
    ``bound_err * (|scale * b~| + |shift|)`` with ``bound_err`` covering all
    steps since the last reset, which matters only where the affine form
    cancels (bounds near zero; e.g. a point sitting on its center).
    """

    def __init__(self, k: int):
        self.ub_scale = np.ones(k)
        self.ub_shift = np.zeros(k)
        self.lb_scale = 1.0
        self.lb_shift = 0.0
        self.version = 0
        self.steps = 0

    def relax(self, old_infl, new_infl, moves) -> bool:
        if relax_is_identity(old_infl, new_infl, moves):
            return False
        ratio = old_infl / new_infl
        shift = moves / new_infl
        self.ub_scale = self.ub_scale * ratio * UB_SLACK
        self.ub_shift = (self.ub_shift * ratio + shift) * UB_SLACK
        rmin = float(ratio.min())
        smax = float(shift.max())
        self.lb_scale = float(self.lb_scale * rmin * LB_SLACK)
        self.lb_shift = float((self.lb_shift * rmin + smax) * LB_SLACK)
        self.version += 1
        self.steps += 1
        return True

    @property
    def bound_err(self) -> float:
        return (4.0 * self.steps + 16.0) * 2.0 ** -52

    def device_params(self):
        """Float32 parameters of the device bound arithmetic, rounded outward.

        Returns (ub_eval (k,4), ub_norm (k,4), lb_a, lb_b, lb_inva, lb_blo) with
          ub <= fmaf_ru(ub~ >= 0 ? E.x : E.y, ub~, E.z)   (E = ub_eval[a])
          lb >= max(fmaf_rd(lb_a, lb~, -lb_b), 0)
        covering the composition error of the float64 maps (bound_err), and the
        normalisation constants (1/S up/down, T down, 1/A down, B down).
        """
        e = self.bound_err
        S, T = self.ub_scale, self.ub_shift
        k = S.shape[0]
        ev = np.zeros((k, 4), dtype=np.float32)
        ev[:, 0] = _f32_up(S * (1.0 + e))
        ev[:, 1] = _f32_down(S * (1.0 - e))
        ev[:, 2] = _f32_up(T * (1.0 + e))
        nm = np.zeros((k, 4), dtype=np.float32)
        inv = 1.0 / S
        nm[:, 0] = _f32_up(np.nextafter(inv, np.inf))
        nm[:, 1] = _f32_down(np.nextafter(inv, 0.0))
        nm[:, 2] = _f32_down(T)
        A, B = self.lb_scale, self.lb_shift
        lb_a = float(_f32_down(np.array([A * (1.0 - e)]))[0])
        lb_b = float(_f32_up(np.array([B * (1.0 + e)]))[0])
        lb_inva = float(_f32_down(np.array([np.nextafter(1.0 / A, 0.0)]))[0])
        lb_blo = float(_f32_down(np.array([B]))[0])
        return ev, nm, lb_a, lb_b, lb_inva, lb_blo

    def needs_rebase(self, scale_hint: float) -> bool:
        lim = 1e6
        s = self.ub_scale
        return bool(
            s.min() < 1 / lim or s.max() > lim or not (1 / lim < self.lb_scale < lim)
            or self.ub_shift.max() > 64.0 * scale_hint or self.lb_shift > 64.0 * scale_hint
        )

    def reset(self):
        self.ub_scale[:] = 1.0
        self.ub_shift[:] = 0.0
        self.lb_scale = 1.0
        self.lb_shift = 0.0
        self.version += 1
        self.steps = 0
