"""CPU oracle for the Geographer balanced k-means hot path.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_1805_01208_b200`` imports,
links or executes this module; only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s CPU-baseline / ``--impl reference`` leg may use it, and
only as the checker or the timed CPU baseline.

This is a numpy restatement of the reference path
(``/root/reference/pkg/src/geopart``), written as one straight-line module
for a single logical rank.  The reference's results are identical for every
simulated rank count p dividing 256 (``ranksim.py:9-17``), so a single-rank
restatement reproduces them bit for bit; ``scan_chunks`` only changes how the
per-point scan prunes (the per-rank boxes of ``kmeans.py:315-319``), never its
result, and lets the oracle run at the reference's fastest setting.

Pinning: ``tests/test_oracle_golden.py`` checks this module against golden
vectors produced by the live reference (``tests/golden/make_golden.py``):
Hilbert keys, SFC order, initial centers, and complete partitions with
per-iteration statistics, bit for bit.

Numerics that matter for bit-exactness (all plain numpy, exactly as the
reference computes them):
  * effective distance = sqrt(einsum('ij,ij->i', diff, diff)) / influence
    (``kmeans.py:157-159``); einsum's 3-D summation order is host dependent.
  * segment-resolved sums: 256 equal position ranges, sequential
    ``bincount`` folds inside a segment, then a sequential fold over
    segments (``ranksim.py:173-197``, ``kmeans.py:368-374``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

SEGMENTS = 256  # ranksim.py:38
DEFAULT_DEPTH = {2: 31, 3: 20}  # geometry.py:28
UB_SLACK = 1.0 + 1e-12  # kmeans.py:61
LB_SLACK = 1.0 - 1e-12  # kmeans.py:62


class OracleError(ValueError):
    pass


# --------------------------------------------------------------------------
# SFC stage
# --------------------------------------------------------------------------

def grid_cells(points: np.ndarray, lo: np.ndarray, hi: np.ndarray, depth: int) -> np.ndarray:
    """Integer cell per axis (geometry.py:112-132): floor((p-lo)/ext * 2^depth), clipped."""
    ext = hi - lo
    safe = np.where(ext > 0, ext, 1.0)
    side = float(1 << depth)
    scaled = (points - lo) / safe * side
    cells = np.clip(np.floor(scaled), 0.0, side - 1.0)
    return cells.astype(np.uint64)


def hilbert_from_cells(cells: np.ndarray, depth: int) -> np.ndarray:
    """Hilbert index of integer cells (geometry.py:135-179).

    Skilling's transpose form: inverse-undo pass over bit planes Q = 2^(depth-1)..2,
    Gray encoding across axes, the t-correction from the last axis, then bit
    interleaving with axis 0 most significant.
    """
    X = [cells[:, a].astype(np.uint64) for a in range(cells.shape[1])]
    d = len(X)
    one = np.uint64(1)
    q = 1 << (depth - 1)
    while q > 1:
        Q = np.uint64(q)
        P = np.uint64(q - 1)
        for a in range(d):
            hit = (X[a] & Q) != 0
            x0 = np.where(hit, X[0] ^ P, X[0])
            swap = np.where(hit, np.uint64(0), (x0 ^ X[a]) & P)
            X[0] = x0 ^ swap
            X[a] = X[a] ^ swap
        q >>= 1
    for a in range(1, d):
        X[a] = X[a] ^ X[a - 1]
    t = np.zeros_like(X[0])
    q = 1 << (depth - 1)
    while q > 1:
        t = np.where((X[d - 1] & np.uint64(q)) != 0, t ^ np.uint64(q - 1), t)
        q >>= 1
    X = [x ^ t for x in X]
    key = np.zeros_like(X[0])
    for bit in range(depth - 1, -1, -1):
        b = np.uint64(bit)
        for a in range(d):
            key = (key << one) | ((X[a] >> b) & one)
    return key


def hilbert_keys(points: np.ndarray, lo: np.ndarray, hi: np.ndarray, depth: int) -> np.ndarray:
    return hilbert_from_cells(grid_cells(points, lo, hi, depth), depth)


def sfc_order(keys: np.ndarray) -> np.ndarray:
    """Order by (key, gid); gids are arange(n) so a stable key sort is the same (ranksim.py:158)."""
    return np.argsort(keys, kind="stable")


def center_positions(n: int, k: int) -> np.ndarray:
    """kmeans.py:170-173."""
    i = np.arange(k, dtype=np.int64)
    return ((2 * i + 1) * n) // (2 * k)


# --------------------------------------------------------------------------
# k-sized control math (kmeans.py:176-239, metrics.py:26-40)
# --------------------------------------------------------------------------

def balance_target(total: float, k: int) -> float:
    if float(total).is_integer():
        return float(-(-int(total) // k))
    return float(math.ceil(total / k))


def imbalance(bw: np.ndarray) -> float:
    total = float(bw.sum())
    if total <= 0:
        raise OracleError("total weight must be positive")
    return float(bw.max() / balance_target(total, bw.shape[0]) - 1.0)


def adapted_influence(infl, block_w, target, cap, d):
    with np.errstate(divide="ignore"):
        gamma = np.where(block_w > 0, target / np.where(block_w > 0, block_w, 1.0), np.inf)
    return infl * np.clip(gamma ** (1.0 / d), 1.0 - cap, 1.0 + cap)


def eroded_influence(infl, moves, beta):
    alpha = 2.0 / (1.0 + np.exp(-moves / beta)) - 1.0
    return infl ** (1.0 - alpha)


def relax(ub, lb, a, infl_old, infl_new, moves):
    """kmeans.py:208-239 (returns new arrays; identity when nothing changed)."""
    if not moves.any() and np.array_equal(infl_old, infl_new):
        return ub, lb
    ratio = infl_old / infl_new
    shift = moves / infl_new
    has = a >= 0
    c = np.where(has, a, 0)
    ub2 = np.where(has, (ub * ratio[c] + shift[c]) * UB_SLACK, ub)
    lb2 = np.maximum((lb * ratio.min() - shift.max()) * LB_SLACK, 0.0)
    return ub2, lb2


# --------------------------------------------------------------------------
# n-sized passes
# --------------------------------------------------------------------------

def effdist(pts: np.ndarray, center: np.ndarray, infl: float) -> np.ndarray:
    """kmeans.py:157-159 — the exact arithmetic every comparison uses."""
    diff = pts - center
    return np.sqrt(np.einsum("ij,ij->i", diff, diff)) / infl


def box_lower_bounds(lo, hi, centers, infl):
    """geometry.py:98-101 divided by influence (kmeans.py:317)."""
    near = np.clip(centers, lo, hi)
    return np.linalg.norm(centers - near, axis=1) / infl


@dataclass
class Tally:
    skips: int = 0
    decisions: int = 0
    evals: int = 0


def scan(points, idx, a, ub, lb, centers, infl, tally):
    """One rank's scan (kmeans.py:297-344); updates a/ub/lb in place."""
    k = centers.shape[0]
    prev = a[idx]
    tally.decisions += idx.size
    keep = (prev >= 0) & (ub[idx] < lb[idx])
    tally.skips += int(np.count_nonzero(keep))
    todo = idx[~keep]
    if todo.size == 0:
        return
    pts = points[todo]
    bound = box_lower_bounds(pts.min(axis=0), pts.max(axis=0), centers, infl)
    order = np.lexsort((np.arange(k), bound))
    best = np.full(todo.size, np.inf)
    second = np.full(todo.size, np.inf)
    arg = np.zeros(todo.size, dtype=np.int64)
    live = np.arange(todo.size)
    for c in order:
        live = live[bound[c] <= second[live]]
        if live.size == 0:
            break
        dist = effdist(pts[live], centers[c], infl[c])
        tally.evals += live.size
        b, s, bi = best[live], second[live], arg[live]
        win = (dist < b) | ((dist == b) & (c < bi))
        second[live] = np.where(win, b, np.minimum(s, dist))
        best[live] = np.where(win, dist, b)
        arg[live] = np.where(win, c, bi)
    a[todo] = arg
    ub[todo] = best
    lb[todo] = second


def segment_sums(seg_of, a, values, k):
    """Per-(segment, block) sequential folds then a sequential fold over segments.

    ranksim.py:173-197 + allreduce (rank order) + np.add.reduce(axis=0)
    (kmeans.py:374, ranksim.py:420-422).  values: (n,) or (n, c).
    """
    ok = a >= 0
    key = seg_of[ok] * k + a[ok]
    if values.ndim == 1:
        per = np.bincount(key, weights=values[ok], minlength=SEGMENTS * k).reshape(SEGMENTS, k)
    else:
        per = np.stack(
            [np.bincount(key, weights=values[ok, j], minlength=SEGMENTS * k)
             for j in range(values.shape[1])],
            axis=1,
        ).reshape(SEGMENTS, k, values.shape[1])
    return np.add.reduce(per, axis=0)


def sample_ranks(n: int, seed: int) -> np.ndarray:
    """Inverse of default_rng(seed).permutation(n) (kmeans.py:564-567)."""
    perm = np.random.default_rng(seed).permutation(n)
    r = np.empty(n, dtype=np.int64)
    r[perm] = np.arange(n, dtype=np.int64)
    return r


def sample_sizes(n: int, init_sample: int) -> list[int]:
    """kmeans.py:456-460."""
    if init_sample <= 0 or n <= init_sample:
        return []
    return [init_sample * 2**j for j in range(math.ceil(math.log2(n / init_sample)))]


# --------------------------------------------------------------------------
# driver
# --------------------------------------------------------------------------

@dataclass
class Knobs:
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


@dataclass
class OracleResult:
    assignment: np.ndarray          # int64, by original id
    centers: np.ndarray             # final_state.centers
    influence: np.ndarray
    block_weights: np.ndarray
    balance_failed: bool
    converged: bool
    empty_blocks: np.ndarray
    keys: np.ndarray                # Hilbert keys by original id
    order: np.ndarray               # gids in SFC order
    init_centers: np.ndarray
    records: list = field(default_factory=list)  # per movement iteration dicts
    balance_history: list = field(default_factory=list)  # imbalance per round


def run(points, weights, knobs: Knobs, scan_chunks: int = 1) -> OracleResult:
    """The whole partition (kmeans.py:502-512 -> 537-650) for one logical rank."""
    pts_in = np.asarray(points, dtype=np.float64)
    n, d = pts_in.shape
    k = knobs.k
    if k > n:
        raise OracleError(f"k={k} exceeds the number of points {n}")
    depth = knobs.sfc_depth if knobs.sfc_depth is not None else DEFAULT_DEPTH[d]
    w_in = np.ones(n) if weights is None else np.asarray(weights, dtype=np.float64)

    lo, hi = pts_in.min(axis=0), pts_in.max(axis=0)
    keys = hilbert_keys(pts_in, lo, hi, depth)
    order = sfc_order(keys)
    pts = pts_in[order]
    w = w_in[order]
    seg_bounds = (np.arange(SEGMENTS + 1, dtype=np.int64) * n) // SEGMENTS
    seg_of = np.searchsorted(seg_bounds, np.arange(n), side="right") - 1
    chunk_bounds = (np.arange(scan_chunks + 1, dtype=np.int64) * n) // scan_chunks

    centers = pts[center_positions(n, k)].copy()
    init_centers = centers.copy()
    infl = np.ones(k)
    block_w = np.zeros(k)
    threshold = knobs.delta_threshold
    if threshold is None:
        threshold = 1e-4 * float(np.linalg.norm(hi - lo))
    rank_sfc = sample_ranks(n, knobs.seed)[order]

    a = np.full(n, -1, dtype=np.int64)
    ub = np.full(n, np.inf)
    lb = np.zeros(n)
    wx = pts * w[:, None]
    plan = [("sample", s) for s in sample_sizes(n, knobs.init_sample)]
    plan += [("full", None)] * knobs.max_iter
    records, history = [], []
    fallback = None
    converged = False
    final_imb = math.inf
    for it, (phase, size) in enumerate(plan):
        active = None if size is None else rank_sfc < size
        idx_chunks = []
        for c in range(scan_chunks):
            lo_c, hi_c = chunk_bounds[c], chunk_bounds[c + 1]
            if active is None:
                idx_chunks.append(np.arange(lo_c, hi_c))
            else:
                idx_chunks.append(lo_c + np.flatnonzero(active[lo_c:hi_c]))
        # ---- assign and balance (kmeans.py:377-453)
        tally = Tally()
        best_imb = math.inf
        step = knobs.influence_step_cap
        regress = 0
        rounds = 0
        for rnd in range(knobs.max_balance_iter):
            rounds += 1
            for idx in idx_chunks:
                scan(pts, idx, a, ub, lb, centers, infl, tally)
            a_act = a if active is None else np.where(active, a, -1)
            block_w = segment_sums(seg_of, a_act, w, k)
            final_imb = imbalance(block_w)
            history.append(final_imb)
            if final_imb <= knobs.epsilon or rnd == knobs.max_balance_iter - 1:
                break
            if final_imb > best_imb:
                regress += 1
                if regress >= 2:
                    step *= 0.5
            best_imb = min(best_imb, final_imb)
            new_infl = adapted_influence(infl, block_w, float(block_w.sum()) / k, step, d)
            ub, lb = relax(ub, lb, a, infl, new_infl, np.zeros(k))
            infl = new_infl
        if phase == "full" and final_imb <= knobs.epsilon:
            fallback = (a.copy(), centers, infl, block_w, final_imb)
        # ---- movement (kmeans.py:585-626)
        a_act = a if active is None else np.where(active, a, -1)
        sums = segment_sums(seg_of, a_act, wx, k)
        tot = segment_sums(seg_of, a_act, w, k)
        empty = tot == 0
        new_centers = sums / np.where(empty, 1.0, tot)[:, None]
        new_centers[empty] = centers[empty]
        moves = np.linalg.norm(new_centers - centers, axis=1)
        ok = a_act >= 0
        diff = pts[ok] - centers[a_act[ok]]
        sq = np.einsum("ij,ij->i", diff, diff)
        objective = float((sq * w[ok]).sum())
        records.append(dict(
            phase=phase,
            active_points=n if active is None else int(active.sum()),
            balance_rounds=rounds,
            imbalance=final_imb,
            skip_decisions=tally.skips,
            total_decisions=tally.decisions,
            distance_evals=tally.evals,
            objective=objective,
            max_move=float(moves.max()),
        ))
        last = it == len(plan) - 1
        converged = phase == "full" and float(moves.max()) < threshold
        if converged or last:
            break
        old_infl = infl
        nxt = old_infl * np.where(empty, 1.0 + knobs.influence_step_cap, 1.0)
        if knobs.erosion:
            ext = np.zeros(k)
            np.maximum.at(ext, a_act[ok], np.sqrt(sq))
            nonempty = block_w > 0
            beta = float(2.0 * ext[nonempty].mean()) if nonempty.any() else 0.0
            if beta > 0:
                nxt = eroded_influence(nxt, moves, beta)
        ub, lb = relax(ub, lb, a, old_infl, nxt, moves)
        centers = new_centers
        infl = nxt

    if final_imb > knobs.epsilon and fallback is not None:
        a, centers, infl, block_w, final_imb = fallback
    failed = final_imb > knobs.epsilon
    out = np.empty(n, dtype=np.int64)
    out[order] = a
    return OracleResult(
        assignment=out,
        centers=centers,
        influence=infl,
        block_weights=block_w,
        balance_failed=failed,
        converged=converged,
        empty_blocks=np.flatnonzero(block_w == 0),
        keys=keys,
        order=order,
        init_centers=init_centers,
        records=records,
        balance_history=history,
    )


def brute_labels(points, centers, infl):
    """Weighted-Voronoi argmin with the scan's arithmetic, lowest index on ties."""
    best = np.full(points.shape[0], np.inf)
    arg = np.zeros(points.shape[0], dtype=np.int64)
    for c in range(centers.shape[0]):
        dist = effdist(points, centers[c], infl[c])
        win = dist < best
        best = np.where(win, dist, best)
        arg = np.where(win, c, arg)
    return arg


def brute_labels_blocked(points, centers, infl, block=256):
    """brute_labels for large k: effdist's exact arithmetic (kmeans.py:157-159,
    the same einsum over rows of diff) on (block x k) tiles; np.argmin keeps the
    first (lowest-index) minimum, the reference's tie-break."""
    points = np.asarray(points, dtype=np.float64)
    n, d = points.shape
    k = centers.shape[0]
    out = np.empty(n, dtype=np.int64)
    for s in range(0, n, block):
        p = points[s:s + block]
        diff = (p[:, None, :] - centers[None, :, :]).reshape(-1, d)
        dist = np.sqrt(np.einsum("ij,ij->i", diff, diff)).reshape(p.shape[0], k) / infl[None, :]
        out[s:s + block] = np.argmin(dist, axis=1)
    return out


def runner_up_gap(points, centers, infl):
    """Relative gap between the best and second-best effective distance per point."""
    mat = np.stack([effdist(points, centers[c], infl[c]) for c in range(centers.shape[0])], axis=1)
    if mat.shape[1] < 2:
        return np.full(points.shape[0], np.inf)
    part = np.partition(mat, 1, axis=1)
    return (part[:, 1] - part[:, 0]) / np.maximum(part[:, 1], 1e-300)


# --------------------------------------------------------------------------
# Callers of the path: SFC baseline cut and estimator predict
# --------------------------------------------------------------------------

def sfc_labels(coords, weights, k: int, depth: int | None = None) -> np.ndarray:
    """The SFC baseline (baselines.py:62-89): prefix weight strictly before each
    vertex in (key, id) order, block floor(before*k/total) clipped to k-1."""
    coords = np.asarray(coords, dtype=np.float64)
    w_all = np.asarray(weights, dtype=np.float64)
    n, d = coords.shape
    if not 1 <= k <= n:
        raise OracleError(f"k={k} out of range 1..{n}")
    depth = DEFAULT_DEPTH[d] if depth is None else depth
    keys = hilbert_keys(coords, coords.min(axis=0), coords.max(axis=0), depth)
    order = sfc_order(keys)
    w = w_all[order]
    before = np.cumsum(w) - w                      # sequential fold, then one subtraction
    total = float(w.sum())                         # numpy pairwise sum
    block = np.minimum((before * k / total).astype(np.int64), k - 1)
    out = np.empty(n, dtype=np.int64)
    out[order] = block
    return out


def predict_labels(X, centers, infl) -> np.ndarray:
    """GeographerPartitioner.predict (estimators.py:107-114), one center at a
    time: norm = sqrt((dx^2 + dy^2) + dz^2) (linalg.norm's reduction order),
    divided by the influence; argmin keeps the first minimum and a NaN wins."""
    X = np.asarray(X, dtype=np.float64)
    C = np.asarray(centers, dtype=np.float64)
    f = np.asarray(infl, dtype=np.float64)
    best = np.full(X.shape[0], np.inf)
    arg = np.zeros(X.shape[0], dtype=np.int64)
    seen_nan = np.zeros(X.shape[0], dtype=bool)
    with np.errstate(all="ignore"):
        for c in range(C.shape[0]):
            diff = X - C[c]
            sq = diff * diff
            s = sq[:, 0]
            for j in range(1, X.shape[1]):
                s = s + sq[:, j]
            dist = np.sqrt(s) / f[c]
            nan = np.isnan(dist) & ~seen_nan
            win = ((dist < best) & ~seen_nan) | nan
            if c == 0:
                win = np.ones_like(win)
            best = np.where(win, dist, best)
            arg = np.where(win, c, arg)
            seen_nan |= nan
    return arg
