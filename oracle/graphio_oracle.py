"""CPU oracle for the formats and metrics either side of the partition path
(SURVEY §8(f) item 4).  TEST INFRASTRUCTURE ONLY: imported by tests/ and by the callers
bench's cpu leg, never by the product package.

A plain-Python / numpy restatement of what the reference's fileio.py and metrics.py
compute, written for clarity rather than speed (per-line loops, per-vertex sets, a
deque BFS).  Pinned bit for bit to golden fixtures produced by the live reference
(tests/golden/make_golden_graphio.py -> tests/golden/graphio.json): every parsed array,
every error message, every metric.

    parse_metis      fileio.py:70-196      parse_table   np.loadtxt as fileio.py:222, :250
    coords_of        fileio.py:219-237     labels_of     fileio.py:246-263
    format_labels    fileio.py:271-278
    edge_cut         metrics.py:48-60      comm_volumes  metrics.py:63-77
    block_weights    graph.py:165-166      diameters     metrics.py:121-168
    report           metrics.py:253-281
"""

from __future__ import annotations

import io
import math
import warnings
from collections import deque

import numpy as np


class ParseError(ValueError):
    """stands for fileio.MetisParseError: same messages"""


# ---------------------------------------------------------------- METIS graph text
def _weight(tok, no, what):
    # fileio.py:60-67
    try:
        w = float(tok)
    except ValueError:
        raise ParseError(f"line {no}: non-numeric {what} {tok!r}") from None
    if not w > 0 or not math.isfinite(w):
        raise ParseError(f"line {no}: {what} must be strictly positive, got {tok!r}")
    return w


def parse_metis(text: str):
    """fileio.py:70-187 up to (not including) the coordinates: returns
    (offsets, neighbors, vertex_weights, edge_weights or None) or raises ParseError."""
    rows = [(no, ln) for no, ln in enumerate(text.splitlines(), 1)
            if not ln.lstrip().startswith("%")]                      # :85-93
    if not rows:
        raise ParseError("line 1: missing header")
    (hno, head), body = rows[0], rows[1:]
    f = head.split()
    if not 2 <= len(f) <= 4:                                         # :98-99
        raise ParseError(f"line {hno}: header must be 'n m [fmt [ncon]]', got {head!r}")
    try:
        n, m = int(f[0]), int(f[1])
    except ValueError:
        raise ParseError(f"line {hno}: non-numeric vertex or edge count") from None
    if n < 1 or m < 0:
        raise ParseError(f"line {hno}: bad sizes n={n} m={m}")
    fmt = f[2] if len(f) > 2 else "0"
    if not fmt.isdigit():
        raise ParseError(f"line {hno}: non-numeric fmt {fmt!r}")
    vsize, vwgt, ewgt = (c == "1" for c in fmt.zfill(3))             # :109-112
    if vsize:
        raise ParseError(f"line {hno}: vertex sizes (fmt 1xx) are not supported")
    ncon = 1
    if len(f) == 4:
        try:
            ncon = int(f[3])
        except ValueError:
            raise ParseError(f"line {hno}: non-numeric ncon {f[3]!r}") from None
    if vwgt and ncon != 1:
        raise ParseError(
            f"line {hno}: only one vertex weight per vertex is supported, got ncon={ncon}")
    while len(body) > n and not body[-1][1].strip():                 # :124-126
        body.pop()
    if len(body) != n:
        raise ParseError(
            f"line {hno}: header declares {n} vertices but file has {len(body)} vertex lines")

    vw = np.ones(n)
    adj, ews = [], []
    for u, (no, ln) in enumerate(body):                              # :134-160
        t = ln.split()
        if vwgt:
            if not t:
                raise ParseError(f"line {no}: missing vertex weight")
            vw[u] = _weight(t[0], no, "vertex weight")
            t = t[1:]
        if ewgt and len(t) % 2:
            raise ParseError(f"line {no}: dangling neighbor without edge weight")
        ids = t[0::2] if ewgt else t
        mine = []
        for tok in ids:
            try:
                v = int(tok)
            except ValueError:
                raise ParseError(f"line {no}: non-numeric neighbor id {tok!r}") from None
            if not 1 <= v <= n:
                raise ParseError(f"line {no}: neighbor id {v} out of range 1..{n}")
            if v == u + 1:
                raise ParseError(f"line {no}: self loop at vertex {u + 1}")
            mine.append(v - 1)
        if len(set(mine)) != len(mine):
            raise ParseError(
                f"line {no}: duplicate neighbor in adjacency list of vertex {u + 1}")
        adj.append(mine)
        if ewgt:
            ews.append([_weight(x, no, "edge weight") for x in t[1::2]])

    nbrs = np.array([v for a in adj for v in a], dtype=np.int64)
    if nbrs.size != 2 * m:                                           # :163-167
        raise ParseError(f"line {hno}: header declares {m} edges but adjacency lists "
                         f"hold {nbrs.size} entries (expected {2 * m})")
    offsets = np.zeros(n + 1, dtype=np.int64)
    offsets[1:] = np.cumsum([len(a) for a in adj])
    ew = np.array([w for a in ews for w in a], dtype=np.float64) if ewgt else None
    pairs = {(u, v): j for u, a in enumerate(adj) for j, v in
             zip(range(int(offsets[u]), int(offsets[u + 1])), a)}
    lost = sorted(p for p in pairs if (p[1], p[0]) not in pairs)     # :173-183
    if lost:
        u, v = lost[0]
        raise ParseError(
            f"asymmetric adjacency: vertex {u + 1} lists {v + 1} but not vice versa")
    if ew is not None and any(ew[j] != ew[pairs[(v, u)]] for (u, v), j in pairs.items()):
        raise ParseError("edge weight differs between the two directions of an edge")
    return offsets, nbrs, vw, ew


# ---------------------------------------------------------------- np.loadtxt tables
def parse_table(text: str, dtype):
    """What np.loadtxt(f, dtype=dtype) returns for the text (the reference calls numpy
    itself, fileio.py:222 and :250), with its ValueError as ParseError text."""
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")
        return np.loadtxt(io.StringIO(text), dtype=dtype, ndmin=2 if dtype is np.float64 else 1)


def coords_of(text: str, expect_n=None):
    # fileio.py:219-237
    try:
        c = parse_table(text, np.float64)
    except ValueError as e:
        raise ParseError(f"malformed coordinate file: {e}") from None
    if c.size == 0:
        raise ParseError("empty coordinate file")
    if c.shape[1] not in (2, 3):
        raise ParseError(f"coordinates must have 2 or 3 columns, got {c.shape[1]}")
    if expect_n is not None and c.shape[0] != expect_n:
        raise ParseError(f"coordinate file has {c.shape[0]} lines, expected {expect_n}")
    if not np.isfinite(c).all():
        raise ParseError("non-finite coordinate")
    return c


def labels_of(text: str, expect_n=None, k=None):
    # fileio.py:246-263: (labels, k)
    try:
        a = parse_table(text, np.int64)
    except ValueError as e:
        raise ParseError(f"malformed partition file: {e}") from None
    if a.ndim != 1:
        raise ParseError("partition file must hold one block id per line")
    if expect_n is not None and a.shape[0] != expect_n:
        raise ParseError(f"partition file has {a.shape[0]} lines, expected {expect_n}")
    if a.size and a.min() < 0:
        raise ParseError("negative block id")
    return a, (k if k is not None else (int(a.max()) + 1 if a.size else 1))


def format_labels(labels) -> str:
    # fileio.py:271-278
    return "".join(f"{int(x)}\n" for x in labels) if len(labels) else "\n"


# ---------------------------------------------------------------- metrics
def _adj(offsets, nbrs, u):
    return nbrs[offsets[u]:offsets[u + 1]]


def edge_cut(offsets, nbrs, ew, labels) -> float:
    # metrics.py:48-60: each undirected cut edge once; weighted: numpy's sum of the masked array
    n = len(offsets) - 1
    src = np.repeat(np.arange(n), np.diff(offsets))
    mask = (labels[src] != labels[nbrs]) & (src < nbrs)
    return float(np.count_nonzero(mask)) if ew is None else float(ew[mask].sum())


def comm_volumes(offsets, nbrs, labels, k):
    # metrics.py:63-77: per vertex, the OTHER blocks among its neighbors
    per = np.zeros(k)
    for u in range(len(offsets) - 1):
        per[labels[u]] += len({int(labels[v]) for v in _adj(offsets, nbrs, u)} - {int(labels[u])})
    return float(per.max()), float(per.sum()), per


def block_weights(labels, vw, k):
    # graph.py:165-166: sequential accumulation in vertex order
    out = np.zeros(k)
    for u, b in enumerate(labels):
        out[b] += vw[u]
    return out


def _levels(offsets, nbrs, labels, root):
    """hop distance from root inside root's block (metrics.py:91-117)"""
    lev = {root: 0}
    q = deque([root])
    while q:
        u = q.popleft()
        for v in _adj(offsets, nbrs, u):
            v = int(v)
            if labels[v] == labels[root] and v not in lev:
                lev[v] = lev[u] + 1
                q.append(v)
    return lev


def diameters(offsets, nbrs, labels, k, refinement_rounds=3):
    # metrics.py:121-168
    out = np.zeros(k)
    for b in range(k):
        members = [int(u) for u in np.flatnonzero(labels == b)]
        if not members:
            out[b] = math.inf
            continue
        if len(members) == 1:
            continue
        lev0 = _levels(offsets, nbrs, labels, members[0])
        if len(lev0) < len(members):
            out[b] = math.inf
            continue
        far = lambda lev: min(lev, key=lambda u: (-lev[u], u))  # noqa: E731
        a = far(lev0)
        lev_a = _levels(offsets, nbrs, labels, a)
        best = max(lev_a.values())
        fringe = [u for u in sorted(members, key=lambda u: (-lev_a[u], u)) if u != a]
        for root in fringe[:refinement_rounds]:
            best = max(best, max(_levels(offsets, nbrs, labels, root).values()))
        out[b] = best
    return out


def report(offsets, nbrs, vw, ew, labels, k):
    # metrics.py:253-281 (the numeric fields of MetricsReport)
    bw = block_weights(labels, vw, k)
    cmax, ctot, per = comm_volumes(offsets, nbrs, labels, k)
    dia = diameters(offsets, nbrs, labels, k)
    with np.errstate(divide="ignore"):
        r = np.where(np.isinf(dia), 0.0, np.divide(1.0, dia))
    denom = r.sum()
    total = float(bw.sum())
    target = float(-(-int(total) // k)) if total.is_integer() else float(math.ceil(total / k))
    return {
        "edge_cut": edge_cut(offsets, nbrs, ew, labels), "comm_max": cmax, "comm_total": ctot,
        "imbalance": float(bw.max() / target - 1.0),
        "harmonic_diameter": math.inf if denom == 0.0 else float(len(dia) / denom),
        "block_weights": bw.tolist(), "block_comm": per.tolist(), "block_diameters": dia.tolist(),
    }
