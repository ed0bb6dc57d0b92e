"""Shared helpers for the graph I/O and metrics tests: the golden fixture made by
tests/golden/make_golden_graphio.py from the live reference, and seeded graph builders."""
import json
import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "graphio.json")


def golden():
    with open(GOLDEN) as f:
        return json.load(f)


def arr(rec):
    if rec is None:
        return None
    if "f64_hex" in rec:
        return np.array([float.fromhex(x) for x in rec["f64_hex"]],
                        dtype=np.float64).reshape(rec["shape"])
    return np.array(rec["i64"], dtype=np.int64).reshape(rec["shape"])


def same_bits(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()


def grid_graph(w, h):
    """(n, CSR offsets, neighbors, coords) of a w x h grid mesh, neighbor lists sorted."""
    idx = np.arange(w * h, dtype=np.int64).reshape(h, w)
    e = np.concatenate([np.stack([idx[:, :-1].ravel(), idx[:, 1:].ravel()], 1),
                        np.stack([idx[:-1, :].ravel(), idx[1:, :].ravel()], 1)])
    ys, xs = np.divmod(np.arange(w * h), w)
    return csr_from_edges(w * h, e) + (np.stack([xs, ys], 1).astype(np.float64),)


def csr_from_edges(n, e):
    src = np.concatenate([e[:, 0], e[:, 1]])
    dst = np.concatenate([e[:, 1], e[:, 0]])
    order = np.lexsort((dst, src))
    off = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(np.bincount(src, minlength=n), out=off[1:])
    return n, off, dst[order]


def random_geometric(n, seed, deg=8.0):
    """2D random geometric graph by cell binning (numpy only): (n, offsets, neighbors, coords)"""
    rng = np.random.default_rng(seed)
    pts = rng.random((n, 2))
    r = np.sqrt(deg / (np.pi * n))
    g = max(1, int(1.0 / r))
    cell = np.minimum((pts * g).astype(np.int64), g - 1)
    cid = cell[:, 0] * g + cell[:, 1]
    order = np.argsort(cid, kind="stable")
    start = np.searchsorted(cid[order], np.arange(g * g + 1))
    pairs = []
    for dx, dy in ((0, 0), (0, 1), (1, -1), (1, 0), (1, 1)):
        for cx in range(g):
            nx = cx + dx
            if nx >= g:
                continue
            for cy in range(g):
                ny = cy + dy
                if not 0 <= ny < g:
                    continue
                a = order[start[cx * g + cy]:start[cx * g + cy + 1]]
                b = order[start[nx * g + ny]:start[nx * g + ny + 1]]
                if not a.size or not b.size:
                    continue
                d2 = ((pts[a][:, None, :] - pts[b][None, :, :]) ** 2).sum(-1)
                ia, ib = np.nonzero(d2 < r * r)
                u, v = a[ia], b[ib]
                keep = u < v if (dx, dy) == (0, 0) else np.ones(u.size, bool)
                pairs.append(np.stack([u[keep], v[keep]], 1))
    e = np.concatenate(pairs) if pairs else np.empty((0, 2), np.int64)
    return csr_from_edges(n, e) + (pts,)


def metis_text(n, off, nbrs, vw=None, ew=None):
    """METIS text of a CSR graph (the layout fileio.py:199-216 writes)."""
    tok = lambda x: str(int(x)) if float(x).is_integer() else repr(float(x))  # noqa: E731
    head = f"{n} {len(nbrs) // 2}"
    if vw is not None or ew is not None:
        head += f" 0{int(vw is not None)}{int(ew is not None)}"
    lines = [head]
    for u in range(n):
        t = [tok(vw[u])] if vw is not None else []
        for j in range(off[u], off[u + 1]):
            t.append(str(int(nbrs[j]) + 1))
            if ew is not None:
                t.append(tok(ew[j]))
        lines.append(" ".join(t))
    return "\n".join(lines) + "\n"
