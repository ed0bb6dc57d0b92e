"""Seeded input recipes shared by the golden generator and the parity tests."""

from __future__ import annotations

import hashlib

import numpy as np


def key_inputs():
    """Hilbert-key golden inputs: (points, lo, hi, depth)."""
    out = {}
    rng = np.random.default_rng(101)
    for d, depth in ((2, 31), (3, 20), (2, 12), (3, 7), (2, 1), (3, 1)):
        pts = rng.random((4096, d))
        out[f"rand_d{d}_depth{depth}"] = (pts, pts.min(axis=0), pts.max(axis=0), depth)
    # offset, anisotropic box with points on the upper faces (clamp into last cell)
    pts = rng.uniform([-3.0, 10.0, 0.5], [4.0, 10.001, 900.0], size=(2048, 3))
    lo, hi = pts.min(axis=0), pts.max(axis=0)
    pts[:64] = hi
    pts[64:128, 0] = hi[0]
    pts[128:192] = lo
    out["faces_d3_depth20"] = (pts, lo, hi, 20)
    # degenerate axis (zero extent)
    pts = rng.random((1024, 2))
    pts[:, 1] = 0.25
    out["flat_d2_depth31"] = (pts, pts.min(axis=0), pts.max(axis=0), 31)
    # coarse-to-fine mixture with many equal keys
    pts = np.round(rng.random((3000, 2)) * 8) / 8
    out["dup_d2_depth31"] = (pts, pts.min(axis=0), pts.max(axis=0), 31)
    return out


def _points(kind, n, d, rng):
    if kind == "uniform":
        return rng.random((n, d))
    if kind == "clouds":
        cs = rng.random((5, d)) * 10
        return cs[rng.integers(0, 5, n)] + rng.normal(0, 0.05, (n, d))
    if kind == "coincident":
        return np.zeros((n, d))
    if kind == "collinear":
        return np.stack([np.linspace(0, 1, n)] + [np.zeros(n)] * (d - 1), axis=1)
    if kind == "dupsites":
        return np.repeat(rng.random((5, d)), n // 5, axis=0)
    if kind == "uneven":
        return np.concatenate([rng.normal(0, 0.01, (n - n // 10, d)),
                               rng.normal(10, 0.01, (n // 10, d))])
    raise ValueError(kind)


def partition_inputs(spec):
    if spec.get("config"):
        import sys
        import os

        sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", ".."))
        from paper_1805_01208_b200.workloads import GENERATORS

        return GENERATORS[spec["config"]](seed=spec.get("gen_seed", 0))
    rng = np.random.default_rng(spec["gen_seed"])
    pts = _points(spec["kind"], spec["n"], spec["d"], rng)
    wk = spec.get("weights")
    if wk is None:
        w = None
    elif wk == "int":
        w = rng.integers(1, 6, spec["n"]).astype(float)
    elif wk == "f32":
        w = rng.uniform(1.0, 4.0, spec["n"]).astype(np.float32).astype(np.float64)
    elif wk == "real":
        w = rng.uniform(0.1, 3.0, spec["n"])
    else:
        raise ValueError(wk)
    return pts, w


def _p(name, n, d, k, kind="uniform", weights=None, gen_seed=0, **settings):
    settings = dict(k=k, **settings)
    settings.setdefault("seed", gen_seed)
    return dict(name=name, n=n, d=d, kind=kind, weights=weights, gen_seed=gen_seed,
                settings=settings)


PARTITION_CASES = [
    _p("u2_k7", 2000, 2, 7, gen_seed=0),
    _p("u3_k9_int", 3000, 3, 9, weights="int", gen_seed=1),
    _p("u2_k16_f32", 6000, 2, 16, weights="f32", gen_seed=2),
    _p("u3_k33_real", 5000, 3, 33, weights="real", gen_seed=3),
    _p("u2_k5_nowarm", 500, 2, 5, gen_seed=4, init_sample=0),
    _p("clouds2_k5", 1500, 2, 5, kind="clouds", gen_seed=5),
    _p("u2_k1", 300, 2, 1, gen_seed=6),
    _p("u2_keqn", 12, 2, 12, gen_seed=7, init_sample=0),
    _p("coincident_k4", 40, 2, 4, kind="coincident", gen_seed=8, init_sample=0),
    _p("collinear_k4", 100, 2, 4, kind="collinear", gen_seed=9),
    _p("dupsites_k5", 150, 2, 5, kind="dupsites", gen_seed=10, init_sample=0),
    _p("uneven_fail", 100, 2, 2, kind="uneven", gen_seed=11, epsilon=0.01, max_iter=1,
       max_balance_iter=1, init_sample=0),
    _p("lloyd_noerosion", 600, 2, 6, gen_seed=12, init_sample=0, max_balance_iter=1,
       erosion=False, max_iter=30),
    _p("u3_k64_audit", 4000, 3, 64, gen_seed=13, audit_bounds=True),
    _p("u2_k40_thresh", 8000, 2, 40, gen_seed=14, delta_threshold=0.0, max_iter=8),
    _p("u3_k20_depth5", 2500, 3, 20, gen_seed=15, sfc_depth=5),
    _p("u2_k200", 20000, 2, 200, gen_seed=16, max_iter=12),
    dict(name="C1", config="C1", gen_seed=0, settings=dict(k=16, epsilon=0.03, seed=0)),
]

SFC_CASES = [
    dict(name="C1", config="C1", gen_seed=0, settings=dict(k=16)),
    dict(name="C2", config="C2", gen_seed=0, settings=dict(k=64)),
    dict(name="C3", config="C3", gen_seed=0, settings=dict(k=256)),
]


def numerics_fingerprint():
    """Host numpy numerics the reference's results depend on."""
    rng = np.random.default_rng(5)
    x = rng.uniform(1e-3, 1e3, 4096)
    y = rng.uniform(-1.0, 1.0, 4096)
    diff = rng.random((4096, 3)) - 0.5
    e3 = np.einsum("ij,ij->i", diff, diff)
    h = hashlib.sha256()
    for arr in (x ** (1.0 / 3.0), np.exp(y), x ** (1.0 - np.abs(y))):
        h.update(arr.tobytes())
    return dict(pow_exp=h.hexdigest()[:16],
                einsum3=hashlib.sha256(e3.tobytes()).hexdigest()[:16],
                numpy=np.__version__)


# ---------------------------------------------------------------- callers (§8f)
def sfc_cut_inputs():
    """SFC-baseline cases: name -> (coords, weights, k, depth)."""
    rng = np.random.default_rng(202)
    out = {}
    out["u2_unit_k6"] = (rng.random((120, 2)), np.ones(120), 6, None)
    out["u2_int_k7"] = (rng.random((3001, 2)), rng.integers(1, 61, 3001).astype(float), 7, None)
    out["u3_f32w_k33"] = (rng.random((4099, 3)),
                          rng.uniform(1, 4, 4099).astype(np.float32).astype(np.float64), 33, None)
    # inexact weights: the pairwise total and the sequential cumsum decide the bits
    out["u2_f64w_k50"] = (rng.random((20000, 2)), rng.random(20000) * 3 + 1e-3, 50, None)
    out["u3_f64w_k5"] = (rng.random((777, 3)), rng.exponential(1.0, 777), 5, None)
    out["line_heavy_k2"] = (np.stack([np.linspace(0.01, 0.99, 4), np.full(4, 0.5)], axis=1),
                            np.array([3.0, 1.0, 1.0, 1.0]), 2, None)
    out["keqn_k7"] = (rng.random((7, 2)), np.ones(7), 7, None)
    out["k1"] = (rng.random((50, 2)), rng.random(50), 1, None)
    out["depth10_k4"] = (rng.random((400, 2)), np.ones(400), 4, 10)
    grid = np.stack(np.meshgrid(np.arange(9.0), np.arange(9.0), np.arange(9.0),
                                indexing="ij"), axis=-1).reshape(-1, 3)
    out["grid3_dups_k3"] = (np.concatenate([grid, grid[:100]]), np.ones(829), 3, None)
    return out


def predict_inputs():
    """predict cases: name -> (X, centers, influence)."""
    rng = np.random.default_rng(303)
    out = {}
    for d, k, n in ((2, 5, 400), (3, 17, 2000), (2, 64, 5000), (3, 300, 3000), (2, 1, 10)):
        X = rng.random((n, d))
        C = rng.random((k, d))
        f = rng.uniform(0.7, 1.4, k)
        out[f"d{d}_k{k}"] = (X, C, f)
    # duplicated centers with equal influence (exact ties -> lowest index),
    # points on centers, points outside the box
    C = rng.random((12, 2))
    C[7] = C[3]
    C[11] = C[3]
    f = np.ones(12)
    X = np.concatenate([rng.random((500, 2)), C, rng.normal(0.5, 3.0, (200, 2))])
    out["ties_d2"] = (X, C, f)
    C = rng.random((9, 3))
    C[8] = C[2]
    f = rng.uniform(0.9, 1.1, 9)
    f[8] = f[2]
    X = np.concatenate([rng.random((700, 3)), C])
    out["ties_d3"] = (X, C, f)
    return out
