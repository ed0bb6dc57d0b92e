"""Seeded synthetic point sets standing in for the paper's meshes.

BASELINE.json names five configurations; none of the paper's inputs ship
with the reference (``PAPER.md:631-645``), so these recipes
generate inputs with the stated shapes, sizes and value distributions.
C1-C4 are host numpy (PCG64, platform independent) so the CPU oracle and the
device path see identical arrays; C5 (2^30 points, 16 GiB) is generated on
the device by :func:`c5_device` with the same distribution family.
"""

from __future__ import annotations

import numpy as np

CONFIGS = {
    "C1": dict(n=100_000, d=2, k=16, epsilon=0.03),
    "C2": dict(n=1 << 20, d=2, k=64, epsilon=0.03),
    "C3": dict(n=1 << 21, d=3, k=256, epsilon=0.03),
    "C4": dict(n=1 << 24, d=3, k=1024, epsilon=0.05),
    "C5": dict(n=1 << 30, d=2, k=16384, epsilon=0.03),
}


def _mixture(rng, n, d, ncomp, smin, smax):
    means = rng.random((ncomp, d))
    sig = rng.uniform(smin, smax, ncomp)
    parts, have = [], 0
    while have < n:
        m = n - have
        comp = rng.integers(0, ncomp, m)
        p = means[comp] + sig[comp, None] * rng.standard_normal((m, d))
        p = p[np.all((p >= 0.0) & (p <= 1.0), axis=1)]
        parts.append(p)
        have += p.shape[0]
    return np.concatenate(parts)[:n]


def c1(seed=0, n=100_000):
    rng = np.random.default_rng(seed)
    return rng.random((n, 2)), None


def c2(seed=0, n=1 << 20):
    """2.5D ocean-style mixture with integer topography weights 1..60."""
    rng = np.random.default_rng(seed)
    pts = _mixture(rng, n, 2, 32, 0.01, 0.1)
    c = rng.random((16, 2))
    s = rng.uniform(0.05, 0.3, 16)
    a = rng.uniform(0.2, 1.0, 16)
    f = np.zeros(n)
    for j in range(16):
        f += a[j] * np.exp(-((pts - c[j]) ** 2).sum(1) / (2 * s[j] ** 2))
    w = 1.0 + np.rint(59.0 * (f - f.min()) / (f.max() - f.min()))
    return pts, w


def c3(seed=0, side=128):
    """Jittered 128^3 lattice, row-major (i, j, k) order, unit weights."""
    rng = np.random.default_rng(seed)
    g = np.stack(np.meshgrid(*[np.arange(side)] * 3, indexing="ij"), -1).reshape(-1, 3)
    g = g.astype(np.float64)
    return (g + 0.5 + rng.uniform(-0.3, 0.3, g.shape)) / side, None


def c4(seed=0, n=1 << 24):
    """Radially refined 3D cloud (density ~ 1/(r+0.01)^2), float32 weights in [1, 4)."""
    rng = np.random.default_rng(seed)
    cen = rng.random((4, 3))
    parts, have = [], 0
    while have < n:
        m = 2 * (n - have)
        r = rng.uniform(0, 1.0, m)
        r = r[rng.random(m) < (r / (r + 0.01)) ** 2]
        v = rng.standard_normal((r.size, 3))
        v /= np.linalg.norm(v, axis=1, keepdims=True)
        p = cen[rng.integers(0, 4, r.size)] + r[:, None] * v
        p = p[np.all((p >= 0) & (p <= 1), axis=1)]
        parts.append(p)
        have += p.shape[0]
    pts = np.concatenate(parts)[:n]
    w = rng.uniform(1.0, 4.0, n).astype(np.float32).astype(np.float64)
    return pts, w


def c5_host(seed=0, n=1 << 30):
    """Half uniform, half a 1024-component mixture (sigma 0.002-0.02); unit weights."""
    rng = np.random.default_rng(seed)
    u = rng.random((n // 2, 2))
    m = _mixture(rng, n - n // 2, 2, 1024, 0.002, 0.02)
    return np.concatenate([u, m]), None


def c5_device(n=1 << 30, seed=0, device="cuda", ncomp=1024):
    """C5's distribution generated on the GPU (torch Philox), SoA layout (2, n).

    Not numpy-identical (C5 has no CPU oracle: the reference cannot run it);
    same shape, size and value distribution as :func:`c5_host`.
    """
    import torch

    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = torch.empty((2, n), dtype=torch.float64, device=device)
    half = n // 2
    out[:, :half].uniform_(0.0, 1.0, generator=g)
    means = torch.rand((ncomp, 2), generator=g, device=device, dtype=torch.float64)
    sig = 0.002 + 0.018 * torch.rand((ncomp,), generator=g, device=device, dtype=torch.float64)
    pos = half
    chunk = 1 << 26
    while pos < n:
        m = min(chunk, n - pos)
        comp = torch.randint(0, ncomp, (m,), generator=g, device=device)
        p = means[comp] + sig[comp, None] * torch.randn((m, 2), generator=g, device=device,
                                                        dtype=torch.float64)
        keep = ((p >= 0) & (p <= 1)).all(dim=1)
        p = p[keep]
        take = min(p.shape[0], n - pos)
        out[:, pos:pos + take] = p[:take].t()
        pos += take
    return out


GENERATORS = {"C1": c1, "C2": c2, "C3": c3, "C4": c4, "C5": c5_host}
