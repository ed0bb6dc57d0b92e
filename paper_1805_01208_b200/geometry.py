"""Device-backed Hilbert keys with the reference's API (geometry.py:182-206).

hilbert_keys(points, box, depth) returns the same uint64 keys as
geopart.geometry.hilbert_keys, computed by the gp_hilbert_keys kernel.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .types import BoundingBox, GeometryError

DEFAULT_DEPTH = {2: 31, 3: 20}
_CLAMP_RTOL = 1e-9  # geometry.py:32


class SfcKey:
    def __init__(self, value: int, depth: int):
        self.value, self.depth = value, depth

    def __eq__(self, other):
        return (self.value, self.depth) == (other.value, other.depth)

    def __repr__(self):
        return f"SfcKey(value={self.value}, depth={self.depth})"


def hilbert_keys(points, box: BoundingBox, depth: int | None = None, device="cuda"):
    pts = np.asarray(points, dtype=np.float64)
    if pts.ndim != 2:
        raise GeometryError("points must be an (n, d) array")
    d = pts.shape[1]
    if depth is None:
        if d not in DEFAULT_DEPTH:
            raise GeometryError(f"unsupported dimension {d}")
        depth = DEFAULT_DEPTH[d]
    if pts.shape[1] != box.dim:
        raise GeometryError("points must be (n, d) matching the box dimension")
    if depth < 1:
        raise GeometryError("curve depth must be >= 1")
    if d not in (2, 3):
        raise GeometryError(f"unsupported dimension {d}")
    if d * depth > 62:
        raise GeometryError(f"depth {depth} out of range for dimension {d}")
    ext = box.hi - box.lo
    margin = _CLAMP_RTOL * np.maximum(ext, 1.0)
    if ((pts < box.lo - margin) | (pts > box.hi + margin)).any():
        raise GeometryError("point lies outside the box")
    n = pts.shape[0]
    if n == 0:
        return np.zeros(0, dtype=np.uint64)
    dev = torch.device(device)
    p = torch.from_numpy(np.ascontiguousarray(pts)).to(dev)
    lohi = torch.from_numpy(np.concatenate([box.lo, box.hi])).to(dev)
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    N.call("gp_hilbert_keys", p.data_ptr(), n, d, d, 1, lohi.data_ptr(), depth,
           keys.data_ptr(), None, 0, torch.cuda.current_stream(dev).cuda_stream)
    return keys.cpu().numpy().view(np.uint64)


def hilbert_key(p, box: BoundingBox, depth: int | None = None) -> SfcKey:
    p = np.asarray(p, dtype=np.float64)
    if p.ndim != 1:
        raise GeometryError("expected a single point")
    d = p.shape[0]
    if depth is None:
        if d not in DEFAULT_DEPTH:
            raise GeometryError(f"unsupported dimension {d}")
        depth = DEFAULT_DEPTH[d]
    return SfcKey(value=int(hilbert_keys(p[None, :], box, depth)[0]), depth=depth)
