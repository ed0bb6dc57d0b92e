"""SFC baseline partitioner on the device (reference baselines.py:62-101).

sfc_labels cuts the Hilbert-sorted vertex sequence at weight multiples of
total/k.  On B200 it reuses the partition path's bootstrap kernels (K1 box, K2
keys, K3 stable radix sort) and adds one cut step (gp_sfc_cut), so the labels
equal the reference's bit for bit:

    keys  = hilbert_keys(coords, BoundingBox.of_points(coords), depth)  # K1+K2
    order = lexsort((arange(n), keys))                                    # K3
    before = cumsum(w[order]) - w[order];  total = w.sum()                # gp_sfc_cut
    labels[order] = minimum((before * k / total).astype(int64), k - 1)

rcb_labels / rcb_partition (baselines.py:14-59) are not part of this build
(DESIGN.md §7).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native as N
from .control import imbalance
from .geometry import DEFAULT_DEPTH
from .types import GeometryError, Partition

__all__ = ["sfc_labels", "sfc_partition"]


def _weight_scale(w: torch.Tensor | None, n: int, sh) -> float:
    """Exact fixed-point scale of the weights (gp_weight_probe), 0.0 if none exists."""
    if w is None:
        return 1.0
    out = torch.empty(3, dtype=torch.int64, device=w.device)
    N.call("gp_weight_probe", w.data_ptr(), n, out.data_ptr(), sh)
    flags, low, mx_bits = (int(v) for v in out.cpu().tolist())
    if flags & 1:
        return 0.0  # non-finite weights: the literal summation orders reproduce numpy's NaN/inf
    mx = np.array([mx_bits], dtype=np.int64).view(np.float64)[0]
    s = max(0, -low) if low < 4096 else 0
    # every |w|*2^s is an integer and any partial sum stays below 2^53 units
    return 2.0 ** s if s <= 1000 and mx * 2.0 ** s * n < 2.0 ** 53 else 0.0


def sfc_labels_device(coords, weights, k: int, depth: int | None = None, device=None):
    """Device int64 labels by original vertex id (see sfc_labels)."""
    dev = torch.device(device if device is not None else "cuda")
    if isinstance(coords, torch.Tensor):
        pts = coords.to(device=dev, dtype=torch.float64)
    else:
        pts = torch.from_numpy(np.ascontiguousarray(np.asarray(coords, dtype=np.float64))).to(dev)
    if pts.dim() != 2:
        raise GeometryError("points must be an (n, d) array")
    n, d = pts.shape
    if not 1 <= k <= n:
        raise ValueError(f"k={k} out of range 1..{n}")
    if depth is None:
        depth = DEFAULT_DEPTH.get(d)
        if depth is None:
            raise GeometryError(f"unsupported dimension {d}")
    if d not in (2, 3):
        raise GeometryError(f"unsupported dimension {d}")
    if depth < 1:
        raise GeometryError("curve depth must be >= 1")
    if d * depth > 62:
        raise GeometryError(f"depth {depth} out of range for dimension {d}")
    w = None
    if weights is not None:
        if isinstance(weights, torch.Tensor):
            w = weights.to(device=dev, dtype=torch.float64).contiguous()
        else:
            w = torch.from_numpy(np.ascontiguousarray(np.asarray(weights, dtype=np.float64)))
            w = w.to(dev)
        if w.shape != (n,):
            raise ValueError(f"weights must have shape ({n},)")
    sh = torch.cuda.current_stream(dev).cuda_stream
    sp, sd = pts.stride()
    # K1: BoundingBox.of_points (baselines.py:82)
    lohi = torch.empty(2 * d, dtype=torch.float64, device=dev)
    bad = torch.empty(1, dtype=torch.int32, device=dev)
    N.call("gp_box_minmax", pts.data_ptr(), n, d, sp, sd, lohi.data_ptr(), bad.data_ptr(), sh)
    if int(bad.item()):
        raise GeometryError("non-finite box corner")
    # K2 + K3: keys and lexsort((arange(n), keys)) (baselines.py:82-83)
    keys = torch.empty(n, dtype=torch.int64, device=dev)
    gids = torch.empty(n, dtype=torch.int32, device=dev)
    N.call("gp_hilbert_keys", pts.data_ptr(), n, d, sp, sd, lohi.data_ptr(), depth,
           keys.data_ptr(), gids.data_ptr(), 0, sh)
    keys_s = torch.empty_like(keys)
    gids_s = torch.empty_like(gids)
    wsb = N.size_query("gp_sort_workspace_bytes", n)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    N.call("gp_sort_pairs", keys.data_ptr(), gids.data_ptr(), keys_s.data_ptr(),
           gids_s.data_ptr(), n, d * depth, ws.data_ptr(), wsb, sh)
    del keys, keys_s, gids, ws
    # the cut (baselines.py:84-89)
    scale = _weight_scale(w, n, sh)
    cwb = N.size_query("gp_sfc_cut_workspace_bytes", n)
    cws = torch.empty(max(cwb, 1), dtype=torch.uint8, device=dev)
    labels = torch.empty(n, dtype=torch.int64, device=dev)
    N.call("gp_sfc_cut", gids_s.data_ptr(), None if w is None else w.data_ptr(), n, int(k),
           float(scale), labels.data_ptr(), cws.data_ptr(), cwb, sh)
    return labels


def sfc_labels(coords: np.ndarray, weights: np.ndarray, k: int,
               depth: int | None = None) -> np.ndarray:
    """Cut the Hilbert-sorted vertex sequence at weight multiples of total/k
    (baselines.py:62-89): a vertex whose prefix weight (weight strictly before it
    in curve order) is w lands in block floor(w * k / total), clipped to k-1."""
    coords = np.asarray(coords, dtype=np.float64)
    weights = np.asarray(weights, dtype=np.float64)
    return sfc_labels_device(coords, weights, k, depth).cpu().numpy()


def sfc_partition(graph, k: int, depth: int | None = None,
                  epsilon: float | None = None) -> Partition:
    """Space-filling-curve partition of a graph's vertex set (baselines.py:92-101)."""
    labels = sfc_labels(graph.coords, graph.vertex_weights, k, depth)
    bw = np.bincount(labels, weights=graph.vertex_weights, minlength=k)
    failed = imbalance(bw) > epsilon if epsilon is not None else False
    return Partition(assignment=labels, k=k, balance_failed=failed,
                     empty_blocks=np.flatnonzero(bw == 0))
