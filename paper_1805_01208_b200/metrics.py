"""Partition quality metrics on the GPU (the reference's metrics.py):
edge cut, communication volume, balance, per-block diameter lower bounds.

Same functions, results and report type as the reference.  The n- and m-sized passes are
the kernels of csrc/graphs.cu behind the C ABI; only k-sized arithmetic stays in numpy:

  edge_cut                      gp_edge_cut      (metrics.py:48-60)
  comm_volumes                  gp_comm_volumes  (metrics.py:63-77)
  Partition.block_weights       gp_block_weights (graph.py:165-166)
  block_diameter_lower_bounds   gp_block_bfs + gp_block_level_top (metrics.py:121-168):
                                the reference's BFS sweeps of one block after another
                                run here for all blocks at once (five sweeps in all)
"""

from __future__ import annotations

import json
import math
from dataclasses import asdict, dataclass

import numpy as np

from .control import balance_target, imbalance  # noqa: F401  (same definitions as metrics.py)
from .types import GraphError, Partition

__all__ = [
    "balance_target", "imbalance", "edge_cut", "comm_volumes", "block_diameter_lower_bounds",
    "block_weights", "geometric_mean", "harmonic_mean_diameters", "MetricsReport", "evaluate",
    "DeviceGraph",
]


class DeviceGraph:
    """CSR arrays of a graph and a partition's labels in device memory, uploaded once
    per evaluate() and shared by the metric kernels."""

    def __init__(self, graph, partition=None):
        import torch

        self.n = int(graph.n)
        self.nnz = int(graph.neighbors.shape[0])
        self.offsets = _dev(graph.offsets, np.int64)
        self.neighbors = _dev(graph.neighbors, np.int64) if self.nnz else \
            torch.empty(1, dtype=torch.int64, device="cuda")
        self.edge_weights = None if graph.edge_weights is None else \
            _dev(graph.edge_weights, np.float64)
        self.vertex_weights = _dev(graph.vertex_weights, np.float64)
        self.labels = None
        if partition is not None:
            self.set_partition(partition)

    def set_partition(self, partition):
        a = np.asarray(partition.assignment)
        self.labels = _dev(a, np.int32)
        self.k = int(partition.k)


def _dev(x, dtype):
    import torch

    from . import staging

    a = np.ascontiguousarray(x, dtype=dtype)
    out = torch.empty(a.shape, dtype=torch.from_numpy(a[:0]).dtype, device="cuda")
    if a.size:
        staging.h2d_into(out, a)
    return out


def _stream():
    import torch

    return torch.cuda.current_stream().cuda_stream


def _exact_scale(w, n: int) -> float:
    """2^s with every w * 2^s an integer and any partial sum below 2^53 units, or 0.0
    (gp_weight_probe; the exact int64 accumulation then equals numpy's fp64 sums)."""
    import torch

    from . import _native as N

    if w is None or n == 0:
        return 1.0
    out = torch.empty(3, dtype=torch.int64, device="cuda")
    N.call("gp_weight_probe", w.data_ptr(), n, out.data_ptr(), _stream())
    flags, low, mx_bits = (int(v) for v in out.cpu().tolist())
    if flags & 1:
        return 0.0
    mx = np.array([mx_bits], dtype=np.int64).view(np.float64)[0]
    s = max(0, -low) if low < 4096 else 0
    return 2.0 ** s if s <= 1000 and mx * 2.0 ** s * n < 2.0 ** 53 else 0.0


def _on_device(graph, partition) -> DeviceGraph:
    if isinstance(graph, DeviceGraph):
        if partition is not None and graph.labels is None:
            graph.set_partition(partition)
        return graph
    return DeviceGraph(graph, partition)


def edge_cut(graph, partition: Partition) -> float:
    """Total weight of edges whose endpoints lie in different blocks; each undirected
    edge counted once, unweighted edges count 1 (metrics.py:48-60)."""
    import torch

    from . import _native as N

    if not isinstance(graph, DeviceGraph):
        partition.validate(graph.n)
    g = _on_device(graph, partition)
    wsb = N.size_query("gp_edge_cut_workspace_bytes", g.n, g.nnz)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    out = torch.empty(1, dtype=torch.float64, device="cuda")
    scale = _exact_scale(g.edge_weights, g.nnz)
    N.call("gp_edge_cut", g.offsets.data_ptr(), g.neighbors.data_ptr(),
           None if g.edge_weights is None else g.edge_weights.data_ptr(), float(scale),
           g.labels.data_ptr(), g.n, g.nnz, out.data_ptr(), ws.data_ptr(), wsb, _stream())
    return float(out.item())


def comm_volumes(graph, partition: Partition):
    """(max_volume, total_volume, per_block): a vertex contributes, to its own block, the
    number of OTHER blocks among its neighbors (metrics.py:63-77)."""
    import torch

    from . import _native as N

    if not isinstance(graph, DeviceGraph):
        partition.validate(graph.n)
    g = _on_device(graph, partition)
    per = torch.empty(g.k, dtype=torch.int64, device="cuda")
    scratch = torch.empty(g.n + 1, dtype=torch.int64, device="cuda")
    N.call("gp_comm_volumes", g.offsets.data_ptr(), g.neighbors.data_ptr(), g.labels.data_ptr(),
           g.n, g.k, per.data_ptr(), scratch.data_ptr(), _stream())
    per_block = per.cpu().numpy().astype(np.float64)
    return float(per_block.max()), float(per_block.sum()), per_block


def block_weights(graph, partition: Partition) -> np.ndarray:
    """partition.block_weights(graph.vertex_weights) (graph.py:165-166) on the device."""
    import torch

    from . import _native as N

    g = _on_device(graph, partition)
    wsb = N.size_query("gp_block_weights_workspace_bytes", g.n, g.k)
    ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
    out = torch.empty(g.k, dtype=torch.float64, device="cuda")
    scale = _exact_scale(g.vertex_weights, g.n)
    N.call("gp_block_weights", g.vertex_weights.data_ptr(), g.labels.data_ptr(), g.n, g.k,
           float(scale), out.data_ptr(), ws.data_ptr(), wsb, _stream())
    return out.cpu().numpy()


def block_diameter_lower_bounds(graph, partition: Partition,
                                refinement_rounds: int = 3) -> np.ndarray:
    """Per-block diameter lower bounds in hop distance (metrics.py:121-168): a double
    sweep (BFS from the block's lowest-id vertex, then from the farthest vertex found)
    and up to ``refinement_rounds`` more sweeps rooted at the deepest vertices of the
    second one.  A disconnected or empty block gets inf."""
    import torch

    from . import _native as N

    if not isinstance(graph, DeviceGraph):
        partition.validate(graph.n)
    g = _on_device(graph, partition)
    k, n, sh = g.k, g.n, _stream()
    level = torch.empty(n, dtype=torch.int32, device="cuda")
    key = torch.empty(k, dtype=torch.int64, device="cuda")      # uint64 bit patterns < 2^63
    LOW = (1 << 32) - 1
    sizes = torch.bincount(g.labels.to(torch.int64), minlength=k)
    qbase = torch.zeros(k + 1, dtype=torch.int64, device="cuda")
    qbase[1:] = torch.cumsum(sizes, 0)
    queue = torch.empty(n, dtype=torch.int64, device="cuda")

    def bfs(roots, lev):
        """one sweep of every block: (largest level, its lowest vertex, vertices reached)"""
        depth = torch.empty(k, dtype=torch.int32, device="cuda")
        far = torch.empty(k, dtype=torch.int64, device="cuda")
        reached = torch.empty(k, dtype=torch.int64, device="cuda")
        N.call("gp_block_bfs", g.offsets.data_ptr(), g.neighbors.data_ptr(), g.labels.data_ptr(),
               n, k, roots.data_ptr(), qbase.data_ptr(), queue.data_ptr(), lev.data_ptr(),
               depth.data_ptr(), far.data_ptr(), reached.data_ptr(), sh)
        return depth.to(torch.int64), far, reached

    def top(lev, exclude=None, below=None):
        """per block: (key, vertex) of the deepest vertex, lowest id first"""
        N.call("gp_block_level_top", lev.data_ptr(), g.labels.data_ptr(), n, k,
               None if exclude is None else exclude.data_ptr(),
               None if below is None else below.data_ptr(), key.data_ptr(), None, sh)
        kk = key.clone()
        vert = LOW - (kk & LOW)
        return kk, torch.where(kk > 0, vert, torch.full_like(vert, -1))

    # lowest-id member of every block: the deepest-vertex key of an all-unreached array
    level.fill_(-1)
    _, first = top(level)
    _, a, reached = bfs(first, level)
    disconnected = reached < sizes
    lev_a = torch.empty_like(level)
    best, _, _ = bfs(a, lev_a)
    # fringe refinement: the next deepest vertices of the second sweep, low id first
    below = torch.full((k,), torch.iinfo(torch.int64).max, dtype=torch.int64, device="cuda")
    for _ in range(max(0, int(refinement_rounds))):
        kr, root = top(lev_a, exclude=a, below=below)
        if not bool((root >= 0).any().item()):
            break
        below = kr  # 0 where the block has no further vertex: nothing lies below it
        ecc, _, _ = bfs(root, level)
        best = torch.where(root >= 0, torch.maximum(best, ecc), best)
    out = best.to(torch.float64)
    out = torch.where(disconnected | (sizes == 0), torch.full_like(out, math.inf), out)
    out = torch.where(sizes == 1, torch.zeros_like(out), out)
    return out.cpu().numpy()


def geometric_mean(values) -> float:
    v = np.asarray(values, dtype=np.float64)
    if v.size == 0 or not (v > 0).all():
        raise ValueError("geometric mean needs positive values")
    return float(np.exp(np.mean(np.log(v))))


def harmonic_mean_diameters(values) -> float:
    """Harmonic mean where unbounded (inf) entries contribute 0 reciprocal."""
    v = np.asarray(values, dtype=np.float64)
    if v.size == 0 or (v < 0).any():
        raise ValueError("harmonic mean needs nonnegative values")
    with np.errstate(divide="ignore"):
        recip = np.where(np.isinf(v), 0.0, np.divide(1.0, v))
    denom = recip.sum()
    return math.inf if denom == 0.0 else float(v.size / denom)


def _fmt(x) -> str:
    if isinstance(x, float) and math.isinf(x):
        return "unbounded"
    if isinstance(x, float) and x.is_integer():
        return str(int(x))
    return repr(x)


def _json_num(x):
    return "unbounded" if isinstance(x, float) and math.isinf(x) else x


@dataclass
class MetricsReport:
    """Quality summary of one partition of one graph (metrics.py:198-250)."""

    n: int
    m: int
    k: int
    edge_cut: float
    comm_max: float
    comm_total: float
    imbalance: float
    harmonic_diameter: float
    block_weights: list
    block_comm: list
    block_diameters: list

    def to_text(self) -> str:
        head = [("vertices", self.n), ("edges", self.m), ("blocks", self.k),
                ("edge_cut", self.edge_cut), ("comm_max", self.comm_max),
                ("comm_total", self.comm_total), ("imbalance", self.imbalance),
                ("harmonic_diameter", self.harmonic_diameter)]
        lines = [f"{name}: {_fmt(v) if isinstance(v, float) else v}" for name, v in head]
        lines += [f"block {i}: weight {_fmt(self.block_weights[i])} comm "
                  f"{_fmt(self.block_comm[i])} diameter {_fmt(self.block_diameters[i])}"
                  for i in range(self.k)]
        return "\n".join(lines)

    def to_json(self) -> str:
        d = asdict(self)
        d["harmonic_diameter"] = _json_num(d["harmonic_diameter"])
        d["block_diameters"] = [_json_num(x) for x in d["block_diameters"]]
        return json.dumps(d, indent=2)

    @classmethod
    def from_json(cls, text: str) -> "MetricsReport":
        d = json.loads(text)
        un = lambda x: math.inf if x == "unbounded" else float(x)  # noqa: E731
        d["harmonic_diameter"] = un(d["harmonic_diameter"])
        d["block_diameters"] = [un(x) for x in d["block_diameters"]]
        return cls(**d)


def evaluate(graph, partition: Partition, diameters: bool = True) -> MetricsReport:
    """The full metrics report for one (graph, partition) pair (metrics.py:253-281); the
    graph and the labels go to the device once."""
    partition.validate(graph.n)
    g = DeviceGraph(graph, partition)
    bw = block_weights(g, partition)
    cmax, ctot, per_block = comm_volumes(g, partition)
    if diameters:
        dia = block_diameter_lower_bounds(g, partition)
        harm = harmonic_mean_diameters(dia)
    else:
        dia = np.full(partition.k, np.nan)
        harm = math.nan
    if not float(bw.sum()) > 0:
        raise GraphError("total weight must be positive")
    return MetricsReport(
        n=graph.n, m=graph.m, k=partition.k, edge_cut=edge_cut(g, partition), comm_max=cmax,
        comm_total=ctot, imbalance=imbalance(bw), harmonic_diameter=harm,
        block_weights=[float(x) for x in bw], block_comm=[float(x) for x in per_block],
        block_diameters=[float(x) for x in dia])
