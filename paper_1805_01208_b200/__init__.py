"""B200-native Geographer balanced k-means hot path (arXiv 1805.01208).

Drop-in for the reference package's partition entry points
(geopart.kmeans.balanced_kmeans_points / balanced_kmeans) with the n-sized
work in hand-written sm_100a CUDA behind a C ABI (include/geopart_b200.h).

Importing the value types and host control math works anywhere; the entry
points load the native library on first use and raise if it is missing.
"""

from .types import (  # noqa: F401
    BalanceInfo,
    BoundingBox,
    ClusterState,
    GeometryError,
    GraphError,
    IterationRecord,
    KMeansSettings,
    KMeansStats,
    Partition,
    PointBounds,
)
from .control import (  # noqa: F401
    adapt_influence,
    balance_target,
    effective_distance,
    erode_influence,
    imbalance,
    initial_center_positions,
    relax_bounds,
)

__version__ = "0.1.0"

_LAZY = {
    "balanced_kmeans_points": "kmeans",
    "balanced_kmeans": "kmeans",
    "partition_device": "kmeans",
    "RankWorld": "kmeans",
    "hilbert_keys": "geometry",
    "hilbert_key": "geometry",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(name)
    import importlib

    return getattr(importlib.import_module(f".{mod}", __name__), name)


__all__ = [
    "KMeansSettings", "ClusterState", "PointBounds", "BalanceInfo", "IterationRecord",
    "KMeansStats", "Partition", "BoundingBox", "GeometryError", "GraphError",
    "balanced_kmeans_points", "balanced_kmeans", "partition_device", "RankWorld",
    "hilbert_keys", "hilbert_key", "adapt_influence", "erode_influence", "relax_bounds",
    "effective_distance", "initial_center_positions", "imbalance", "balance_target",
]
