"""The reference-side shim (paper_1805_01208_b200.integration) on CPU: names swapped in
a module namespace, results converted to the reference's Partition type."""

from dataclasses import dataclass, field

import numpy as np

from paper_1805_01208_b200 import integration
from paper_1805_01208_b200.types import KMeansStats, Partition


@dataclass
class RefPartition:  # stands in for geopart.graph.Partition (graph.py:131-150)
    assignment: np.ndarray
    k: int
    balance_failed: bool = False
    empty_blocks: np.ndarray = field(default_factory=lambda: np.array([], dtype=np.int64))


def test_install_swaps_namespace_names():
    ns = {"balanced_kmeans_points": "ref_bkp", "balanced_kmeans": "ref_bk", "other": 1}
    old = integration.install(ns)
    assert old == {"balanced_kmeans_points": "ref_bkp", "balanced_kmeans": "ref_bk"}
    from paper_1805_01208_b200 import kmeans as bk

    assert ns["balanced_kmeans_points"].__wrapped__ is bk.balanced_kmeans_points
    assert ns["balanced_kmeans"].__wrapped__ is bk.balanced_kmeans
    assert ns["other"] == 1


def test_results_become_reference_partitions():
    p = Partition(assignment=np.array([0, 1, 1]), k=3, balance_failed=True,
                  empty_blocks=np.array([2]))
    calls = {}
    f = integration.wrap(lambda *a, **kw: p, RefPartition, calls, "balanced_kmeans_points")
    r = f()
    assert isinstance(r, RefPartition) and r.k == 3 and r.balance_failed
    assert np.array_equal(r.assignment, p.assignment)
    assert np.array_equal(r.empty_blocks, [2])
    st = KMeansStats()
    g = integration.wrap(lambda *a, **kw: (p, st), RefPartition, calls, "balanced_kmeans_points")
    r2, s2 = g()
    assert isinstance(r2, RefPartition) and s2 is st
    assert calls["balanced_kmeans_points"] == 2
