"""`balanced_kmeans_points(..., p)` with p > 1 drives p GPU workers (pool.py).

On a one-GPU box the workers share GPU 0 (GP_POOL_SHARE_GPU=1, gloo collectives
through the host); the sharded run must equal the single-GPU run bit for bit
(ACCEPT-07, pkg/tests/test_acceptance.py:213-231: identical partitions for every
rank count), and argument errors must surface from the pool the way the
single-GPU path raises them, leaving the pool usable.
"""
import numpy as np
import pytest

from conftest import has_cuda

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _shared_pool():
    if not has_cuda():
        pytest.fail("CUDA device required for -m gpu tests")
    mp = pytest.MonkeyPatch()
    mp.setenv("GP_POOL_SHARE_GPU", "1")
    yield
    from paper_1805_01208_b200 import pool

    pool.shutdown()
    mp.undo()


@pytest.mark.parametrize("p,dim,weighted,k", [(2, 2, True, 24), (3, 3, False, 150),
                                              (4, 2, False, 300)])
def test_pool_bit_identical_to_one_gpu(p, dim, weighted, k):
    from paper_1805_01208_b200 import KMeansSettings, balanced_kmeans_points

    rng = np.random.default_rng(40 + p)
    n = 90_001
    pts = rng.random((n, dim))
    w = rng.integers(1, 7, n).astype(float) if weighted else None
    s = KMeansSettings(k=k, seed=1, max_iter=12)
    a1, st1 = balanced_kmeans_points(pts, w, s, p=1, return_stats=True)
    ap, stp = balanced_kmeans_points(pts, w, s, p=p, return_stats=True)
    assert np.array_equal(ap.assignment, a1.assignment)
    assert np.array_equal(stp.final_state.centers, st1.final_state.centers)
    assert np.array_equal(stp.final_state.influence, st1.final_state.influence)
    assert np.array_equal(stp.final_state.block_weights, st1.final_state.block_weights)
    assert ap.balance_failed == a1.balance_failed
    for g, r in zip(stp.iterations, st1.iterations):
        for key in ("phase", "active_points", "balance_rounds", "imbalance", "total_decisions",
                    "max_move"):
            assert vars(g)[key] == vars(r)[key], key


def test_pool_errors_match_single_gpu_and_pool_survives():
    from paper_1805_01208_b200 import GeometryError, KMeansSettings, balanced_kmeans_points
    from paper_1805_01208_b200 import pool

    rng = np.random.default_rng(0)
    with pytest.raises(GeometryError):
        balanced_kmeans_points(rng.random((500, 4)), None, KMeansSettings(k=3), p=2)
    with pytest.raises(ValueError):
        balanced_kmeans_points(rng.random((5, 2)), None, KMeansSettings(k=6), p=2)
    with pytest.raises(IndexError):
        balanced_kmeans_points(rng.random((50, 2)), np.ones(40), KMeansSettings(k=3), p=2)
    bad = rng.random((400, 2))
    bad[7, 0] = np.inf
    with pytest.raises(GeometryError):
        balanced_kmeans_points(bad, None, KMeansSettings(k=3), p=2)
    assert pool._POOL is not None and pool._POOL.alive()
    pts = rng.random((3000, 2))
    a = balanced_kmeans_points(pts, None, KMeansSettings(k=5), p=2).assignment
    b = balanced_kmeans_points(pts, None, KMeansSettings(k=5), p=1).assignment
    assert np.array_equal(a, b)
