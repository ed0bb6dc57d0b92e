"""Host control math and API validation (no GPU): same behaviour as the reference."""
import math

import numpy as np
import pytest

from paper_1805_01208_b200 import (
    ClusterState, KMeansSettings, PointBounds, adapt_influence, erode_influence,
    initial_center_positions, relax_bounds, imbalance, effective_distance,
)
from paper_1805_01208_b200.control import BoundMaps, sample_schedule
from paper_1805_01208_b200.numerics import einsum_order3


def st(influence, weights=None, dim=2, moves=None):
    k = len(influence)
    return ClusterState(np.zeros((k, dim)), np.asarray(influence, float),
                        np.asarray(weights if weights is not None else np.ones(k), float),
                        np.asarray(moves if moves is not None else np.zeros(k), float))


def test_settings_validation_matches_reference():
    for bad in (dict(k=0), dict(k=2, epsilon=-0.1), dict(k=2, influence_step_cap=1.5),
                dict(k=2, max_iter=0), dict(k=2, delta_threshold=-1.0), dict(k=2, init_sample=-1),
                dict(k=2, sfc_depth=0)):
        with pytest.raises(ValueError):
            KMeansSettings(**bad)


def test_frozen_influence_constants():
    # reference tests/test_influence.py:77-107, :140-152
    assert adapt_influence(st([1.0], [200.0]), 100.0, 0.05).influence[0] == 0.95
    v = adapt_influence(st([1.0], [104.0]), 100.0, 0.05).influence[0]
    assert v == pytest.approx(0.9805806756909202, rel=1e-10)
    assert adapt_influence(st([1.0, 1.0], [0.0, 200.0]), 100.0, 0.05).influence[0] == 1.05
    v3 = adapt_influence(st([1.0], [104.0], dim=3), 100.0, 0.05).influence[0]
    assert v3 == pytest.approx((100.0 / 104.0) ** (1.0 / 3.0), rel=1e-10)
    e = erode_influence(st([4.0], moves=[1.0]), beta=1.0).influence[0]
    assert e == pytest.approx(2.1078404750300304, rel=1e-10)
    assert list(initial_center_positions(100, 4)) == [12, 37, 62, 87]
    assert effective_distance(np.zeros(2), np.array([0.0, 2.0]), 2.0) == 1.0


def test_control_math_bit_identical_to_oracle():
    from oracle import geographer_oracle as O

    rng = np.random.default_rng(7)
    for dim in (2, 3):
        infl = rng.uniform(0.05, 20, 1000)
        bw = rng.uniform(0, 1e6, 1000)
        bw[::17] = 0
        a = adapt_influence(st(infl, bw, dim=dim), 1234.5, 0.05).influence
        b = O.adapted_influence(infl, bw, 1234.5, 0.05, dim)
        assert np.array_equal(a, b)
    moves = rng.uniform(0, 5, 1000)
    assert np.array_equal(erode_influence(st(infl, moves=moves), 2.5).influence,
                          O.eroded_influence(infl, moves, 2.5))
    w = rng.integers(1, 9, 64).astype(float)
    assert imbalance(w) == O.imbalance(w)


def test_relax_bounds_identity_and_floor():
    b = PointBounds(np.array([1.5, 2.0]), np.array([0.5, 0.25]))
    infl = np.array([1.0, 2.0])
    out = relax_bounds(b, np.array([0, 1]), infl, infl.copy(), np.zeros(2))
    assert out is b
    out = relax_bounds(PointBounds(np.array([1.0]), np.array([0.5])), np.array([0]),
                       np.ones(1), np.ones(1), np.array([10.0]))
    assert out.lower[0] == 0.0 and out.upper[0] == pytest.approx(11.0, rel=1e-9)


def _f32(x):
    return np.asarray(x, dtype=np.float32)


def test_lazy_bound_maps_are_sound_against_eager_relaxation():
    """Device float32 bound arithmetic (emulated in float64 on the outward-rounded
    parameters) never gives a tighter bound than the reference's eager relaxation."""
    rng = np.random.default_rng(3)
    k, m = 7, 400
    maps = BoundMaps(k)
    a = rng.integers(0, k, m)
    best = rng.uniform(0.0, 1.0, m)
    best[:20] = 0.0  # points sitting on their center (cancellation case)
    second = best + rng.uniform(0.0, 1.0, m)
    ub_eager, lb_eager = best.copy(), second.copy()
    ev, nm, la, lb, linv, lblo = maps.device_params()
    num = best - nm[a, 2].astype(np.float64)
    ub_t = num * np.where(num >= 0, nm[a, 0], nm[a, 1]).astype(np.float64)
    ub_t = np.nextafter(ub_t.astype(np.float32), np.float32(np.inf)).astype(np.float64)
    lb_t = (second + lblo) * linv
    lb_t = np.nextafter(lb_t.astype(np.float32), np.float32(-np.inf)).astype(np.float64)
    infl = np.ones(k)
    for step in range(300):
        new = infl * rng.uniform(0.95, 1.05, k)
        moves = rng.uniform(0, 0.01, k) * (step % 3 == 0)
        b2 = relax_bounds(PointBounds(ub_eager, lb_eager), a, infl, new, moves)
        ub_eager, lb_eager = b2.upper, b2.lower
        maps.relax(infl, new, moves)
        infl = new
        ev, nm, la, lb, linv, lblo = maps.device_params()
        E = ev[a].astype(np.float64)
        ub_lazy = np.where(ub_t >= 0, E[:, 0], E[:, 1]) * ub_t + E[:, 2]
        lb_lazy = np.maximum(la * lb_t - lb, 0.0)
        assert np.all(ub_lazy >= ub_eager * (1 - 1e-12))
        assert np.all(lb_lazy <= lb_eager * (1 + 1e-12) + 1e-300)
        # and still tight to float32 precision
        assert np.all(ub_lazy <= ub_eager * (1 + 1e-5) + 1e-6)


def test_sample_schedule():
    assert sample_schedule(100000, 100) == [100 * 2 ** j for j in range(10)]
    assert sample_schedule(100, 100) == []
    assert sample_schedule(5000, 0) == []


def test_einsum_order_probe():
    assert einsum_order3() in (0, 1, 2)


def test_row_norms_bit_identical_to_linalg_norm():
    import numpy as np

    from paper_1805_01208_b200.control import row_norms

    rng = np.random.default_rng(12)
    for d in (2, 3):
        for scale in (1e-9, 1.0, 1e7):
            x = (rng.random((20_000, d)) - 0.5) * scale
            x[:7] = 0.0
            assert np.array_equal(row_norms(x), np.linalg.norm(x, axis=1))
