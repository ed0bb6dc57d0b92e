"""Device-side balance decisions (gp_balance_decide) and the device center grid."""
import ctypes

import pytest

from conftest import has_cuda

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_cuda():
        pytest.fail("CUDA device required for -m gpu tests")


@pytest.mark.parametrize("k,weights", [(16, None), (300, "int")])
def test_balance_drivers_bit_identical(monkeypatch, k, weights):
    """The balance-round drivers (host loop with on-device decisions, host loop with
    host numpy decisions) give the same partition, state and per-iteration records
    bit for bit, and the oracle's."""
    import numpy as np

    from oracle import geographer_oracle as O
    from paper_1805_01208_b200 import KMeansSettings, balanced_kmeans_points

    rng = np.random.default_rng(5)
    pts = rng.random((40_000, 2))
    w = rng.integers(1, 7, 40_000).astype(float) if weights else None
    s = KMeansSettings(k=k, seed=0, max_iter=10)
    runs = {}
    for mode in ("0", "host"):
        monkeypatch.setenv("GP_DEVICE_DECIDE", "0" if mode == "host" else "1")
        runs[mode] = balanced_kmeans_points(pts, w, s, return_stats=True)
    ref = O.run(pts, w, O.Knobs(k=k, seed=0, max_iter=10), scan_chunks=16)
    for mode, (part, stats) in runs.items():
        assert np.array_equal(part.assignment, ref.assignment), mode
        assert np.array_equal(stats.final_state.centers, ref.centers), mode
        assert np.array_equal(stats.final_state.influence, ref.influence), mode
        for g, r in zip(stats.iterations, ref.records):
            for key in ("balance_rounds", "imbalance", "total_decisions", "active_points"):
                assert vars(g)[key] == r[key], (mode, key)
        base = runs["0"][1]
        assert [vars(i)["skip_decisions"] for i in stats.iterations] == \
            [vars(i)["skip_decisions"] for i in base.iterations], mode


def test_balance_decide_matches_host_numpy():
    """gp_balance_decide reproduces the host round decision bit for bit: imbalance,
    stop test, step halving after the second regression, next influences."""
    import numpy as np
    import torch

    from paper_1805_01208_b200 import _native as N
    from paper_1805_01208_b200.control import imbalance, influence_factor

    rng = np.random.default_rng(3)
    k, scale, eps, mr = 777, 4.0, 0.03, 20
    infl = rng.uniform(0.8, 1.25, k)
    bal = torch.zeros(8 + 3 * mr, dtype=torch.float64, device="cuda")
    bal[0], bal[2] = 0.05, float("inf")
    cur = torch.from_numpy(infl).cuda()
    nxt = torch.zeros(k, dtype=torch.float64, device="cuda")
    cap, best, regressions = 0.05, float("inf"), 0
    for rnd, spread in enumerate([0.3, 0.5, 0.6, 0.2, 0.01]):
        units = rng.integers(1000, int(1000 * (1 + spread)) + 2, k).astype(np.int64)
        units[rng.integers(0, k)] = 0                          # an empty block
        red = torch.from_numpy(np.concatenate([units, [11, 22, 33]])).cuda()
        N.check(N.lib.gp_balance_decide(red.data_ptr(), k, scale, eps, mr, bal.data_ptr(),
                                        cur.data_ptr(), nxt.data_ptr(), None), "decide")
        torch.cuda.synchronize()
        b = bal.cpu().numpy()
        bw = units.astype(np.float64) / scale
        imb = imbalance(bw)
        assert b[8 + rnd] == imb
        stop = imb <= eps or rnd == mr - 1
        assert bool(b[5]) == stop
        if stop:
            break
        if imb > best:
            regressions += 1
            if regressions >= 2:
                cap *= 0.5
        best = min(best, imb)
        target = float(bw.sum()) / k
        want = infl * influence_factor(bw, target, cap, 2)
        assert np.array_equal(nxt.cpu().numpy(), want)
        assert b[0] == cap
        infl = want
        cur.copy_(nxt)


def test_center_grid_matches_host_build():
    """gp_center_grid: the cell counts and per-cell center sets of the host numpy build."""
    import numpy as np
    import torch

    from paper_1805_01208_b200 import _native as N

    rng = np.random.default_rng(4)
    for d, k, G in ((2, 5000, 50), (3, 999, 8), (2, 3, 1)):
        centers = rng.random((k, d))
        lo, h = np.zeros(d), 1.0 / G * (1 + 1e-12)
        cell = np.clip(np.floor((centers - lo) / h).astype(np.int64), 0, G - 1)
        flat = cell[:, 0]
        for j in range(1, d):
            flat = flat * G + cell[:, j]
        start = np.zeros(G ** d + 1, dtype=np.int64)
        np.cumsum(np.bincount(flat, minlength=G ** d), out=start[1:])
        items = np.argsort(flat, kind="stable")
        wsb = N.size_query("gp_center_grid_workspace_bytes", k)
        ws = torch.empty(wsb, dtype=torch.uint8, device="cuda")
        out = torch.empty(G ** d + 1 + k, dtype=torch.int32, device="cuda")
        lo3 = (ctypes.c_double * 3)(*list(lo) + [0.0] * (3 - d))
        c_d = torch.from_numpy(centers).cuda()
        N.check(N.lib.gp_center_grid(c_d.data_ptr(), k, d, lo3, h, G, out.data_ptr(),
                                     out.data_ptr() + 4 * (G ** d + 1), ws.data_ptr(), wsb,
                                     None), "grid")
        o = out.cpu().numpy()
        assert np.array_equal(o[:G ** d + 1], start)
        assert np.array_equal(o[G ** d + 1:], items)   # stable radix sort == stable argsort
