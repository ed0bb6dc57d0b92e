"""Device-resident loop graphs (gp_loop_graph_*): a conditional WHILE node whose
body is captured from stream work runs until a body kernel stops it."""
import ctypes

import pytest

from conftest import has_cuda

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not has_cuda():
        pytest.fail("CUDA device required for -m gpu tests")


def test_while_graph_countdown():
    import torch

    from paper_1805_01208_b200 import _native as N

    s = torch.cuda.Stream()
    cnt = torch.tensor([7], dtype=torch.int32, device="cuda")
    hits = torch.zeros(1, dtype=torch.int32, device="cuda")
    torch.cuda.synchronize()
    ctx = ctypes.c_void_p()
    N.check(N.lib.gp_loop_graph_begin(s.cuda_stream, ctypes.byref(ctx)), "begin")
    h = N.lib.gp_loop_graph_handle(ctx)
    with torch.cuda.stream(s):
        hits.add_(1)                       # torch work is captured into the body too
    N.check(N.lib.gp_loop_test_countdown(cnt.data_ptr(), h, s.cuda_stream), "countdown")
    N.check(N.lib.gp_loop_graph_end(ctx), "end")
    for rep in range(2):
        cnt.fill_(7 + rep)
        hits.zero_()
        torch.cuda.synchronize()
        N.check(N.lib.gp_loop_graph_launch(ctx, s.cuda_stream), "launch")
        s.synchronize()
        assert int(cnt.item()) == 0
        assert int(hits.item()) == 7 + rep
    N.lib.gp_loop_graph_destroy(ctx)


@pytest.mark.parametrize("k,weights", [(16, None), (300, "int")])
def test_balance_graph_modes_bit_identical(monkeypatch, k, weights):
    """The balance-round drivers (loop graph in every phase or the full phase only,
    host loop with on-device decisions, host loop with host numpy decisions) give
    the same partition, state and per-iteration records bit for bit, and the
    oracle's."""
    import numpy as np

    from oracle import geographer_oracle as O
    from paper_1805_01208_b200 import KMeansSettings, balanced_kmeans_points

    rng = np.random.default_rng(5)
    pts = rng.random((40_000, 2))
    w = rng.integers(1, 7, 40_000).astype(float) if weights else None
    s = KMeansSettings(k=k, seed=0, max_iter=10)
    runs = {}
    for mode in ("0", "full", "all", "host"):
        monkeypatch.setenv("GP_BALANCE_GRAPH", "0" if mode == "host" else mode)
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
