"""Multi-rank device path on ONE GPU: 2 and 4 processes (gloo collectives staged through
the host; no kernel waits on another rank, so sharing the GPU is safe) must give the
single-GPU result bit for bit - labels, final state and per-iteration statistics."""
import os
import socket

import numpy as np
import pytest

from conftest import has_cuda

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, n, k, dim, weighted, q):
    import torch
    import torch.distributed as dist

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1805_01208_b200 import KMeansSettings
        from paper_1805_01208_b200.kmeans import partition_distributed

        rng = np.random.default_rng(3)
        pts = rng.random((n, dim))
        w = rng.integers(1, 9, n).astype(float) if weighted else None
        rows = np.array_split(np.arange(n), world)[rank]
        lab, stats = partition_distributed(pts[rows], None if w is None else w[rows],
                                           KMeansSettings(k=k, seed=0))
        st = stats.final_state
        q.put((rank, lab.cpu().numpy(), st.centers, st.influence,
               [vars(r) for r in stats.iterations], stats.balance_failed))
    except Exception as e:
        q.put((rank, e, None, None, None, None))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n,k,dim,weighted", [(2, 120_000, 40, 2, True),
                                                    (4, 60_000, 300, 3, False)])
def test_multirank_bit_identical_to_one_gpu(world, n, k, dim, weighted):
    if not has_cuda():
        pytest.fail("CUDA device required")
    import torch.multiprocessing as mp

    from paper_1805_01208_b200 import KMeansSettings, balanced_kmeans_points

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_rank_main, args=(r, world, port, n, k, dim, weighted, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = dict((r[0], r[1:]) for r in (q.get(timeout=600) for _ in range(world)))
    for p in procs:
        p.join(timeout=120)
    for r in range(world):
        if isinstance(res[r][0], Exception):
            raise res[r][0]
    labels = np.concatenate([res[r][0] for r in range(world)])

    rng = np.random.default_rng(3)
    pts = rng.random((n, dim))
    w = rng.integers(1, 9, n).astype(float) if weighted else None
    part, stats = balanced_kmeans_points(pts, w, KMeansSettings(k=k, seed=0), return_stats=True)
    assert np.array_equal(labels, part.assignment)
    for r in range(world):
        _, centers, infl, recs, failed = res[r]
        assert np.array_equal(centers, stats.final_state.centers)
        assert np.array_equal(infl, stats.final_state.influence)
        assert failed == part.balance_failed
        for a, b in zip(recs, [vars(x) for x in stats.iterations]):
            for key in ("phase", "active_points", "balance_rounds", "imbalance",
                        "total_decisions", "max_move"):
                assert a[key] == b[key], key
