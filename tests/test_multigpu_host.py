"""Multi-rank protocol on CPU with gloo (world_size 2 and 3): sharding, exact-rank
splitters + all-to-all redistribution, fold-partial exchange.  The per-rank compute is
the CPU oracle here (the kernels need a GPU); the protocol code is the product's
(paper_1805_01208_b200/parallel.py).  Results must equal one rank's, bit for bit, as
the reference's rank invariance demands (ranksim.py:9-17, test_ranksim.py:107-118)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1805_01208_b200.parallel import SEGMENTS, shard_bounds


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, fn, args, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world, *args)))
    except Exception as e:  # surface worker errors in the test
        q.put((rank, e))
    finally:
        dist.destroy_process_group()


def run_ranks(world, fn, *args):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, args, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=300) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    for r, v in out.items():
        if isinstance(v, Exception):
            raise v
    return [out[r] for r in range(world)]


def test_shard_bounds_are_segment_aligned():
    for n in (1000, 100_000, 1 << 20, 12345):
        seg = (np.arange(SEGMENTS + 1) * n) // SEGMENTS
        for world in (1, 2, 3, 4, 8):
            b = shard_bounds(n, world)
            assert b[0] == 0 and b[-1] == n and np.all(np.diff(b) >= 0)
            assert set(b.tolist()) <= set(seg.tolist())
            if SEGMENTS % world == 0:
                assert np.array_equal(b, (np.arange(world + 1) * n) // world)


def _redistribute_case(rank, world, n, dup):
    from oracle import geographer_oracle as O
    from paper_1805_01208_b200.parallel import Comm, input_offsets, sfc_redistribute

    rng = np.random.default_rng(5)
    pts = rng.random((n, 2))
    if dup:
        pts = np.round(pts * 4) / 4       # many equal keys across ranks
    comm = Comm()
    rows = np.array_split(np.arange(n), world)[rank]
    off, n_glob = input_offsets(len(rows), comm)
    assert off == rows[0] and n_glob == n
    lo = torch.tensor(pts[rows].min(axis=0))
    hi = torch.tensor(pts[rows].max(axis=0))
    comm.allreduce(lo, dist.ReduceOp.MIN)
    comm.allreduce(hi, dist.ReduceOp.MAX)
    keys = O.hilbert_keys(pts[rows], lo.numpy(), hi.numpy(), 31).astype(np.int64)
    order = np.argsort(keys, kind="stable")
    ks = torch.from_numpy(keys[order])
    gids = torch.from_numpy((rows[order]).astype(np.int64))
    xs = torch.from_numpy(pts[rows][order])
    k2, (g2, x2) = sfc_redistribute(ks, [gids, xs], n, comm, 62,
                                    lambda k: torch.sort(k, stable=True).indices)
    return k2.numpy(), g2.numpy(), x2.numpy()


@pytest.mark.parametrize("world,n,dup", [(2, 5000, False), (2, 4096, True), (3, 7001, False)])
def test_sample_sort_redistribution_matches_one_rank(world, n, dup):
    from oracle import geographer_oracle as O

    parts = run_ranks(world, _redistribute_case, n, dup)
    rng = np.random.default_rng(5)
    pts = rng.random((n, 2))
    if dup:
        pts = np.round(pts * 4) / 4
    keys = O.hilbert_keys(pts, pts.min(axis=0), pts.max(axis=0), 31)
    order = O.sfc_order(keys)
    b = shard_bounds(n, world)
    for r, (k2, g2, x2) in enumerate(parts):
        assert len(g2) == b[r + 1] - b[r]
        assert np.array_equal(g2, order[b[r]:b[r + 1]])
        assert np.array_equal(k2.astype(np.uint64), keys[order[b[r]:b[r + 1]]])
        assert np.array_equal(x2, pts[order[b[r]:b[r + 1]]])


def _fold_case(rank, world, n, k):
    """Per-rank (segment, block) partials of w*x -> gather -> segment-order fold."""
    from paper_1805_01208_b200.parallel import Comm, gather_fold_pairs

    rng = np.random.default_rng(9)
    x = rng.random(n) * np.power(10.0, rng.integers(-6, 7, n))
    a = rng.integers(0, k, n)
    comm = Comm()
    b = shard_bounds(n, world)
    seg_b = (np.arange(SEGMENTS + 1) * n) // SEGMENTS
    keys, vals = [], []
    for s in range(SEGMENTS):
        if not (b[rank] <= seg_b[s] and seg_b[s + 1] <= b[rank + 1]) or seg_b[s] == seg_b[s + 1]:
            continue
        for c in range(k):
            sel = a[seg_b[s]:seg_b[s + 1]] == c
            if sel.any():
                acc = 0.0
                for v in x[seg_b[s]:seg_b[s + 1]][sel]:   # the bincount fold order
                    acc += v
                keys.append(s * k + c)
                vals.append(acc)
    kt = torch.tensor(keys, dtype=torch.int64)
    vt = torch.tensor(vals, dtype=torch.float64).reshape(-1, 1)
    K, V = gather_fold_pairs(kt, vt, comm)
    # combine: per block, fold present segments in global order (gp_fold_combine)
    out = np.zeros(k)
    order = np.argsort(K.numpy(), kind="stable")
    for j in order:
        c = int(K[j]) % k
        out[c] = out[c] + float(V[j, 0])
    return out


@pytest.mark.parametrize("world", [2, 4])
def test_fold_partials_combine_bit_identical_to_one_rank(world):
    n, k = 3000, 7
    outs = run_ranks(world, _fold_case, n, k)
    ref = run_ranks(1, _fold_case, n, k)[0]
    for o in outs:
        assert np.array_equal(o, ref)
    # and the reference's own sequential segment fold (ranksim.py:173-222)
    rng = np.random.default_rng(9)
    x = rng.random(n) * np.power(10.0, rng.integers(-6, 7, n))
    a = rng.integers(0, k, n)
    seg = np.searchsorted((np.arange(SEGMENTS + 1) * n) // SEGMENTS, np.arange(n), "right") - 1
    per = np.bincount(seg * k + a, weights=x, minlength=SEGMENTS * k).reshape(SEGMENTS, k)
    assert np.array_equal(ref, np.add.reduce(per, axis=0))
