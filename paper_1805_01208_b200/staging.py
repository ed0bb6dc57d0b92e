"""Host <-> device copies of the caller's numpy arrays at DMA speed.

The reference takes plain numpy arrays (`kmeans.py:510`, `np.asarray`), which
live in pageable memory.  A pageable cudaMemcpy goes through the driver's
small bounce buffer at a fraction of the link rate, so large inputs are
staged here instead: a ring of pinned chunks, each filled by a few host
threads (numpy copies release the GIL) while the DMA of the previous chunk
runs on the stream.  Page-locked inputs (a pinned torch tensor's numpy view)
are copied directly.
"""

from __future__ import annotations

import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np
import torch

CHUNK = 64 << 20        # bytes per pinned chunk
NBUF = 4                # chunks in the ring
MIN_STAGED = 32 << 20   # below this a plain copy is as fast
_ring = None
_pool = None


def _threads() -> ThreadPoolExecutor:
    global _pool
    if _pool is None:
        try:
            cores = len(os.sched_getaffinity(0))
        except AttributeError:
            cores = os.cpu_count() or 1
        # GP_STAGE_THREADS: host copy threads filling / draining the pinned ring
        want = int(os.environ.get("GP_STAGE_THREADS", "8"))
        _pool = ThreadPoolExecutor(max(1, min(want, cores)))
    return _pool


def _bufs():
    global _ring
    if _ring is None:
        _ring = ([torch.empty(CHUNK, dtype=torch.uint8, pin_memory=True) for _ in range(NBUF)],
                 [None] * NBUF)
    return _ring


def _par_copy(dst: np.ndarray, src: np.ndarray):
    """dst[:] = src (1-D uint8 views) split over the host threads."""
    n = dst.shape[0]
    pool = _threads()
    parts = pool._max_workers
    step = max(1 << 20, (n + parts - 1) // parts)
    futs = [pool.submit(np.copyto, dst[o:o + step], src[o:o + step]) for o in range(0, n, step)]
    for f in futs:
        f.result()


def is_pinned(a: np.ndarray) -> bool:
    from . import _native as N

    return bool(N.lib.gp_host_is_pinned(C_void(a.ctypes.data)))


def C_void(p):
    import ctypes

    return ctypes.c_void_p(p)


def h2d_into(dst: torch.Tensor, src: np.ndarray):
    """dst (contiguous CUDA tensor) <- src (contiguous host array of the same bytes),
    stream-ordered on dst's current stream."""
    stream = torch.cuda.current_stream(dst.device)
    sb = np.ascontiguousarray(src).reshape(-1).view(np.uint8)
    db = dst.reshape(-1).view(torch.uint8)
    nbytes = sb.shape[0]
    if nbytes < MIN_STAGED:
        db.copy_(torch.from_numpy(sb))
        return
    bufs, evs = _bufs()
    for j, off in enumerate(range(0, nbytes, CHUNK)):
        i = j % NBUF
        if evs[i] is not None:
            evs[i].synchronize()
        m = min(CHUNK, nbytes - off)
        _par_copy(bufs[i].numpy()[:m], sb[off:off + m])
        db[off:off + m].copy_(bufs[i][:m], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        evs[i] = ev


def d2h_into(dst: np.ndarray, src: torch.Tensor):
    """dst (contiguous host array) <- src (contiguous CUDA tensor of the same bytes);
    returns after the data is in dst."""
    stream = torch.cuda.current_stream(src.device)
    db = dst.reshape(-1).view(np.uint8)
    sb = src.reshape(-1).view(torch.uint8)
    nbytes = db.shape[0]
    if nbytes < MIN_STAGED:
        torch.from_numpy(db).copy_(sb)
        return
    bufs, evs = _bufs()
    for e in evs:
        if e is not None:
            e.synchronize()
    offs = list(range(0, nbytes, CHUNK))
    pend = {}

    def issue(j):
        i = j % NBUF
        off = offs[j]
        m = min(CHUNK, nbytes - off)
        bufs[i][:m].copy_(sb[off:off + m], non_blocking=True)
        ev = torch.cuda.Event()
        ev.record(stream)
        pend[j] = ev

    for j in range(min(NBUF, len(offs))):
        issue(j)
    for j, off in enumerate(offs):
        pend.pop(j).synchronize()
        m = min(CHUNK, nbytes - off)
        _par_copy(db[off:off + m], bufs[j % NBUF].numpy()[:m])
        if j + NBUF < len(offs):
            issue(j + NBUF)
    for i in range(NBUF):
        evs[i] = None
