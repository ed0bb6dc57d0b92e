"""`p` GPUs behind one call: a persistent pool of one worker process per GPU.

The reference's `balanced_kmeans_points(points, weights, settings, p)`
(`kmeans.py:502-512`) deals the rows over `p` simulated ranks
(`RankWorld.from_points`, `ranksim.py:89-108`).  Here `p` is the GPU count:
`balanced_kmeans_points(..., p=G)` with G > 1 visible GPUs runs the sharded
partition (`kmeans.DistributedPartitioner`: SFC-range shards, k-sized NCCL
exchanges per round) on min(p, GPUs) devices.  Results are bit-identical for
every p, as in the reference.

Design:
* The workers are spawned once (first use) and kept: each sets its device,
  joins one NCCL process group (created once, `init_process_group` over TCP
  on 127.0.0.1), then serves partition tasks from its queue.
* Inputs never go through host shared memory: the caller's process copies
  row block g (rows `[g n/G, (g+1) n/G)`, the reference's `_split_bounds`
  dealing, `ranksim.py:74-75`) to GPU g and hands the device tensor to
  worker g through CUDA IPC (torch.multiprocessing); worker g returns the
  int64 labels of its rows the same way.
* Errors: argument errors are agreed by all ranks before any other
  collective (`DistributedPartitioner.bootstrap`), so every worker reports
  the same exception and the pool stays usable; any other failure shuts the
  pool down and re-raises.

`GP_POOL_SHARE_GPU=1` (tests) runs the workers on GPU 0 with gloo collectives
staged through the host, so the pool is exercised on a one-GPU box; no kernel
waits on another rank, so sharing one device is safe.
"""

from __future__ import annotations

import atexit
import os
import queue as _queue
import socket
import traceback

import numpy as np
import torch

_POOL = None
TASK_TIMEOUT_S = float(os.environ.get("GP_POOL_TIMEOUT", "3600"))


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, share, tasks, results):
    import torch.distributed as dist

    dev = torch.device("cuda", 0 if share else rank)
    torch.cuda.set_device(dev)
    backend = "gloo" if share else "nccl"
    kw = {} if share else {"device_id": dev}
    dist.init_process_group(backend, init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=world, **kw)
    from .kmeans import partition_distributed

    results.put(("ready", rank, None))
    while True:
        task = tasks.get()
        if task is None:
            break
        tid, pts, w, settings = task
        try:
            lab, stats = partition_distributed(pts, w, settings, device=dev)
            torch.cuda.current_stream(dev).synchronize()
            results.put((tid, rank, (lab, stats if rank == 0 else None)))
            # the caller copies the labels out before the next task; keep them alive
            # until then (CUDA IPC: the producer owns the memory)
            keep = lab  # noqa: F841
        except Exception as e:   # every rank raises the same argument errors together
            results.put((tid, rank, e if _picklable(e) else RuntimeError(traceback.format_exc())))
        del pts, w
    dist.destroy_process_group()


def _picklable(e) -> bool:
    import pickle

    try:
        pickle.dumps(e)
        return True
    except Exception:
        return False


class GpuPool:
    """World of `G` worker processes, one per GPU (or all on GPU 0 when shared)."""

    def __init__(self, G: int, share: bool):
        import torch.multiprocessing as mp

        self.G, self.share = G, share
        ctx = mp.get_context("spawn")
        self.results = ctx.Queue()
        self.tasks = [ctx.Queue() for _ in range(G)]
        port = _free_port()
        self.procs = [ctx.Process(target=_worker, args=(r, G, port, share, self.tasks[r],
                                                        self.results), daemon=True)
                      for r in range(G)]
        for p in self.procs:
            p.start()
        self.next_id = 0
        for _ in range(G):
            msg = self._get()
            if msg[0] != "ready":
                self.close()
                raise RuntimeError(f"GPU pool worker failed to start: {msg}")

    def _get(self):
        try:
            return self.results.get(timeout=TASK_TIMEOUT_S)
        except _queue.Empty:
            self.close()
            raise RuntimeError("GPU pool: a worker did not answer in time; pool shut down")

    def alive(self) -> bool:
        return all(p.is_alive() for p in self.procs)

    def run(self, points, weights, settings):
        """Partition (n, d) points with the workers; returns (int64 labels on the
        caller's current device's host, KMeansStats)."""
        n = int(points.shape[0])
        G = self.G
        bounds = [(g * n) // G for g in range(G + 1)]
        tid = self.next_id
        self.next_id += 1
        held = []
        for g in range(G):
            dev = torch.device("cuda", 0 if self.share else g)
            lo, hi = bounds[g], bounds[g + 1]
            pts_g = _to_device(points, lo, hi, dev)
            w_g = None if weights is None else _to_device(weights, lo, hi, dev)
            torch.cuda.synchronize(dev)
            held.append((pts_g, w_g))
            self.tasks[g].put((tid, pts_g, w_g, settings))
        out = np.empty(n, dtype=np.int64)
        stats, errors = None, []
        for _ in range(G):
            msg = self._get()
            t, rank, payload = msg
            if t != tid:
                self.close()
                raise RuntimeError("GPU pool: out-of-order result; pool shut down")
            if isinstance(payload, BaseException):
                errors.append((rank, payload))
                continue
            lab, st = payload
            out[bounds[rank]:bounds[rank + 1]] = lab.cpu().numpy()
            del lab
            if st is not None:
                stats = st
        del held
        if errors:
            errors.sort(key=lambda e: e[0])
            raise errors[0][1]
        return out, stats

    def close(self):
        for q in self.tasks:
            try:
                q.put(None)
            except Exception:
                pass
        for p in self.procs:
            p.join(timeout=10)
            if p.is_alive():
                p.terminate()


def _to_device(a, lo, hi, dev):
    if isinstance(a, torch.Tensor):
        return a[lo:hi].to(device=dev, dtype=torch.float64).contiguous()
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a[lo:hi], dtype=np.float64))).to(dev)


def gpu_count_for(p: int) -> int:
    """How many GPUs a call with `p` ranks uses: min(p, visible GPUs); the
    shared-GPU test mode uses p workers on GPU 0."""
    if os.environ.get("GP_POOL_SHARE_GPU") == "1":
        return p
    return max(1, min(p, torch.cuda.device_count()))


def get_pool(G: int) -> GpuPool:
    global _POOL
    share = os.environ.get("GP_POOL_SHARE_GPU") == "1"
    if _POOL is not None and (_POOL.G != G or _POOL.share != share or not _POOL.alive()):
        _POOL.close()
        _POOL = None
    if _POOL is None:
        _POOL = GpuPool(G, share)
    return _POOL


def shutdown():
    global _POOL
    if _POOL is not None:
        _POOL.close()
        _POOL = None


atexit.register(shutdown)
