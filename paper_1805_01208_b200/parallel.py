"""Multi-GPU protocol: SFC-range sharding with only k-sized exchanges per round.

One process per GPU (torch.distributed; NCCL over NVLink on B200s, gloo on CPU for the
host-logic tests).  The reference simulates ranks in one process with deterministic
collectives (ranksim.py); here they are real:

  reference                                 here
  ----------------------------------------  ------------------------------------------
  RankWorld shards, _split_bounds           shard_bounds(): contiguous SFC ranges on the
    (ranksim.py:74-75, :159-167)              256-segment boundaries (bit-identical folds)
  allreduce_extreme (kmeans.py:546-548)     Comm.allreduce(MIN/MAX) of 2d doubles
  global_sort_redistribute (ranksim.py:143) exact_cuts() + Comm.alltoall() (sample sort
                                              with exact-rank splitters, §DESIGN 6)
  gather_rows (kmeans.py:558)               Comm.allgather_var()
  allreduce_sum of block weights            Comm.allreduce(SUM) of k int64 (exact)
    (kmeans.py:373)
  weighted_mean_reduce partials             gather_fold_pairs(): the (segment, block)
    (ranksim.py:200-222)                      partials, folded in global segment order

Every function here works on torch tensors of any device, so the same code runs with
gloo on CPU (tests/test_multigpu_host.py) and with NCCL on GPUs.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

SEGMENTS = 256  # ranksim.py:38


class Comm:
    """Collectives of one process group (None: the default group).

    NCCL takes device tensors directly.  With gloo (CPU tests, or several processes
    sharing one GPU in the single-GPU multi-rank test) device tensors are staged
    through host memory."""

    def __init__(self, group=None):
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        self.device = torch.device("cuda", torch.cuda.current_device()) \
            if self.backend == "nccl" or torch.cuda.is_available() else torch.device("cpu")

    def _host(self, t):
        return self.backend != "nccl" and t.is_cuda

    def allreduce(self, t: torch.Tensor, op=dist.ReduceOp.SUM) -> torch.Tensor:
        if self._host(t):
            h = t.cpu()
            dist.all_reduce(h, op=op, group=self.group)
            t.copy_(h)
            return t
        dist.all_reduce(t, op=op, group=self.group)
        return t

    def allgather_var(self, t: torch.Tensor) -> list[torch.Tensor]:
        """All ranks' tensors (variable first dimension), in rank order."""
        if self._host(t):
            return [o.to(t.device) for o in self.allgather_var(t.cpu())]
        n = torch.tensor([t.shape[0]], dtype=torch.int64, device=t.device)
        sizes = [torch.empty_like(n) for _ in range(self.world)]
        dist.all_gather(sizes, n, group=self.group)
        sizes = [int(s.item()) for s in sizes]
        mx = max(sizes)
        pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
        pad[: t.shape[0]] = t
        outs = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(outs, pad, group=self.group)
        return [o[:s] for o, s in zip(outs, sizes)]

    def alltoall(self, t: torch.Tensor, send_counts: list[int]) -> tuple[torch.Tensor, list[int]]:
        """Rows [sum(send[:g]), sum(send[:g+1])) of t go to rank g; returns the received
        rows concatenated in source-rank order and the per-source counts."""
        if self._host(t):
            out, rc = self.alltoall(t.cpu(), send_counts)
            return out.to(t.device), rc
        sc = torch.tensor(send_counts, dtype=torch.int64, device=t.device)
        rc = torch.empty_like(sc)
        dist.all_to_all_single(rc, sc, group=self.group)
        recv_counts = [int(v) for v in rc.tolist()]
        row = int(np.prod(t.shape[1:])) if t.dim() > 1 else 1
        flat = t.reshape(-1)
        out = torch.empty(sum(recv_counts) * row, dtype=t.dtype, device=t.device)
        dist.all_to_all_single(out, flat, output_split_sizes=[c * row for c in recv_counts],
                               input_split_sizes=[c * row for c in send_counts],
                               group=self.group)
        return out.reshape((-1,) + tuple(t.shape[1:])), recv_counts


def shard_bounds(n: int, world: int) -> np.ndarray:
    """Contiguous ranges of the global SFC order on segment boundaries.

    For world | 256 these are exactly floor(g n / world) (ranksim.py:74-75); every
    (segment, block) fold then lives on one rank, so the movement sums are bit-identical
    to one shard's."""
    seg = (np.arange(SEGMENTS + 1, dtype=np.int64) * n) // SEGMENTS
    idx = (np.arange(world + 1, dtype=np.int64) * SEGMENTS) // world
    return seg[idx]


def input_offsets(n_local: int, comm: Comm) -> tuple[int, int]:
    """(global offset of this rank's original rows, global n): ranks hold contiguous
    original rows in rank order, as RankWorld.from_points deals them."""
    counts = comm.allgather_var(torch.tensor([n_local], dtype=torch.int64, device=comm.device))
    counts = [int(c.item()) for c in counts]
    return sum(counts[: comm.rank]), sum(counts)


def exact_cuts(keys_sorted: torch.Tensor, targets: np.ndarray, comm: Comm,
               key_bits: int) -> np.ndarray:
    """Local cut indices for global (key, gid)-order positions.

    keys_sorted: this rank's keys sorted stably (so ties are in gid order).  For every
    global target position t, returns how many of this rank's elements precede it.
    Ties in key are broken by gid, and gids are contiguous per rank in rank order, so
    among equal keys the lower rank comes first: a binary search over the key space
    (counts all-reduced) finds each target's key, then the per-rank counts of that key
    split it exactly.
    """
    T = len(targets)
    dev = keys_sorted.device
    tgt = torch.tensor(targets, dtype=torch.int64, device=dev)
    lo = torch.zeros(T, dtype=torch.int64, device=dev)
    hi = torch.full((T,), (1 << key_bits) - 1, dtype=torch.int64, device=dev)
    # largest key K with count(keys < K) <= t
    for _ in range(key_bits + 1):
        mid = lo + (hi - lo + 1) // 2
        cnt = torch.searchsorted(keys_sorted, mid, right=False).to(torch.int64)
        comm.allreduce(cnt)
        ok = cnt <= tgt
        lo = torch.where(ok, mid, lo)
        hi = torch.where(ok, hi, mid - 1)
        if bool((lo >= hi).all()):
            break
    K = lo
    below = torch.searchsorted(keys_sorted, K, right=False).to(torch.int64)   # local < K
    equal = torch.searchsorted(keys_sorted, K, right=True).to(torch.int64) - below
    g_below = comm.allreduce(below.clone())
    rem = tgt - g_below                       # how many key == K elements precede t
    eq_all = torch.stack(comm.allgather_var(equal.reshape(1, -1))).reshape(comm.world, T)
    before = eq_all[: comm.rank].sum(dim=0) if comm.rank > 0 else torch.zeros_like(rem)
    take = torch.clamp(rem - before, min=0)
    take = torch.minimum(take, equal)
    return (below + take).cpu().numpy()


def sfc_redistribute(keys_sorted, payload_sorted: list[torch.Tensor], n_global: int,
                     comm: Comm, key_bits: int, local_sort):
    """Exchange so that rank g holds global SFC positions shard_bounds(n)[g:g+2].

    keys_sorted / payload_sorted: this rank's rows in local (key, gid) order.
    local_sort(keys) -> stable permutation (device radix sort on GPUs).
    Returns (keys, payload) of the new shard, in global (key, gid) order.
    """
    bounds = shard_bounds(n_global, comm.world)
    cuts = exact_cuts(keys_sorted, bounds[1:-1], comm, key_bits)
    cuts = np.concatenate([[0], cuts, [keys_sorted.shape[0]]]).astype(np.int64)
    send = np.diff(cuts).tolist()
    keys_r, _ = comm.alltoall(keys_sorted, send)
    pay_r = [comm.alltoall(t, send)[0] for t in payload_sorted]
    # received runs come in source-rank order = gid order among equal keys; a stable
    # key sort therefore restores the global (key, gid) order
    perm = local_sort(keys_r)
    return keys_r[perm], [t[perm] for t in pay_r]


def gather_fold_pairs(keys: torch.Tensor, vals: torch.Tensor, comm: Comm):
    """All ranks' (segment, block) fold partials, concatenated (order irrelevant: the
    combine indexes them by key and folds in global segment order)."""
    ks = comm.allgather_var(keys)
    vs = comm.allgather_var(vals)
    return torch.cat(ks), torch.cat(vs)
