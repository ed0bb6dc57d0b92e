"""Drop-in balanced k-means partitioner on B200 (arXiv 1805.01208, Alg. 1 + Alg. 2).

Public entry points keep the reference's signatures
(``balanced_kmeans_points`` kmeans.py:502-512, ``balanced_kmeans``
kmeans.py:515-534).  The host loop below mirrors ``_run_pipeline``
(kmeans.py:537-650) and ``assign_and_balance`` (kmeans.py:377-453) line for
line for every k-sized decision, in host numpy; every n-sized pass runs in the
sm_100a kernels of ``csrc/`` through the C ABI:

  reference pass                                 device call
  ---------------------------------------------  ---------------------------
  min/max + allreduce_extreme  kmeans.py:546-548 gp_box_minmax
  hilbert_keys                 geometry.py:182   gp_hilbert_keys
  global_sort_redistribute     ranksim.py:143    gp_sort_pairs + gp_gather_points
  gather_rows (initial centers) kmeans.py:552    gp_gather_rows
  active = rank < size         kmeans.py:579     gp_compact_active
  _scan_rank + relax_bounds + _global_block_weights
                               kmeans.py:297-453 gp_assign_round (per balance round)
  _weighted_center_partials + weighted_mean_reduce + _cluster_extents + _objective
                               kmeans.py:463-499 gp_movement_fold
  _audit_rank                  kmeans.py:347     gp_audit
  full_assignment[gids] = a    kmeans.py:637     gp_scatter_by_gid

There is no CPU fallback: without the built extension the import fails.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import weakref
from dataclasses import dataclass

import numpy as np
import torch

from . import _native as N
from .control import (
    BoundMaps,
    row_norms,
    imbalance,
    influence_factor,
    eroded,
    initial_center_positions,
    sample_schedule,
)
from .numerics import einsum_order3
from .types import (
    BalanceInfo,
    BoundingBox,
    ClusterState,
    GeometryError,
    GraphError,
    IterationRecord,
    KMeansSettings,
    KMeansStats,
    Partition,
)

DEFAULT_DEPTH = {2: 31, 3: 20}  # geometry.py:28


def check_weights(n: int, weights) -> None:
    """Weights must be 1-D with at least n entries (extra ones are ignored, as the
    reference's shard slices ignore them, ranksim.py:101-106)."""
    shape = tuple(weights.shape) if hasattr(weights, "shape") else np.shape(weights)
    if len(shape) != 1:
        raise ValueError(f"weights must be a 1-D array of length {n}, got shape {shape}")
    if shape[0] < n:
        # the reference fails in its redistribution gather (ranksim.py:160-168)
        raise IndexError(f"weights has {shape[0]} entries for {n} points")


def _host_to_device(a: np.ndarray, dev) -> torch.Tensor:
    """Copy a host array to the device: one DMA when it is page-locked, else staged
    through pinned chunks (staging.py), so a plain numpy input also moves at link rate."""
    from . import staging

    t = torch.from_numpy(a)
    if a.nbytes < staging.MIN_STAGED or staging.is_pinned(a):
        return t.to(dev, non_blocking=True)
    out = torch.empty(a.shape, dtype=t.dtype, device=dev)
    staging.h2d_into(out, a)
    return out


# GP_NVTX=1: every assign round inside an NVTX range "round<N>" (N counts the rounds of
# the process), so an ncu capture can select one round (--nvtx --nvtx-include round550/)
_NVTX = os.environ.get("GP_NVTX") == "1"
_ROUNDS = [0]


def _round_counter() -> int:
    _ROUNDS[0] += 1
    return _ROUNDS[0] - 1


_FOLDS = [0]


def _fold_counter() -> int:
    _FOLDS[0] += 1
    return _FOLDS[0] - 1


def _ptr(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


class RankWorld:
    """Rank-count descriptor kept for API parity with ranksim.RankWorld.

    Results are identical for every p (as in the reference).  p is the GPU count:
    balanced_kmeans_points(..., p) shards the run over min(p, visible GPUs) devices
    (pool.py), by SFC range with k-sized NCCL exchanges (parallel.py).
    """

    def __init__(self, n: int, dim: int, p: int, coords=None, weights=None):
        self.n, self.dim, self.p = n, dim, p
        self.coords, self.weights = coords, weights

    @classmethod
    def from_points(cls, points, weights=None, p: int = 1) -> "RankWorld":
        n = int(points.shape[0])
        if p < 1 or p > n:
            raise ValueError(f"rank count {p} out of range 1..{n}")
        dim = int(points.shape[1]) if len(points.shape) > 1 else 0
        return cls(n, dim, p, points, weights)

    @classmethod
    def from_graph(cls, graph, p: int = 1) -> "RankWorld":
        return cls.from_points(graph.coords, graph.vertex_weights, p)


@dataclass
class _WeightPlan:
    mode: int          # GP_W_*
    exact: bool        # block-weight sums exact in int64 units of 1/scale
    scale: float       # 2^s


class _Timer:
    """Optional CUDA-event timing of the assign kernel (for bench.py's roofline)."""

    def __init__(self):
        self.events = []
        self.mids = []
        self.rounds = []   # (n_active, n_scanned, n_evals) per assign launch
        self.scan = []     # gp_scan_stats per round (GP_SCAN_STATS=1)

    def mark(self, stream):
        ev = torch.cuda.Event(enable_timing=True)
        ev.record(stream)
        return ev

    def begin(self, stream, aargs):
        """Events around one gp_assign_round, plus one the library records between
        its filter and scan launches (gp_assign_args.split_event)."""
        e0 = self.mark(stream)
        mid = self.mark(stream)          # recorded once so the CUDA event exists
        aargs.split_event = mid.cuda_event
        return e0, mid

    def end(self, stream, aargs, tok):
        aargs.split_event = None
        self.events.append((tok[0], self.mark(stream)))
        self.mids.append(tok[1])

    def total_ms(self) -> float:
        torch.cuda.synchronize()
        return sum(a.elapsed_time(b) for a, b in self.events)

    def split_ms(self) -> tuple[float, float]:
        """(filter, scan) milliseconds summed over the assign rounds."""
        torch.cuda.synchronize()
        f = sum(a.elapsed_time(m) for (a, _), m in zip(self.events, self.mids))
        s = sum(m.elapsed_time(b) for (_, b), m in zip(self.events, self.mids))
        return f, s


def sort_pairs(keys: torch.Tensor, vals: torch.Tensor | None, keys_out: torch.Tensor | None,
               vals_out: torch.Tensor, key_bits: int, stream) -> None:
    """(key, val) pairs in stable key order (np.lexsort((gids, keys)), ranksim.py:158,
    when vals are the input positions): the onesweep device radix sort, gp_sort_pairs.
    vals None means val = input index."""
    n = keys.shape[0]
    dev = keys.device
    ko = keys_out if keys_out is not None else torch.empty_like(keys)
    wsb = N.size_query("gp_sort_workspace_bytes", n)
    ws = torch.empty(max(wsb, 1), dtype=torch.uint8, device=dev)
    # vals None: the sort numbers the pairs itself (no n-sized index array to fill and read)
    N.call("gp_sort_pairs", keys.data_ptr(), _ptr(vals), ko.data_ptr(), vals_out.data_ptr(),
           n, key_bits, ws.data_ptr(), wsb, stream)


def sample_ranks_device(n: int, seed: int, device, stream) -> torch.Tensor:
    """Inverse of numpy.random.default_rng(seed).permutation(n), computed on the GPU.

    Bit-exact with numpy (gp_sample_ranks reproduces PCG64 + the masked
    rejection draws + the descending Fisher-Yates swaps); set
    GP_HOST_PERMUTATION=1 to compute it with host numpy instead (verification).
    """
    if os.environ.get("GP_HOST_PERMUTATION") == "1":
        perm = np.random.default_rng(seed).permutation(n)
        rank = np.empty(n, dtype=np.int32)
        rank[perm] = np.arange(n, dtype=np.int32)
        return torch.from_numpy(rank).to(device)
    st = np.random.PCG64(seed).state["state"]
    m64 = (1 << 64) - 1
    words = (C.c_uint64 * 4)(st["state"] >> 64, st["state"] & m64, st["inc"] >> 64,
                             st["inc"] & m64)
    rank = torch.empty(n, dtype=torch.int32, device=device)
    wsb = N.size_query("gp_sample_ranks_workspace_bytes", n)
    ws = torch.empty(wsb, dtype=torch.uint8, device=device)
    N.call("gp_sample_ranks", words, n, rank.data_ptr(), ws.data_ptr(), wsb, stream)
    return rank


# warm-up samples with at most WALK_RATIO active points per center (and k >=
# WALK_MIN_K) assign by warp-per-point grid walks instead of per-unit candidate
# selection over the k centers (GP_WALK_RATIO=0 disables)
WALK_RATIO = float(os.environ.get("GP_WALK_RATIO", "32"))
WALK_MIN_K = 256


def full_scan_regions(n: int, k: int) -> int:
    """Full-phase scan unit in 256-entry filter regions: about 1/8 of a block's
    points (SFC-compact units whose boxes stay small against a block), 1..32."""
    if os.environ.get("GP_FULL_SREG"):   # tuning override
        return int(os.environ["GP_FULL_SREG"])
    target = max(1, n // (8 * k))
    r = 1
    while r < 32 and 256 * r * 2 <= target:
        r *= 2
    return r


class _Hierarchy:
    """Group-level candidate lists (gp_group_boxes / gp_group_candidates).

    Super groups of 2^14 active entries take their candidates from mega groups
    of 2^20 entries (k > 4096) or from all k; tiles of the assign kernel then
    start from their super group's list instead of all k centers.
    """

    SUPER_SHIFT, MEGA_SHIFT, GIGA_SHIFT = 14, 20, 24
    SUPER_CAP, MEGA_CAP, GIGA_CAP = 1024, 4096, 8192

    def __init__(self, eng, use_mega: bool):
        self.eng = weakref.proxy(eng)  # no engine <-> hierarchy cycle keeping GBs alive
        self.use_mega = use_mega
        self.key = None
        if os.environ.get("GP_SUPER_SHIFT"):   # tuning override
            self.SUPER_SHIFT = int(os.environ["GP_SUPER_SHIFT"])

    def prepare(self, list_ptr, m):
        """Boxes of the groups of the current active list (once per active set)."""
        eng = self.eng
        key = (eng.aargs.X, list_ptr, m)
        if self.key == key:
            return
        self.key = key
        dev, d = eng.device, eng.d
        self.ns = max(1, (m + (1 << self.SUPER_SHIFT) - 1) >> self.SUPER_SHIFT)
        self.nm = max(1, (m + (1 << self.MEGA_SHIFT) - 1) >> self.MEGA_SHIFT)
        self.sbox = torch.empty(self.ns * 2 * d, dtype=torch.float64, device=dev)
        self.slist = torch.empty(self.ns * self.SUPER_CAP, dtype=torch.int32, device=dev)
        self.scount = torch.empty(self.ns, dtype=torch.int32, device=dev)
        N.call("gp_group_boxes", eng.aargs.X, eng.ldx, d, list_ptr, m, self.SUPER_SHIFT,
               self.sbox.data_ptr(), eng.sh)
        if self.use_mega:
            self.mlist = torch.empty(self.nm * self.MEGA_CAP, dtype=torch.int32, device=dev)
            self.mcount = torch.empty(self.nm, dtype=torch.int32, device=dev)
            # mega boxes = unions of their 64 super boxes (min / max are exact: the same
            # boxes as a second pass over the points, without reading them again)
            self.mbox = self._unions(self.sbox, self.ns, self.MEGA_SHIFT - self.SUPER_SHIFT,
                                     self.nm, d)
        # a third level (2^24 entries) when there are many mega groups: the mega
        # lists then start from a giga list instead of all k
        self.use_giga = self.use_mega and m > (1 << (self.GIGA_SHIFT + 1))
        if self.use_giga:
            self.ng = (m + (1 << self.GIGA_SHIFT) - 1) >> self.GIGA_SHIFT
            self.glist = torch.empty(self.ng * self.GIGA_CAP, dtype=torch.int32, device=dev)
            self.gcount = torch.empty(self.ng, dtype=torch.int32, device=dev)
            # giga boxes = unions of their 16 mega boxes
            self.gbox = self._unions(self.mbox, self.nm, self.GIGA_SHIFT - self.MEGA_SHIFT,
                                     self.ng, d)
        a = eng.aargs
        a.group_list, a.group_count = self.slist.data_ptr(), self.scount.data_ptr()
        a.group_cap, a.group_shift = self.SUPER_CAP, self.SUPER_SHIFT

    @staticmethod
    def _unions(child, n_child, ratio_log2, n_parent, d):
        """Boxes of groups made of 2^ratio_log2 consecutive child groups (k-sized torch
        reductions; a missing child is the empty box +inf / -inf)."""
        r = 1 << ratio_log2
        cb = child.view(n_child, 2, d)
        pad = n_parent * r - n_child
        if pad:
            fill = torch.empty((pad, 2, d), dtype=torch.float64, device=child.device)
            fill[:, 0], fill[:, 1] = math.inf, -math.inf
            cb = torch.cat([cb, fill])
        cb = cb.view(n_parent, r, 2, d)
        return torch.stack([cb[:, :, 0].amin(dim=1), cb[:, :, 1].amax(dim=1)],
                           dim=1).contiguous().view(-1)

    def refresh(self):
        """Candidate lists under the current centers and influences (every round)."""
        eng = self.eng
        d, k = eng.d, eng.settings.k
        cen = eng.centers_d.data_ptr()
        i2lo, i2hi = eng.aargs.inv2_lo, eng.aargs.inv2_hi
        parent, pcount, pcap = None, None, 0
        if self.use_giga:
            N.call("gp_group_candidates", self.gbox.data_ptr(), self.ng, d, k, cen, i2lo, i2hi,
                   None, None, 0, 0, self.glist.data_ptr(), self.gcount.data_ptr(),
                   self.GIGA_CAP, eng.sh)
            parent, pcount, pcap = self.glist.data_ptr(), self.gcount.data_ptr(), self.GIGA_CAP
        if self.use_mega:
            N.call("gp_group_candidates", self.mbox.data_ptr(), self.nm, d, k, cen, i2lo, i2hi,
                   parent, pcount, pcap, self.GIGA_SHIFT - self.MEGA_SHIFT if parent else 0,
                   self.mlist.data_ptr(), self.mcount.data_ptr(), self.MEGA_CAP, eng.sh)
            parent, pcount, pcap = self.mlist.data_ptr(), self.mcount.data_ptr(), self.MEGA_CAP
        N.call("gp_group_candidates", self.sbox.data_ptr(), self.ns, d, k, cen, i2lo, i2hi,
               parent, pcount, pcap, self.MEGA_SHIFT - self.SUPER_SHIFT,
               self.slist.data_ptr(), self.scount.data_ptr(), self.SUPER_CAP, eng.sh)


class DevicePartitioner:
    """One partition run on one GPU (the whole point set is one SFC shard)."""

    def __init__(self, settings: KMeansSettings, device=None, timer: _Timer | None = None,
                 keep_keys: bool = False):
        self.settings = settings
        self.keep_keys = keep_keys
        self.device = torch.device(device if device is not None else "cuda")
        self.timer = timer
        self.order3 = einsum_order3()
        self.stream = torch.cuda.current_stream(self.device)
        self.sh = self.stream.cuda_stream

    # ------------------------------------------------------------ bootstrap
    def _input(self, points, weights):
        dev = self.device
        if isinstance(points, torch.Tensor):
            pts = points.to(device=dev, dtype=torch.float64)
        else:
            pts = _host_to_device(np.ascontiguousarray(np.asarray(points, dtype=np.float64)), dev)
        if pts.dim() != 2:
            raise GeometryError("points must be an (n, d) array")
        w = None
        if weights is not None:
            n = pts.shape[0]
            check_weights(n, weights)
            if isinstance(weights, torch.Tensor):
                w = weights[:n].to(device=dev, dtype=torch.float64).contiguous()
            else:
                # extra entries are ignored, as the reference's shard slices do
                # (ranksim.py:101-106)
                w = _host_to_device(
                    np.ascontiguousarray(np.asarray(weights, dtype=np.float64)[:n]), dev)
        return pts, w

    def _weight_plan(self, w: torch.Tensor | None, n: int) -> _WeightPlan:
        if w is None:
            return _WeightPlan(0, True, 1.0)
        out = torch.empty(3, dtype=torch.int64, device=self.device)
        N.call("gp_weight_probe", w.data_ptr(), n, out.data_ptr(), self.sh)
        flags, low, mx_bits = (int(v) for v in out.cpu().tolist())
        mx = np.array([mx_bits], dtype=np.int64).view(np.float64)[0]
        mode = 2 if flags & 2 else 1
        if flags & 1:
            return _WeightPlan(2, False, 1.0)
        s = max(0, -low) if low < 4096 else 0
        exact = (s <= 1000 and mx * 2.0 ** s * n < 2.0 ** 53)
        return _WeightPlan(mode, bool(exact), 2.0 ** s if exact else 1.0)

    def bootstrap(self, points, weights):
        if _NVTX:
            torch.cuda.nvtx.range_push("bootstrap")
        try:
            return self._bootstrap(points, weights)
        finally:
            if _NVTX:
                torch.cuda.nvtx.range_pop()

    def _bootstrap(self, points, weights):
        st = self.settings
        pts, w = self._input(points, weights)
        n, d = pts.shape
        self.n, self.d = n, d
        self.n_global, self.pos0 = n, 0
        k = st.k
        if k > n:
            raise ValueError(f"k={k} exceeds the number of points {n}")
        depth = st.sfc_depth if st.sfc_depth is not None else DEFAULT_DEPTH.get(d)
        if depth is None or d not in (2, 3):
            raise GeometryError(f"unsupported dimension {d}")
        if d * depth > 62:
            raise GeometryError(f"depth {depth} out of range for dimension {d}")
        dev, sh = self.device, self.sh
        sp, sd = pts.stride()
        # K1: global box (kmeans.py:546-548)
        lohi = torch.empty(2 * d, dtype=torch.float64, device=dev)
        bad = torch.empty(1, dtype=torch.int32, device=dev)
        N.call("gp_box_minmax", pts.data_ptr(), n, d, sp, sd, lohi.data_ptr(), bad.data_ptr(), sh)
        lohi_h = lohi.cpu().numpy()
        if int(bad.item()):
            raise GeometryError("non-finite box corner")
        self.box = BoundingBox(lohi_h[:d].copy(), lohi_h[d:].copy())
        # weights plan
        self.wplan = self._weight_plan(w, n)
        # K2 keys + K3 sort + payload gather (geometry.py:182, ranksim.py:143-170)
        keys = torch.empty(n, dtype=torch.int64, device=dev)
        N.call("gp_hilbert_keys", pts.data_ptr(), n, d, sp, sd, lohi.data_ptr(), depth,
               keys.data_ptr(), None, 0, sh)
        # gids are the input positions (ranksim.py:98-107): the sort's implicit vals
        self.gids = torch.empty(n, dtype=torch.int32, device=dev)
        keys_s = torch.empty_like(keys) if self.keep_keys else None
        sort_pairs(keys, None, keys_s, self.gids, d * depth, sh)
        self.keys_sorted = keys_s
        del keys, keys_s
        self.ldx = d
        self.X = torch.empty((n, d), dtype=torch.float64, device=dev)  # AoS, SFC order
        self.W = None
        if w is not None:
            self.W = torch.empty(n, dtype=torch.float32 if self.wplan.mode == 1 else torch.float64,
                                 device=dev)
        N.call("gp_gather_points", pts.data_ptr(), sp, sd, d, self.gids.data_ptr(), n,
               self.X.data_ptr(), self.ldx, _ptr(w), self.wplan.mode if w is not None else 0,
               _ptr(self.W), sh)
        # K4 initial centers (kmeans.py:552-558)
        pos = torch.from_numpy(initial_center_positions(n, k)).to(dev)
        cen = torch.empty((k, d), dtype=torch.float64, device=dev)
        N.call("gp_gather_rows", self.X.data_ptr(), self.ldx, d, pos.data_ptr(), k,
               cen.data_ptr(), sh)
        self.centers_d = cen
        self.init_centers = cen.cpu().numpy().copy()
        # sample ranks in SFC order (kmeans.py:564-568)
        self.sizes = sample_schedule(n, st.init_sample)
        if self.sizes:
            rank_d = sample_ranks_device(n, st.seed, dev, sh)
            self.rank_sfc = torch.empty(n, dtype=torch.int32, device=dev)
            N.call("gp_gather_ranks", rank_d.data_ptr(), self.gids.data_ptr(), n,
                   self.rank_sfc.data_ptr(), sh)
            cwb = N.size_query("gp_compact_workspace_bytes", n)
            self.compact_ws = torch.empty(max(cwb, 8), dtype=torch.uint8, device=dev)
            self.active_idx = torch.empty(n, dtype=torch.int32, device=dev)
            self.active_cnt = torch.empty(1, dtype=torch.int64, device=dev)
            del rank_d
        del pts, w
        return self

    # ------------------------------------------------------------ helpers
    def _cold_bounds(self):
        """ub~ = +inf, lb~ = 0 for every entry: one fill of the packed fp16 pair
        (0x7C00 | 0 << 16) instead of two strided ones."""
        self.UBLB.view(torch.int32).fill_(0x7C00)

    def _alloc_state(self):
        n, k, d, dev = self.n, self.settings.k, self.d, self.device
        self.A = torch.full((n,), -1, dtype=torch.int32, device=dev)
        # (ub~, lb~) fp16 pairs (scaled by bound_scale): ub~ = +inf (unassigned), lb~ = 0
        # (kmeans.py:146-147)
        self.UBLB = torch.empty((n, 2), dtype=torch.float16, device=dev)
        self._cold_bounds()
        # influences (ping-pong) | inv2_lo | inv2_hi | moves   (float64)
        self.kstate = torch.empty(5 * k, dtype=torch.float64, device=dev)
        # device bound maps S[k] | T[k] | A | B | steps, and their float32 parameters
        self.mapstate = torch.empty(4 * k + 8, dtype=torch.float64, device=dev)
        self.kmaps = torch.empty(8 * k + 4, dtype=torch.float32, device=dev)
        self.mapflag = torch.zeros(1, dtype=torch.int32, device=dev)
        self.red = torch.zeros(k + 3, dtype=torch.int64, device=dev)      # block_w | counters
        # pinned staging for the per-round k-sized transfers
        self.red_h = torch.empty(k + 3, dtype=torch.int64, pin_memory=True)
        self.infl_h = torch.empty(k, dtype=torch.float64, pin_memory=True)
        self.moves_h = torch.empty(k, dtype=torch.float64, pin_memory=True)
        self.cur = 0
        self.audit_out = torch.zeros(3, dtype=torch.int64, device=dev)
        self.fold_out = torch.empty(k * (d + 3), dtype=torch.float64, device=dev)
        fwb = N.size_query("gp_fold_workspace_bytes", n, self.pos0, self.n_global, k)
        self.fold_ws = torch.empty(max(fwb, 8), dtype=torch.uint8, device=dev)
        a = N.AssignArgs()
        a.X, a.ldx, a.d, a.k, a.order3 = self.X.data_ptr(), self.ldx, d, k, self.order3
        a.wmode = self.wplan.mode if self.W is not None else 0
        a.w = _ptr(self.W)
        a.wscale = self.wplan.scale
        a.a, a.ublb = self.A.data_ptr(), self.UBLB.data_ptr()
        # stored bounds are fp16 times a power of two near 1 / the box diagonal
        e = -int(round(math.log2(max(self.box.diagonal(), 1e-30))))
        a.bound_scale = 2.0 ** max(-60, min(60, e))
        a.centers = self.centers_d.data_ptr()
        base = self.kstate.data_ptr()
        a.infl, a.inv2_lo, a.inv2_hi = base, base + 16 * k, base + 24 * k
        mb = self.kmaps.data_ptr()
        a.ub_eval, a.ub_norm, a.lb_par = mb, mb + 16 * k, mb + 32 * k
        a.inv2_min_dev = self.mapstate.data_ptr() + 8 * (2 * k + 7)   # kept by gp_update_maps
        a.block_w = self.red.data_ptr()
        a.counters = self.red.data_ptr() + 8 * k
        awb = N.size_query("gp_assign_workspace_bytes", n)
        self.assign_ws = torch.empty(awb, dtype=torch.uint8, device=dev)
        a.workspace, a.workspace_bytes = self.assign_ws.data_ptr(), awb
        # scan statistics for tools/kprof.py (debugging aid; costs a sync per round)
        a.flags = 1 if self.timer is not None and os.environ.get("GP_SCAN_STATS") else 0
        self.aargs = a
        self.hier = _Hierarchy(self, use_mega=k > 4096) if k > 128 else None
        self.rmaps = None          # region-local lower-bound maps (full phase)
        self.lists_fresh = False   # candidate lists already match the current parameters
        self.walk = False          # sparse warm-up rounds use the walk kernel (flags bit 1)
        f = N.FoldArgs()
        f.X, f.ldx, f.d, f.k, f.order3 = self.X.data_ptr(), self.ldx, d, k, self.order3
        f.wmode, f.w, f.a = a.wmode, a.w, self.A.data_ptr()
        f.n_local, f.pos0, f.n_global = n, self.pos0, self.n_global
        f.centers = self.centers_d.data_ptr()
        fo = self.fold_out.data_ptr()
        f.sums, f.wsum, f.extent, f.objective = fo, fo + 8 * k * d, fo + 8 * k * (d + 1), \
            fo + 8 * k * (d + 2)
        f.workspace, f.workspace_bytes = self.fold_ws.data_ptr(), self.fold_ws.numel()
        self.fargs = f

    def _infl_ptr(self, which):
        return self.kstate.data_ptr() + 8 * self.settings.k * which

    def _set_influence(self, new_infl, moves=None, reset=False):
        """Upload the next influences (pinned, async) and compose the bound maps on the
        device (gp_update_maps): the relaxation of kmeans.py:208-239, lazily."""
        k = self.settings.k
        nxt = 1 - self.cur
        self.infl_h.numpy()[:] = new_infl
        self.kstate[nxt * k:(nxt + 1) * k].copy_(self.infl_h, non_blocking=True)
        mv = None
        if moves is not None:
            self.moves_h.numpy()[:] = moves
            self.kstate[4 * k:5 * k].copy_(self.moves_h, non_blocking=True)
            mv = self.kstate.data_ptr() + 32 * k
        old = self._infl_ptr(nxt if reset else self.cur)
        mb = self.kmaps.data_ptr()
        N.call("gp_update_maps", old, self._infl_ptr(nxt), mv, k, self.mapstate.data_ptr(),
               self.aargs.inv2_lo, self.aargs.inv2_hi, mb, mb + 16 * k, mb + 32 * k,
               self.mapflag.data_ptr(), 1 if reset else 0, self.scale_hint, self.sh)
        self.cur = nxt
        self.aargs.infl = self._infl_ptr(nxt)
        self.aargs.inv2_min = 1.0 / float(np.max(new_infl)) ** 2 * (1.0 - 1e-15)
        if self.rmaps is not None:
            self._relax_regions(old, self._infl_ptr(nxt), mv, reset)

    def _enter_region_maps(self, infl):
        """Full phase with a candidate hierarchy: every super group gets its own
        lower-bound map (gp_region_maps).  Bounds are materialised under the global
        maps first, then every map restarts from identity."""
        a = self.aargs
        N.count("gp_rebase_bounds")
        N.check(N.lib.gp_rebase_bounds(C.byref(a), self.sh), "gp_rebase_bounds")
        self.mapflag.zero_()
        self._alloc_region_maps(self.hier.ns)
        self._set_influence(infl, reset=True)
        a.lb_rpar, a.lb_rshift = self.rpar.data_ptr(), self.hier.SUPER_SHIFT

    def _relax_regions(self, old_ptr, new_ptr, moves_ptr, reset):
        h = self.hier
        if not reset:
            h.refresh()                # the lists under the new centers and influences
            self.lists_fresh = True
        N.call("gp_region_maps", self.mapstate.data_ptr(), self.settings.k,
               h.slist.data_ptr(), h.scount.data_ptr(), h.SUPER_CAP, self.rmaps,
               self.rstate.data_ptr(), self.rpar.data_ptr(), self.mapflag.data_ptr(),
               1 if reset else 0, self.scale_hint, self.sh)

    def _upload_centers(self, centers: np.ndarray):
        """Stream-ordered async H2D of the next centers through a pinned buffer."""
        if getattr(self, "cen_h", None) is None:
            self.cen_h = torch.empty(centers.shape, dtype=torch.float64, pin_memory=True)
            self.cen_evt = None
        if self.cen_evt is not None:
            self.cen_evt.synchronize()
        self.cen_h.numpy()[:] = centers
        self.centers_d.copy_(self.cen_h, non_blocking=True)
        self.cen_evt = torch.cuda.Event()
        self.cen_evt.record(self.stream)

    def _build_grid(self, centers: np.ndarray):
        """Uniform grid over the point box holding the centers (gp_center_grid on the
        device copy of the centers), walked by scan units whose candidate set
        overflows and by the walk kernel (gp_assign_args.grid_*)."""
        k, d = centers.shape
        lo = self.box.lo
        ext = float((self.box.hi - self.box.lo).max())
        G = int(np.ceil((k / 2.0) ** (1.0 / d)))
        G = max(1, min(G, 1024 if d == 2 else 128))
        h = ext / G * (1.0 + 1e-12) if ext > 0 else 1.0
        ncell = G ** d
        if getattr(self, "grid_cap", (0, 0)) != (ncell, k):
            self.grid_cap = (ncell, k)
            self.grid_dev = torch.empty(ncell + 1 + k, dtype=torch.int32, device=self.device)
            gwb = N.size_query("gp_center_grid_workspace_bytes", k)
            self.grid_ws = torch.empty(gwb, dtype=torch.uint8, device=self.device)
        self.grid_start = self.grid_dev[:ncell + 1]
        self.grid_items = self.grid_dev[ncell + 1:]
        lo3 = (C.c_double * 3)(*[float(v) for v in lo] + [0.0] * (3 - d))
        N.call("gp_center_grid", self.centers_d.data_ptr(), k, d, lo3, h, G,
               self.grid_start.data_ptr(), self.grid_items.data_ptr(), self.grid_ws.data_ptr(),
               self.grid_ws.numel(), self.sh)
        a = self.aargs
        a.grid_n, a.grid_h = G, h
        a.grid_start, a.grid_items = self.grid_start.data_ptr(), self.grid_items.data_ptr()
        for j in range(d):
            a.grid_lo[j] = float(lo[j])

    def _set_active(self, size):
        m = self._set_active_list(size)
        # (general-weight mode folds block weights from the full arrays every round)
        dense = size is not None and self.wplan.exact
        if dense:
            self._enter_dense(m)
        # sparse warm-up samples (few points per center): warp-per-point grid walks
        # (gp_assign_args.flags bit 1) need no candidate lists, unit boxes or region maps
        a = self.aargs
        k = self.settings.k
        # decided on the global sample size, so every rank of a sharded run agrees
        self.walk = (size is not None and a.grid_n > 0 and k >= WALK_MIN_K
                     and size <= WALK_RATIO * k)
        a.flags = (a.flags & ~2) | (2 if self.walk else 0)
        if self.walk:
            return m
        if self.hier is not None:
            self.hier.prepare(self.aargs.list, m)
        self._unit_boxes(m)
        if dense and self.hier is not None:
            self._sample_region_maps()
        return m

    def _alloc_region_maps(self, R):
        if getattr(self, "rcap", 0) < R:
            self.rcap = R
            self.rstate = torch.empty(3 * R, dtype=torch.float64, device=self.device)
            self.rpar = torch.empty(4 * R, dtype=torch.float32, device=self.device)
        self.rmaps = R

    def _sample_region_maps(self):
        """Dense warm-up sample: region-local lower-bound maps over the sample's super
        groups for this step's balance rounds (lower bounds materialised under the
        global map on entry, renormalised to it in _leave_dense)."""
        a = self.aargs
        N.call("gp_lb_remap", C.byref(a), 0, self.sh)
        self._alloc_region_maps(self.hier.ns)
        N.call("gp_region_maps", None, self.settings.k, None, None, 0, self.rmaps,
               self.rstate.data_ptr(), self.rpar.data_ptr(), self.mapflag.data_ptr(), 1,
               self.scale_hint, self.sh)
        a.lb_rpar, a.lb_rshift = self.rpar.data_ptr(), self.hier.SUPER_SHIFT

    def _unit_boxes(self, m):
        """Static box of every scan unit over its active entries (once per active set)."""
        a = self.aargs
        shift = 8 + (a.scan_regions.bit_length() - 1)
        key = (a.X, a.list, m, shift)
        if getattr(self, "ubox_key", None) == key:   # the full phase's set never changes
            a.unit_boxes, a.unit_shift = self.ubox.data_ptr(), shift
            return
        self.ubox_key = key
        nu = max(1, (m + (1 << shift) - 1) >> shift)
        if getattr(self, "ubox_cap", 0) < nu:
            self.ubox_cap = max(nu, (self.n + 255) >> 8)
            self.ubox = torch.empty(self.ubox_cap * 2 * self.d, dtype=torch.float64,
                                    device=self.device)
        N.call("gp_group_boxes", a.X, self.ldx, self.d, a.list, m, shift, self.ubox.data_ptr(),
               self.sh)
        a.unit_boxes, a.unit_shift = self.ubox.data_ptr(), shift

    def _enter_dense(self, m):
        """Sample phase: gather the active entries' state into dense arrays so the
        ~20 balance rounds of this movement iteration stream contiguous memory."""
        d, dev = self.d, self.device
        if getattr(self, "dense_cap", 0) < m:
            cap = max(self.sizes)
            self.dense_cap = cap
            self.A_d = torch.empty(cap, dtype=torch.int32, device=dev)
            self.UBLB_d = torch.empty((cap, 2), dtype=torch.float16, device=dev)
            self.X_d = torch.empty((cap, d), dtype=torch.float64, device=dev)
            self.W_d = None if self.W is None else torch.empty(cap, dtype=self.W.dtype, device=dev)
        wbytes = 0 if self.W is None else self.W.element_size()
        N.call("gp_gather_state", self.active_idx.data_ptr(), m, d, self.A.data_ptr(),
               self.UBLB.data_ptr(), self.X.data_ptr(), _ptr(self.W), wbytes,
               self.A_d.data_ptr(), self.UBLB_d.data_ptr(), self.X_d.data_ptr(), _ptr(self.W_d),
               self.sh)
        a = self.aargs
        a.X, a.a, a.ublb, a.w = (self.X_d.data_ptr(), self.A_d.data_ptr(),
                                 self.UBLB_d.data_ptr(), _ptr(self.W_d))
        a.list, a.m = None, m
        a.scan_regions = full_scan_regions(m, self.settings.k)  # dense SFC-ordered entries
        self.dense_m = m

    def _leave_dense(self):
        """Write the dense sample state back and point the kernels at the full arrays.
        The movement fold that follows still reads the dense arrays (gp_fold_args.list)."""
        if not getattr(self, "dense_m", 0):
            self.fold_dense = None
            return
        self.fold_dense = self.dense_m
        if self.rmaps is not None:
            # region maps end with the sample step: back to the global lower-bound map
            N.call("gp_lb_remap", C.byref(self.aargs), 1, self.sh)
            self.aargs.lb_rpar = None
            self.rmaps = None
        N.call("gp_scatter_state", self.active_idx.data_ptr(), self.dense_m, self.A_d.data_ptr(),
               self.UBLB_d.data_ptr(), self.A.data_ptr(), self.UBLB.data_ptr(), self.sh)
        a = self.aargs
        a.X, a.a, a.ublb, a.w = (self.X.data_ptr(), self.A.data_ptr(), self.UBLB.data_ptr(),
                                 _ptr(self.W))
        self.dense_m = 0

    def _set_active_list(self, size):
        a = self.aargs
        if size is None:
            a.list, a.m = None, self.n
            a.scan_regions = full_scan_regions(self.n_global, self.settings.k)
            return self.n
        a.scan_regions = 1       # sparse warm-up sample: 256-entry units
        ranks, pos, cnt = self._sample_candidates(size)
        N.call("gp_compact_candidates", ranks.data_ptr(), _ptr(pos), cnt, size,
               self.active_idx.data_ptr(), self.active_cnt.data_ptr(),
               self.compact_ws.data_ptr(), self.compact_ws.numel(), self.sh)
        m = int(self.active_cnt.item())
        a.list, a.m = self.active_idx.data_ptr(), m
        return m

    # sample sizes below these limits are compacted from a candidate list (the positions
    # and ranks of the entries with rank < limit, built once) instead of all n ranks
    CANDIDATE_TIERS = (1 << 26, 1 << 22)

    def _sample_candidates(self, size):
        """(ranks, positions or None, count) to compact the sample `rank < size` from."""
        if getattr(self, "cand_tiers", None) is None:
            self.cand_tiers = []
            ranks, pos, cnt = self.rank_sfc, None, self.n
            for limit in self.CANDIDATE_TIERS:       # large to small, each from the last
                if cnt < 8 * limit:
                    continue
                idx = torch.empty(limit, dtype=torch.int32, device=self.device)
                N.call("gp_compact_candidates", ranks.data_ptr(), _ptr(pos), cnt, limit,
                       idx.data_ptr(), self.active_cnt.data_ptr(), self.compact_ws.data_ptr(),
                       self.compact_ws.numel(), self.sh)
                c = int(self.active_cnt.item())
                pos = idx[:c]
                ranks = self.rank_sfc[pos.long()].contiguous()
                cnt = c
                self.cand_tiers.append((limit, ranks, pos, c))
        best = (self.rank_sfc, None, self.n)
        for limit, ranks, pos, c in self.cand_tiers:
            if size <= limit:
                best = (ranks, pos, c)
        return best

    def _assign(self):
        if self.hier is not None and not self.lists_fresh and not self.walk:
            self.hier.refresh()
        self.lists_fresh = False
        self.red.zero_()
        if self.timer is not None:
            tok = self.timer.begin(self.stream, self.aargs)
        if _NVTX:
            torch.cuda.nvtx.range_push(f"round{_round_counter()}")
        N.count("gp_assign_round")
        N.check(N.lib.gp_assign_round(C.byref(self.aargs), self.sh), "gp_assign_round")
        if _NVTX:
            torch.cuda.nvtx.range_pop()
        if self.timer is not None:
            self.timer.end(self.stream, self.aargs, tok)
        self._reduce_round()
        self.red_h.copy_(self.red, non_blocking=True)
        self.stream.synchronize()
        host = self.red_h.numpy()
        k = self.settings.k
        cnt = host[k:k + 3].copy()
        cnt[1] = self.m_global  # every active entry is one decision (kmeans.py:309)
        if self.timer is not None:
            self.timer.rounds.append((int(cnt[1]), int(cnt[1] - cnt[0]), int(cnt[2])))
            if self.aargs.flags & 1:
                st = np.zeros(8, dtype=np.uint64)
                N.check(N.lib.gp_scan_stats(st.ctypes.data, 1), "gp_scan_stats")
                self.timer.scan.append(st)
        return host[:k].copy(), cnt

    # ---- hooks the multi-GPU partitioner overrides (one shard: nothing to exchange)
    def _reduce_round(self):
        pass

    def _audit_totals(self):
        return self.audit_out.cpu().numpy()

    def _global_count(self, m):
        return m

    def _fold(self, weights_only):
        f = self.fargs
        f.weights_only = weights_only
        m = getattr(self, "fold_dense", None) if not weights_only else None
        if m:
            # warm-up sample: fold the dense active entries (SFC order) at their positions
            f.X, f.a, f.w = self.X_d.data_ptr(), self.A_d.data_ptr(), _ptr(self.W_d)
            f.list, f.m = self.active_idx.data_ptr(), m
        else:
            f.X, f.a, f.w = self.X.data_ptr(), self.A.data_ptr(), _ptr(self.W)
            f.list, f.m = None, 0
        if _NVTX:
            torch.cuda.nvtx.range_push(f"fold{_fold_counter()}")
        N.count("gp_movement_fold")
        N.check(N.lib.gp_movement_fold(C.byref(f), self.sh), "gp_movement_fold")
        if _NVTX:
            torch.cuda.nvtx.range_pop()

    def _block_weights(self, blk_int):
        if self.wplan.exact:
            return blk_int.astype(np.float64) / self.wplan.scale
        self._fold(1)
        k = self.settings.k
        return self.fold_out[k * self.d:k * (self.d + 1)].cpu().numpy().copy()

    # ------------------------------------------------------------ main loop
    def run(self):
        st, n, d, k = self.settings, self.n, self.d, self.settings.k
        self._alloc_state()
        centers = self.init_centers.copy()
        infl = np.ones(k)
        block_w = np.zeros(k)
        last_move = np.zeros(k)
        self.scale_hint = max(self.box.diagonal(), 1e-300)
        self._set_influence(infl, reset=True)
        self._build_grid(centers)
        threshold = st.delta_threshold
        if threshold is None:
            threshold = 1e-4 * self.box.diagonal()
        stats = KMeansStats()
        plan = [("sample", s) for s in self.sizes] + [("full", None)] * st.max_iter
        info = None
        fallback = None
        for step, (phase, size) in enumerate(plan):
            m = self._set_active(size)
            self.m_global = self._global_count(m)
            if phase == "full" and self.hier is not None and self.rmaps is None:
                self._enter_region_maps(infl)
            # ---------------- assign_and_balance (kmeans.py:377-453)
            if self._device_decide_ok():
                info, infl = self._balance_device(infl)
            else:
                info, infl = self._balance_host(infl)
            block_w = info.block_weights
            self._leave_dense()
            if phase == "full" and info.imbalance <= st.epsilon:
                # the assignment at this point is the exact argmin under (centers, infl);
                # it is recomputed from them only if the fallback is taken (no n-sized copy)
                fallback = (ClusterState(centers.copy(), infl.copy(), block_w.copy(),
                                         last_move.copy()), info.imbalance)
            # ---------------- movement (kmeans.py:585-626)
            self._fold(0)
            if getattr(self, "fold_h", None) is None:
                self.fold_h = torch.empty(self.fold_out.numel(), dtype=torch.float64,
                                          pin_memory=True)
            self.fold_h.copy_(self.fold_out, non_blocking=True)
            self.stream.synchronize()
            red = self.fold_h.numpy()   # read before the next fold overwrites it
            sums = red[:k * d].reshape(k, d)
            totals = red[k * d:k * (d + 1)]
            extents = red[k * (d + 1):k * (d + 2)]
            obj_parts = red[k * (d + 2):k * (d + 3)]
            empty = totals == 0
            any_empty = bool(empty.any())
            if any_empty:
                safe = np.where(empty, 1.0, totals)
                new_centers = sums / safe[:, None]
                new_centers[empty] = centers[empty]
            else:   # the common case, same bits: no block lost all its points
                new_centers = sums / totals[:, None]
            moves = row_norms(new_centers - centers)
            stats.iterations.append(IterationRecord(
                phase=phase, active_points=self.m_global, balance_rounds=info.rounds,
                imbalance=info.imbalance, skip_decisions=info.skip_decisions,
                total_decisions=info.total_decisions, distance_evals=info.distance_evals,
                objective=float(obj_parts.sum()), max_move=float(moves.max())))
            last = step == len(plan) - 1
            converged = phase == "full" and float(moves.max()) < threshold
            if converged or last:
                stats.converged = converged
                break
            old_infl = infl
            # (x * 1.0 is x: without empty blocks the influences enter the erosion as is)
            nxt = old_infl * np.where(empty, 1.0 + st.influence_step_cap, 1.0) if any_empty \
                else old_infl.copy()
            if st.erosion:
                nonempty = block_w > 0
                if nonempty.all():   # the mean of the same elements in the same order
                    beta = float(2.0 * extents.mean())
                else:
                    beta = float(2.0 * extents[nonempty].mean()) if nonempty.any() else 0.0
                if beta > 0:
                    nxt = eroded(nxt, moves, beta)
            centers = new_centers
            infl = nxt
            last_move = moves
            self._upload_centers(centers)
            self._build_grid(centers)
            self._set_influence(infl, moves=moves)
            if int(self.mapflag.item()):
                # cumulative maps drifted out of range: materialise every bound and restart
                # from identity maps (result-invariant; only skip tightness changes)
                a = self.aargs
                lst, mm = a.list, a.m
                a.list, a.m = None, n
                N.count("gp_rebase_bounds")
                N.check(N.lib.gp_rebase_bounds(C.byref(a), self.sh), "gp_rebase_bounds")
                a.list, a.m = lst, mm
                self.mapflag.zero_()
                self._set_influence(infl, reset=True)

        final_state = ClusterState(centers, infl, block_w, last_move)
        final_imb = info.imbalance
        A = self.A
        if final_imb > st.epsilon and fallback is not None:
            final_state, final_imb = fallback
            A = self._recompute(final_state)
        stats.balance_failed = final_imb > st.epsilon
        stats.final_state = final_state
        if st.audit_bounds:
            aud = self._audit_totals()
            stats.audited_point_iterations = int(aud[0])
            stats.bound_violations = int(aud[1])
            stats.skip_check_failures = int(aud[2])
        out = self._deliver(A)
        self.release()
        return out, stats

    def _device_decide_ok(self) -> bool:
        """d = 2 (the influence step is a sqrt), exact integer block weights, no audit
        or per-round scan statistics: the round's decision and influence step run on
        the device (gp_balance_decide) and the host only reads a few scalars per
        round.  Sharded runs all-reduce the k + 3 int64 sums first, so every rank takes
        the same decision.  GP_DEVICE_DECIDE=0 turns it off."""
        return (self.d == 2 and self.wplan.exact
                and not self.settings.audit_bounds and not (self.aargs.flags & 1)
                and os.environ.get("GP_DEVICE_DECIDE", "1") != "0")

    def _balance_device(self, infl):
        """assign_and_balance (kmeans.py:377-453) driven by the host, decided on the
        device: per round the assign kernels, gp_balance_decide (imbalance, stop
        test, step halving and the next influences), a read-back of its record
        (6 doubles) and, when the loop goes on, the bound-map / candidate-list /
        region-map update from the device influences.  No k-sized host math or
        transfers inside the loop."""
        st, k, a = self.settings, self.settings.k, self.aargs
        mr = st.max_balance_iter
        if getattr(self, "bal", None) is None or self.bal.numel() < 8 + 3 * mr:
            self.bal = torch.empty(8 + 3 * mr, dtype=torch.float64, device=self.device)
            self.bal_h = torch.empty(8 + 3 * mr, dtype=torch.float64, pin_memory=True)
            self.bal_init = torch.empty(8, dtype=torch.float64, pin_memory=True)
        cur, nxt = self.cur, 1 - self.cur
        cur_p, nxt_p = self._infl_ptr(cur), self._infl_ptr(nxt)
        cur_t = self.kstate[cur * k:(cur + 1) * k]
        nxt_t = self.kstate[nxt * k:(nxt + 1) * k]
        self.bal_init.numpy()[:] = [st.influence_step_cap, 0.0, math.inf, 0.0, 0.0, 0.0, 0.0, 0.0]
        self.bal[:8].copy_(self.bal_init, non_blocking=True)
        mb = self.kmaps.data_ptr()
        bh = self.bal_h.numpy()
        rounds = 0
        for rnd in range(mr):
            if rnd > 0:
                # the influence step decided last round (kmeans.py:437-443)
                N.call("gp_update_maps", cur_p, nxt_p, None, k, self.mapstate.data_ptr(),
                       a.inv2_lo, a.inv2_hi, mb, mb + 16 * k, mb + 32 * k,
                       self.mapflag.data_ptr(), 0, self.scale_hint, self.sh)
                if self.rmaps is not None:
                    self._relax_regions(cur_p, nxt_p, None, False)
                cur_t.copy_(nxt_t)
            if self.hier is not None and not self.lists_fresh and not self.walk:
                self.hier.refresh()
            self.lists_fresh = False
            self.red.zero_()
            if self.timer is not None:
                tok = self.timer.begin(self.stream, a)
            if _NVTX:
                torch.cuda.nvtx.range_push(f"round{_round_counter()}")
            N.count("gp_assign_round")
            N.check(N.lib.gp_assign_round(C.byref(a), self.sh), "gp_assign_round")
            if _NVTX:
                torch.cuda.nvtx.range_pop()
            if self.timer is not None:
                self.timer.end(self.stream, a, tok)
            self._reduce_round()   # sharded runs: every rank decides on the global sums
            N.call("gp_balance_decide", self.red.data_ptr(), k, float(self.wplan.scale),
                   float(st.epsilon), mr, self.bal.data_ptr(), cur_p, nxt_p, self.sh)
            self.bal_h[:8].copy_(self.bal[:8], non_blocking=True)
            self.stream.synchronize()
            rounds += 1
            if bh[4] == 1.0:     # imbalance() of metrics.py:33-40
                raise GraphError("total weight must be positive")
            if bh[4] != 0.0:
                raise ValueError("target weight must be positive")
            if bh[5] != 0.0:    # stop (the next influences were not written)
                break
        self.red_h.copy_(self.red, non_blocking=True)
        self.bal_h.copy_(self.bal, non_blocking=True)
        self.stream.synchronize()
        bal = self.bal_h.numpy()
        hist = [float(v) for v in bal[8:8 + rounds]]
        skips_r = bal[8 + mr:8 + mr + rounds].astype(np.int64)
        evals_r = bal[8 + 2 * mr:8 + 2 * mr + rounds].astype(np.int64)
        block_w = self._block_weights(self.red_h.numpy()[:k].copy())
        if rounds > 1:   # the influences the last round used
            infl = cur_t.cpu().numpy().copy()
            a.inv2_min = 1.0 / float(np.max(infl)) ** 2 * (1.0 - 1e-15)
        if self.timer is not None:
            for sk, ev in zip(skips_r, evals_r):
                self.timer.rounds.append((self.m_global, int(self.m_global - sk), int(ev)))
        info = BalanceInfo(rounds, hist[-1], block_w, int(skips_r.sum()),
                           rounds * self.m_global, int(evals_r.sum()), hist)
        return info, infl

    def _balance_host(self, infl):
        """assign_and_balance (kmeans.py:377-453) with one host round trip per round."""
        st, d, k = self.settings, self.d, self.settings.k
        skips = decisions = evals = 0
        final_imb = math.inf
        best_imb = math.inf
        cap = st.influence_step_cap
        regressions = 0
        history = []
        rounds = 0
        for rnd in range(st.max_balance_iter):
            rounds += 1
            if st.audit_bounds:
                N.count("gp_audit")
                N.check(N.lib.gp_audit(C.byref(self.aargs), self.audit_out.data_ptr(), self.sh),
                        "gp_audit")
            blk, cnt = self._assign()
            skips += int(cnt[0])
            decisions += int(cnt[1])
            evals += int(cnt[2])
            block_w = self._block_weights(blk)
            final_imb = imbalance(block_w)
            history.append(final_imb)
            if final_imb <= st.epsilon or rnd == st.max_balance_iter - 1:
                break
            if final_imb > best_imb:
                regressions += 1
                if regressions >= 2:
                    cap *= 0.5
            best_imb = min(best_imb, final_imb)
            target = float(block_w.sum()) / k
            if not target > 0:
                raise ValueError("target weight must be positive")
            new_infl = infl * influence_factor(block_w, target, cap, d)
            infl = new_infl
            self._set_influence(infl)
        info = BalanceInfo(rounds, final_imb, block_w, skips, decisions, evals, history)
        return info, infl

    def _recompute(self, state: ClusterState):
        """The fallback assignment (kmeans.py:583-584, 627-630): one assign round from
        cold bounds under the fallback centers and influences reproduces it exactly."""
        self.centers_d.copy_(torch.from_numpy(np.ascontiguousarray(state.centers)))
        self._build_grid(state.centers)
        self._set_influence(state.influence, reset=True)
        self._cold_bounds()
        self.lists_fresh = False
        self._assign()
        return self.A

    def _deliver(self, A):
        """int64 assignment by original id (kmeans.py:637-641)."""
        if _NVTX:
            torch.cuda.nvtx.range_push("deliver")
        try:
            return self._deliver_ids(A)
        finally:
            if _NVTX:
                torch.cuda.nvtx.range_pop()

    def _deliver_ids(self, A):
        out = torch.empty(self.n, dtype=torch.int64, device=self.device)
        # one shard: the gids are a permutation of 0..n-1, delivered without random writes
        # (radix-grouped windows); the sort scratch reuses the buffers the run is done with
        for name in ("UBLB", "A_d", "UBLB_d", "X_d", "W_d", "rank_sfc", "active_idx", "assign_ws",
                     "fold_ws"):
            if hasattr(self, name):
                setattr(self, name, None)
        wsb = N.size_query("gp_deliver_workspace_bytes", self.n)
        ws = torch.empty(max(wsb, 8), dtype=torch.uint8, device=self.device)
        N.call("gp_deliver_permutation", A.data_ptr(), self.gids.data_ptr(), self.n,
               out.data_ptr(), ws.data_ptr(), wsb, self.sh)
        return out

    def release(self):
        """Drop every n-sized device buffer (the caller keeps only the result)."""
        for name in ("X", "W", "A", "UBLB", "A_d", "UBLB_d", "X_d", "W_d", "gids", "rank_sfc", "active_idx",
                     "assign_ws", "fold_ws", "compact_ws", "keys_sorted", "hier", "grid_start",
                     "grid_items", "ubox", "rstate", "rpar", "cand_tiers"):
            if hasattr(self, name):
                setattr(self, name, None)


class DistributedPartitioner(DevicePartitioner):
    """One shard of a multi-GPU partition (one process per GPU, torch.distributed).

    Every rank passes its own contiguous block of the original rows (in rank order,
    like RankWorld.from_points deals them).  The SFC bootstrap redistributes points into
    contiguous ranges of the global (key, gid) order on 256-segment boundaries
    (parallel.sfc_redistribute); each balance round all-reduces the k exact int64 block
    weights; each movement iteration gathers the (segment, block) fold partials and folds
    them in global segment order.  All k-sized host math is identical on every rank, so
    the result is bit-identical to one GPU's (and to the reference's).
    """

    def __init__(self, settings, comm, device=None, timer=None):
        super().__init__(settings, device=device, timer=timer)
        self.comm = comm

    # ---------------------------------------------------------------- bootstrap
    def _device_sort(self, keys: torch.Tensor) -> torch.Tensor:
        """Stable permutation sorting int64 keys (device radix sort, sort_pairs)."""
        m = keys.shape[0]
        vo = torch.empty(m, dtype=torch.int32, device=keys.device)
        sort_pairs(keys.contiguous(), None, None, vo, self.key_bits, self.sh)
        return vo.long()

    def bootstrap(self, points, weights):
        from . import parallel as P

        st, comm = self.settings, self.comm
        pts, w = self._input(points, weights)
        n_in, d = pts.shape
        self.d = d
        # local argument errors are agreed on before any other collective, so every rank
        # raises the same error instead of one rank leaving the others blocked
        chk = torch.tensor([1 if n_in < 1 else 0, 1 if w is None else 0, 1 if w is not None else 0,
                            d], dtype=torch.int64, device=self.device)
        mx = comm.allreduce(chk.clone(), P.dist.ReduceOp.MAX).cpu().tolist()
        mn = comm.allreduce(chk.clone(), P.dist.ReduceOp.MIN).cpu().tolist()
        if mx[0]:
            raise ValueError("every rank needs at least one point")
        if mx[1] and mx[2]:
            raise ValueError("weights must be given on every rank or on none")
        if mx[3] != mn[3]:
            raise GeometryError("all ranks must pass points of the same dimension")
        off, n = P.input_offsets(n_in, comm)
        self.in_offset, self.n_in = off, n_in
        k = st.k
        if k > n:
            raise ValueError(f"k={k} exceeds the number of points {n}")
        depth = st.sfc_depth if st.sfc_depth is not None else DEFAULT_DEPTH.get(d)
        if depth is None or d not in (2, 3):
            raise GeometryError(f"unsupported dimension {d}")
        if d * depth > 62:
            raise GeometryError(f"depth {depth} out of range for dimension {d}")
        self.key_bits = d * depth
        dev, sh = self.device, self.sh
        sp, sd = pts.stride()
        # K1 box: local min/max + allreduce MIN/MAX (kmeans.py:546-548)
        lohi = torch.empty(2 * d, dtype=torch.float64, device=dev)
        bad = torch.empty(1, dtype=torch.int32, device=dev)
        N.call("gp_box_minmax", pts.data_ptr(), n_in, d, sp, sd, lohi.data_ptr(), bad.data_ptr(), sh)
        comm.allreduce(lohi[:d], P.dist.ReduceOp.MIN)
        comm.allreduce(lohi[d:], P.dist.ReduceOp.MAX)
        comm.allreduce(bad, P.dist.ReduceOp.MAX)
        lohi_h = lohi.cpu().numpy()
        if int(bad.item()):
            raise GeometryError("non-finite box corner")
        self.box = BoundingBox(lohi_h[:d].copy(), lohi_h[d:].copy())
        # weight plan agreed by all ranks
        self.wplan = self._weight_plan_global(w, n_in, n)
        # K2 keys (gids = global ids) + local sort
        keys = torch.empty(n_in, dtype=torch.int64, device=dev)
        gids = torch.empty(n_in, dtype=torch.int32, device=dev)
        N.call("gp_hilbert_keys", pts.data_ptr(), n_in, d, sp, sd, lohi.data_ptr(), depth,
               keys.data_ptr(), gids.data_ptr(), off, sh)
        perm = self._device_sort(keys)
        keys_s = keys[perm]
        gids_s = gids[perm]
        local_idx = (gids_s - off).to(torch.int32)
        X_s = torch.empty((n_in, d), dtype=torch.float64, device=dev)
        W_s = None
        if w is not None:
            W_s = torch.empty(n_in, dtype=torch.float32 if self.wplan.mode == 1 else torch.float64,
                              device=dev)
        N.call("gp_gather_points", pts.data_ptr(), sp, sd, d, local_idx.data_ptr(), n_in,
               X_s.data_ptr(), d, _ptr(w), self.wplan.mode if w is not None else 0, _ptr(W_s), sh)
        payload = [gids_s, X_s] + ([W_s] if W_s is not None else [])
        keys_r, pay_r = P.sfc_redistribute(keys_s, payload, n, comm, self.key_bits,
                                           self._device_sort)
        del keys, gids, perm, keys_s, gids_s, local_idx, X_s, W_s, payload
        bounds = P.shard_bounds(n, comm.world)
        self.n, self.pos0, self.n_global = int(keys_r.shape[0]), int(bounds[comm.rank]), n
        assert self.n == bounds[comm.rank + 1] - bounds[comm.rank]
        self.gids = pay_r[0].contiguous()
        self.X = pay_r[1].contiguous()
        self.W = pay_r[2].contiguous() if w is not None else None
        self.ldx = d
        self.keys_sorted = keys_r if self.keep_keys else None
        # K4 initial centers: the owner of each global position contributes its rows
        pos = initial_center_positions(n, k)
        mine = pos[(pos >= self.pos0) & (pos < self.pos0 + self.n)] - self.pos0
        rows = self.X[torch.from_numpy(mine).to(dev)] if len(mine) else \
            torch.empty((0, d), dtype=torch.float64, device=dev)
        cen = torch.cat(comm.allgather_var(rows)).contiguous()
        self.centers_d = cen
        self.init_centers = cen.cpu().numpy().copy()
        # warm-up sample order over all n (every rank derives the same permutation)
        self.sizes = sample_schedule(n, st.init_sample)
        if self.sizes:
            rank_d = sample_ranks_device(n, st.seed, dev, sh)
            self.rank_sfc = torch.empty(self.n, dtype=torch.int32, device=dev)
            N.call("gp_gather_ranks", rank_d.data_ptr(), self.gids.data_ptr(), self.n,
                   self.rank_sfc.data_ptr(), sh)
            cwb = N.size_query("gp_compact_workspace_bytes", self.n)
            self.compact_ws = torch.empty(max(cwb, 8), dtype=torch.uint8, device=dev)
            self.active_idx = torch.empty(self.n, dtype=torch.int32, device=dev)
            self.active_cnt = torch.empty(1, dtype=torch.int64, device=dev)
            del rank_d
        del pts, w
        return self

    def _weight_plan_global(self, w, n_in, n) -> _WeightPlan:
        from . import parallel as P

        flags = torch.zeros(4, dtype=torch.float64, device=self.device)
        has = torch.tensor([0.0 if w is None else 1.0], dtype=torch.float64, device=self.device)
        self.comm.allreduce(has, P.dist.ReduceOp.MAX)
        if float(has.item()) == 0.0:
            return _WeightPlan(0, True, 1.0)
        assert w is not None   # agreed in bootstrap()
        out = torch.empty(3, dtype=torch.int64, device=self.device)
        N.call("gp_weight_probe", w.data_ptr(), n_in, out.data_ptr(), self.sh)
        fl, low, mxb = (int(v) for v in out.cpu().tolist())
        mx = float(np.array([mxb], dtype=np.int64).view(np.float64)[0])
        flags[0] = float(fl & 1)
        flags[1] = float((fl >> 1) & 1)
        flags[2] = float(-low)
        flags[3] = mx
        self.comm.allreduce(flags, P.dist.ReduceOp.MAX)
        f = flags.cpu().numpy()
        if f[0]:
            return _WeightPlan(2, False, 1.0)
        mode = 2 if f[1] else 1
        low = -int(f[2])
        s = max(0, -low) if low < 4096 else 0
        exact = s <= 1000 and f[3] * 2.0 ** s * n < 2.0 ** 53
        return _WeightPlan(mode, bool(exact), 2.0 ** s if exact else 1.0)

    # ---------------------------------------------------------------- exchanges
    def _reduce_round(self):
        self.comm.allreduce(self.red)

    def _global_count(self, m):
        t = torch.tensor([m], dtype=torch.int64, device=self.device)
        return int(self.comm.allreduce(t).item())

    def _audit_totals(self):
        return self.comm.allreduce(self.audit_out.clone()).cpu().numpy()

    def _fold(self, weights_only):
        from . import parallel as P

        super()._fold(weights_only)
        k, d = self.settings.k, self.d
        if not hasattr(self, "pair_keys"):
            cap = min((256 // self.comm.world + 2) * k, self.n + 1)
            self.pair_keys = torch.empty(cap, dtype=torch.int64, device=self.device)
            self.pair_vals = torch.empty((cap, 6), dtype=torch.float64, device=self.device)
            self.pair_n = torch.empty(1, dtype=torch.int64, device=self.device)
            cb = N.size_query("gp_fold_combine_bytes", k)
            self.combine_ws = torch.empty(cb, dtype=torch.uint8, device=self.device)
        N.call("gp_fold_export", C.byref(self.fargs), self.pair_keys.data_ptr(),
               self.pair_vals.data_ptr(), self.pair_n.data_ptr(), self.sh)
        npairs = int(self.pair_n.item())
        keys, vals = P.gather_fold_pairs(self.pair_keys[:npairs], self.pair_vals[:npairs],
                                         self.comm)
        keys, vals = keys.contiguous(), vals.contiguous()
        fo = self.fold_out.data_ptr()
        N.call("gp_fold_combine", keys.data_ptr(), vals.data_ptr(), keys.shape[0], k, d,
               weights_only, fo, fo + 8 * k * d, fo + 8 * k * (d + 1), fo + 8 * k * (d + 2),
               self.combine_ws.data_ptr(), self.combine_ws.numel(), self.sh)

    def _recompute(self, state: ClusterState):
        """The fallback assignment (kmeans.py:583-584, 627-630): one assign round from
        cold bounds under the fallback centers and influences reproduces it exactly."""
        self.centers_d.copy_(torch.from_numpy(np.ascontiguousarray(state.centers)))
        self._build_grid(state.centers)
        self._set_influence(state.influence, reset=True)
        self._cold_bounds()
        self.lists_fresh = False
        self._assign()
        return self.A

    def _deliver(self, A):
        """Labels of this rank's own input rows, routed back from the SFC shards."""
        from . import parallel as P

        comm = self.comm
        offs = torch.tensor([t.item() for t in comm.allgather_var(
            torch.tensor([self.in_offset], dtype=torch.int64, device=self.device))] + [
            self.n_global], dtype=torch.int64, device=self.device)
        g = self.gids.long()
        owner = torch.searchsorted(offs, g, right=True) - 1
        order = torch.sort(owner, stable=True).indices
        send = torch.bincount(owner, minlength=comm.world).tolist()
        pair = torch.stack([g[order], A.long()[order]], dim=1)
        recv, _ = comm.alltoall(pair, send)
        out = torch.empty(self.n_in, dtype=torch.int64, device=self.device)
        out[recv[:, 0] - self.in_offset] = recv[:, 1]
        return out

    def release(self):
        super().release()
        for name in ("pair_keys", "pair_vals", "combine_ws"):
            if hasattr(self, name):
                setattr(self, name, None)


def partition_distributed(points, weights, settings: KMeansSettings, group=None, device=None,
                          timer=None):
    """Multi-GPU partition: this rank's contiguous block of original rows in, their
    int64 labels (device tensor) and the (global, rank-identical) KMeansStats out."""
    from .parallel import Comm

    eng = DistributedPartitioner(settings, Comm(group), device=device, timer=timer)
    eng.bootstrap(points, weights)
    return eng.run()


def partition_device(points, weights, settings: KMeansSettings, device=None, timer=None):
    """Run on one GPU; returns (device int64 assignment by original id, KMeansStats)."""
    eng = DevicePartitioner(settings, device=device, timer=timer)
    eng.bootstrap(points, weights)
    return eng.run()


def _finish(assign_dev, stats, k, return_stats):
    # int64 result (kmeans.py:637-641) into page-locked memory: one DMA, and the
    # numpy array keeps the pinned tensor alive
    host = torch.empty(assign_dev.shape, dtype=torch.int64, pin_memory=True)
    host.copy_(assign_dev)
    assignment = host.numpy()
    part = Partition(assignment=assignment, k=k, balance_failed=stats.balance_failed,
                     empty_blocks=np.flatnonzero(stats.final_state.block_weights == 0))
    return (part, stats) if return_stats else part


def balanced_kmeans_points(points, weights, settings: KMeansSettings, p: int = 1,
                           return_stats: bool = False):
    """Partition a raw point set (kmeans.py:502-512); identical results for every p.

    p is the GPU count: p > 1 shards the run over min(p, visible GPUs) devices
    (pool.py: one worker process per GPU, SFC-range shards, NCCL), p = 1 runs on
    the current device."""
    if not isinstance(points, torch.Tensor):
        points = np.asarray(points, dtype=np.float64)
    RankWorld.from_points(points, weights, p)  # rank-count validation (ranksim.py:98-100)
    G = 1
    if p > 1:
        from . import pool

        G = pool.gpu_count_for(p)
    if G > 1:
        if len(points.shape) != 2:
            raise GeometryError("points must be an (n, d) array")
        if weights is not None:
            check_weights(int(points.shape[0]), weights)
            weights = weights[:points.shape[0]]
        labels, stats = pool.get_pool(G).run(points, weights, settings)
        part = Partition(assignment=labels, k=settings.k, balance_failed=stats.balance_failed,
                         empty_blocks=np.flatnonzero(stats.final_state.block_weights == 0))
        return (part, stats) if return_stats else part
    assign_dev, stats = partition_device(points, weights, settings)
    return _finish(assign_dev, stats, settings.k, return_stats)


def balanced_kmeans(graph, settings: KMeansSettings, world: RankWorld | None = None,
                    return_stats: bool = False):
    """Partition a geometric graph's vertices (kmeans.py:515-534)."""
    if world is None:
        world = RankWorld.from_graph(graph)
    elif world.n != graph.n:
        raise ValueError("world does not match the graph")
    # the reference runs the pipeline on the world's own shards (kmeans.py:531-534), so a
    # world built from other coordinates or weights (same n) partitions those
    coords, weights = _world_arrays(world, graph)
    return balanced_kmeans_points(coords, weights, settings, p=world.p,
                                  return_stats=return_stats)


def _world_arrays(world, graph):
    """(coords, weights) a world partitions: this module's RankWorld carries them; a
    reference ``ranksim.RankWorld`` (reached through the INTEGRATION.md shim, e.g. from
    ``cli.py:110-111``) holds them as shards whose gids index the original rows
    (``ranksim.py:53-108``)."""
    shards = getattr(world, "shards", None)
    if shards is None:
        return (world.coords if world.coords is not None else graph.coords), world.weights
    n, d = int(world.n), int(world.dim)
    coords = np.empty((n, d), dtype=np.float64)
    weights = np.empty(n, dtype=np.float64)
    for sh in shards:
        g = np.asarray(sh.gids, dtype=np.int64)
        coords[g] = np.asarray(sh.points, dtype=np.float64)
        weights[g] = np.asarray(sh.weights, dtype=np.float64)
    return coords, weights
