/*
 * geopart_b200 — C ABI of the B200-native Geographer balanced k-means hot path.
 *
 * The reference (geopart, pure Python/numpy) has no FFI: its hot path is a set
 * of per-rank numpy passes plus simulated collectives.  Each entry point below
 * replaces one of those passes; the reference function it stands in for is
 * cited next to it (paths relative to /root/reference/pkg/src/geopart).
 *
 * Conventions
 *  - All pointers named in a signature are DEVICE pointers unless documented
 *    otherwise; sizes are int64_t; `stream` is a cudaStream_t passed as void*.
 *  - Every call is asynchronous on `stream` and returns GP_OK (0) or an error
 *    code; gp_last_error() returns the thread-local message of the last error.
 *  - The library never allocates or frees caller buffers.  Scratch is sized by
 *    the *_workspace_bytes queries and passed in.
 *  - Not re-entrant on the same buffers.
 *  - Coordinates are float64.  Inputs in the caller's layout are described by
 *    (stride_pt, stride_dim) in elements: AoS (n,d) row-major is (d, 1), SoA
 *    (d,n) is (1, ld).  The library's own working layout is AoS in SFC order:
 *    point i at X[i*ldx .. i*ldx+d) with ldx = d (one 16-byte load per 2D point).
 */
#ifndef GEOPART_B200_H
#define GEOPART_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define GP_OK 0
#define GP_ERR_INVALID 1
#define GP_ERR_CUDA 2
#define GP_ERR_NCCL 3

#define GP_SEGMENTS 256 /* ranksim.py:38 */

/* weight storage modes */
#define GP_W_UNIT 0 /* weights None -> ones (ranksim.py:101-102) */
#define GP_W_F32 1  /* every weight exactly representable as float32 */
#define GP_W_F64 2

const char* gp_last_error(void);
int gp_abi_version(void);
/* sizeof(gp_assign_args), sizeof(gp_fold_args): lets bindings verify struct layouts. */
void gp_args_sizes(size_t* assign_args, size_t* fold_args);
/* 1 when host pointer p lies in page-locked (cudaHostAlloc / registered) memory, so a
 * host<->device copy of it is one DMA; 0 for pageable memory. */
int gp_host_is_pinned(const void* p);

/* K1  global bounding box: replaces the per-shard min/max + allreduce_extreme
 * of kmeans.py:546-548.  lohi[0:d] = min, lohi[d:2d] = max (device, doubles).
 * *nonfinite (device int32) is set to 1 if any coordinate is NaN/inf. */
int gp_box_minmax(const double* pts, int64_t n, int d, int64_t stride_pt, int64_t stride_dim,
                  double* lohi, int32_t* nonfinite, void* stream);

/* Weight probe (device): out[0] = flags (bit0 non-finite, bit1 not float32-exact),
 * out[1] = min over nonzero |w| of the exponent of the lowest set mantissa bit,
 * out[2] = bits of max |w| (double).  Used to choose exact integer block-weight
 * accumulation. */
int gp_weight_probe(const double* w, int64_t n, int64_t* out, void* stream);

/* K2  Hilbert keys: replaces geometry.py:112-132 (point_cells) +
 * geometry.py:135-179 (hilbert_cell_keys) + geometry.py:182-192.  Bit-exact.
 * gids (nullable) receives gid_base + i. */
/* Host-only check of the table form of the key (gp_hilbert_keys runs the transpose
 * as a finite-state machine, several levels per lookup): rebuilds the tables for
 * dimension d and compares them with gp_hilbert_cell_key_host on random cells at every
 * depth.  0 = they agree. */
int gp_hilbert_fsm_selfcheck(int d);
int gp_hilbert_keys(const double* pts, int64_t n, int d, int64_t stride_pt, int64_t stride_dim,
                    const double* lohi, int depth, uint64_t* keys, uint32_t* gids,
                    uint32_t gid_base, void* stream);

/* Host-side scalar helper (host pointers): Hilbert key of integer cells, same
 * algorithm as the kernel; used by the host-logic tests. */
uint64_t gp_hilbert_cell_key_host(const uint32_t* cells, int d, int depth);

/* K3  stable radix sort of (key, gid) pairs on the low key_bits bits:
 * replaces np.lexsort((gids, keys)) in ranksim.py:158 (gids arrive in
 * increasing order, so a stable key sort is the same total order).  Hand-written
 * (csrc/radix.cu): onesweep LSD passes over the top key bits, then one pass that
 * orders each top-bits bucket by the full key.  vals_in NULL: val = input position.
 * keys_out must not alias keys_in; the inputs are left intact. */
int gp_sort_workspace_bytes(int64_t n, size_t* bytes);
int gp_sort_pairs(const uint64_t* keys_in, const uint32_t* vals_in, uint64_t* keys_out,
                  uint32_t* vals_out, int64_t n, int key_bits, void* workspace,
                  size_t workspace_bytes, void* stream);

/* Payload gather after the sort: replaces the fancy-indexing redistribution of
 * ranksim.py:159-168.  X (AoS, point stride ldx) <- pts[gids]; w_out (float or
 * double per wmode; ignored for GP_W_UNIT) <- w_in[gids]. */
int gp_gather_points(const double* pts, int64_t stride_pt, int64_t stride_dim, int d,
                     const uint32_t* gids, int64_t n, double* X, int64_t ldx,
                     const double* w_in, int wmode, void* w_out, void* stream);

/* K4  initial centers: rows[i] = X[positions[i], :] (kmeans.py:552-558). */
int gp_gather_rows(const double* X, int64_t ldx, int d, const int64_t* positions, int k,
                   double* rows, void* stream);

/* K5  sample-phase active list: idx <- positions i (increasing) with
 * rank[i] < size; *count (device int64).  Replaces kmeans.py:579 + the
 * flatnonzero of kmeans.py:405-408. */
int gp_compact_workspace_bytes(int64_t n, size_t* bytes);
int gp_compact_active(const int32_t* rank, int64_t n, int64_t size, int32_t* idx,
                      int64_t* count, void* workspace, size_t workspace_bytes, void* stream);
/* The same over a candidate subset: idx <- positions[j] (increasing) with rank[j] < size,
 * where (positions, rank) list the entries of a larger sample in position order (the
 * warm-up sizes double, so small samples are compacted from a list of a few million
 * candidates instead of all n ranks).  positions NULL: gp_compact_active. */
int gp_compact_candidates(const int32_t* rank, const int32_t* positions, int64_t n, int64_t size,
                          int32_t* idx, int64_t* count, void* workspace, size_t workspace_bytes,
                          void* stream);

/* Dense view of a sample phase's active entries (the ~20 balance rounds of one
 * movement iteration then stream contiguous arrays instead of gathering through
 * the active list): gp_gather_state copies A, UBLB (4-byte bound pairs), X (AoS, d
 * columns) and W (wbytes per point, 0 = none) of list[0..m) into dense arrays;
 * gp_scatter_state writes A and UBLB back. */
int gp_gather_state(const int32_t* list, int64_t m, int d, const int32_t* a, const void* ublb,
                    const double* X, const void* w, int wbytes, int32_t* a_out, void* ublb_out,
                    double* X_out, void* w_out, void* stream);
int gp_scatter_state(const int32_t* list, int64_t m, const int32_t* a_dense,
                     const void* ublb_dense, int32_t* a, void* ublb, void* stream);

/* K5b warm-up sample order, bit-exact with numpy: rank[perm[t]] = t for
 * perm = numpy.random.default_rng(seed).permutation(n) (kmeans.py:564-567).
 * pcg_state is a HOST array {state_hi, state_lo, inc_hi, inc_lo} of the
 * generator's PCG64 state (np.random.PCG64(seed).state).  Synchronises the
 * stream (its acceptance and reservation loops read back small counters). */
int gp_sample_ranks_workspace_bytes(int64_t n, size_t* bytes);
int gp_sample_ranks(const uint64_t* pcg_state, int64_t n, int32_t* rank, void* workspace,
                    size_t workspace_bytes, void* stream);

/* K6  one assign round over the active points of one shard.  Replaces
 * _scan_rank (kmeans.py:297-344) for every rank, the bound relaxations of
 * kmeans.py:438-443 / :622-625 (applied lazily through per-cluster affine
 * maps), and the block-weight segment sums of _global_block_weights
 * (kmeans.py:368-374, ranksim.py:173-197) as exact int64 accumulation.
 * The result per point is the lowest-index argmin of the reference's
 * effective distance, bit for bit. */
typedef struct gp_assign_args {
  const double* X;        /* AoS coordinates in SFC order, point stride ldx */
  int64_t ldx;
  int32_t d;
  int32_t k;
  int32_t order3;         /* einsum summation order for d == 3 (see common.cuh) */
  int32_t wmode;          /* GP_W_* */
  const void* w;          /* weights (float or double) or NULL for unit */
  double wscale;          /* exact scale 2^s: block weight units = w * wscale */
  const int32_t* list;    /* active positions (NULL: all positions 0..m-1) */
  int64_t m;              /* number of active entries */
  int32_t* a;             /* assignment per position (-1 = unassigned) */
  void* ublb;             /* per position (ub~, lb~) * bound_scale: normalised bounds as
                             an IEEE fp16 pair (4 bytes), rounded outward (ub~ up,
                             lb~ down) */
  const double* centers;  /* k x d row-major */
  const double* infl;     /* k influences */
  const double* inv2_lo;  /* k: lower bound of 1/infl^2 (outward-rounded on the host) */
  const double* inv2_hi;  /* k: upper bound of 1/infl^2 */
  /* Lazily relaxed Hamerly bounds, float32, rounded outward:
   *   ub = fmaf_ru(ub~ >= 0 ? E.x : E.y, ub~, E.z)      E = ub_eval[4a .. 4a+3]
   *   lb = max(fmaf_rd(lb_a, lb~, -lb_b), 0)
   * and after a scan with best/second effective distances b, s:
   *   ub~ = (b - N.z) * (b - N.z >= 0 ? N.x : N.y)  rounded up, N = ub_norm[4c ..]
   *   lb~ = (s + lb_blo) * lb_inva                 rounded down. */
  const float* ub_eval;   /* k x 4 */
  const float* ub_norm;   /* k x 4 */
  const float* lb_par;    /* 4 floats: lb_a, lb_b, lb_inva, lb_blo */
  long long* block_w;     /* out: k exact block weights (units of 1/wscale), accumulated */
  unsigned long long* counters; /* out: [skips, decisions, evals], accumulated */
  /* optional hierarchical candidate source (gp_group_candidates): entry li of
   * the active list belongs to group li >> group_shift, whose candidate centers
   * are group_list[g*group_cap .. +group_count[g]); group_count[g] < 0 means
   * "all k".  NULL group_list: every tile starts from all k centers. */
  const int32_t* group_list;
  const int32_t* group_count;
  int32_t group_cap;
  int32_t group_shift;
  /* scratch of gp_assign_workspace_bytes(m) bytes (filter -> scan hand-off) */
  void* workspace;
  size_t workspace_bytes;
  /* scan unit = scan_regions x 256 consecutive entries (1..4; 0 = automatic).
   * Dense (full-phase) lists want 4, sparse warm-up samples 1. */
  int32_t scan_regions;
  /* uniform grid over the centers (built on the host per movement iteration):
   * cell (i0,i1[,i2]) covers [lo + i*h, lo + (i+1)*h); its centers are
   * grid_items[grid_start[cell] .. grid_start[cell+1]).  Used for scan units whose
   * candidate set overflows (sparse warm-up samples).  grid_n = 0: no grid. */
  int32_t grid_n;
  const int32_t* grid_start;
  const int32_t* grid_items;
  double grid_lo[3];
  double grid_h;
  double inv2_min;        /* lower bound of min_c 1/infl_c^2 */
  /* static box of every scan unit (gp_group_boxes over the active entries with
   * shift = unit_shift = log2(scan_regions * 256)); NULL: boxes of the scanned
   * points are computed per round */
  const double* unit_boxes;
  int32_t unit_shift;
  int32_t flags;          /* bit 0: accumulate scan statistics (gp_scan_stats);
                             bit 1: sparse round: one warp per rescanned point walks
                             the center grid (needs grid_n > 0) instead of the
                             per-unit candidate scan */
  /* region-local lower-bound maps (gp_region_maps): entry li uses the float4
   * lb_rpar[li >> lb_rshift] instead of lb_par; NULL: the global lb_par */
  const float* lb_rpar;
  int32_t lb_rshift;
  /* power of two applied to the stored fp16 bounds (keeps them in fp16's normal range;
   * about 1 / the box diagonal) */
  float bound_scale;
  /* device copy of inv2_min kept by gp_update_maps (map_state + 2k + 7); when set it
   * replaces inv2_min, so a captured loop graph sees every round's value */
  const double* inv2_min_dev;
  /* optional cudaEvent_t recorded on the stream between the filter and the scan
   * launches (per-kernel timing); NULL: none */
  void* split_event;
} gp_assign_args;
int gp_assign_workspace_bytes(int64_t m, size_t* bytes);
int gp_assign_round(const gp_assign_args* args, void* stream);

/* Hierarchical candidate lists (a B200 replacement for the reference's one
 * box per rank, kmeans.py:315-319).  Entries of the active list are grouped in
 * aligned runs of 2^shift (SFC-contiguous, so each group is spatially
 * compact).
 *  gp_group_boxes: per group the bounding box of its points, boxes[g*2d ..]
 *    = (lo[0..d), hi[0..d)); computed once per active set.
 *  gp_group_candidates: per group, every center whose box lower bound does not
 *    exceed the second smallest box upper bound (a sound superset of each
 *    member point's best and runner-up center under the current influences),
 *    taken from the parent level's list (parent_list/parent_count with
 *    parent_shift >= shift) or from all k when parent_list is NULL.  A group
 *    whose list would exceed cap gets count -1 ("all k"). */
int gp_group_boxes(const double* X, int64_t ldx, int d, const int32_t* list, int64_t m,
                   int shift, double* boxes, void* stream);
int gp_group_candidates(const double* boxes, int64_t ngroups, int d, int k,
                        const double* centers, const double* inv2_lo, const double* inv2_hi,
                        const int32_t* parent_list, const int32_t* parent_count, int parent_cap,
                        int parent_ratio_log2, int32_t* list, int32_t* count, int cap,
                        void* stream);

/* Device-side bound-map bookkeeping (control.BoundMaps on the GPU): compose one
 * relaxation (kmeans.py:208-239) old_infl -> new_infl with center moves `moves`
 * (NULL = zero moves) into the cumulative maps `state` (4k + 8 doubles: S[k], T[k],
 * A, B, steps, 5 scratch (min ratio, max shift, changed, max influence, inv2_min =
 * 1 / max(infl)^2 * (1 - 1e-15)), then this relaxation's per-cluster ratio
 * I_old/I_new [k] and shift move/I_new [k]), unless it is the reference's identity
 * early return, and
 * derive every parameter the kernels read: inv2_lo/inv2_hi (k), ub_eval/ub_norm
 * (k x 4 floats), lb_par (4 floats).  flags[0] is set to 1 when the maps should
 * be re-based (gp_rebase_bounds + gp_reset_maps).  reset != 0 starts from
 * identity maps (first call / after a rebase). */
int gp_update_maps(const double* old_infl, const double* new_infl, const double* moves, int k,
                   double* state, double* inv2_lo, double* inv2_hi, float* ub_eval,
                   float* ub_norm, float* lb_par, int32_t* flags, int reset, double scale_hint,
                   void* stream);

/* Region-local lower-bound maps (full phase, B200 extension of kmeans.py:229-236).
 * The reference relaxes every lower bound by the smallest influence ratio and the
 * largest center shift over all k centers.  For the entries of super group r only
 * the centers of its candidate list (gp_group_candidates, under the NEW centers
 * and influences) can be the nearest or the runner-up: every other center is
 * farther than the group's second-smallest upper bound, which bounds the
 * runner-up of every entry.  So the relaxation over the list alone is sound.
 * map_state: the state of the gp_update_maps call for the same relaxation (its
 * per-cluster ratios and shifts are gathered over the lists).
 * rstate: nregions x 3 doubles (A, B, steps); rpar: nregions x float4 in the
 * layout of lb_par.  reset = 1: identity maps.  flags[0] = 1 when a map leaves
 * the float32 range (the caller rebases). */
/* Lower bounds of the active entries between the maps: mode 0 materialises them
 * under the global map (lb_par; identity region maps follow), mode 1 renormalises
 * them from the region maps (lb_rpar) to the global map. */
int gp_lb_remap(const gp_assign_args* args, int mode, void* stream);

int gp_region_maps(const double* map_state, int k, const int32_t* group_list,
                   const int32_t* group_count, int group_cap, int64_t nregions, double* rstate,
                   float* rpar, int32_t* flags, int reset, double scale_hint, void* stream);

/* Re-express every bound under identity maps (when the host's cumulative
 * maps drift out of range).  Same bound semantics as gp_assign_args. */
int gp_rebase_bounds(const gp_assign_args* args, void* stream);

/* K7  movement reduction of one shard, bit-exact with the reference:
 * per-(segment, block) sequential folds of w*x and w in SFC order
 * (ranksim.py:173-197, kmeans.py:463-471), the sequential fold over segments
 * (ranksim.py:218-222), per-block max distance to the old centers
 * (_cluster_extents, kmeans.py:474-487) and the objective terms
 * (kmeans.py:490-499).  Positions pos0..pos0+n_local-1 of a global sequence of
 * n_global points; points with a < 0 are excluded.  Synchronises the stream
 * once (it reads back the number of runs to size the run sort). */
typedef struct gp_fold_args {
  const double* X;
  int64_t ldx;
  int32_t d;
  int32_t k;
  int32_t order3;
  int32_t wmode;
  const void* w;
  const int32_t* a;
  int64_t n_local;
  int64_t pos0;           /* global position of local position 0 */
  int64_t n_global;
  const double* centers;  /* OLD centers (k x d) for extents and objective */
  int32_t weights_only;   /* 1: fold only w (block weights in general-weight mode) */
  /* outputs (device) */
  double* sums;           /* k x d  : sum of w*x per block (only if !weights_only) */
  double* wsum;           /* k      : sum of w per block */
  double* extent;         /* k      : max distance to old center (only if !weights_only) */
  double* objective;      /* k      : per-block objective partial (only if !weights_only) */
  /* scratch */
  void* workspace;
  size_t workspace_bytes;
  /* optional dense entry list: when list != NULL the entries are i = 0..m-1 at
   * local positions list[i] (ascending), and X, w, a are indexed by i (the dense
   * warm-up sample arrays); NULL: entry i is local position i, i < n_local */
  const int32_t* list;
  int64_t m;
} gp_fold_args;
int gp_fold_workspace_bytes(int64_t n_local, int64_t pos0, int64_t n_global, int k,
                            size_t* bytes);
int gp_movement_fold(const gp_fold_args* args, void* stream);
/* Multi-GPU movement reduction.  After gp_movement_fold on a shard,
 * gp_fold_export writes the shard's (segment, block) partials: keys[p] =
 * global_segment * k + block, vals[p*6 .. p*6+6) = (w*x_0..w*x_{d-1}, w, objective
 * padded to 5 columns, extent) and *npairs (device int64).  Every rank then
 * gathers all ranks' partials and gp_fold_combine folds them per block in global
 * segment order (the same sequential order as one shard), writing sums / wsum /
 * extent / objective like gp_movement_fold.  workspace: gp_fold_combine_bytes. */
int gp_fold_export(const gp_fold_args* args, int64_t* keys, double* vals, int64_t* npairs,
                   void* stream);
int gp_fold_combine_bytes(int k, size_t* bytes);
int gp_fold_combine(const int64_t* keys, const double* vals, int64_t npairs, int k, int d,
                    int weights_only, double* sums, double* wsum, double* extent,
                    double* objective, void* workspace, size_t workspace_bytes, void* stream);

/* Debugging aid (synchronises the device): out[4] = {runs, work cursor, valid runs,
 * pairs} of the last gp_movement_fold call. */
int gp_fold_stats(int64_t* out);

/* Debugging aid (synchronises the device): out[8] = scan statistics summed over the
 * gp_assign_round calls made with flags bit 0 since the last reset: {units with
 * points, scanned points, candidate source entries, staged candidates, overflow
 * units, exact evaluations, candidate walk steps, point passes}. */
int gp_scan_stats(uint64_t* out, int reset);

/* K8  bound audit (kmeans.py:347-365): brute-force n x k recheck of the
 * bound contracts for the active points; out[3] += {audited, violations,
 * bad_skips}.  Uses the same args as gp_assign_round (nothing written but out). */
int gp_audit(const gp_assign_args* args, unsigned long long* out, void* stream);

/* K9  result delivery: out[gids[i]] = a[i] (kmeans.py:637-641). */
int gp_scatter_by_gid(const int32_t* a, const uint32_t* gids, int64_t n, int64_t* out,
                      void* stream);
/* The same delivery when gids is a permutation of 0..n-1 (one shard holding every point),
 * without random writes: two radix passes on the high gid bits group the (gid, block)
 * pairs into windows of 2^14 consecutive ids, then one CTA per window places its pairs in
 * shared memory and writes the window's labels as one contiguous run. */
int gp_deliver_workspace_bytes(int64_t n, size_t* bytes);
int gp_deliver_permutation(const int32_t* a, const uint32_t* gids, int64_t n, int64_t* out,
                           void* workspace, size_t workspace_bytes, void* stream);

/* Sample-rank delivery in SFC order: out[i] = rank_by_gid[gids[i]]
 * (kmeans.py:568). */
int gp_gather_ranks(const int32_t* rank_by_gid, const uint32_t* gids, int64_t n, int32_t* out,
                    void* stream);

/* Uniform grid over the centers for the scan's overflow walk and the walk kernel:
 * cell of center c = clip(floor((centers[c] - lo) / h), 0, G - 1) per axis
 * (row-major flat index), items = the centers sorted stably by cell, start[cell]
 * = first item of the cell (G^d + 1 entries).  lo is a HOST array of d doubles.
 * workspace: gp_center_grid_workspace_bytes(k). */
int gp_center_grid_workspace_bytes(int k, size_t* bytes);
int gp_center_grid(const double* centers, int k, int d, const double* lo, double h, int G,
                   int32_t* start, int32_t* items, void* workspace, size_t workspace_bytes,
                   void* stream);

/* ---- device-side balance decision ----------------------------------------- */
/* One balance-round decision of assign_and_balance (kmeans.py:425-443) on the
 * device (d = 2, exact block weights): from the round's
 * block-weight units and counters red[k + 3] (gp_assign_round), the block
 * weights units / wscale, imbalance (metrics.py:33-40), the stop test
 * (imbalance <= eps or the last round), the step halving from the second
 * regression, and, when the loop goes on, next[c] = cur[c] * clip(sqrt(target /
 * w_c), 1 - cap, 1 + cap) (kmeans.py:176-191 with d = 2: numpy's x ** 0.5 is
 * sqrt).  bal (doubles): [0] cap, [1] regressions, [2] best imbalance, [3] rounds
 * done, [4] error (1: total <= 0, 2: target <= 0), [5] stop, [6..7] unused, then the per-round
 * imbalance, skips and distance evaluations (max_rounds each). */
int gp_balance_decide(const long long* red, int k, double wscale, double eps, int max_rounds,
                      double* bal, const double* infl_cur, double* infl_next, void* stream);

/* ---- callers of the path ---------------------------------- */

/* SFC baseline cut (baselines.py:62-89, replaces lines 84-89 after the key sort
 * of lines 82-83): for curve position i (gids = the stable key sort's values)
 *   before = cumsum(w)[i] - w[i], total = w.sum(),
 *   labels[gids[i]] = min((int64)(before * k / total), k - 1).
 * w is by original id (NULL = unit weights, then scale must be 1).
 * scale > 0: every weight times scale is an exact integer and the total of those
 *   integers is below 2^53 (gp_weight_probe), so the prefix sums are exact.
 * scale == 0: the reference's summation orders are restated literally (numpy's
 *   pairwise w.sum() and a sequential cumsum).
 * workspace: gp_sfc_cut_workspace_bytes(n). */
int gp_sfc_cut_workspace_bytes(int64_t n, size_t* bytes);
int gp_sfc_cut(const uint32_t* gids, const double* w, int64_t n, int k, double scale,
               int64_t* labels, void* workspace, size_t workspace_bytes, void* stream);

/* GeographerPartitioner.predict (estimators.py:107-114):
 *   labels[i] = argmin_c norm(X[i] - centers[c]) / influence[c]
 * with linalg.norm's (dx^2 + dy^2) + dz^2 order and numpy argmin semantics
 * (first minimum; a NaN wins).  X is AoS (n, d).  safe_influence != 0 asserts
 * every influence is finite and in [1e-150, 1e150] (enables the fp64 ranking
 * pass; otherwise every point is evaluated with the exact arithmetic). */
int gp_predict(const double* X, int64_t n, int d, const double* centers, const double* influence,
               int k, int safe_influence, int64_t* labels, void* stream);

/* ---- formats and evaluation either side of the path -------- */

/* token kinds written by gp_text_tokens */
#define GP_TOK_INT 0     /* [+-]?digits, at most 18 significant: value = the int64 */
#define GP_TOK_REAL 1    /* plain decimal real: value = bits of the correctly rounded double */
#define GP_TOK_PERCENT 2 /* starts with '%' (a METIS comment line when first on its line) */
#define GP_TOK_SUSPECT 3 /* anything else (nan, 1_000, > 19 digits, ...): the host decides */

/* Host helper (host pointers): the tokenizer's number conversion for one token; returns
 * the kind.  Used by the CPU tests to pin the decimal -> binary64 conversion to Python's
 * float() without a GPU. */
int gp_parse_number_host(const char* text, int len, int64_t* value);

/* Line and token index of a text file held in device memory (fileio.py:83 `f.read()
 * .splitlines()` + `line.split()`, and np.loadtxt's rows in fileio.py:222, :250).
 * Lines end at '\n', '\r\n' or a lone '\r'; tokens are separated by blanks and tabs.
 * comment_char != 0 ('#' for the np.loadtxt formats): the rest of a line from that
 * character is ignored.  gp_text_index writes counts[0..3) = {lines, tokens, bytes that
 * are not printable ASCII, tab or a line end} (device); after reading them the caller sizes the outputs of gp_text_tokens:
 *   line_off[l]  (lines + 1)  byte offset of line l (sentinel: len)
 *   line_tok0[l] (lines + 1)  index of the first token at or after line l (sentinel: tokens)
 *   tok_val / tok_kind (tokens)  value and GP_TOK_* kind of every token
 * The same workspace (gp_text_index_workspace_bytes) must be passed to both calls. */
int gp_text_index_workspace_bytes(int64_t len, size_t* bytes);
int gp_text_index(const uint8_t* text, int64_t len, int comment_char, int64_t* counts,
                  void* workspace, size_t workspace_bytes, void* stream);
int gp_text_tokens(const uint8_t* text, int64_t len, int comment_char, const void* workspace,
                   int64_t n_lines, int64_t n_tokens, int64_t* line_off, int64_t* line_tok0,
                   int64_t* tok_val, uint8_t* tok_kind, void* stream);

/* METIS adjacency file -> CSR (fileio.py:70-170).
 * gp_metis_lines: drops '%' comment lines (fileio.py:85-93); info (device) = {non-comment
 *   lines, line of the header, 1 + index of the last vertex line holding a token};
 *   body_line[v] = line of vertex v (the v+1-th non-comment line after the header).
 * gp_metis_offsets: offsets[0..n] from the token counts (fileio.py:131-149, :163-164);
 *   flags[v] = 1 where the line lacks its vertex weight or ends in a dangling neighbor.
 * gp_metis_fill: neighbors (0-based), edge and vertex weights; flags[v] |= 1 for every
 *   line the reference rejects for a bad token, an id out of range, a self loop or a
 *   non-positive weight.  Flagged lines are re-read by the host for the message (and for
 *   tokens only Python's int()/float() accept).  Duplicates are left to gp_graph_check. */
int gp_metis_workspace_bytes(int64_t n_lines, size_t* bytes);
int gp_metis_lines(const int64_t* line_tok0, const uint8_t* tok_kind, int64_t n_lines,
                   int64_t* body_line, int64_t body_cap, int64_t* info, void* workspace,
                   size_t workspace_bytes, void* stream);
int gp_metis_offsets(const int64_t* line_tok0, const int64_t* body_line, int64_t n, int has_vw,
                     int has_ew, int64_t* offsets, uint8_t* flags, void* workspace,
                     size_t workspace_bytes, void* stream);
int gp_metis_fill(const int64_t* line_tok0, const int64_t* body_line, const int64_t* tok_val,
                  const uint8_t* tok_kind, int64_t n, int has_vw, int has_ew,
                  const int64_t* offsets, int64_t* neighbors, double* edge_weights,
                  double* vertex_weights, uint8_t* flags, void* stream);

/* Whitespace table (np.loadtxt in fileio.py:222 and :250): out[t] = value of token t as
 * double (want_int 0) or int64 (want_int 1) -- the row-major table once every non-blank
 * line has as many tokens as the first.  info (device) = {rows, first line with another
 * token count or -1, first token that is not a plain number of the wanted type or -1,
 * columns}. */
int gp_table_values(const int64_t* line_tok0, int64_t n_lines, const int64_t* tok_val,
                    const uint8_t* tok_kind, int64_t n_tokens, int want_int, void* out,
                    int64_t* info, void* stream);

/* Partition writer (fileio.py:271-278): one decimal per line.  _plan computes the byte
 * position of every value and *out_len (device); _write fills out[0, out_len) using the
 * same workspace. */
int gp_format_ints_workspace_bytes(int64_t n, size_t* bytes);
int gp_format_ints_plan(const int64_t* values, int64_t n, int64_t* out_len, void* workspace,
                        size_t workspace_bytes, void* stream);
int gp_format_ints_write(const int64_t* values, int64_t n, uint8_t* out, const void* workspace,
                         void* stream);

/* Structural check of a CSR graph (graph.py:85-128, fileio.py:173-187).  result (device):
 * result[0] = bit flags {1 neighbor out of range, 2 self loop, 4 parallel edge,
 * 8 asymmetric, 16 edge weight differs between directions, 32 non-positive edge weight,
 * 64 offsets malformed}; result[1] = the smallest directed-edge key u*n+v whose reverse
 * is missing (fileio.py:180-183), or -1.  vertex_flags (nullable, n bytes): set to 1 for
 * every vertex listing a neighbor twice. */
int gp_graph_check_workspace_bytes(int64_t nnz, size_t* bytes);
int gp_graph_check(const int64_t* offsets, const int64_t* neighbors, const double* edge_weights,
                   int64_t n, int64_t nnz, uint8_t* vertex_flags, int64_t* result,
                   void* workspace, size_t workspace_bytes, void* stream);

/* metrics.py:48-60.  edge_weights NULL: the number of cut edges.  scale > 0: every edge
 * weight times scale is an exact integer (gp_weight_probe) and the cut is summed in
 * int64; scale == 0: numpy's pairwise sum of the masked weights in CSR order (this
 * variant synchronises the stream).  *out is a device double. */
int gp_edge_cut_workspace_bytes(int64_t n, int64_t nnz, size_t* bytes);
int gp_edge_cut(const int64_t* offsets, const int64_t* neighbors, const double* edge_weights,
                double scale, const int32_t* assignment, int64_t n, int64_t nnz, double* out,
                void* workspace, size_t workspace_bytes, void* stream);

/* metrics.py:63-77: per_block[b] = sum over the vertices of block b of the number of other
 * blocks among their neighbors.  heavy_scratch: n + 1 int64. */
int gp_comm_volumes(const int64_t* offsets, const int64_t* neighbors, const int32_t* assignment,
                    int64_t n, int k, int64_t* per_block, int64_t* heavy_scratch, void* stream);

/* graph.py:165-166: np.bincount(assignment, weights, minlength=k).  weights NULL = ones.
 * scale > 0: exact integer units; scale == 0: the sequential fold in vertex order. */
int gp_block_weights_workspace_bytes(int64_t n, int k, size_t* bytes);
int gp_block_weights(const double* weights, const int32_t* assignment, int64_t n, int k,
                     double scale, double* out, void* workspace, size_t workspace_bytes,
                     void* stream);

/* metrics.py:80-168: BFS inside every block at once from roots[b] (-1 = none), hop levels
 * into level (int32, -1 = unreached); one CTA per block, one launch per sweep.  qbase
 * (k + 1) = exclusive prefix sums of the block sizes; queue = n int64 of scratch.  Per
 * block: depth[b] = the largest level, far[b] = the lowest vertex id on it
 * (metrics.py:115-118), reached[b] = vertices reached (a block is connected iff it equals
 * the block size).
 * gp_block_level_top: out[b] = max over the block's vertices v != exclude[b] with key <
 * below[b] of key = (level + 1) << 32 | (2^32 - 1 - v), i.e. the deepest vertex, lowest id
 * first (metrics.py:152); unreached[b] (nullable) = vertices of b with level -1. */
int gp_block_bfs(const int64_t* offsets, const int64_t* neighbors, const int32_t* assignment,
                 int64_t n, int k, const int64_t* roots, const int64_t* qbase, int64_t* queue,
                 int32_t* level, int32_t* depth, int64_t* far, int64_t* reached, void* stream);
int gp_block_level_top(const int32_t* level, const int32_t* assignment, int64_t n, int k,
                       const int64_t* exclude, const uint64_t* below, uint64_t* out,
                       uint64_t* unreached, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* GEOPART_B200_H */
