// K7 movement reduction, bit-exact with the reference.
//
// The reference sums w*x and w per (segment, block) with sequential bincount
// folds in SFC order (ranksim.py:173-197), then folds the 256 segment partials
// sequentially (np.add.reduce(axis=0), ranksim.py:218-222 / kmeans.py:374).
// A sequential fold cannot be parallelised, but the folds of different
// (segment, block) pairs are independent, and SFC order keeps each block in a
// short span of positions.  So:
//   discover : per (segment, block) the first/last local position (warp
//              aggregated atomics on a dense S x k table);
//   pairs    : compact the non-empty (segment, block) cells into a work list;
//   fold     : one warp per pair walks its span in 32-wide chunks, stages the
//              chunk's values in shared memory and lets lane j fold column j
//              in position order (the exact bincount order); extents (max
//              distance to the old center, kmeans.py:474-487) and the
//              objective terms (kmeans.py:490-499) are computed in parallel
//              by all lanes of the chunk;
//   combine  : per block, fold the pair partials in segment order.
#include "common.cuh"

namespace gp {

struct Pair {
  int32_t key;  // local_segment * k + block
  int32_t first;
  int32_t last;
  int32_t pad;
};

constexpr int FT = 256;           // threads per fold CTA (8 warps)
constexpr int MAXCOL = 5;         // d wx columns + w + objective (d <= 3)

struct FoldLayout {
  int64_t s0, nseg, cells, max_pairs;
  size_t off_first, off_last, off_slot, off_pairs, off_out, off_counters, total;
};

static FoldLayout layout(int64_t n_local, int64_t pos0, int64_t n_global, int k) {
  FoldLayout L;
  auto seg = [&](int64_t pos) { return ((pos + 1) * (int64_t)GP_SEGMENTS - 1) / n_global; };
  L.s0 = n_local > 0 ? seg(pos0) : 0;
  int64_t s1 = n_local > 0 ? seg(pos0 + n_local - 1) : 0;
  L.nseg = n_local > 0 ? s1 - L.s0 + 1 : 1;
  L.cells = L.nseg * k;
  L.max_pairs = L.cells < n_local ? L.cells : (n_local > 0 ? n_local : 1);
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  size_t o = 0;
  L.off_first = o; o = al(o + L.cells * sizeof(int32_t));
  L.off_last = o; o = al(o + L.cells * sizeof(int32_t));
  L.off_slot = o; o = al(o + L.cells * sizeof(int32_t));
  L.off_pairs = o; o = al(o + L.max_pairs * sizeof(Pair));
  L.off_out = o; o = al(o + L.max_pairs * (MAXCOL + 1) * sizeof(double));
  L.off_counters = o; o = al(o + 4 * sizeof(int64_t));
  L.total = o;
  return L;
}

__global__ void fold_init(int32_t* first, int32_t* last, int64_t cells, int64_t* counters) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cells;
       i += (int64_t)gridDim.x * blockDim.x) {
    first[i] = 0x7fffffff;
    last[i] = -1;
  }
  if (blockIdx.x == 0 && threadIdx.x < 4) counters[threadIdx.x] = 0;
}

__global__ void fold_discover(const int32_t* __restrict__ a, int64_t n_local, int64_t pos0,
                              int64_t n_global, int64_t s0, int k, int32_t* first,
                              int32_t* last) {
  int lane = threadIdx.x & 31;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t base = blockIdx.x * (int64_t)blockDim.x; base < n_local; base += stride) {
    int64_t i = base + threadIdx.x;
    int key = -1;
    if (i < n_local) {
      int c = a[i];
      if (c >= 0) key = (int)((segment_of(pos0 + i, n_global) - s0) * k + c);
    }
    unsigned grp = __match_any_sync(FULL, key);
    if (key >= 0 && lane == __ffs(grp) - 1) {
      int hi_lane = 31 - __clz(grp);
      atomicMin(&first[key], (int32_t)i);
      atomicMax(&last[key], (int32_t)(i - lane + hi_lane));
    }
  }
}

__global__ void fold_pairs(const int32_t* __restrict__ first, const int32_t* __restrict__ last,
                           int64_t cells, int32_t* slot, Pair* pairs, int64_t* counters) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < cells;
       i += (int64_t)gridDim.x * blockDim.x) {
    int32_t l = last[i];
    if (l >= 0) {
      int64_t p = atomicAdd((unsigned long long*)&counters[0], 1ull);
      pairs[p] = Pair{(int32_t)i, first[i], l, 0};
      slot[i] = (int32_t)p;
    } else {
      slot[i] = -1;
    }
  }
}

// One warp per (segment, block) pair.  The span [first, last] is walked in
// batches of FB chunks of 32 positions: every load of a batch is issued before
// any of its values is consumed (one memory latency per batch instead of one
// per chunk), then lane j folds column j over the matched positions in order.
constexpr int FB = 4;

template <int D>
__global__ void __launch_bounds__(FT) fold_kernel(gp_fold_args f, const Pair* __restrict__ pairs,
                                                  int64_t* counters, double* out) {
  __shared__ double sm[FT / 32][MAXCOL][FB * 32 + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ncols = f.weights_only ? 1 : D + 2;
  const int64_t npairs = counters[0];
  for (;;) {
    int64_t pi;
    if (lane == 0) pi = (int64_t)atomicAdd((unsigned long long*)&counters[1], 1ull);
    pi = __shfl_sync(FULL, pi, 0);
    if (pi >= npairs) break;
    const Pair pr = pairs[pi];
    const int c = pr.key % f.k;
    double cold[D];
    if (!f.weights_only) {
#pragma unroll
      for (int j = 0; j < D; ++j) cold[j] = f.centers[c * D + j];
    }
    double acc = 0.0;  // lane j < ncols folds column j; bincount starts from 0.0
    double ext = 0.0;
    for (int64_t base = pr.first; base <= pr.last; base += FB * 32) {
      int av[FB];
      double xv[FB][D], wv[FB];
#pragma unroll
      for (int b = 0; b < FB; ++b) {
        int64_t i = base + b * 32 + lane;
        bool in = i <= pr.last;
        av[b] = in ? f.a[i] : -1;
        wv[b] = in ? load_weight(f.w, f.wmode, i) : 0.0;
        if (!f.weights_only) {
#pragma unroll
          for (int j = 0; j < D; ++j) xv[b][j] = in ? f.X[j * f.ldx + i] : 0.0;
        }
      }
      unsigned masks[FB];
#pragma unroll
      for (int b = 0; b < FB; ++b) {
        bool valid = av[b] == c;
        masks[b] = __ballot_sync(FULL, valid);
        const int slot = b * 32 + lane;
        if (f.weights_only) {
          sm[warp][0][slot] = wv[b];
        } else {
          double diff[D];
#pragma unroll
          for (int j = 0; j < D; ++j) {
            sm[warp][j][slot] = __dmul_rn(xv[b][j], wv[b]);  // wx = points * weights[:, None]
            diff[j] = __dsub_rn(xv[b][j], cold[j]);
          }
          double sq = sqnorm_rn(diff, D, f.order3);
          sm[warp][D][slot] = wv[b];
          sm[warp][D + 1][slot] = __dmul_rn(sq, wv[b]);
          if (valid) ext = fmax(ext, __dsqrt_rn(sq));
        }
      }
      __syncwarp();
      if (lane < ncols) {
        const double* col = sm[warp][lane];
#pragma unroll
        for (int b = 0; b < FB; ++b) {
          unsigned m = masks[b];
          if (m == FULL) {
#pragma unroll
            for (int t = 0; t < 32; ++t) acc = __dadd_rn(acc, col[b * 32 + t]);
          } else {
            while (m) {
              int t = __ffs(m) - 1;
              m &= m - 1;
              acc = __dadd_rn(acc, col[b * 32 + t]);
            }
          }
        }
      }
      __syncwarp();
    }
    for (int o = 16; o; o >>= 1) ext = fmax(ext, __shfl_xor_sync(FULL, ext, o));
    double* po = out + pi * (MAXCOL + 1);
    if (lane < ncols) po[lane] = acc;
    if (lane == 0) po[MAXCOL] = ext;
  }
}

// One warp per block: gather the block's pair partials over the segments
// (independent loads), then fold them in segment order (np.add.reduce(axis=0)).
template <int D>
__global__ void fold_combine(gp_fold_args f, const int32_t* __restrict__ slot, int64_t nseg,
                             const double* __restrict__ out) {
  __shared__ int32_t s_slot[4][GP_SEGMENTS];
  __shared__ int s_cnt[4];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * 4 + warp;
  if (c >= f.k) return;
  // ordered compaction of the present segments
  if (lane == 0) s_cnt[warp] = 0;
  __syncwarp();
  int base = 0;
  for (int64_t s0 = 0; s0 < nseg; s0 += 32) {
    int64_t s = s0 + lane;
    int32_t p = s < nseg ? slot[s * f.k + c] : -1;
    unsigned m = __ballot_sync(FULL, p >= 0);
    if (p >= 0) s_slot[warp][base + __popc(m & ((1u << lane) - 1))] = p;
    base += __popc(m);
  }
  __syncwarp();
  const int np = base;
  const int ncols = f.weights_only ? 1 : D + 2;
  if (lane < ncols) {
    double acc = 0.0;
    for (int i = 0; i < np; ++i) acc = __dadd_rn(acc, out[(int64_t)s_slot[warp][i] * (MAXCOL + 1) + lane]);
    if (f.weights_only) {
      f.wsum[c] = acc;
    } else if (lane < D) {
      f.sums[c * D + lane] = acc;
    } else if (lane == D) {
      f.wsum[c] = acc;
    } else {
      f.objective[c] = acc;
    }
  }
  if (!f.weights_only) {
    double ext = 0.0;
    for (int i = lane; i < np; i += 32) ext = fmax(ext, out[(int64_t)s_slot[warp][i] * (MAXCOL + 1) + MAXCOL]);
    for (int o = 16; o; o >>= 1) ext = fmax(ext, __shfl_xor_sync(FULL, ext, o));
    if (lane == 0) f.extent[c] = ext;
  }
}

}  // namespace gp

using namespace gp;

extern "C" {

int gp_fold_workspace_bytes(int64_t n_local, int64_t pos0, int64_t n_global, int k,
                            size_t* bytes) {
  GP_REQUIRE(n_global >= 1 && k >= 1, "gp_fold_workspace_bytes: bad sizes");
  *bytes = layout(n_local, pos0, n_global, k).total;
  return GP_OK;
}

int gp_movement_fold(const gp_fold_args* f, void* stream) {
  GP_REQUIRE(f && (f->d == 2 || f->d == 3) && f->k >= 1, "gp_movement_fold: bad args");
  GP_REQUIRE(f->n_local >= 0 && f->n_local < (1ll << 31), "gp_movement_fold: n out of range");
  GP_REQUIRE(f->wmode == GP_W_UNIT || f->w != nullptr, "gp_movement_fold: weights missing");
  GP_REQUIRE(f->wsum != nullptr, "gp_movement_fold: wsum missing");
  GP_REQUIRE(f->weights_only || (f->sums && f->extent && f->objective && f->centers),
             "gp_movement_fold: outputs missing");
  FoldLayout L = layout(f->n_local, f->pos0, f->n_global, f->k);
  GP_REQUIRE(f->workspace_bytes >= L.total, "gp_movement_fold: workspace too small (%zu < %zu)",
             f->workspace_bytes, L.total);
  GP_REQUIRE(L.cells < (1ll << 31), "gp_movement_fold: segment x block table too large");
  cudaStream_t s = (cudaStream_t)stream;
  char* ws = (char*)f->workspace;
  int32_t* first = (int32_t*)(ws + L.off_first);
  int32_t* last = (int32_t*)(ws + L.off_last);
  int32_t* slot = (int32_t*)(ws + L.off_slot);
  Pair* pairs = (Pair*)(ws + L.off_pairs);
  double* out = (double*)(ws + L.off_out);
  int64_t* counters = (int64_t*)(ws + L.off_counters);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);

  fold_init<<<grid_for(L.cells, 256, sms * 8), 256, 0, s>>>(first, last, L.cells, counters);
  if (f->n_local > 0)
    fold_discover<<<grid_for(f->n_local, 256, sms * 16), 256, 0, s>>>(
        f->a, f->n_local, f->pos0, f->n_global, L.s0, f->k, first, last);
  fold_pairs<<<grid_for(L.cells, 256, sms * 8), 256, 0, s>>>(first, last, L.cells, slot, pairs,
                                                             counters);
  if (f->d == 2) {
    fold_kernel<2><<<sms * 8, FT, 0, s>>>(*f, pairs, counters, out);
    fold_combine<2><<<grid_for(f->k, 4), 128, 0, s>>>(*f, slot, L.nseg, out);
  } else {
    fold_kernel<3><<<sms * 8, FT, 0, s>>>(*f, pairs, counters, out);
    fold_combine<3><<<grid_for(f->k, 4), 128, 0, s>>>(*f, slot, L.nseg, out);
  }
  return check_launch("movement_fold");
}

}  // extern "C"
