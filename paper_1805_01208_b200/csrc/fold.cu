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

template <int D>
__global__ void __launch_bounds__(FT) fold_kernel(gp_fold_args f, const Pair* __restrict__ pairs,
                                                  int64_t* counters, double* out) {
  __shared__ double sm[FT / 32][MAXCOL][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ncols = f.weights_only ? 1 : D + 2;
  const int64_t npairs = counters[0];
  for (;;) {
    int64_t pi;
    if (lane == 0) pi = (int64_t)atomicAdd((unsigned long long*)&counters[1], 1ull);
    pi = __shfl_sync(FULL, pi, 0);
    if (pi >= npairs) break;
    Pair pr = pairs[pi];
    const int c = pr.key % f.k;
    double cold[D];
    if (!f.weights_only) {
#pragma unroll
      for (int j = 0; j < D; ++j) cold[j] = f.centers[c * D + j];
    }
    double acc = 0.0;   // lane j < ncols folds column j (bincount starts from 0.0)
    double ext = 0.0;
    for (int64_t base = pr.first; base <= pr.last; base += 32) {
      int64_t i = base + lane;
      bool valid = i <= pr.last && f.a[i] == c;
      if (valid) {
        double w = load_weight(f.w, f.wmode, i);
        if (f.weights_only) {
          sm[warp][0][lane] = w;
        } else {
          double x[D], diff[D];
#pragma unroll
          for (int j = 0; j < D; ++j) {
            x[j] = f.X[j * f.ldx + i];
            sm[warp][j][lane] = __dmul_rn(x[j], w);  // wx = points * weights[:, None]
            diff[j] = __dsub_rn(x[j], cold[j]);
          }
          double sq = sqnorm_rn(diff, D, f.order3);
          sm[warp][D][lane] = w;
          sm[warp][D + 1][lane] = __dmul_rn(sq, w);
          ext = fmax(ext, __dsqrt_rn(sq));
        }
      }
      unsigned m = __ballot_sync(FULL, valid);
      __syncwarp();
      if (lane < ncols) {
        if (m == FULL) {
#pragma unroll
          for (int b = 0; b < 32; ++b) acc = __dadd_rn(acc, sm[warp][lane][b]);
        } else {
          while (m) {
            int b = __ffs(m) - 1;
            m &= m - 1;
            acc = __dadd_rn(acc, sm[warp][lane][b]);
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

template <int D>
__global__ void fold_combine(gp_fold_args f, const int32_t* __restrict__ slot, int64_t nseg,
                             const double* __restrict__ out) {
  int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= f.k) return;
  if (f.weights_only) {
    double w = 0.0;
    for (int64_t s = 0; s < nseg; ++s) {
      int32_t p = slot[s * f.k + c];
      if (p >= 0) w = __dadd_rn(w, out[(int64_t)p * (MAXCOL + 1)]);
    }
    f.wsum[c] = w;
    return;
  }
  double acc[D + 2];
#pragma unroll
  for (int j = 0; j < D + 2; ++j) acc[j] = 0.0;
  double ext = 0.0;
  for (int64_t s = 0; s < nseg; ++s) {
    int32_t p = slot[s * f.k + c];
    if (p >= 0) {
      const double* po = out + (int64_t)p * (MAXCOL + 1);
#pragma unroll
      for (int j = 0; j < D + 2; ++j) acc[j] = __dadd_rn(acc[j], po[j]);
      ext = fmax(ext, po[MAXCOL]);
    }
  }
#pragma unroll
  for (int j = 0; j < D; ++j) f.sums[c * D + j] = acc[j];
  f.wsum[c] = acc[D];
  f.objective[c] = acc[D + 1];
  f.extent[c] = ext;
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
    fold_combine<2><<<grid_for(f->k, 128), 128, 0, s>>>(*f, slot, L.nseg, out);
  } else {
    fold_kernel<3><<<sms * 8, FT, 0, s>>>(*f, pairs, counters, out);
    fold_combine<3><<<grid_for(f->k, 128), 128, 0, s>>>(*f, slot, L.nseg, out);
  }
  return check_launch("movement_fold");
}

}  // extern "C"
