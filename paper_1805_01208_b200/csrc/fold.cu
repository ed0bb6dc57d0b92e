// K7 movement reduction, bit-exact with the reference.
//
// The reference sums w*x and w per (segment, block) with sequential bincount
// folds in SFC order (ranksim.py:173-197), then folds the 256 segment partials
// sequentially (np.add.reduce(axis=0), ranksim.py:218-222 / kmeans.py:374).
// A sequential fold cannot be parallelised, but the folds of different
// (segment, block) pairs are independent.  SFC order keeps a block in a few
// runs of consecutive positions, so:
//   runs     : every maximal run of positions with the same (segment, block)
//              key (stable compaction of the key-change positions);
//   group    : stable radix sort of the runs by key -> each pair's runs in
//              position order; pair boundaries -> work list;
//   fold     : one warp per pair walks its runs in order, stages each chunk's
//              values in shared memory and lets lane j fold column j in
//              position order (the exact bincount order); extents (max
//              distance to the old center, kmeans.py:474-487) and the
//              objective terms (kmeans.py:490-499) are computed in parallel
//              by all lanes of the chunk;
//   combine  : per block, fold the pair partials in segment order.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include "common.cuh"

namespace gp {

constexpr int FT = 256;     // threads per fold CTA (8 warps)
constexpr int MAXCOL = 5;   // d wx columns + w + objective (d <= 3)
constexpr int FB = 4;       // chunks of 32 positions prefetched per batch

// counters[]: 0 runs, 1 work cursor, 2 valid runs, 3 pairs
struct FoldLayout {
  int64_t s0, nseg, cells, cap, pcap;
  size_t off_flags, off_starts, off_rkey, off_skey, off_sidx, off_ridx, off_pbeg, off_slot,
      off_out, off_counters, off_cub, cub_bytes, off_rpre, off_spos, off_skey_final, total;
};

static FoldLayout layout(int64_t n_local, int64_t pos0, int64_t n_global, int k) {
  FoldLayout L;
  auto seg = [&](int64_t pos) { return ((pos + 1) * (int64_t)GP_SEGMENTS - 1) / n_global; };
  L.s0 = n_local > 0 ? seg(pos0) : 0;
  int64_t s1 = n_local > 0 ? seg(pos0 + n_local - 1) : 0;
  L.nseg = n_local > 0 ? s1 - L.s0 + 1 : 1;
  L.cells = L.nseg * k;
  L.cap = n_local > 0 ? n_local : 1;
  L.pcap = L.cells < L.cap ? L.cells : L.cap;  // pairs <= min(segments x blocks, runs)
  size_t b1 = 0, b2 = 0, b3 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b3, (const int64_t*)nullptr, (int64_t*)nullptr,
                                (int)L.cap + 1);
  cub::DeviceSelect::Flagged(nullptr, b1, cub::CountingInputIterator<int32_t>(0),
                             (const uint8_t*)nullptr, (int32_t*)nullptr, (int64_t*)nullptr,
                             (int)L.cap);
  cub::DoubleBuffer<uint32_t> kb(nullptr, nullptr);
  cub::DoubleBuffer<int32_t> vb(nullptr, nullptr);
  cub::DeviceRadixSort::SortPairs(nullptr, b2, kb, vb, (int)L.cap, 0, 32);
  L.cub_bytes = b1 > b2 ? b1 : b2;
  if (b3 > L.cub_bytes) L.cub_bytes = b3;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  size_t o = 0;
  L.off_flags = o; o = al(o + L.cap);
  L.off_starts = o; o = al(o + (L.cap + 1) * 4);
  L.off_rkey = o; o = al(o + L.cap * 4);
  L.off_skey = o; o = al(o + L.cap * 4);
  L.off_skey_final = L.off_skey;
  L.off_sidx = o; o = al(o + L.cap * 4);
  L.off_ridx = o; o = al(o + L.cap * 4);
  L.off_pbeg = o; o = al(o + (L.pcap + 1) * 4);
  L.off_slot = o; o = al(o + L.cells * 4);
  L.off_out = o; o = al(o + L.pcap * (MAXCOL + 1) * sizeof(double));
  L.off_counters = o; o = al(o + 8 * sizeof(int64_t));
  L.off_cub = o; o = al(o + L.cub_bytes);
  L.off_rpre = o; o = al(o + (L.cap + 1) * 8);
  L.off_spos = o; o = al(o + L.cap * 4);
  L.total = o;
  return L;
}

__device__ __forceinline__ int32_t fold_key(const int32_t* a, int64_t i, int64_t pos0,
                                            int64_t n_global, int64_t s0, int k) {
  int c = a[i];
  return c >= 0 ? (int32_t)((segment_of(pos0 + i, n_global) - s0) * k + c) : -1;
}

// flag every position whose key differs from its predecessor's (run starts);
// each thread handles MK consecutive positions with one segment computation
constexpr int MK = 8;
__global__ void fold_mark(const int32_t* __restrict__ a, int64_t n_local, int64_t pos0,
                          int64_t n_global, int64_t s0, int k, uint8_t* __restrict__ flags) {
  const int64_t nt = (n_local + MK - 1) / MK;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < nt;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i0 = t * MK;
    int seg = segment_of(pos0 + i0, n_global);
    int64_t next_b = seg + 1 < GP_SEGMENTS ? ((int64_t)(seg + 1) * n_global >> 8) - pos0
                                            : INT64_MAX;  // local position of the next segment
    int prev_key = i0 > 0 ? fold_key(a, i0 - 1, pos0, n_global, s0, k) : -2;
    uint8_t f[MK];
#pragma unroll
    for (int e = 0; e < MK; ++e) {
      const int64_t i = i0 + e;
      if (i >= n_local) break;
      while (i >= next_b) {
        ++seg;
        next_b = seg + 1 < GP_SEGMENTS ? ((int64_t)(seg + 1) * n_global >> 8) - pos0 : INT64_MAX;
      }
      const int c = a[i];
      const int key = c >= 0 ? (int)((seg - s0) * k + c) : -1;
      f[e] = key != prev_key;
      prev_key = key;
    }
    if (i0 + MK <= n_local) {
      uint2 v;
      v.x = f[0] | (f[1] << 8) | (f[2] << 16) | ((unsigned)f[3] << 24);
      v.y = f[4] | (f[5] << 8) | (f[6] << 16) | ((unsigned)f[7] << 24);
      *reinterpret_cast<uint2*>(flags + i0) = v;
    } else {
      for (int e = 0; i0 + e < n_local; ++e) flags[i0 + e] = f[e];
    }
  }
}

// run r -> (key, r); runs with key -1 (unassigned / inactive) sort last
__global__ void fold_run_keys(const int32_t* __restrict__ a, int32_t* __restrict__ starts,
                              int64_t R, int64_t* counters, int64_t n_local, int64_t pos0,
                              int64_t n_global, int64_t s0, int k, uint32_t* __restrict__ rkey,
                              int32_t* __restrict__ ridx) {
  if (blockIdx.x == 0 && threadIdx.x == 0) starts[R] = (int32_t)n_local;  // sentinel end
  int valid = 0;
  for (int64_t r = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; r < R;
       r += (int64_t)gridDim.x * blockDim.x) {
    int32_t key = fold_key(a, starts[r], pos0, n_global, s0, k);
    rkey[r] = (uint32_t)key;  // -1 -> 0xffffffff
    ridx[r] = (int32_t)r;
    valid += key >= 0;
  }
  for (int o = 16; o; o >>= 1) valid += __shfl_xor_sync(FULL, valid, o);
  if ((threadIdx.x & 31) == 0 && valid)
    atomicAdd((unsigned long long*)&counters[2], (unsigned long long)valid);
}

// first sorted run of every pair (valid runs occupy the first counters[2] slots)
__global__ void fold_pair_flags(const uint32_t* __restrict__ skey, int64_t R,
                                const int64_t* counters, uint8_t* __restrict__ flags) {
  const int64_t V = counters[2];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < R;
       j += (int64_t)gridDim.x * blockDim.x)
    flags[j] = j < V && (j == 0 || skey[j] != skey[j - 1]);
}

// length of the j-th sorted run (valid runs only; 0 beyond)
__global__ void fold_run_len(const int32_t* __restrict__ starts, const int32_t* __restrict__ sidx,
                             int64_t R, const int64_t* counters, int64_t* __restrict__ len) {
  const int64_t V = counters[2];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j <= R;
       j += (int64_t)gridDim.x * blockDim.x) {
    int64_t l = 0;
    if (j < V) {
      const int r = sidx[j];
      l = starts[r + 1] - starts[r];
    }
    len[j] = l;
  }
}

// sorted positions: every valid position, grouped by pair, in position order
// within the pair (one warp per sorted run)
__global__ void fold_expand(const int32_t* __restrict__ starts, const int32_t* __restrict__ sidx,
                            const int64_t* __restrict__ pre, const int64_t* counters,
                            int32_t* __restrict__ spos) {
  const int64_t V = counters[2];
  const int lane = threadIdx.x & 31;
  const int64_t nw = (int64_t)gridDim.x * (blockDim.x / 32);
  for (int64_t j = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) / 32; j < V; j += nw) {
    const int r = sidx[j];
    const int32_t b = starts[r], e = starts[r + 1];
    const int64_t o = pre[j];
    for (int32_t t = lane; t < e - b; t += 32) spos[o + t] = b + t;
  }
}

__global__ void fold_slots(const uint32_t* __restrict__ skey, int32_t* __restrict__ pbeg,
                           const int64_t* counters, int32_t* __restrict__ slot) {
  const int64_t P = counters[3];
  if (blockIdx.x == 0 && threadIdx.x == 0) pbeg[P] = (int32_t)counters[2];  // sentinel end
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x)
    slot[skey[pbeg[p]]] = (int32_t)p;
}

// One warp per (segment, block) pair: its positions (contiguous in spos, in
// position order) in batches of FB*32; the loads of batch b+1 are issued before
// batch b is folded, so the serial fold (lane j folds column j) overlaps them.
template <int D>
__device__ __forceinline__ void fold_load(const gp_fold_args& f, const int32_t* spos, int64_t v0,
                                          int64_t v1, int lane, double (&xv)[FB][D],
                                          double (&wv)[FB]) {
#pragma unroll
  for (int b = 0; b < FB; ++b) {
    const int64_t v = v0 + b * 32 + lane;
    const bool in = v < v1;
    const int i = in ? spos[v] : 0;
    wv[b] = in ? load_weight(f.w, f.wmode, i) : 0.0;
    if (!f.weights_only) {
      if (in) load_point<D>(f.X, f.ldx, i, xv[b]);
      else
#pragma unroll
        for (int j = 0; j < D; ++j) xv[b][j] = 0.0;
    }
  }
}

template <int D>
__global__ void __launch_bounds__(FT) fold_kernel(gp_fold_args f, const int32_t* __restrict__ spos,
                                                  const int64_t* __restrict__ pre,
                                                  const uint32_t* __restrict__ skey,
                                                  const int32_t* __restrict__ pbeg,
                                                  int64_t* counters, double* __restrict__ out) {
  __shared__ double sm[FT / 32][MAXCOL][FB * 32 + 1];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ncols = f.weights_only ? 1 : D + 2;
  const int64_t npairs = counters[3];
  for (;;) {
    int64_t pi;
    if (lane == 0) pi = (int64_t)atomicAdd((unsigned long long*)&counters[1], 1ull);
    pi = __shfl_sync(FULL, pi, 0);
    if (pi >= npairs) break;
    const int j0 = pbeg[pi], j1 = pbeg[pi + 1];
    const int c = (int)(skey[j0] % (uint32_t)f.k);
    const int64_t v0 = pre[j0], v1 = pre[j1];
    double cold[D];
    if (!f.weights_only) {
#pragma unroll
      for (int j = 0; j < D; ++j) cold[j] = f.centers[c * D + j];
    }
    double acc = 0.0;  // lane j < ncols folds column j; bincount starts from 0.0
    double ext = 0.0;
    double xv[FB][D], wv[FB];
    fold_load<D>(f, spos, v0, v1, lane, xv, wv);
    for (int64_t base = v0; base < v1; base += FB * 32) {
      // stage the current batch, then issue the next batch's loads
#pragma unroll
      for (int b = 0; b < FB; ++b) {
        const int slot = b * 32 + lane;
        const bool in = base + slot < v1;
        if (f.weights_only) {
          sm[warp][0][slot] = wv[b];
        } else {
          double diff[D];
#pragma unroll
          for (int j = 0; j < D; ++j) {
            sm[warp][j][slot] = __dmul_rn(xv[b][j], wv[b]);  // wx = points * weights[:, None]
            diff[j] = __dsub_rn(xv[b][j], cold[j]);
          }
          const double sq = sqnorm_rn(diff, D, f.order3);
          sm[warp][D][slot] = wv[b];
          sm[warp][D + 1][slot] = __dmul_rn(sq, wv[b]);
          if (in) ext = fmax(ext, __dsqrt_rn(sq));
        }
      }
      __syncwarp();
      if (base + FB * 32 < v1) fold_load<D>(f, spos, base + FB * 32, v1, lane, xv, wv);
      const int cnt = (int)min((int64_t)(FB * 32), v1 - base);
      if (lane < ncols) {
        const double* col = sm[warp][lane];
        if (cnt == FB * 32) {
#pragma unroll 32
          for (int t = 0; t < FB * 32; ++t) acc = __dadd_rn(acc, col[t]);
        } else {
          for (int t = 0; t < cnt; ++t) acc = __dadd_rn(acc, col[t]);
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
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * 4 + warp;
  if (c >= f.k) return;
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
    for (int i = 0; i < np; ++i)
      acc = __dadd_rn(acc, out[(int64_t)s_slot[warp][i] * (MAXCOL + 1) + lane]);
    if (f.weights_only) f.wsum[c] = acc;
    else if (lane < D) f.sums[c * D + lane] = acc;
    else if (lane == D) f.wsum[c] = acc;
    else f.objective[c] = acc;
  }
  if (!f.weights_only) {
    double ext = 0.0;
    for (int i = lane; i < np; i += 32)
      ext = fmax(ext, out[(int64_t)s_slot[warp][i] * (MAXCOL + 1) + MAXCOL]);
    for (int o = 16; o; o >>= 1) ext = fmax(ext, __shfl_xor_sync(FULL, ext, o));
    if (lane == 0) f.extent[c] = ext;
  }
}

__global__ void fold_export_kernel(const uint32_t* __restrict__ skey,
                                   const int32_t* __restrict__ pbeg,
                                   const int64_t* __restrict__ counters,
                                   const double* __restrict__ out, int64_t s0, int k,
                                   int64_t* __restrict__ keys, double* __restrict__ vals,
                                   int64_t* npairs) {
  const int64_t P = counters[3];
  if (blockIdx.x == 0 && threadIdx.x == 0) *npairs = P;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t key = skey[pbeg[p]];
    const int64_t seg = key / (uint32_t)k + s0, c = key % (uint32_t)k;
    keys[p] = seg * k + c;
#pragma unroll
    for (int j = 0; j < MAXCOL + 1; ++j) vals[p * (MAXCOL + 1) + j] = out[p * (MAXCOL + 1) + j];
  }
}

__global__ void combine_slots(const int64_t* __restrict__ keys, int64_t npairs,
                              int32_t* __restrict__ slot) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npairs;
       p += (int64_t)gridDim.x * blockDim.x)
    slot[keys[p]] = (int32_t)p;
}

}  // namespace gp

using namespace gp;

static int64_t* g_last_counters = nullptr;

extern "C" {

int gp_fold_stats(int64_t* out) {
  // debugging aid: {runs, cursor, valid runs, pairs} of the last gp_movement_fold (syncs)
  if (!g_last_counters) return GP_ERR_INVALID;
  GP_CUDA(cudaDeviceSynchronize());
  GP_CUDA(cudaMemcpy(out, g_last_counters, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost));
  return GP_OK;
}

int gp_fold_export(const gp_fold_args* f, int64_t* keys, double* vals, int64_t* npairs,
                   void* stream) {
  GP_REQUIRE(f && keys && vals && npairs, "gp_fold_export: bad args");
  FoldLayout L = layout(f->n_local, f->pos0, f->n_global, f->k);
  char* ws = (char*)f->workspace;
  fold_export_kernel<<<grid_for(L.pcap, 256, 148 * 8), 256, 0, (cudaStream_t)stream>>>(
      (const uint32_t*)(ws + L.off_skey_final), (const int32_t*)(ws + L.off_pbeg),
      (const int64_t*)(ws + L.off_counters), (const double*)(ws + L.off_out), L.s0, f->k, keys,
      vals, npairs);
  return check_launch("fold_export");
}

int gp_fold_combine_bytes(int k, size_t* bytes) {
  GP_REQUIRE(k >= 1, "gp_fold_combine_bytes: bad k");
  *bytes = (size_t)GP_SEGMENTS * k * sizeof(int32_t);
  return GP_OK;
}

int gp_fold_combine(const int64_t* keys, const double* vals, int64_t npairs, int k, int d,
                    int weights_only, double* sums, double* wsum, double* extent,
                    double* objective, void* workspace, size_t workspace_bytes, void* stream) {
  GP_REQUIRE(d == 2 || d == 3, "gp_fold_combine: bad d");
  GP_REQUIRE(workspace_bytes >= (size_t)GP_SEGMENTS * k * sizeof(int32_t),
             "gp_fold_combine: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  int32_t* slot = (int32_t*)workspace;
  GP_CUDA(cudaMemsetAsync(slot, 0xff, (size_t)GP_SEGMENTS * k * sizeof(int32_t), s));
  if (npairs > 0)
    combine_slots<<<grid_for(npairs, 256, 148 * 8), 256, 0, s>>>(keys, npairs, slot);
  gp_fold_args f{};
  f.d = d;
  f.k = k;
  f.weights_only = weights_only;
  f.sums = sums;
  f.wsum = wsum;
  f.extent = extent;
  f.objective = objective;
  if (d == 2) fold_combine<2><<<grid_for(k, 4), 128, 0, s>>>(f, slot, GP_SEGMENTS, vals);
  else fold_combine<3><<<grid_for(k, 4), 128, 0, s>>>(f, slot, GP_SEGMENTS, vals);
  return check_launch("fold_combine");
}

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
  uint8_t* flags = (uint8_t*)(ws + L.off_flags);
  int32_t* starts = (int32_t*)(ws + L.off_starts);
  uint32_t* rkey = (uint32_t*)(ws + L.off_rkey);
  uint32_t* skey = (uint32_t*)(ws + L.off_skey);
  int32_t* sidx = (int32_t*)(ws + L.off_sidx);
  int32_t* ridx = (int32_t*)(ws + L.off_ridx);
  int32_t* pbeg = (int32_t*)(ws + L.off_pbeg);
  int32_t* slot = (int32_t*)(ws + L.off_slot);
  double* out = (double*)(ws + L.off_out);
  int64_t* counters = (int64_t*)(ws + L.off_counters);
  int64_t* rpre = (int64_t*)(ws + L.off_rpre);
  int32_t* spos = (int32_t*)(ws + L.off_spos);
  g_last_counters = counters;
  void* cub_tmp = ws + L.off_cub;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t n = f->n_local;

  GP_CUDA(cudaMemsetAsync(counters, 0, 8 * sizeof(int64_t), s));
  GP_CUDA(cudaMemsetAsync(slot, 0xff, L.cells * sizeof(int32_t), s));
  if (n > 0) {
    fold_mark<<<grid_for((n + MK - 1) / MK, 256, sms * 16), 256, 0, s>>>(f->a, n, f->pos0, f->n_global, L.s0,
                                                          f->k, flags);
    size_t b = L.cub_bytes;
    GP_CUDA(cub::DeviceSelect::Flagged(cub_tmp, b, cub::CountingInputIterator<int32_t>(0), flags,
                                       starts, counters + 0, (int)n, s));
    int64_t R = 0;
    GP_CUDA(cudaMemcpyAsync(&R, counters, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    GP_CUDA(cudaStreamSynchronize(s));
    fold_run_keys<<<grid_for(R, 256, sms * 16), 256, 0, s>>>(
        f->a, starts, R, counters, n, f->pos0, f->n_global, L.s0, f->k, rkey, ridx);
    // stable LSD radix sort with ping-pong buffers (no n-sized CUB scratch)
    cub::DoubleBuffer<uint32_t> kb(rkey, skey);
    cub::DoubleBuffer<int32_t> vb(ridx, sidx);
    b = L.cub_bytes;
    GP_CUDA(cub::DeviceRadixSort::SortPairs(cub_tmp, b, kb, vb, (int)R, 0, 32, s));
    skey = kb.Current();
    sidx = vb.Current();
    if (skey != (uint32_t*)(ws + L.off_skey_final)) {
      // keep the sorted keys where gp_fold_export expects them
      GP_CUDA(cudaMemcpyAsync(ws + L.off_skey_final, skey, R * sizeof(uint32_t),
                              cudaMemcpyDeviceToDevice, s));
      skey = (uint32_t*)(ws + L.off_skey_final);
    }
    fold_pair_flags<<<grid_for(R, 256, sms * 16), 256, 0, s>>>(skey, R, counters, flags);
    b = L.cub_bytes;
    GP_CUDA(cub::DeviceSelect::Flagged(cub_tmp, b, cub::CountingInputIterator<int32_t>(0), flags,
                                       pbeg, counters + 3, (int)R, s));
    fold_slots<<<grid_for(R, 256, sms * 8), 256, 0, s>>>(skey, pbeg, counters, slot);
    // positions grouped by pair: prefix of the sorted run lengths, then expansion
    fold_run_len<<<grid_for(R + 1, 256, sms * 8), 256, 0, s>>>(starts, sidx, R, counters, rpre);
    b = L.cub_bytes;
    GP_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, b, rpre, rpre, (int)(R + 1), s));
    fold_expand<<<grid_for(R * 32, 256, sms * 16), 256, 0, s>>>(starts, sidx, rpre, counters,
                                                                spos);
  }
  if (f->d == 2) {
    fold_kernel<2><<<sms * 6, FT, 0, s>>>(*f, spos, rpre, skey, pbeg, counters, out);
    fold_combine<2><<<grid_for(f->k, 4), 128, 0, s>>>(*f, slot, L.nseg, out);
  } else {
    fold_kernel<3><<<sms * 6, FT, 0, s>>>(*f, spos, rpre, skey, pbeg, counters, out);
    fold_combine<3><<<grid_for(f->k, 4), 128, 0, s>>>(*f, slot, L.nseg, out);
  }
  return check_launch("movement_fold");
}

}  // extern "C"
