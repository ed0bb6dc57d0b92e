// SFC bootstrap kernels: bounding box, Hilbert keys, radix sort, payload
// gather, initial centers, sample-phase compaction, result scatter.
//
// Reference semantics: geometry.py:112-192 (cells + Hilbert keys),
// ranksim.py:143-170 (global sort + redistribution), kmeans.py:546-568.

#include <cstdarg>
#include <cstdio>

#include <cub/device/device_scan.cuh>

#include <utility>
#include <vector>

#include "common.cuh"
#include "radix.cuh"

namespace gp {

static thread_local char g_err[512] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    set_error("%s launch failed: %s", what, cudaGetErrorString(e));
    return GP_ERR_CUDA;
  }
  return GP_OK;
}

// ---------------------------------------------------------------- K1 box
__global__ void box_kernel(const double* __restrict__ pts, int64_t n, int d, int64_t sp,
                           int64_t sd, unsigned long long* keys, int32_t* nonfinite) {
  double lo[3] = {INFINITY, INFINITY, INFINITY};
  double hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  int bad = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    for (int j = 0; j < d; ++j) {
      double v = pts[i * sp + j * sd];
      bad |= !isfinite(v);
      lo[j] = fmin(lo[j], v);
      hi[j] = fmax(hi[j], v);
    }
  }
  for (int j = 0; j < d; ++j) {
    for (int o = 16; o; o >>= 1) {
      lo[j] = fmin(lo[j], __shfl_xor_sync(FULL, lo[j], o));
      hi[j] = fmax(hi[j], __shfl_xor_sync(FULL, hi[j], o));
    }
  }
  bad = __any_sync(FULL, bad);
  if ((threadIdx.x & 31) == 0) {
    for (int j = 0; j < d; ++j) {
      atomicMin(&keys[j], dkey(lo[j]));
      atomicMax(&keys[d + j], dkey(hi[j]));
    }
    if (bad) atomicOr(nonfinite, 1);
  }
}

// the common layout, AoS (n, 2) rows: 16-byte loads, four independent points per step
__global__ void box_kernel_aos2(const double2* __restrict__ pts, int64_t n,
                                unsigned long long* keys, int32_t* nonfinite) {
  double lo0 = INFINITY, lo1 = INFINITY, hi0 = -INFINITY, hi1 = -INFINITY;
  int bad = 0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += 4 * stride) {
    double2 v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t i = i0 + u * stride;
      v[u] = (u == 0 || i < n) ? pts[i] : v[0];   // past the end: repeat the step's first point
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      bad |= !isfinite(v[u].x) | !isfinite(v[u].y);
      lo0 = fmin(lo0, v[u].x); hi0 = fmax(hi0, v[u].x);
      lo1 = fmin(lo1, v[u].y); hi1 = fmax(hi1, v[u].y);
    }
  }
  for (int o = 16; o; o >>= 1) {
    lo0 = fmin(lo0, __shfl_xor_sync(FULL, lo0, o)); hi0 = fmax(hi0, __shfl_xor_sync(FULL, hi0, o));
    lo1 = fmin(lo1, __shfl_xor_sync(FULL, lo1, o)); hi1 = fmax(hi1, __shfl_xor_sync(FULL, hi1, o));
  }
  bad = __any_sync(FULL, bad);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&keys[0], dkey(lo0)); atomicMin(&keys[1], dkey(lo1));
    atomicMax(&keys[2], dkey(hi0)); atomicMax(&keys[3], dkey(hi1));
    if (bad) atomicOr(nonfinite, 1);
  }
}

__global__ void box_finalize(unsigned long long* keys, int d) {
  int j = threadIdx.x;
  if (j < 2 * d) {
    double v = dkey_inv(keys[j]);
    reinterpret_cast<double*>(keys)[j] = v;
  }
}

// ------------------------------------------------------- weight probe
__global__ void weight_probe_kernel(const double* __restrict__ w, int64_t n,
                                    unsigned long long* out) {
  unsigned long long flags = 0;
  int low = 4096;
  double mx = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double v = w[i];
    if (!isfinite(v)) { flags |= 1; continue; }
    if ((double)(float)v != v) flags |= 2;
    double av = fabs(v);
    mx = fmax(mx, av);
    if (av != 0.0) {
      // exponent of the lowest set bit: av = m * 2^e with m odd
      int e;
      double m = frexp(av, &e);  // av = m * 2^e, m in [0.5, 1)
      // ldexp(m, 53) is an integer in [2^52, 2^53) (exact): av = iv * 2^(e-53)
      unsigned long long iv = (unsigned long long)ldexp(m, 53);
      int tz = __ffsll((long long)iv) - 1;
      low = min(low, e - 53 + tz);
    }
  }
  for (int o = 16; o; o >>= 1) {
    flags |= __shfl_xor_sync(FULL, flags, o);
    low = min(low, __shfl_xor_sync(FULL, low, o));
    mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicOr(&out[0], flags);
    atomicMin((long long*)&out[1], (long long)low);
    atomicMax(&out[2], (unsigned long long)__double_as_longlong(mx));
  }
}

// -------------------------------------------------------- K2 Hilbert keys
__device__ __forceinline__ uint64_t spread2(uint32_t x) {
  uint64_t v = x;
  v = (v | (v << 16)) & 0x0000FFFF0000FFFFull;
  v = (v | (v << 8)) & 0x00FF00FF00FF00FFull;
  v = (v | (v << 4)) & 0x0F0F0F0F0F0F0F0Full;
  v = (v | (v << 2)) & 0x3333333333333333ull;
  v = (v | (v << 1)) & 0x5555555555555555ull;
  return v;
}
__device__ __forceinline__ uint64_t spread3(uint32_t x) {
  uint64_t v = x & 0x1fffffu;
  v = (v | (v << 32)) & 0x001f00000000ffffull;
  v = (v | (v << 16)) & 0x001f0000ff0000ffull;
  v = (v | (v << 8)) & 0x100f00f00f00f00full;
  v = (v | (v << 4)) & 0x10c30c30c30c30c3ull;
  v = (v | (v << 2)) & 0x1249249249249249ull;
  return v;
}

// geometry.py:135-179 on 32-bit lanes (cells < 2^depth <= 2^31).
template <int D>
__host__ __device__ __forceinline__ void hilbert_transpose(uint32_t* X, int depth) {
  for (uint32_t Q = 1u << (depth - 1); Q > 1; Q >>= 1) {
    uint32_t P = Q - 1;
#pragma unroll
    for (int i = 0; i < D; ++i) {
      uint32_t t = (X[0] ^ X[i]) & P;
      bool flip = (X[i] & Q) != 0;
      X[0] ^= flip ? P : t;
      if (!flip) X[i] ^= t;
    }
  }
#pragma unroll
  for (int i = 1; i < D; ++i) X[i] ^= X[i - 1];
  uint32_t t = 0;
  for (uint32_t Q = 1u << (depth - 1); Q > 1; Q >>= 1)
    if (X[D - 1] & Q) t ^= Q - 1;
#pragma unroll
  for (int i = 0; i < D; ++i) X[i] ^= t;
}

template <int D>
__device__ __forceinline__ uint64_t interleave(const uint32_t* X) {
  if (D == 2) return (spread2(X[0]) << 1) | spread2(X[1]);
  return (spread3(X[0]) << 2) | (spread3(X[1]) << 1) | spread3(X[2]);
}

// The transpose above as a finite-state machine over levels, top level first (the
// form the kernel runs).  Processing level b with the cells' raw bits r:
//   t = g(r)                  bits as transformed by the operations of the levels above;
//   G = gray(t)               G_0 = t_0, G_i = t_i ^ G_{i-1}       (the Gray loop);
//   F = G ^ par               par = xor of G_{d-1} over the levels above (the t loop);
//   key <- key . F_0 .. F_{d-1}                                     (the interleave);
//   g <- h(t) o g             h: for i = 0..d-1, invert axis 0 if t_i, else swap
//                             axes 0 and i (the operations on the lower bits);
//   par <- par ^ G_{d-1}.
// g ranges over a few signed axis permutations, so (g, par) is a small state and L
// levels at a time become one table lookup: entry [state][d*L raw bits] = the d*L key
// bits | next state << (d*L).  The tables are built on the host from this definition
// (hilbert_fsm_tables) and checked against the transpose at load (gp_hilbert_keys).
struct HFsm {
  int states;
  int L;                           // levels per multi-level lookup
  uint16_t multi[96 * 256];        // [state][raw chunk]
  uint16_t single[96 * 8];         // [state][raw level]
};
__device__ HFsm g_hfsm[2];         // d = 2, d = 3

static void hilbert_fsm_tables(int d, HFsm& T) {
  const int nv = 1 << d;
  std::vector<std::vector<int>> gs;   // reachable transforms (maps on d-bit vectors)
  std::vector<int> ident(nv);
  for (int v = 0; v < nv; ++v) ident[v] = v;
  gs.push_back(ident);
  auto level_op = [&](int t) {
    std::vector<int> h(nv);
    for (int v = 0; v < nv; ++v) {
      int bits[3] = {v & 1, (v >> 1) & 1, (v >> 2) & 1};
      for (int i = 0; i < d; ++i) {
        if ((t >> i) & 1) bits[0] ^= 1;
        else std::swap(bits[0], bits[i]);
      }
      h[v] = bits[0] | (bits[1] << 1) | (bits[2] << 2);
    }
    return h;
  };
  auto index_of = [&](const std::vector<int>& g) {
    for (size_t k = 0; k < gs.size(); ++k)
      if (gs[k] == g) return (int)k;
    gs.push_back(g);
    return (int)gs.size() - 1;
  };
  // one level from (g index, par) with raw bits r: out F bits (axis 0 most significant),
  // next (g index, par)
  auto step = [&](int gi, int par, int r, int& F, int& ngi, int& npar) {
    const std::vector<int> g = gs[gi];
    const int t = g[r];
    int G[3], prev = 0;
    for (int i = 0; i < d; ++i) {
      G[i] = ((t >> i) & 1) ^ (i ? prev : 0);
      prev = G[i];
    }
    F = 0;
    for (int i = 0; i < d; ++i) F = (F << 1) | (G[i] ^ par);
    const std::vector<int> h = level_op(t);
    std::vector<int> ng(nv);
    for (int v = 0; v < nv; ++v) ng[v] = h[g[v]];
    ngi = index_of(ng);
    npar = par ^ G[d - 1];
  };
  for (size_t gi = 0; gi < gs.size(); ++gi)      // close the state set
    for (int r = 0; r < nv; ++r) {
      int F, ngi, np;
      step((int)gi, 0, r, F, ngi, np);
    }
  T.states = 2 * (int)gs.size();
  T.L = d == 2 ? 4 : 2;
  const int L = T.L, nin = 1 << (d * L);
  for (int st = 0; st < T.states; ++st) {
    for (int r = 0; r < nv; ++r) {
      int F, ngi, np;
      step(st >> 1, st & 1, r, F, ngi, np);
      T.single[st * 8 + r] = (uint16_t)(F | ((2 * ngi + np) << d));
    }
    for (int c = 0; c < nin; ++c) {
      int gi = st >> 1, par = st & 1, key = 0;
      for (int l = 0; l < L; ++l) {   // top level of the chunk first
        int r = 0;
        for (int i = 0; i < d; ++i) r |= ((c >> (i * L + (L - 1 - l))) & 1) << i;
        int F, ngi, np;
        step(gi, par, r, F, ngi, np);
        key = (key << d) | F;
        gi = ngi;
        par = np;
      }
      T.multi[st * 256 + c] = (uint16_t)(key | ((2 * gi + par) << (d * L)));
    }
  }
}

template <int D>
__global__ void hilbert_kernel(const double* __restrict__ pts, int64_t n, int64_t sp, int64_t sd,
                               const double* __restrict__ lohi, int depth,
                               uint64_t* __restrict__ keys, uint32_t* __restrict__ gids,
                               uint32_t gid_base) {
  __shared__ uint16_t s_multi[96 * 64 > 16 * 256 ? 96 * 64 : 16 * 256];
  __shared__ uint16_t s_single[96 * 8];
  const HFsm& T = g_hfsm[D - 2];
  constexpr int L = D == 2 ? 4 : 2;
  constexpr int NIN = 1 << (D * L);
  const int S = T.states;
  for (int e = threadIdx.x; e < S * NIN; e += blockDim.x)
    s_multi[e] = T.multi[(e / NIN) * 256 + (e % NIN)];
  for (int e = threadIdx.x; e < S * 8; e += blockDim.x) s_single[e] = T.single[e];
  __syncthreads();
  double lo[D], safe[D];
  const double side = (double)(1ull << depth);
  const double top = side - 1.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    lo[j] = lohi[j];
    double ext = __dsub_rn(lohi[D + j], lo[j]);
    safe[j] = ext > 0.0 ? ext : 1.0;
  }
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t X[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      // geometry.py:129-132: (p - lo) / ext * 2^depth, floor, clip to [0, side-1]
      double s = __dmul_rn(__ddiv_rn(__dsub_rn(pts[i * sp + j * sd], lo[j]), safe[j]), side);
      double c = fmin(fmax(floor(s), 0.0), top);
      X[j] = (uint32_t)c;
    }
    // the transpose + interleave as table steps, top level first
    uint64_t key = 0;
    int st = 0;
    int b = depth - 1;                     // next level to consume
    for (; b + 1 >= L; b -= L) {
      int c = 0;
#pragma unroll
      for (int j = 0; j < D; ++j) c |= (int)((X[j] >> (b + 1 - L)) & ((1u << L) - 1)) << (j * L);
      const unsigned e = s_multi[st * NIN + c];
      key = (key << (D * L)) | (e & ((1u << (D * L)) - 1));
      st = (int)(e >> (D * L));
    }
    for (; b >= 0; --b) {
      int r = 0;
#pragma unroll
      for (int j = 0; j < D; ++j) r |= (int)((X[j] >> b) & 1u) << j;
      const unsigned e = s_single[st * 8 + r];
      key = (key << D) | (e & ((1u << D) - 1));
      st = (int)(e >> D);
    }
    keys[i] = key;
    if (gids) gids[i] = gid_base + (uint32_t)i;
  }
}

// ---------------------------------------------------------- payload gather
// Four independent elements per thread and iteration: the random reads of a
// thread (gids, then the points) are all in flight together.
__global__ void gather_points_kernel(const double* __restrict__ pts, int64_t sp, int64_t sd, int d,
                                     const uint32_t* __restrict__ gids, int64_t n,
                                     double* __restrict__ X, int64_t ldx,
                                     const double* __restrict__ w_in, int wmode, void* w_out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if (d == 2 && ldx == 2 && sp == 2 && sd == 1 && wmode == GP_W_UNIT &&
      (((uintptr_t)pts | (uintptr_t)X) & 15) == 0) {
    // the common layout: one 16-byte load and store per point, eight gathers in flight
    constexpr int UA = 8;
    const double2* src = reinterpret_cast<const double2*>(pts);
    double2* dst = reinterpret_cast<double2*>(X);
    for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += UA * stride) {
      uint32_t g[UA];
#pragma unroll
      for (int u = 0; u < UA; ++u) g[u] = i0 + u * stride < n ? gids[i0 + u * stride] : 0u;
      double2 v[UA];
#pragma unroll
      for (int u = 0; u < UA; ++u) v[u] = src[g[u]];
#pragma unroll
      for (int u = 0; u < UA; ++u)
        if (i0 + u * stride < n) dst[i0 + u * stride] = v[u];
    }
    return;
  }
  constexpr int U = 4;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    int64_t g[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      g[u] = i < n ? (int64_t)gids[i] : 0;
    }
    double v[U][3];
    double wv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
#pragma unroll
      for (int j = 0; j < 3; ++j) v[u][j] = (i < n && j < d) ? pts[g[u] * sp + j * sd] : 0.0;
      wv[u] = (i < n && wmode != GP_W_UNIT) ? w_in[g[u]] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      if (i >= n) continue;
      if (d == 2 && ldx == 2) {
        reinterpret_cast<double2*>(X)[i] = make_double2(v[u][0], v[u][1]);
      } else {
        for (int j = 0; j < d; ++j) X[i * ldx + j] = v[u][j];
      }
      if (wmode == GP_W_F32) ((float*)w_out)[i] = (float)wv[u];
      else if (wmode == GP_W_F64) ((double*)w_out)[i] = wv[u];
    }
  }
}

__global__ void gather_rows_kernel(const double* __restrict__ X, int64_t ldx, int d,
                                   const int64_t* __restrict__ pos, int k, double* rows) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < k)
    for (int j = 0; j < d; ++j) rows[i * d + j] = X[pos[i] * ldx + j];
}

// ------------------------------------------------------- K5 compaction
// Ordered compaction of {i : rank[i] < size} in ONE pass (rank is read once): persistent
// CTAs take tiles of CT = 4096 consecutive entries in order from a ticket counter; a
// tile's threads count their 16 consecutive entries, a block scan orders them, the tile's
// place in the output comes from a decoupled look-back over the earlier tiles' published
// counts (one 64-bit status word per tile: flag in the top two bits), and the selected
// indices are staged in shared memory and written out as one contiguous run.
constexpr int CTH = 256;            // threads per CTA
constexpr int CPER = 16;            // consecutive entries per thread (32: 44 vs 31 ms at C5)
constexpr int CT = CTH * CPER;      // entries per tile
constexpr unsigned long long ST_AGG = 1ull << 62, ST_INC = 2ull << 62, ST_VAL = ST_AGG - 1;

__global__ void __launch_bounds__(CTH) compact_onepass(const int32_t* __restrict__ rank,
                                                       const int32_t* __restrict__ pos, int64_t n,
                                                       int64_t size, int64_t ntiles,
                                                       unsigned long long* __restrict__ ticket,
                                                       unsigned long long* __restrict__ status,
                                                       int32_t* __restrict__ idx,
                                                       int64_t* __restrict__ total) {
  __shared__ int32_t s_out[CT];
  __shared__ int s_warp[CTH / 32];
  __shared__ long long s_tile, s_base;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (;;) {
    __syncthreads();   // the previous tile's staging buffer and cursors are free
    if (tid == 0) s_tile = (long long)atomicAdd(ticket, 1ull);
    __syncthreads();
    const long long tile = s_tile;
    if (tile >= ntiles) return;
    const long long e0 = tile * CT + (long long)tid * CPER;
    // this thread's entries as a bit mask
    unsigned sel = 0;
    if (e0 + CPER <= n) {
      const int4* p = reinterpret_cast<const int4*>(rank + e0);
#pragma unroll
      for (int v = 0; v < CPER / 4; ++v) {
        const int4 r = p[v];
        sel |= (unsigned)(r.x < size) << (4 * v) | (unsigned)(r.y < size) << (4 * v + 1) |
               (unsigned)(r.z < size) << (4 * v + 2) | (unsigned)(r.w < size) << (4 * v + 3);
      }
    } else {
      for (int j = 0; j < CPER; ++j)
        if (e0 + j < n && rank[e0 + j] < size) sel |= 1u << j;
    }
    const int mine = __popc(sel);
    int incl = mine;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_warp[warp] = incl;
    __syncthreads();
    int before = incl - mine, tile_count = 0;
#pragma unroll
    for (int w2 = 0; w2 < CTH / 32; ++w2) {
      if (w2 < warp) before += s_warp[w2];
      tile_count += s_warp[w2];
    }
    // publish this tile's count, then look back for the tiles before it (warp 0)
    if (warp == 0) {
      if (lane == 0)
        atomicExch(&status[tile], (tile == 0 ? ST_INC : ST_AGG) | (unsigned long long)tile_count);
      long long base = 0;
      if (tile > 0) {
        long long t = tile - 1;
        for (;;) {
          // lanes look at 32 earlier tiles at once; the nearest inclusive prefix ends it
          const long long tt = t - lane;
          unsigned long long st = 0;
          if (tt >= 0) {
            do {
              st = atomicAdd(&status[tt], 0ull);
            } while (!(st >> 62));
          } else {
            st = ST_INC;   // before the first tile: an inclusive prefix of zero
          }
          const unsigned inc = __ballot_sync(FULL, (st >> 62) == 2);
          const int stop = inc ? __ffs(inc) - 1 : 32;   // lanes 0..stop contribute
          long long v = lane <= stop ? (long long)(st & ST_VAL) : 0;
          for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(FULL, v, o);
          base += v;
          if (inc) break;
          t -= 32;
        }
        if (lane == 0)
          atomicExch(&status[tile], ST_INC | (unsigned long long)(base + tile_count));
      }
      if (lane == 0) {
        s_base = base;
        if (tile == ntiles - 1) *total = base + tile_count;
      }
    }
    // stage the selected indices in entry order, then one contiguous copy
    int o = before;
    unsigned m = sel;
    while (m) {
      const int j = __ffs(m) - 1;
      m &= m - 1;
      s_out[o++] = pos ? pos[e0 + j] : (int32_t)(e0 + j);
    }
    __syncthreads();
    const long long base = s_base;
    for (int i = tid; i < tile_count; i += CTH) idx[base + i] = s_out[i];
  }
}

__global__ void scatter_gid_kernel(const int32_t* __restrict__ a, const uint32_t* __restrict__ g,
                                   int64_t n, int64_t* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    out[g[i]] = a[i];
}

// labels of one window of 2^DW_SHIFT consecutive ids: the window's pairs (grouped by the
// radix passes on the high id bits) are placed by id in shared memory, then written out
constexpr int DW_SHIFT = 14, DW = 1 << DW_SHIFT;
__global__ void __launch_bounds__(512) deliver_window_kernel(const uint32_t* __restrict__ g,
                                                             const int32_t* __restrict__ a,
                                                             int64_t n, int64_t* __restrict__ out) {
  extern __shared__ int32_t s_lab[];
  const int64_t w0 = (int64_t)blockIdx.x << DW_SHIFT;
  const int cnt = (int)(n - w0 < DW ? n - w0 : DW);
  for (int i = threadIdx.x; i < cnt; i += blockDim.x)
    s_lab[g[w0 + i] & (DW - 1)] = a[w0 + i];
  __syncthreads();
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) out[w0 + i] = s_lab[i];
}

__global__ void gather_ranks_kernel(const int32_t* __restrict__ r, const uint32_t* __restrict__ g,
                                    int64_t n, int32_t* __restrict__ out) {
  constexpr int U = 8;   // random 4-byte gathers in flight per thread
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i0 = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i0 < n; i0 += U * stride) {
    uint32_t gg[U];
#pragma unroll
    for (int u = 0; u < U; ++u) gg[u] = i0 + u * stride < n ? g[i0 + u * stride] : 0u;
    int32_t v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = i0 + u * stride < n ? r[gg[u]] : 0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (i0 + u * stride < n) out[i0 + u * stride] = v[u];
  }
}

__global__ void gather_state_kernel(const int32_t* __restrict__ list, int64_t m, int d,
                                    const int32_t* __restrict__ a, const uint32_t* __restrict__ ublb,
                                    const double* __restrict__ X, const uint8_t* __restrict__ w,
                                    int wbytes, int32_t* __restrict__ a_out,
                                    uint32_t* __restrict__ ublb_out, double* __restrict__ X_out,
                                    uint8_t* __restrict__ w_out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = list[i];
    a_out[i] = a[q];
    ublb_out[i] = ublb[q];
    for (int j = 0; j < d; ++j) X_out[i * d + j] = X[q * d + j];
    if (wbytes == 4) reinterpret_cast<float*>(w_out)[i] = reinterpret_cast<const float*>(w)[q];
    else if (wbytes == 8)
      reinterpret_cast<double*>(w_out)[i] = reinterpret_cast<const double*>(w)[q];
  }
}

__global__ void scatter_state_kernel(const int32_t* __restrict__ list, int64_t m,
                                     const int32_t* __restrict__ a_dense,
                                     const uint32_t* __restrict__ ublb_dense, int32_t* __restrict__ a,
                                     uint32_t* __restrict__ ublb) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t q = list[i];
    a[q] = a_dense[i];
    ublb[q] = ublb_dense[i];
  }
}

static unsigned stride_grid(int64_t n) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t want = (n + 255) / 256;
  int64_t cap = (int64_t)sms * 8;
  return (unsigned)(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace gp

using namespace gp;

extern "C" {

const char* gp_last_error(void) { return g_err; }
int gp_abi_version(void) { return 2; }
int gp_host_is_pinned(const void* p) {
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return at.type == cudaMemoryTypeHost ? 1 : 0;
}
void gp_args_sizes(size_t* a, size_t* f) {
  *a = sizeof(gp_assign_args);
  *f = sizeof(gp_fold_args);
}

int gp_box_minmax(const double* pts, int64_t n, int d, int64_t stride_pt, int64_t stride_dim,
                  double* lohi, int32_t* nonfinite, void* stream) {
  GP_REQUIRE(n >= 1, "gp_box_minmax: n must be >= 1");
  GP_REQUIRE(d == 2 || d == 3, "gp_box_minmax: d must be 2 or 3");
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long* keys = reinterpret_cast<unsigned long long*>(lohi);
  GP_CUDA(cudaMemsetAsync(keys, 0xff, d * sizeof(double), s));
  GP_CUDA(cudaMemsetAsync(keys + d, 0x00, d * sizeof(double), s));
  GP_CUDA(cudaMemsetAsync(nonfinite, 0, sizeof(int32_t), s));
  if (d == 2 && stride_pt == 2 && stride_dim == 1 && ((uintptr_t)pts & 15) == 0) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t want = (n + 1023) / 1024;
    box_kernel_aos2<<<(unsigned)(want < sms * 8 ? want : sms * 8), 256, 0, s>>>(
        (const double2*)pts, n, keys, nonfinite);
  } else {
    box_kernel<<<stride_grid(n), 256, 0, s>>>(pts, n, d, stride_pt, stride_dim, keys, nonfinite);
  }
  box_finalize<<<1, 32, 0, s>>>(keys, d);
  return check_launch("box");
}

int gp_weight_probe(const double* w, int64_t n, int64_t* out, void* stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int64_t init[3] = {0, 4096, 0};
  GP_CUDA(cudaMemcpyAsync(out, init, sizeof(init), cudaMemcpyHostToDevice, s));
  if (n > 0)
    weight_probe_kernel<<<stride_grid(n), 256, 0, s>>>(w, n, (unsigned long long*)out);
  return check_launch("weight_probe");
}

// build the tables for dimension d and check them against the transpose on random
// cells at every depth (host only)
static uint64_t fsm_key(const HFsm& T, int d, int depth, const uint32_t* X) {
  uint64_t key = 0;
  int st = 0, b = depth - 1;
  const int L = T.L;
  for (; b + 1 >= L; b -= L) {
    int ch = 0;
    for (int j = 0; j < d; ++j) ch |= (int)((X[j] >> (b + 1 - L)) & ((1u << L) - 1)) << (j * L);
    const unsigned e = T.multi[st * 256 + ch];
    key = (key << (d * L)) | (e & ((1u << (d * L)) - 1));
    st = (int)(e >> (d * L));
  }
  for (; b >= 0; --b) {
    int r = 0;
    for (int j = 0; j < d; ++j) r |= (int)((X[j] >> b) & 1u) << j;
    const unsigned e = T.single[st * 8 + r];
    key = (key << d) | (e & ((1u << d) - 1));
    st = (int)(e >> d);
  }
  return key;
}

static int hilbert_fsm_checked(int d, HFsm& T) {
  hilbert_fsm_tables(d, T);
  GP_REQUIRE(T.states <= (d == 2 ? 16 : 96), "hilbert tables: unexpected state count");
  uint64_t rs = 0x243F6A8885A308D3ull;
  for (int dep = 1; d * dep <= 62; ++dep)
    for (int trial = 0; trial < 512; ++trial) {
      uint32_t c[3];
      for (int j = 0; j < d; ++j) {
        rs = rs * 6364136223846793005ull + 1442695040888963407ull;
        c[j] = (uint32_t)(rs >> 33) & (uint32_t)((1ull << dep) - 1);
      }
      const uint64_t want = gp_hilbert_cell_key_host(c, d, dep);
      GP_REQUIRE(fsm_key(T, d, dep, c) == want,
                 "hilbert tables disagree with the transpose (d=%d depth=%d)", d, dep);
    }
  return GP_OK;
}

int gp_hilbert_fsm_selfcheck(int d) {
  GP_REQUIRE(d == 2 || d == 3, "gp_hilbert_fsm_selfcheck: d must be 2 or 3");
  static HFsm T;
  return hilbert_fsm_checked(d, T);
}

int gp_hilbert_keys(const double* pts, int64_t n, int d, int64_t stride_pt, int64_t stride_dim,
                    const double* lohi, int depth, uint64_t* keys, uint32_t* gids,
                    uint32_t gid_base, void* stream) {
  GP_REQUIRE(d == 2 || d == 3, "gp_hilbert_keys: unsupported dimension %d", d);
  GP_REQUIRE(depth >= 1 && d * depth <= 62, "gp_hilbert_keys: depth %d out of range for d=%d",
             depth, d);
  if (n == 0) return GP_OK;
  static bool tables = false;
  if (!tables) {
    for (int dd = 2; dd <= 3; ++dd) {
      static HFsm T;
      int rc = hilbert_fsm_checked(dd, T);
      if (rc) return rc;
      GP_CUDA(cudaMemcpyToSymbol(g_hfsm, &T, sizeof(HFsm), (dd - 2) * sizeof(HFsm)));
    }
    tables = true;
  }
  cudaStream_t s = (cudaStream_t)stream;
  if (d == 2)
    hilbert_kernel<2><<<stride_grid(n), 256, 0, s>>>(pts, n, stride_pt, stride_dim, lohi, depth,
                                                     keys, gids, gid_base);
  else
    hilbert_kernel<3><<<stride_grid(n), 256, 0, s>>>(pts, n, stride_pt, stride_dim, lohi, depth,
                                                     keys, gids, gid_base);
  return check_launch("hilbert_keys");
}

uint64_t gp_hilbert_cell_key_host(const uint32_t* cells, int d, int depth) {
  uint32_t X[3] = {cells[0], cells[1], d == 3 ? cells[2] : 0u};
  if (d == 2) hilbert_transpose<2>(X, depth);
  else hilbert_transpose<3>(X, depth);
  uint64_t key = 0;
  for (int j = depth - 1; j >= 0; --j)
    for (int i = 0; i < d; ++i) key = (key << 1) | ((X[i] >> j) & 1u);
  return key;
}

int gp_sort_workspace_bytes(int64_t n, size_t* bytes) {
  GP_REQUIRE(n >= 0 && n < (1ll << 31), "gp_sort: n out of range");
  *bytes = radix::workspace_bytes(n, 8, 4);
  return GP_OK;
}

int gp_sort_pairs(const uint64_t* keys_in, const uint32_t* vals_in, uint64_t* keys_out,
                  uint32_t* vals_out, int64_t n, int key_bits, void* workspace,
                  size_t workspace_bytes, void* stream) {
  GP_REQUIRE(key_bits >= 1 && key_bits <= 64, "gp_sort: key_bits out of range");
  return radix::sort_pairs<uint64_t, uint32_t>(keys_in, vals_in, keys_out, vals_out, n, 0,
                                               key_bits, workspace, workspace_bytes,
                                               (cudaStream_t)stream, true);
}

int gp_gather_points(const double* pts, int64_t stride_pt, int64_t stride_dim, int d,
                     const uint32_t* gids, int64_t n, double* X, int64_t ldx, const double* w_in,
                     int wmode, void* w_out, void* stream) {
  GP_REQUIRE(d == 2 || d == 3, "gp_gather_points: bad d");
  GP_REQUIRE(wmode == GP_W_UNIT || (w_in && w_out), "gp_gather_points: weights missing");
  if (n == 0) return GP_OK;
  gather_points_kernel<<<stride_grid(n), 256, 0, (cudaStream_t)stream>>>(
      pts, stride_pt, stride_dim, d, gids, n, X, ldx, w_in, wmode, w_out);
  return check_launch("gather_points");
}

int gp_gather_rows(const double* X, int64_t ldx, int d, const int64_t* positions, int k,
                   double* rows, void* stream) {
  GP_REQUIRE(k >= 1, "gp_gather_rows: k must be >= 1");
  gather_rows_kernel<<<grid_for(k, 256), 256, 0, (cudaStream_t)stream>>>(X, ldx, d, positions, k,
                                                                          rows);
  return check_launch("gather_rows");
}

int gp_compact_workspace_bytes(int64_t n, size_t* bytes) {
  const int64_t nt = (n + CT - 1) / CT;
  *bytes = 256 + ((size_t)(nt + 1) * sizeof(unsigned long long) + 255) / 256 * 256;
  return GP_OK;
}

int gp_compact_active(const int32_t* rank, int64_t n, int64_t size, int32_t* idx, int64_t* count,
                      void* workspace, size_t workspace_bytes, void* stream) {
  return gp_compact_candidates(rank, nullptr, n, size, idx, count, workspace, workspace_bytes,
                               stream);
}

int gp_compact_candidates(const int32_t* rank, const int32_t* positions, int64_t n, int64_t size,
                          int32_t* idx, int64_t* count, void* workspace, size_t workspace_bytes,
                          void* stream) {
  size_t need = 0;
  gp_compact_workspace_bytes(n, &need);
  GP_REQUIRE(workspace_bytes >= need, "gp_compact_active: workspace too small");
  GP_REQUIRE(((uintptr_t)rank & 15) == 0, "gp_compact_active: rank must be 16-byte aligned");
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) {
    GP_CUDA(cudaMemsetAsync(count, 0, sizeof(int64_t), s));
    return GP_OK;
  }
  const int64_t nt = (n + CT - 1) / CT;
  GP_CUDA(cudaMemsetAsync(workspace, 0, need, s));   // ticket and every tile's status
  unsigned long long* ticket = (unsigned long long*)workspace;
  unsigned long long* status = (unsigned long long*)((char*)workspace + 256);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t cap = (int64_t)sms * 6;
  compact_onepass<<<(unsigned)(nt < cap ? nt : cap), CTH, 0, s>>>(rank, positions, n, size, nt,
                                                                 ticket, status, idx, count);
  return check_launch("compact_active");
}

int gp_gather_state(const int32_t* list, int64_t m, int d, const int32_t* a, const void* ublb,
                    const double* X, const void* w, int wbytes, int32_t* a_out, void* ublb_out,
                    double* X_out, void* w_out, void* stream) {
  GP_REQUIRE(d == 2 || d == 3, "gp_gather_state: bad d");
  GP_REQUIRE(wbytes == 0 || wbytes == 4 || wbytes == 8, "gp_gather_state: bad wbytes");
  if (m == 0) return GP_OK;
  gather_state_kernel<<<stride_grid(m), 256, 0, (cudaStream_t)stream>>>(
      list, m, d, a, (const uint32_t*)ublb, X, (const uint8_t*)w, wbytes, a_out, (uint32_t*)ublb_out,
      X_out, (uint8_t*)w_out);
  return check_launch("gather_state");
}

int gp_scatter_state(const int32_t* list, int64_t m, const int32_t* a_dense,
                     const void* ublb_dense, int32_t* a, void* ublb, void* stream) {
  if (m == 0) return GP_OK;
  scatter_state_kernel<<<stride_grid(m), 256, 0, (cudaStream_t)stream>>>(
      list, m, a_dense, (const uint32_t*)ublb_dense, a, (uint32_t*)ublb);
  return check_launch("scatter_state");
}

int gp_scatter_by_gid(const int32_t* a, const uint32_t* gids, int64_t n, int64_t* out,
                      void* stream) {
  if (n == 0) return GP_OK;
  scatter_gid_kernel<<<stride_grid(n), 256, 0, (cudaStream_t)stream>>>(a, gids, n, out);
  return check_launch("scatter_by_gid");
}

int gp_deliver_workspace_bytes(int64_t n, size_t* bytes) {
  GP_REQUIRE(n >= 0 && n < (1ll << 31), "gp_deliver: n out of range");
  *bytes = 2 * (((size_t)n * 4 + 255) & ~(size_t)255) + radix::workspace_bytes(n, 4, 4);
  return GP_OK;
}

int gp_deliver_permutation(const int32_t* a, const uint32_t* gids, int64_t n, int64_t* out,
                           void* workspace, size_t workspace_bytes, void* stream) {
  if (n == 0) return GP_OK;
  int bits = 1;
  while (bits < 32 && ((uint64_t)(n - 1) >> bits) != 0) ++bits;
  if (bits <= DW_SHIFT)   // one window: the plain scatter stays inside shared-memory reach
    return gp_scatter_by_gid(a, gids, n, out, stream);
  size_t need = 0;
  gp_deliver_workspace_bytes(n, &need);
  GP_REQUIRE(workspace_bytes >= need, "gp_deliver_permutation: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t arr = ((size_t)n * 4 + 255) & ~(size_t)255;
  uint32_t* gs = (uint32_t*)workspace;
  int32_t* as = (int32_t*)((char*)workspace + arr);
  void* rws = (char*)workspace + 2 * arr;
  int rc = radix::sort_pairs<uint32_t, int32_t>(gids, a, gs, as, n, DW_SHIFT, bits, rws,
                                                workspace_bytes - 2 * arr, s, false);
  if (rc) return rc;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(deliver_window_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         DW * (int)sizeof(int32_t));
    attr = true;
  }
  const int64_t nw = (n + DW - 1) >> DW_SHIFT;
  deliver_window_kernel<<<(unsigned)nw, 512, DW * sizeof(int32_t), s>>>(gs, as, n, out);
  return check_launch("deliver_permutation");
}

int gp_gather_ranks(const int32_t* rank_by_gid, const uint32_t* gids, int64_t n, int32_t* out,
                    void* stream) {
  if (n == 0) return GP_OK;
  gather_ranks_kernel<<<stride_grid(n), 256, 0, (cudaStream_t)stream>>>(rank_by_gid, gids, n,
                                                                        out);
  return check_launch("gather_ranks");
}

}  // extern "C"

// ------------------------------------------------ center grid (scan overflow, walk)
namespace gp {

template <int D>
__global__ void center_cells_kernel(const double* __restrict__ centers, int k, double lo0,
                                    double lo1, double lo2, double h, int G,
                                    uint64_t* __restrict__ keys, uint32_t* __restrict__ vals) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= k) return;
  const double lo[3] = {lo0, lo1, lo2};
  uint64_t flat = 0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    // np.clip(np.floor((centers - lo) / h), 0, G - 1)
    double f = floor(__ddiv_rn(__dsub_rn(centers[c * D + j], lo[j]), h));
    f = fmin(fmax(f, 0.0), (double)(G - 1));
    flat = flat * (uint64_t)G + (uint64_t)f;
  }
  keys[c] = flat;
  vals[c] = (uint32_t)c;
}

// start[cell] = first sorted position with key >= cell (lower bound), start[G^d] = k
__global__ void cell_starts_kernel(const uint64_t* __restrict__ skeys, int k, int64_t ncell,
                                   int32_t* __restrict__ start) {
  const int64_t cell = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (cell > ncell) return;
  int lo = 0, hi = k;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (skeys[mid] < (uint64_t)cell) lo = mid + 1;
    else hi = mid;
  }
  start[cell] = lo;
}

}  // namespace gp

extern "C" int gp_center_grid_workspace_bytes(int k, size_t* bytes) {
  GP_REQUIRE(k >= 1, "gp_center_grid: k must be >= 1");
  const size_t b = gp::radix::workspace_bytes(k, 8, 4);
  *bytes = 2 * (size_t)k * (sizeof(uint64_t) + sizeof(uint32_t)) + ((b + 255) & ~(size_t)255) + 256;
  return GP_OK;
}

extern "C" int gp_center_grid(const double* centers, int k, int d, const double* lo, double h,
                              int G, int32_t* start, int32_t* items, void* workspace,
                              size_t workspace_bytes, void* stream) {
  GP_REQUIRE(d == 2 || d == 3, "gp_center_grid: bad d");
  GP_REQUIRE(k >= 1 && G >= 1 && h > 0.0, "gp_center_grid: bad sizes");
  size_t need = 0;
  int rc = gp_center_grid_workspace_bytes(k, &need);
  if (rc) return rc;
  GP_REQUIRE(workspace_bytes >= need, "gp_center_grid: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  uint64_t* kin = (uint64_t*)ws;
  uint64_t* kout = kin + k;
  uint32_t* vin = (uint32_t*)(kout + k);
  uint32_t* vout = vin + k;
  void* tmp = (void*)(((uintptr_t)(vout + k) + 255) & ~(uintptr_t)255);
  size_t tb = workspace_bytes - ((char*)tmp - ws);
  int64_t ncell = 1;
  for (int j = 0; j < d; ++j) ncell *= G;
  int bits = 1;
  while (bits < 64 && (1ull << bits) <= (unsigned long long)ncell) ++bits;
  if (d == 2)
    gp::center_cells_kernel<2><<<(k + 255) / 256, 256, 0, s>>>(centers, k, lo[0], lo[1], 0.0, h,
                                                                G, kin, vin);
  else
    gp::center_cells_kernel<3><<<(k + 255) / 256, 256, 0, s>>>(centers, k, lo[0], lo[1], lo[2],
                                                                h, G, kin, vin);
  rc = gp::radix::sort_pairs<uint64_t, uint32_t>(kin, vin, kout, (uint32_t*)items, k, 0, bits, tmp,
                                                 tb, s, false);
  if (rc) return rc;
  gp::cell_starts_kernel<<<(unsigned)((ncell + 1 + 255) / 256), 256, 0, s>>>(kout, k, ncell,
                                                                             start);
  return gp::check_launch("center_grid");
}
