// K6 assign round, K8 audit, bound rebase.
//
// One CTA owns a tile of TILE consecutive active entries (SFC order, so the
// tile is spatially compact).  Per tile:
//   1. skip test per entry with the lazily relaxed Hamerly bounds
//      (reference: kmeans.py:308-311 with relax_bounds kmeans.py:208-239
//      applied through cumulative affine maps);
//   2. box of the entries that must be scanned (kmeans.py:315-316, but per
//      tile instead of per rank);
//   3. candidate centers: every center whose box lower bound does not exceed
//      the second smallest box upper bound (a sound superset of every
//      scanned point's best and second-best center);
//   4. exact scan of the candidates with the reference's arithmetic and
//      (dist, index) lexicographic tie-break (kmeans.py:326-344);
//   5. exact int64 block weights (kmeans.py:368-374) and counters.
#include "common.cuh"

namespace gp {

constexpr int AT = 256;          // threads per CTA
constexpr int PPT = 4;           // max entries per thread (runtime ppt in {1,2,4})
constexpr int TILE_MAX = AT * PPT;
constexpr int CAP = 512;         // candidate centers staged in shared memory
constexpr int HSLOTS = 128;      // per-CTA block-weight cache
constexpr double LO_SLACK = 1.0 - 1e-12;
constexpr double HI_SLACK = 1.0 + 1e-12;
constexpr double Q_TOL = 1e-13;  // prefilter tolerance (>> the q rounding error)

__device__ __forceinline__ void two_min_merge(double& m1, double& m2, double b1, double b2) {
  double lo = fmin(m1, b1);
  double hi = fmin(fmax(m1, b1), fmin(m2, b2));
  m1 = lo;
  m2 = hi;
}

// Rigorous bounds of the effective distance from any point of the box to c:
// lbnd <= effdist <= ubnd (directed rounding plus 1e-12 slack).
template <int D>
__device__ __forceinline__ void box_bounds(const double* c, const double* lo, const double* hi,
                                           double infl, double& lbnd, double& ubnd) {
  double sl = 0.0, su = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double dl = 0.0;
    if (c[j] < lo[j]) dl = __dsub_rd(lo[j], c[j]);
    else if (c[j] > hi[j]) dl = __dsub_rd(c[j], hi[j]);
    sl = __dadd_rd(sl, __dmul_rd(dl, dl));
    double du = fmax(__dsub_ru(c[j], lo[j]), __dsub_ru(hi[j], c[j]));
    su = __dadd_ru(su, __dmul_ru(du, du));
  }
  lbnd = __dmul_rd(__ddiv_rd(__dsqrt_rd(sl), infl), LO_SLACK);
  ubnd = __dmul_ru(__ddiv_ru(__dsqrt_ru(su), infl), HI_SLACK);
}

__device__ __forceinline__ void cache_add(int* ckey, long long* cval, long long* global, int a,
                                          long long v) {
  int slot = a & (HSLOTS - 1);
  int old = atomicCAS(&ckey[slot], -1, a);
  if (old == -1 || old == a) atomicAdd((unsigned long long*)&cval[slot], (unsigned long long)v);
  else atomicAdd((unsigned long long*)&global[a], (unsigned long long)v);
}

template <int D>
struct ScanSmem {
  double c[D][CAP];
  double inf[CAP];
  double i2[CAP];     // 1 / infl^2 for the prefilter
  int cid[CAP];
};

template <int D>
__device__ __forceinline__ void stage_center(ScanSmem<D>& S, int slot, int c, const double* cen,
                                             const double* infl) {
#pragma unroll
  for (int j = 0; j < D; ++j) S.c[j][slot] = cen[c * D + j];
  double I = infl[c];
  S.inf[slot] = I;
  S.i2[slot] = 1.0 / (I * I);
  S.cid[slot] = c;
}

// squared distance / infl^2 (prefilter only; any rounding)
template <int D>
__device__ __forceinline__ double qdist(const double* x, const ScanSmem<D>& S, int i) {
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double t = x[j] - S.c[j][i];
    s = fma(t, t, s);
  }
  return s * S.i2[i];
}

template <int D>
__global__ void __launch_bounds__(AT, 2) assign_kernel(gp_assign_args p, int ppt) {
  __shared__ ScanSmem<D> S;
  __shared__ int s_pos[TILE_MAX];     // positions that need a scan
  __shared__ short s_ent[TILE_MAX];   // their tile-local entry ids
  __shared__ int s_newa[TILE_MAX];
  __shared__ unsigned s_scanned[TILE_MAX / 32];
  __shared__ int s_ckey[HSLOTS];
  __shared__ long long s_cval[HSLOTS];
  __shared__ double s_red[2 * D][AT / 32];
  __shared__ double s_two[2][AT / 32];
  __shared__ int s_nscan, s_ncand;
  __shared__ unsigned long long s_cnt[3];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tile = AT * ppt;
  const int64_t base = (int64_t)blockIdx.x * tile;
  if (tid == 0) {
    s_nscan = 0;
    s_ncand = 0;
    s_cnt[0] = s_cnt[1] = s_cnt[2] = 0;
  }
  for (int i = tid; i < HSLOTS; i += AT) {
    s_ckey[i] = -1;
    s_cval[i] = 0;
  }
  for (int i = tid; i < TILE_MAX / 32; i += AT) s_scanned[i] = 0;
  __syncthreads();

  // ---- 1. skip test with the lazily relaxed bounds (kmeans.py:308-311)
  int pos[PPT], cur[PPT];
  double wv[PPT];
  int nskip = 0, ndec = 0;
#pragma unroll
  for (int e = 0; e < PPT; ++e) {
    pos[e] = -1;
    cur[e] = -1;
    wv[e] = 0.0;
    int ent = e * AT + tid;
    int64_t li = base + ent;
    if (e < ppt && li < p.m) {
      int q = p.list ? p.list[li] : (int)li;
      pos[e] = q;
      int a = p.a[q];
      cur[e] = a;
      wv[e] = load_weight(p.w, p.wmode, q);
      ++ndec;
      bool skip = false;
      if (a >= 0) {
        double ub = ub_eval(p.ub_scale[a], p.ub[q], p.ub_shift[a], p.bound_err);
        double lb = lb_eval(p.lb_scale, p.lb[q], p.lb_shift, p.bound_err);
        skip = ub < lb;
      }
      if (skip) {
        ++nskip;
      } else {
        int slot = atomicAdd(&s_nscan, 1);
        s_pos[slot] = q;
        s_ent[slot] = (short)ent;
        atomicOr(&s_scanned[ent >> 5], 1u << (ent & 31));
      }
    }
  }
  __syncthreads();
  const int nscan = s_nscan;
  unsigned long long nevals = 0;

  if (nscan > 0) {
    // candidate source: the group's hierarchical list, or all k centers
    const int32_t* src = nullptr;
    int nsrc = p.k;
    if (p.group_list) {
      int64_t g = base >> p.group_shift;
      int cnt = p.group_count[g];
      if (cnt >= 0) {
        src = p.group_list + g * (int64_t)p.group_cap;
        nsrc = cnt;
      }
    }
    // ---- 2. box of the scanned points (kmeans.py:315-316, per tile)
    double lo[D], hi[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      lo[j] = INFINITY;
      hi[j] = -INFINITY;
    }
    for (int s = tid; s < nscan; s += AT) {
      int q = s_pos[s];
#pragma unroll
      for (int j = 0; j < D; ++j) {
        double v = p.X[j * p.ldx + q];
        lo[j] = fmin(lo[j], v);
        hi[j] = fmax(hi[j], v);
      }
    }
#pragma unroll
    for (int j = 0; j < D; ++j) {
      for (int o = 16; o; o >>= 1) {
        lo[j] = fmin(lo[j], __shfl_xor_sync(FULL, lo[j], o));
        hi[j] = fmax(hi[j], __shfl_xor_sync(FULL, hi[j], o));
      }
      if (lane == 0) {
        s_red[j][warp] = lo[j];
        s_red[D + j][warp] = hi[j];
      }
    }
    __syncthreads();
#pragma unroll
    for (int j = 0; j < D; ++j) {
      lo[j] = s_red[j][0];
      hi[j] = s_red[D + j][0];
      for (int w = 1; w < AT / 32; ++w) {
        lo[j] = fmin(lo[j], s_red[j][w]);
        hi[j] = fmax(hi[j], s_red[D + j][w]);
      }
    }

    // ---- 3. candidates: lbnd <= second smallest ubnd over the source
    double m1 = INFINITY, m2 = INFINITY;
    for (int i = tid; i < nsrc; i += AT) {
      int c = src ? src[i] : i;
      double cc[D];
#pragma unroll
      for (int j = 0; j < D; ++j) cc[j] = p.centers[c * D + j];
      double lb_, ub_;
      box_bounds<D>(cc, lo, hi, p.infl[c], lb_, ub_);
      two_min_merge(m1, m2, ub_, INFINITY);
    }
    for (int o = 16; o; o >>= 1) {
      double b1 = __shfl_xor_sync(FULL, m1, o);
      double b2 = __shfl_xor_sync(FULL, m2, o);
      two_min_merge(m1, m2, b1, b2);
    }
    if (lane == 0) {
      s_two[0][warp] = m1;
      s_two[1][warp] = m2;
    }
    __syncthreads();
    m1 = s_two[0][0];
    m2 = s_two[1][0];
    for (int w = 1; w < AT / 32; ++w) two_min_merge(m1, m2, s_two[0][w], s_two[1][w]);
    const double U = m2;  // +inf when only one center exists
    for (int i = tid; i < nsrc; i += AT) {
      int c = src ? src[i] : i;
      double cc[D];
#pragma unroll
      for (int j = 0; j < D; ++j) cc[j] = p.centers[c * D + j];
      double lb_, ub_;
      box_bounds<D>(cc, lo, hi, p.infl[c], lb_, ub_);
      if (lb_ <= U) {
        int slot = atomicAdd(&s_ncand, 1);
        if (slot < CAP) stage_center<D>(S, slot, c, p.centers, p.infl);
      }
    }
    __syncthreads();
    const int ncand = s_ncand;
    const bool overflow = ncand > CAP;   // then stream the whole source in chunks
    const int total = overflow ? nsrc : ncand;

    // ---- 4. scan (kmeans.py:326-344) with an approximate prefilter:
    // pass 1 finds the two smallest q = d^2/infl^2; pass 2 evaluates the
    // reference's exact effective distance only where q <= q2 (1 + Q_TOL),
    // a superset of every center whose exact distance is <= the exact runner-up.
    double x[PPT][D], q1[PPT], q2[PPT];
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
      int s = tid + r * AT;
      q1[r] = INFINITY;
      q2[r] = INFINITY;
      if (r < ppt && s < nscan) {
        int q = s_pos[s];
#pragma unroll
        for (int j = 0; j < D; ++j) x[r][j] = p.X[j * p.ldx + q];
      }
    }
    for (int c0 = 0; c0 < total; c0 += CAP) {
      const int cn = min(CAP, total - c0);
      if (overflow) {
        __syncthreads();
        for (int i = tid; i < cn; i += AT) {
          int c = src ? src[c0 + i] : c0 + i;
          stage_center<D>(S, i, c, p.centers, p.infl);
        }
        __syncthreads();
      }
#pragma unroll
      for (int r = 0; r < PPT; ++r) {
        if (r < ppt && tid + r * AT < nscan) {
          double a1 = q1[r], a2 = q2[r];
          int i = 0;
          for (; i + 4 <= cn; i += 4) {
            double t0 = qdist<D>(x[r], S, i), t1 = qdist<D>(x[r], S, i + 1);
            double t2 = qdist<D>(x[r], S, i + 2), t3 = qdist<D>(x[r], S, i + 3);
            a2 = fmin(a2, fmax(a1, t0)); a1 = fmin(a1, t0);
            a2 = fmin(a2, fmax(a1, t1)); a1 = fmin(a1, t1);
            a2 = fmin(a2, fmax(a1, t2)); a1 = fmin(a1, t2);
            a2 = fmin(a2, fmax(a1, t3)); a1 = fmin(a1, t3);
          }
          for (; i < cn; ++i) {
            double t = qdist<D>(x[r], S, i);
            a2 = fmin(a2, fmax(a1, t));
            a1 = fmin(a1, t);
          }
          q1[r] = a1;
          q2[r] = a2;
        }
      }
    }
    double best[PPT], second[PPT], thr[PPT];
    int bi[PPT];
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
      best[r] = INFINITY;
      second[r] = INFINITY;
      bi[r] = 0x7fffffff;
      thr[r] = fma(q2[r], Q_TOL, q2[r]);
    }
    for (int c0 = 0; c0 < total; c0 += CAP) {
      const int cn = min(CAP, total - c0);
      if (overflow) {
        __syncthreads();
        for (int i = tid; i < cn; i += AT) {
          int c = src ? src[c0 + i] : c0 + i;
          stage_center<D>(S, i, c, p.centers, p.infl);
        }
        __syncthreads();
      }
#pragma unroll
      for (int r = 0; r < PPT; ++r) {
        if (r < ppt && tid + r * AT < nscan) {
          for (int i = 0; i < cn; ++i) {
            if (qdist<D>(x[r], S, i) <= thr[r]) {
              double cc[D];
#pragma unroll
              for (int j = 0; j < D; ++j) cc[j] = S.c[j][i];
              double dist = effdist_rn<D>(x[r], cc, S.inf[i], p.order3);
              int cid = S.cid[i];
              bool win = dist < best[r] || (dist == best[r] && cid < bi[r]);
              second[r] = win ? best[r] : fmin(second[r], dist);
              best[r] = win ? dist : best[r];
              bi[r] = win ? cid : bi[r];
              ++nevals;
            }
          }
        }
      }
    }
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
      int s = tid + r * AT;
      if (r < ppt && s < nscan) {
        int q = s_pos[s];
        int c = bi[r];
        p.a[q] = c;
        p.ub[q] = __ddiv_ru(__dsub_ru(best[r], p.ub_shift[c]), p.ub_scale[c]);
        p.lb[q] = __ddiv_rd(__dadd_rd(second[r], p.lb_shift), p.lb_scale);
        s_newa[s_ent[s]] = c;
      }
    }
  }
  __syncthreads();

  // ---- 5. block weights (exact int64, kmeans.py:368-374) + counters
#pragma unroll
  for (int e = 0; e < PPT; ++e) {
    if (e >= ppt) break;
    int ent = e * AT + tid;
    int a = cur[e];
    if (pos[e] >= 0 && ((s_scanned[ent >> 5] >> (ent & 31)) & 1u)) a = s_newa[ent];
    bool valid = pos[e] >= 0 && a >= 0;
    long long v = valid ? (long long)(wv[e] * p.wscale) : 0;
    unsigned grp = __match_any_sync(FULL, valid ? a : -1);
    if (grp == FULL) {
      // SFC order makes whole-warp groups the common case: one smem atomic per warp
      long long gsum = v;
      for (int o = 16; o; o >>= 1) gsum += __shfl_xor_sync(FULL, gsum, o);
      if (lane == 0 && valid) cache_add(s_ckey, s_cval, p.block_w, a, gsum);
    } else if (valid) {
      cache_add(s_ckey, s_cval, p.block_w, a, v);
    }
  }
  unsigned long long c0 = nskip, c1 = ndec, c2 = nevals;
  for (int o = 16; o; o >>= 1) {
    c0 += __shfl_xor_sync(FULL, c0, o);
    c1 += __shfl_xor_sync(FULL, c1, o);
    c2 += __shfl_xor_sync(FULL, c2, o);
  }
  if (lane == 0) {
    atomicAdd(&s_cnt[0], c0);
    atomicAdd(&s_cnt[1], c1);
    atomicAdd(&s_cnt[2], c2);
  }
  __syncthreads();
  for (int i = tid; i < HSLOTS; i += AT)
    if (s_ckey[i] >= 0 && s_cval[i] != 0)
      atomicAdd((unsigned long long*)&p.block_w[s_ckey[i]], (unsigned long long)s_cval[i]);
  if (tid < 3 && s_cnt[tid]) atomicAdd(&p.counters[tid], s_cnt[tid]);
}

// ------------------------------------------------------------------ audit
template <int D>
__global__ void audit_kernel(gp_assign_args p, unsigned long long* out) {
  unsigned long long aud = 0, viol = 0, bad = 0;
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < p.m;
       li += (int64_t)gridDim.x * blockDim.x) {
    int q = p.list ? p.list[li] : (int)li;
    double x[D];
#pragma unroll
    for (int j = 0; j < D; ++j) x[j] = p.X[j * p.ldx + q];
    int a = p.a[q];
    double m1 = INFINITY, m2 = INFINITY, own = 0.0;
    int arg = 0;
    for (int c = 0; c < p.k; ++c) {
      double cc[D];
#pragma unroll
      for (int j = 0; j < D; ++j) cc[j] = p.centers[c * D + j];
      double dist = effdist_rn<D>(x, cc, p.infl[c], p.order3);
      if (c == (a >= 0 ? a : 0)) own = dist;
      if (dist < m1) {
        m2 = m1;
        m1 = dist;
        arg = c;
      } else {
        m2 = fmin(m2, dist);
      }
    }
    double ub = a >= 0 ? ub_eval(p.ub_scale[a], p.ub[q], p.ub_shift[a], p.bound_err) : INFINITY;
    double lb = lb_eval(p.lb_scale, p.lb[q], p.lb_shift, p.bound_err);
    ++aud;
    if (a >= 0 && ub < own) ++viol;
    if (p.k > 1 && lb > m2) ++viol;
    if (a >= 0 && ub < lb && arg != a) ++bad;
  }
  atomicAdd(&out[0], aud);
  atomicAdd(&out[1], viol);
  atomicAdd(&out[2], bad);
}

__global__ void rebase_kernel(gp_assign_args p) {
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < p.m;
       li += (int64_t)gridDim.x * blockDim.x) {
    int q = p.list ? p.list[li] : (int)li;
    int a = p.a[q];
    if (a >= 0) p.ub[q] = ub_eval(p.ub_scale[a], p.ub[q], p.ub_shift[a], p.bound_err);
    p.lb[q] = lb_eval(p.lb_scale, p.lb[q], p.lb_shift, p.bound_err);
  }
}

static int validate(const gp_assign_args* a) {
  GP_REQUIRE(a != nullptr, "null args");
  GP_REQUIRE(a->d == 2 || a->d == 3, "d must be 2 or 3");
  GP_REQUIRE(a->k >= 1, "k must be >= 1");
  GP_REQUIRE(a->m >= 0 && a->m < (1ll << 31), "m out of range");
  GP_REQUIRE(a->wmode == GP_W_UNIT || a->w != nullptr, "weights missing");
  return GP_OK;
}

}  // namespace gp

using namespace gp;

extern "C" {

int gp_assign_round(const gp_assign_args* args, void* stream) {
  int rc = validate(args);
  if (rc) return rc;
  if (args->m == 0) return GP_OK;
  // tile size: 4 entries per thread when the grid is big enough, fewer for the
  // small sample-phase lists so that they still spread over the SMs
  int ppt = args->m >= (int64_t)AT * 4 * 296 ? 4 : (args->m >= (int64_t)AT * 2 * 296 ? 2 : 1);
  if (args->group_list) {
    GP_REQUIRE((int64_t)AT * ppt <= (1ll << args->group_shift),
               "group_shift smaller than the tile");
  }
  unsigned grid = grid_for(args->m, AT * ppt);
  cudaStream_t s = (cudaStream_t)stream;
  if (args->d == 2) assign_kernel<2><<<grid, AT, 0, s>>>(*args, ppt);
  else assign_kernel<3><<<grid, AT, 0, s>>>(*args, ppt);
  return check_launch("assign_round");
}

int gp_rebase_bounds(const gp_assign_args* args, void* stream) {
  int rc = validate(args);
  if (rc) return rc;
  if (args->m == 0) return GP_OK;
  rebase_kernel<<<grid_for(args->m, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(*args);
  return check_launch("rebase_bounds");
}

int gp_audit(const gp_assign_args* args, unsigned long long* out, void* stream) {
  int rc = validate(args);
  if (rc) return rc;
  if (args->m == 0) return GP_OK;
  unsigned grid = grid_for(args->m, 128, 148 * 8);
  cudaStream_t s = (cudaStream_t)stream;
  if (args->d == 2) audit_kernel<2><<<grid, 128, 0, s>>>(*args, out);
  else audit_kernel<3><<<grid, 128, 0, s>>>(*args, out);
  return check_launch("audit");
}

}  // extern "C"

// ----------------------------------------------------- hierarchical groups
namespace gp {

template <int D>
__global__ void group_boxes_kernel(const double* __restrict__ X, int64_t ldx,
                                   const int32_t* __restrict__ list, int64_t m, int shift,
                                   double* __restrict__ boxes) {
  __shared__ double s_red[2 * D][8];
  const int64_t g = blockIdx.x;
  const int64_t b0 = g << shift;
  const int64_t b1 = min(m, (g + 1) << shift);
  double lo[D], hi[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    lo[j] = INFINITY;
    hi[j] = -INFINITY;
  }
  for (int64_t li = b0 + threadIdx.x; li < b1; li += blockDim.x) {
    int64_t q = list ? list[li] : li;
#pragma unroll
    for (int j = 0; j < D; ++j) {
      double v = X[j * ldx + q];
      lo[j] = fmin(lo[j], v);
      hi[j] = fmax(hi[j], v);
    }
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    for (int o = 16; o; o >>= 1) {
      lo[j] = fmin(lo[j], __shfl_xor_sync(FULL, lo[j], o));
      hi[j] = fmax(hi[j], __shfl_xor_sync(FULL, hi[j], o));
    }
    if (lane == 0) {
      s_red[j][warp] = lo[j];
      s_red[D + j][warp] = hi[j];
    }
  }
  __syncthreads();
  if (threadIdx.x < 2 * D) {
    int j = threadIdx.x;
    double v = s_red[j][0];
    for (int w = 1; w < (int)(blockDim.x / 32); ++w)
      v = j < D ? fmin(v, s_red[j][w]) : fmax(v, s_red[j][w]);
    boxes[g * 2 * D + j] = v;
  }
}

template <int D>
__global__ void __launch_bounds__(256) group_candidates_kernel(
    const double* __restrict__ boxes, int k, const double* __restrict__ centers,
    const double* __restrict__ infl, const int32_t* __restrict__ parent_list,
    const int32_t* __restrict__ parent_count, int parent_cap, int ratio_log2,
    int32_t* __restrict__ list, int32_t* __restrict__ count, int cap) {
  __shared__ double s_two[2][8];
  __shared__ int s_n;
  const int64_t g = blockIdx.x;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double lo[D], hi[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    lo[j] = boxes[g * 2 * D + j];
    hi[j] = boxes[g * 2 * D + D + j];
  }
  if (threadIdx.x == 0) s_n = 0;
  if (!(lo[0] <= hi[0])) {  // empty group
    if (threadIdx.x == 0) count[g] = 0;
    return;
  }
  const int32_t* src = nullptr;
  int nsrc = k;
  if (parent_list) {
    int64_t pg = g >> ratio_log2;
    int pc = parent_count[pg];
    if (pc >= 0) {
      src = parent_list + pg * (int64_t)parent_cap;
      nsrc = pc;
    }
  }
  double m1 = INFINITY, m2 = INFINITY;
  for (int i = threadIdx.x; i < nsrc; i += blockDim.x) {
    int c = src ? src[i] : i;
    double lb_, ub_;
    box_bounds<D>(centers + c * D, lo, hi, infl[c], lb_, ub_);
    two_min_merge(m1, m2, ub_, INFINITY);
  }
  for (int o = 16; o; o >>= 1) {
    double b1 = __shfl_xor_sync(FULL, m1, o);
    double b2 = __shfl_xor_sync(FULL, m2, o);
    two_min_merge(m1, m2, b1, b2);
  }
  if (lane == 0) {
    s_two[0][warp] = m1;
    s_two[1][warp] = m2;
  }
  __syncthreads();
  m1 = s_two[0][0];
  m2 = s_two[1][0];
  for (int w = 1; w < (int)(blockDim.x / 32); ++w) two_min_merge(m1, m2, s_two[0][w], s_two[1][w]);
  const double U = m2;
  int32_t* out = list + g * (int64_t)cap;
  for (int i = threadIdx.x; i < nsrc; i += blockDim.x) {
    int c = src ? src[i] : i;
    double lb_, ub_;
    box_bounds<D>(centers + c * D, lo, hi, infl[c], lb_, ub_);
    if (lb_ <= U) {
      int slot = atomicAdd(&s_n, 1);
      if (slot < cap) out[slot] = c;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) count[g] = s_n <= cap ? s_n : -1;
}

}  // namespace gp

extern "C" {

int gp_group_boxes(const double* X, int64_t ldx, int d, const int32_t* list, int64_t m, int shift,
                   double* boxes, void* stream) {
  GP_REQUIRE(d == 2 || d == 3, "gp_group_boxes: bad d");
  GP_REQUIRE(shift >= 5 && shift < 31, "gp_group_boxes: bad shift");
  if (m <= 0) return GP_OK;
  int64_t ng = (m + (1ll << shift) - 1) >> shift;
  cudaStream_t s = (cudaStream_t)stream;
  if (d == 2) group_boxes_kernel<2><<<(unsigned)ng, 256, 0, s>>>(X, ldx, list, m, shift, boxes);
  else group_boxes_kernel<3><<<(unsigned)ng, 256, 0, s>>>(X, ldx, list, m, shift, boxes);
  return check_launch("group_boxes");
}

int gp_group_candidates(const double* boxes, int64_t ngroups, int d, int k,
                        const double* centers, const double* infl, const int32_t* parent_list,
                        const int32_t* parent_count, int parent_cap, int parent_ratio_log2,
                        int32_t* list, int32_t* count, int cap, void* stream) {
  GP_REQUIRE(d == 2 || d == 3, "gp_group_candidates: bad d");
  GP_REQUIRE(cap >= 1 && k >= 1, "gp_group_candidates: bad sizes");
  if (ngroups <= 0) return GP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  if (d == 2)
    group_candidates_kernel<2><<<(unsigned)ngroups, 256, 0, s>>>(
        boxes, k, centers, infl, parent_list, parent_count, parent_cap, parent_ratio_log2, list,
        count, cap);
  else
    group_candidates_kernel<3><<<(unsigned)ngroups, 256, 0, s>>>(
        boxes, k, centers, infl, parent_list, parent_count, parent_cap, parent_ratio_log2, list,
        count, cap);
  return check_launch("group_candidates");
}

}  // extern "C"
