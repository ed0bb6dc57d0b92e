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
constexpr int PPT = 4;           // entries per thread
constexpr int TILE = AT * PPT;   // entries per tile
constexpr int CAP = 512;         // candidate centers staged in shared memory
constexpr int HSLOTS = 128;      // per-CTA block-weight cache
constexpr double LO_SLACK = 1.0 - 1e-12;
constexpr double HI_SLACK = 1.0 + 1e-12;

__device__ __forceinline__ void two_min_merge(double& m1, double& m2, double b1, double b2) {
  double lo = fmin(m1, b1);
  double hi = fmin(fmax(m1, b1), fmin(m2, b2));
  m1 = lo;
  m2 = hi;
}

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
__global__ void __launch_bounds__(AT) assign_kernel(gp_assign_args p) {
  __shared__ double s_c[D][CAP];
  __shared__ double s_inf[CAP];
  __shared__ int s_cid[CAP];
  __shared__ int s_pos[TILE];     // positions that need a scan
  __shared__ short s_ent[TILE];   // their tile-local entry ids
  __shared__ int s_newa[TILE];
  __shared__ int s_ckey[HSLOTS];
  __shared__ long long s_cval[HSLOTS];
  __shared__ double s_red[2 * D][AT / 32];
  __shared__ double s_two[2][AT / 32];
  __shared__ int s_nscan, s_ncand;
  __shared__ unsigned long long s_cnt[3];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t base = (int64_t)blockIdx.x * TILE;
  if (tid == 0) {
    s_nscan = 0;
    s_ncand = 0;
    s_cnt[0] = s_cnt[1] = s_cnt[2] = 0;
  }
  for (int i = tid; i < HSLOTS; i += AT) {
    s_ckey[i] = -1;
    s_cval[i] = 0;
  }
  __syncthreads();

  // ---- 1. skip test (kmeans.py:308-311)
  int pos[PPT], cur[PPT];
  double wv[PPT];
  int nskip = 0, ndec = 0;
#pragma unroll
  for (int e = 0; e < PPT; ++e) {
    int ent = e * AT + tid;
    int64_t li = base + ent;
    pos[e] = -1;
    cur[e] = -1;
    wv[e] = 0.0;
    if (li < p.m) {
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
      }
    }
  }
  __syncthreads();
  const int nscan = s_nscan;
  unsigned long long nevals = 0;

  if (nscan > 0) {
    // ---- 2. box of the scanned points
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

    // ---- 3. candidate threshold: second smallest box upper bound
    double m1 = INFINITY, m2 = INFINITY;
    for (int c = tid; c < p.k; c += AT) {
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
    __syncthreads();  // s_red reuse guard
    if (lane == 0) {
      s_two[0][warp] = m1;
      s_two[1][warp] = m2;
    }
    __syncthreads();
    m1 = s_two[0][0];
    m2 = s_two[1][0];
    for (int w = 1; w < AT / 32; ++w) two_min_merge(m1, m2, s_two[0][w], s_two[1][w]);
    const double U = m2;  // +inf when k == 1

    // collect candidates (lbnd <= U)
    for (int c = tid; c < p.k; c += AT) {
      double cc[D];
#pragma unroll
      for (int j = 0; j < D; ++j) cc[j] = p.centers[c * D + j];
      double lb_, ub_;
      box_bounds<D>(cc, lo, hi, p.infl[c], lb_, ub_);
      if (lb_ <= U) {
        int slot = atomicAdd(&s_ncand, 1);
        if (slot < CAP) {
#pragma unroll
          for (int j = 0; j < D; ++j) s_c[j][slot] = cc[j];
          s_inf[slot] = p.infl[c];
          s_cid[slot] = c;
        }
      }
    }
    __syncthreads();
    const int ncand = s_ncand;
    const bool overflow = ncand > CAP;

    // ---- 4. exact scan (kmeans.py:326-344); each thread owns <= PPT scanned points
    double x[PPT][D], best[PPT], second[PPT];
    int bi[PPT];
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
      int s = tid + r * AT;
      best[r] = INFINITY;
      second[r] = INFINITY;
      bi[r] = 0x7fffffff;
      if (s < nscan) {
        int q = s_pos[s];
#pragma unroll
        for (int j = 0; j < D; ++j) x[r][j] = p.X[j * p.ldx + q];
      }
    }
    const int total = overflow ? p.k : ncand;
    for (int c0 = 0; c0 < total; c0 += CAP) {
      int cn = min(CAP, total - c0);
      if (overflow) {
        __syncthreads();
        for (int i = tid; i < cn; i += AT) {
#pragma unroll
          for (int j = 0; j < D; ++j) s_c[j][i] = p.centers[(c0 + i) * D + j];
          s_inf[i] = p.infl[c0 + i];
          s_cid[i] = c0 + i;
        }
        __syncthreads();
      }
#pragma unroll
      for (int r = 0; r < PPT; ++r) {
        if (tid + r * AT < nscan) {
          for (int i = 0; i < cn; ++i) {
            double cc[D];
#pragma unroll
            for (int j = 0; j < D; ++j) cc[j] = s_c[j][i];
            double dist = effdist_rn<D>(x[r], cc, s_inf[i], p.order3);
            int cid = s_cid[i];
            bool win = dist < best[r] || (dist == best[r] && cid < bi[r]);
            second[r] = win ? best[r] : fmin(second[r], dist);
            best[r] = win ? dist : best[r];
            bi[r] = win ? cid : bi[r];
          }
          nevals += cn;
        }
      }
    }
#pragma unroll
    for (int r = 0; r < PPT; ++r) {
      int s = tid + r * AT;
      if (s < nscan) {
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

  // ---- 5. block weights (exact int64) + counters
  __shared__ unsigned s_scanned[TILE / 32];
  for (int i = tid; i < TILE / 32; i += AT) s_scanned[i] = 0;
  __syncthreads();
  for (int s = tid; s < nscan; s += AT) {
    int ent = s_ent[s];
    atomicOr(&s_scanned[ent >> 5], 1u << (ent & 31));
  }
  __syncthreads();
#pragma unroll
  for (int e = 0; e < PPT; ++e) {
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
  // counters
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
  unsigned grid = grid_for(args->m, TILE);
  cudaStream_t s = (cudaStream_t)stream;
  if (args->d == 2) assign_kernel<2><<<grid, AT, 0, s>>>(*args);
  else assign_kernel<3><<<grid, AT, 0, s>>>(*args);
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
