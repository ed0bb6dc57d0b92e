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

// ------------------------------------------------------------ filter kernel
// Streaming pass over the active entries: skip test with the lazily relaxed
// bounds (kmeans.py:308-311), exact block weights of the points that keep
// their assignment, and compaction of the points that must be scanned.
// Chunk c = entries [c*FCHUNK, (c+1)*FCHUNK); its scanned positions go to
// scan[c*FCHUNK ..] (no global reservation) and runs[c] = their count.
// Persistent CTAs walk contiguous chunk ranges (SFC-contiguous, so the
// per-CTA block-weight cache sees few blocks); each thread owns FPER
// consecutive entries, loaded with 16-byte vector loads in the full phase.
constexpr int FTH = 256;
constexpr int FPER = 8;
constexpr int FCHUNK = FTH * FPER;   // 2048 entries per chunk

struct AssignLayout {
  int64_t nchunks;
  size_t off_list, off_runs, total;
};

static AssignLayout assign_layout(int64_t m) {
  AssignLayout L;
  L.nchunks = (m + FCHUNK - 1) / FCHUNK;
  if (L.nchunks < 1) L.nchunks = 1;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  size_t o = 0;
  L.off_list = o; o = al(o + (size_t)L.nchunks * FCHUNK * 4);
  L.off_runs = o; o = al(o + (size_t)L.nchunks * 4);
  L.total = o;
  return L;
}

// weight in exact integer units of 1/wscale, without fp->int conversions
// (w * wscale is an integer by construction of wscale = 2^s)
template <int WM>
__device__ __forceinline__ long long weight_units(const void* w, int64_t i, int shift) {
  if (WM == GP_W_UNIT) return 1;
  if (WM == GP_W_F32) {
    unsigned b = __float_as_uint(((const float*)w)[i]);
    int e = (b >> 23) & 0xff;
    long long mant = e ? ((b & 0x7fffff) | 0x800000) : (b & 0x7fffff);
    int sh = (e ? e : 1) - 150 + shift;  // value = mant * 2^(e-150) * 2^shift
    long long v = sh >= 0 ? (mant << sh) : (mant >> -sh);
    return (b >> 31) ? -v : v;
  }
  unsigned long long b = (unsigned long long)__double_as_longlong(((const double*)w)[i]);
  int e = (int)((b >> 52) & 0x7ff);
  long long mant = e ? (long long)((b & 0xfffffffffffffull) | 0x10000000000000ull)
                     : (long long)(b & 0xfffffffffffffull);
  int sh = (e ? e : 1) - 1075 + shift;
  long long v = sh >= 0 ? (mant << sh) : (mant >> -sh);
  return (b >> 63) ? -v : v;
}

template <int WM>
__global__ void __launch_bounds__(FTH) filter_kernel(gp_assign_args p, int wshift, int64_t nchunks,
                                                     int32_t* __restrict__ scan,
                                                     int32_t* __restrict__ runs) {
  __shared__ int s_ckey[HSLOTS];
  __shared__ long long s_cval[HSLOTS];
  __shared__ int s_wcnt[FTH / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < HSLOTS; i += FTH) {
    s_ckey[i] = -1;
    s_cval[i] = 0;
  }
  __syncthreads();
  const int64_t per = (nchunks + gridDim.x - 1) / gridDim.x;
  const int64_t cb = blockIdx.x * per, ce = min(nchunks, cb + per);
  unsigned long long nskip = 0;
  for (int64_t c = cb; c < ce; ++c) {
    const int64_t e0 = c * FCHUNK + (int64_t)tid * FPER;   // my first entry
    int a[FPER], q[FPER];
    double ub[FPER], lb[FPER];
    if (p.list == nullptr && e0 + FPER <= p.m) {
      // full phase: positions == entries, 16-byte vector loads
      const int4* ap = reinterpret_cast<const int4*>(p.a + e0);
      int4 a0 = ap[0], a1 = ap[1];
      a[0] = a0.x; a[1] = a0.y; a[2] = a0.z; a[3] = a0.w;
      a[4] = a1.x; a[5] = a1.y; a[6] = a1.z; a[7] = a1.w;
      const double2* up = reinterpret_cast<const double2*>(p.ub + e0);
      const double2* lp = reinterpret_cast<const double2*>(p.lb + e0);
#pragma unroll
      for (int h = 0; h < FPER / 2; ++h) {
        double2 u = up[h], l = lp[h];
        ub[2 * h] = u.x; ub[2 * h + 1] = u.y;
        lb[2 * h] = l.x; lb[2 * h + 1] = l.y;
      }
#pragma unroll
      for (int e = 0; e < FPER; ++e) q[e] = (int)(e0 + e);
    } else {
#pragma unroll
      for (int e = 0; e < FPER; ++e) {
        const int64_t li = e0 + e;
        q[e] = li < p.m ? (p.list ? p.list[li] : (int)li) : -1;
        a[e] = q[e] >= 0 ? p.a[q[e]] : -1;
        ub[e] = q[e] >= 0 ? p.ub[q[e]] : 0.0;
        lb[e] = q[e] >= 0 ? p.lb[q[e]] : 0.0;
      }
    }
    // skip test; run-length accumulation of the kept points' weights
    unsigned need = 0;
    int run_a = -1;
    long long run_w = 0;
    bool broke = false;
#pragma unroll
    for (int e = 0; e < FPER; ++e) {
      if (q[e] < 0) continue;
      bool skip = false;
      const int ae = a[e];
      if (ae >= 0) {
        const double u = ub_eval(p.ub_scale[ae], ub[e], p.ub_shift[ae], p.bound_err);
        const double l = lb_eval(p.lb_scale, lb[e], p.lb_shift, p.bound_err);
        skip = u < l;
      }
      if (!skip) {
        need |= 1u << e;
        continue;
      }
      ++nskip;
      const long long v = weight_units<WM>(p.w, q[e], wshift);
      if (ae == run_a) {
        run_w += v;
      } else {
        if (run_a >= 0) {
          cache_add(s_ckey, s_cval, p.block_w, run_a, run_w);
          broke = true;
        }
        run_a = ae;
        run_w = v;
      }
    }
    // one warp-wide reduction when every lane ends on the same block (common)
    const unsigned grp = __match_any_sync(FULL, run_a);
    const bool uni = grp == FULL && !__any_sync(FULL, broke) && run_a >= 0;
    if (uni) {
      long long g = run_w;
      for (int o = 16; o; o >>= 1) g += __shfl_xor_sync(FULL, g, o);
      if (lane == 0) cache_add(s_ckey, s_cval, p.block_w, run_a, g);
    } else if (run_a >= 0) {
      cache_add(s_ckey, s_cval, p.block_w, run_a, run_w);
    }
    // compaction of the points to scan into the chunk's own slots
    const int mine = __popc(need);
    int incl = mine;
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    if (lane == 31) s_wcnt[warp] = incl;
    __syncthreads();
    int before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < FTH / 32; ++w) {
      const int cw = s_wcnt[w];
      before += w < warp ? cw : 0;
      total += cw;
    }
    int off = before + incl - mine;
    int32_t* dst = scan + c * FCHUNK;
#pragma unroll
    for (int e = 0; e < FPER; ++e)
      if (need & (1u << e)) dst[off++] = q[e];
    if (tid == 0) runs[c] = total;
    __syncthreads();  // s_wcnt reuse
  }
  for (int o = 16; o; o >>= 1) nskip += __shfl_xor_sync(FULL, nskip, o);
  if (lane == 0 && nskip) atomicAdd(&p.counters[0], nskip);
  __syncthreads();
  for (int i = tid; i < HSLOTS; i += FTH)
    if (s_ckey[i] >= 0 && s_cval[i] != 0)
      atomicAdd((unsigned long long*)&p.block_w[s_ckey[i]], (unsigned long long)s_cval[i]);
}

// -------------------------------------------------------------- scan kernel
// One CTA per filter run: box of the run's points (kmeans.py:315-316, per
// run), candidate centers (lbnd <= second smallest ubnd over the group's list
// or all k), then the scan (kmeans.py:326-344) with an approximate prefilter:
// pass 1 finds the two smallest q = d^2/infl^2; pass 2 evaluates the
// reference's exact effective distance only where q <= q2 (1 + Q_TOL), a
// superset of every center whose exact distance is <= the exact runner-up.
constexpr int SPT = 2;             // points per thread per sub-tile
constexpr int STILE = AT * SPT;    // 512

template <int D, int WM>
__global__ void __launch_bounds__(AT, 2) scan_kernel(gp_assign_args p, int wshift, int64_t nchunks,
                                                     const int32_t* __restrict__ scan,
                                                     const int32_t* __restrict__ runs) {
  __shared__ ScanSmem<D> S;
  __shared__ int s_ckey[HSLOTS];
  __shared__ long long s_cval[HSLOTS];
  __shared__ double s_red[2 * D][AT / 32];
  __shared__ double s_two[2][AT / 32];
  __shared__ int s_ncand;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < HSLOTS; i += AT) {
    s_ckey[i] = -1;
    s_cval[i] = 0;
  }
  __syncthreads();
  unsigned long long nevals = 0;
  for (int64_t chunk = blockIdx.x; chunk < nchunks; chunk += gridDim.x) {
  const int cnt = runs[chunk];
  if (cnt == 0) continue;
  const int32_t* cscan = scan + chunk * FCHUNK;
  // candidate source: the group's hierarchical list, or all k centers
  const int32_t* src = nullptr;
  int nsrc = p.k;
  if (p.group_list) {
    const int64_t g = (chunk * FCHUNK) >> p.group_shift;
    const int gc = p.group_count[g];
    if (gc >= 0) {
      src = p.group_list + g * (int64_t)p.group_cap;
      nsrc = gc;
    }
  }
  for (int t0 = 0; t0 < cnt; t0 += STILE) {
    const int tn = min(STILE, cnt - t0);
    __syncthreads();  // previous sub-tile done with s_ncand / S
    if (tid == 0) s_ncand = 0;
    int qpos[SPT];
    double x[SPT][D];
#pragma unroll
    for (int r = 0; r < SPT; ++r) {
      const int s = tid + r * AT;
      qpos[r] = s < tn ? cscan[t0 + s] : -1;
      if (qpos[r] >= 0) {
#pragma unroll
        for (int j = 0; j < D; ++j) x[r][j] = p.X[j * p.ldx + qpos[r]];
      }
    }
    // ---- box of the sub-tile's points
    double lo[D], hi[D];
#pragma unroll
    for (int j = 0; j < D; ++j) {
      lo[j] = INFINITY;
      hi[j] = -INFINITY;
#pragma unroll
      for (int r = 0; r < SPT; ++r)
        if (qpos[r] >= 0) {
          lo[j] = fmin(lo[j], x[r][j]);
          hi[j] = fmax(hi[j], x[r][j]);
        }
      for (int o = 16; o; o >>= 1) {
        lo[j] = fmin(lo[j], __shfl_xor_sync(FULL, lo[j], o));
        hi[j] = fmax(hi[j], __shfl_xor_sync(FULL, hi[j], o));
      }
    }
    __syncthreads();  // previous sub-tile done with s_red / S
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < D; ++j) {
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
    // ---- candidates: lbnd <= second smallest ubnd over the source
    double m1 = INFINITY, m2 = INFINITY;
    for (int i = tid; i < nsrc; i += AT) {
      const int c = src ? src[i] : i;
      double lb_, ub_;
      box_bounds<D>(p.centers + c * D, lo, hi, p.infl[c], lb_, ub_);
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
      const int c = src ? src[i] : i;
      double lb_, ub_;
      box_bounds<D>(p.centers + c * D, lo, hi, p.infl[c], lb_, ub_);
      if (lb_ <= U) {
        const int slot = atomicAdd(&s_ncand, 1);
        if (slot < CAP) stage_center<D>(S, slot, c, p.centers, p.infl);
      }
    }
    __syncthreads();
    const int ncand = s_ncand;
    const bool overflow = ncand > CAP;  // then stream the whole source in chunks
    const int total = overflow ? nsrc : ncand;

    double q1[SPT], q2[SPT];
#pragma unroll
    for (int r = 0; r < SPT; ++r) q1[r] = q2[r] = INFINITY;
    for (int c0 = 0; c0 < total; c0 += CAP) {
      const int cn = min(CAP, total - c0);
      if (overflow) {
        __syncthreads();
        for (int i = tid; i < cn; i += AT)
          stage_center<D>(S, i, src ? src[c0 + i] : c0 + i, p.centers, p.infl);
        __syncthreads();
      }
#pragma unroll
      for (int r = 0; r < SPT; ++r) {
        if (qpos[r] >= 0) {
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
    double best[SPT], second[SPT], thr[SPT];
    int bi[SPT];
#pragma unroll
    for (int r = 0; r < SPT; ++r) {
      best[r] = INFINITY;
      second[r] = INFINITY;
      bi[r] = 0x7fffffff;
      thr[r] = fma(q2[r], Q_TOL, q2[r]);
    }
    for (int c0 = 0; c0 < total; c0 += CAP) {
      const int cn = min(CAP, total - c0);
      if (overflow) {
        __syncthreads();
        for (int i = tid; i < cn; i += AT)
          stage_center<D>(S, i, src ? src[c0 + i] : c0 + i, p.centers, p.infl);
        __syncthreads();
      }
#pragma unroll
      for (int r = 0; r < SPT; ++r) {
        if (qpos[r] >= 0) {
          for (int i = 0; i < cn; ++i) {
            if (qdist<D>(x[r], S, i) <= thr[r]) {
              double cc[D];
#pragma unroll
              for (int j = 0; j < D; ++j) cc[j] = S.c[j][i];
              const double dist = effdist_rn<D>(x[r], cc, S.inf[i], p.order3);
              const int cid = S.cid[i];
              const bool win = dist < best[r] || (dist == best[r] && cid < bi[r]);
              second[r] = win ? best[r] : fmin(second[r], dist);
              best[r] = win ? dist : best[r];
              bi[r] = win ? cid : bi[r];
              ++nevals;
            }
          }
        }
      }
    }
    // ---- write back + block weights of the scanned points
#pragma unroll
    for (int r = 0; r < SPT; ++r) {
      const bool valid = qpos[r] >= 0;
      int c = -1;
      long long v = 0;
      if (valid) {
        const int q = qpos[r];
        c = bi[r];
        p.a[q] = c;
        p.ub[q] = __ddiv_ru(__dsub_ru(best[r], p.ub_shift[c]), p.ub_scale[c]);
        p.lb[q] = __ddiv_rd(__dadd_rd(second[r], p.lb_shift), p.lb_scale);
        v = weight_units<WM>(p.w, q, wshift);
      }
      const unsigned grp = __match_any_sync(FULL, c);
      if (grp == FULL) {
        long long g = v;
        for (int o = 16; o; o >>= 1) g += __shfl_xor_sync(FULL, g, o);
        if (lane == 0 && valid) cache_add(s_ckey, s_cval, p.block_w, c, g);
      } else if (valid) {
        cache_add(s_ckey, s_cval, p.block_w, c, v);
      }
    }
  }
  }  // chunk loop
  for (int o = 16; o; o >>= 1) nevals += __shfl_xor_sync(FULL, nevals, o);
  if (lane == 0 && nevals) atomicAdd(&p.counters[2], nevals);
  __syncthreads();
  for (int i = tid; i < HSLOTS; i += AT)
    if (s_ckey[i] >= 0 && s_cval[i] != 0)
      atomicAdd((unsigned long long*)&p.block_w[s_ckey[i]], (unsigned long long)s_cval[i]);
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

int gp_assign_workspace_bytes(int64_t m, size_t* bytes) {
  GP_REQUIRE(m >= 0 && m < (1ll << 31), "gp_assign_workspace_bytes: m out of range");
  *bytes = assign_layout(m).total;
  return GP_OK;
}

int gp_assign_round(const gp_assign_args* args, void* stream) {
  int rc = validate(args);
  if (rc) return rc;
  if (args->m == 0) return GP_OK;
  AssignLayout L = assign_layout(args->m);
  GP_REQUIRE(args->workspace && args->workspace_bytes >= L.total,
             "gp_assign_round: workspace too small");
  if (args->group_list)
    GP_REQUIRE(FCHUNK <= (1ll << args->group_shift), "group_shift smaller than a filter chunk");
  cudaStream_t s = (cudaStream_t)stream;
  char* ws = (char*)args->workspace;
  int32_t* scan = (int32_t*)(ws + L.off_list);
  int32_t* runs = (int32_t*)(ws + L.off_runs);
  // exact weight units: wscale = 2^wshift
  int wshift = 0;
  frexp(args->wscale, &wshift);
  wshift -= 1;
  GP_REQUIRE(ldexp(1.0, wshift) == args->wscale, "gp_assign_round: wscale must be a power of 2");
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t nc = L.nchunks;
  // persistent grids: exactly the co-resident CTAs (static chunk split in the filter)
  auto fit = [&](const void* fn, int threads) {
    int per_sm = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, 0);
    int64_t g = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
    return (unsigned)(nc < g ? nc : g);
  };
#define GP_LAUNCH_ASSIGN(WM)                                                                     \
  {                                                                                              \
    unsigned gf = fit((const void*)filter_kernel<WM>, FTH);                                      \
    filter_kernel<WM><<<gf, FTH, 0, s>>>(*args, wshift, nc, scan, runs);                         \
    if (args->d == 2) {                                                                          \
      unsigned gs = fit((const void*)scan_kernel<2, WM>, AT);                                    \
      scan_kernel<2, WM><<<gs, AT, 0, s>>>(*args, wshift, nc, scan, runs);                       \
    } else {                                                                                     \
      unsigned gs = fit((const void*)scan_kernel<3, WM>, AT);                                    \
      scan_kernel<3, WM><<<gs, AT, 0, s>>>(*args, wshift, nc, scan, runs);                       \
    }                                                                                            \
  }
  if (args->wmode == GP_W_UNIT) { GP_LAUNCH_ASSIGN(GP_W_UNIT) }
  else if (args->wmode == GP_W_F32) { GP_LAUNCH_ASSIGN(GP_W_F32) }
  else { GP_LAUNCH_ASSIGN(GP_W_F64) }
#undef GP_LAUNCH_ASSIGN
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
