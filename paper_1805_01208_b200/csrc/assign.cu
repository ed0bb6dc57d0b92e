// K6 assign round (filter + scan), K8 audit, bound rebase, group candidates.
//
// One balance round of the reference (kmeans.py:415-425 for every rank:
// _scan_rank kmeans.py:297-344 + _global_block_weights kmeans.py:368-374) is
// two kernels:
//   filter : streams the active entries once (HBM bound): skip test with the
//            lazily relaxed Hamerly bounds (kmeans.py:308-311; relax_bounds
//            kmeans.py:208-239 applied through affine maps),
//            exact int64 block weights of the points that keep their block,
//            and a per-warp compaction of the points that must be scanned;
//   scan   : one warp per 256-entry region: box of the region's scanned
//            points (kmeans.py:315-316, per region instead of per rank),
//            candidate centers (every center whose box lower bound does not
//            exceed the second smallest box upper bound), then the scan with
//            an approximate prefilter and the reference's exact effective
//            distance for the near-contenders, (dist, index) lexicographic
//            tie-break, write-back, block weights of the scanned points.
// The result per point is the lowest-index argmin of the reference's
// effective distance, bit for bit; pruning only decides what is evaluated.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <type_traits>

#include "common.cuh"

namespace gp {

constexpr double LO_SLACK = 1.0 - 1e-12;
constexpr double HI_SLACK = 1.0 + 1e-12;
constexpr double Q_TOL = 1e-13;    // prefilter tolerance (>> the q rounding error)

__device__ __forceinline__ void two_min_merge(double& m1, double& m2, double b1, double b2) {
  double lo = fmin(m1, b1);
  double hi = fmin(fmax(m1, b1), fmin(m2, b2));
  m1 = lo;
  m2 = hi;
}

// Rigorous bounds of the SQUARED effective distance from any point of the box
// [lo, hi] to center c: lsq <= (dist/infl)^2 <= usq, with inv2_lo <= 1/infl^2
// <= inv2_hi (host-rounded outward), directed rounding and 1e-12 slack.
template <int D>
__device__ __forceinline__ void box_bounds_sq(const double* c, const double* lo, const double* hi,
                                              double inv2_lo, double inv2_hi, double& lsq,
                                              double& usq) {
  double sl = 0.0, su = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double dl = 0.0;
    if (c[j] < lo[j]) dl = __dsub_rd(lo[j], c[j]);
    else if (c[j] > hi[j]) dl = __dsub_rd(c[j], hi[j]);
    sl = __fma_rd(dl, dl, sl);
    double du = fmax(__dsub_ru(c[j], lo[j]), __dsub_ru(hi[j], c[j]));
    su = __fma_ru(du, du, su);
  }
  lsq = __dmul_rd(__dmul_rd(sl, inv2_lo), LO_SLACK);
  usq = __dmul_ru(__dmul_ru(su, inv2_hi), HI_SLACK);
}

// the two halves of box_bounds_sq (identical arithmetic), for passes needing one
template <int D>
__device__ __forceinline__ double box_usq(const double* c, const double* lo, const double* hi,
                                          double inv2_hi) {
  double su = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double du = fmax(__dsub_ru(c[j], lo[j]), __dsub_ru(hi[j], c[j]));
    su = __fma_ru(du, du, su);
  }
  return __dmul_ru(__dmul_ru(su, inv2_hi), HI_SLACK);
}
template <int D>
__device__ __forceinline__ double box_lsq(const double* c, const double* lo, const double* hi,
                                          double inv2_lo) {
  double sl = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    double dl = 0.0;
    if (c[j] < lo[j]) dl = __dsub_rd(lo[j], c[j]);
    else if (c[j] > hi[j]) dl = __dsub_rd(c[j], hi[j]);
    sl = __fma_rd(dl, dl, sl);
  }
  return __dmul_rd(__dmul_rd(sl, inv2_lo), LO_SLACK);
}

// fresh best / runner-up effective distances (b rounded up, s rounded down)
// -> normalised float32 bounds under the current maps
__device__ __forceinline__ void store_bounds(const gp_assign_args& p, const float4& L, int64_t q,
                                             int c, float b_up, float s_dn) {
  const float4 N = reinterpret_cast<const float4*>(p.ub_norm)[c];
  reinterpret_cast<unsigned*>(p.ublb)[q] =
      bnd_pack(ub_normf(N, b_up), lb_normf(L.z, L.w, s_dn), p.bound_scale);
}

// lower bound of min_c 1/infl_c^2: the device copy gp_update_maps keeps (so that a
// captured loop graph sees every round's value), else the host scalar
__device__ __forceinline__ double inv2_min_of(const gp_assign_args& p) {
  return p.inv2_min_dev ? *p.inv2_min_dev : p.inv2_min;
}

// lower-bound map parameters (A_lo, B_hi, 1/A_lo, B_lo) of active entry li: its
// region's (gp_region_maps) or the global ones
__device__ __forceinline__ float4 lb_params(const gp_assign_args& p, int64_t li) {
  if (p.lb_rpar) return reinterpret_cast<const float4*>(p.lb_rpar)[li >> p.lb_rshift];
  return *reinterpret_cast<const float4*>(p.lb_par);
}

// Per-warp block-weight table (no atomics, no cross-warp contention): the lanes'
// (block, value) pairs are combined per distinct block in a warp-uniform loop and
// one leader lane updates the warp's table; an evicted entry goes to global memory.
constexpr int WT = 16;
struct WarpTab {
  int key[WT];
  long long val[WT];
};
__device__ __forceinline__ void tab_init(WarpTab& t, int lane) {
  if (lane < WT) {
    t.key[lane] = -1;
    t.val[lane] = 0;
  }
  __syncwarp();
}
template <typename V>
__device__ __forceinline__ void tab_add(WarpTab& t, long long* global, int lane, bool active,
                                        int key, V val) {
  unsigned pend = __ballot_sync(FULL, active);
  while (pend) {
    const int leader = __ffs(pend) - 1;
    const int k = __shfl_sync(FULL, key, leader);
    const bool mine = active && key == k;
    const unsigned m = __ballot_sync(FULL, mine);
    long long sum;
    if (sizeof(V) == 4) {
      sum = (long long)__reduce_add_sync(FULL, mine ? (unsigned)val : 0u);
    } else {
      sum = mine ? (long long)val : 0;
      for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(FULL, sum, o);
    }
    if (lane == leader) {
      const int sl = k & (WT - 1);
      if (t.key[sl] == k) {
        t.val[sl] += sum;
      } else {
        if (t.key[sl] >= 0)
          atomicAdd((unsigned long long*)&global[t.key[sl]], (unsigned long long)t.val[sl]);
        t.key[sl] = k;
        t.val[sl] = sum;
      }
    }
    __syncwarp();
    pend &= ~m;
  }
}
__device__ __forceinline__ void tab_flush(WarpTab& t, long long* global, int lane) {
  __syncwarp();
  if (lane < WT && t.key[lane] >= 0 && t.val[lane] != 0)
    atomicAdd((unsigned long long*)&global[t.key[lane]], (unsigned long long)t.val[lane]);
}

// weight in exact integer units of 1/wscale without fp->int conversions
// (w * 2^shift is an integer by construction)
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

// ------------------------------------------------------------ filter kernel
constexpr int FTH = 256;
constexpr int FPER = 8;
constexpr int WREG = 32 * FPER;       // entries per warp region (256)
constexpr int RPW = 2;                // consecutive regions a warp takes per chunk
constexpr int FCHUNK = FTH * FPER * RPW;   // entries per CTA chunk (4096 = 16 regions)

struct AssignLayout {
  int64_t nchunks, nregions;
  size_t off_list, off_olda, off_runs, off_sched, total;
};

static AssignLayout assign_layout(int64_t m) {
  AssignLayout L;
  L.nchunks = (m + FCHUNK - 1) / FCHUNK;
  if (L.nchunks < 1) L.nchunks = 1;
  L.nregions = L.nchunks * (FCHUNK / WREG);
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  size_t o = 0;
  L.off_list = o; o = al(o + (size_t)L.nregions * WREG * 8);   // int2 (position, old block)
  L.off_olda = o;
  L.off_runs = o; o = al(o + (size_t)L.nregions * 4);
  L.off_sched = o; o = al(o + 8);
  L.total = o;
  return L;
}

// Region r = entries [r*WREG, (r+1)*WREG), owned by one warp.  Lane l owns the
// entry pairs 64h + 2l + {0,1} (h < 4): every warp-wide access is one contiguous
// 256/512-byte line, in global and in shared memory (no bank conflicts).  Its
// scanned positions go, in entry order, to scan[r*WREG ..] and runs[r] = their
// count.  Persistent CTAs walk contiguous chunk ranges (warp w takes region w of
// every chunk).  Dense full regions are streamed by the bulk-copy engine into a
// per-warp ring of FSTAGES shared-memory stages (lane 0 issues cp.async.bulk,
// completion on the stage's mbarrier), so each warp's HBM stream runs ahead of it
// with no CTA-wide barrier; other regions (sparse lists, the tail) use direct loads.
constexpr int FSTAGES = 2;
constexpr int FREG_BYTES = RPW * WREG * 8;   // a (4 B) + packed (ub, lb) (4 B) per entry

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

template <int WM>
__global__ void __launch_bounds__(FTH) filter_kernel(gp_assign_args p, int wshift, int64_t nchunks,
                                                     int2* __restrict__ ent,
                                                     int32_t* __restrict__ runs,
                                                     unsigned long long* __restrict__ sched) {
  typedef typename std::conditional<WM == GP_W_UNIT, int, long long>::type RunW;
  extern __shared__ __align__(128) unsigned char fsm[];   // [warp][stage] regions
  __shared__ __align__(8) uint64_t s_bar[FTH / 32][FSTAGES];
  __shared__ WarpTab s_tab[FTH / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  WarpTab& tab = s_tab[warp];
  if (blockIdx.x == 0 && tid == 0) *sched = 0;  // the scan's work counter
  tab_init(tab, lane);
  const int64_t per = (nchunks + gridDim.x - 1) / gridDim.x;
  const int64_t cb = blockIdx.x * per, ce = min(nchunks, cb + per);
  // regions of chunks [cb, fe) are dense and full: streamed through shared memory
  const int64_t nfull = p.list == nullptr ? p.m / FCHUNK : 0;
  const int64_t fe = max(cb, min(ce, nfull));
  unsigned char* wsm = fsm + (size_t)warp * FSTAGES * FREG_BYTES;
  auto issue = [&](int64_t c, int sg) {
    const int64_t e0 = (c * (FCHUNK / WREG) + RPW * warp) * WREG;
    unsigned char* base = wsm + (size_t)sg * FREG_BYTES;
    mbar_expect_tx(&s_bar[warp][sg], FREG_BYTES);
    bulk_g2s(base, p.a + e0, RPW * WREG * 4, &s_bar[warp][sg]);
    bulk_g2s(base + RPW * WREG * 4, reinterpret_cast<const unsigned*>(p.ublb) + e0,
             RPW * WREG * 4, &s_bar[warp][sg]);
  };
  if (lane == 0) {
    for (int sg = 0; sg < FSTAGES; ++sg) mbar_init(&s_bar[warp][sg], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (int sg = 0; sg < FSTAGES && cb + sg < fe; ++sg) issue(cb + sg, sg);
  }
  __syncwarp();
  unsigned long long nskip = 0;
  const float binv = __frcp_rn(p.bound_scale);   // exact: a power of two
  int st = 0;            // ring stage of the next staged region, and its use parity
  unsigned phase = 0;
  for (int64_t c = cb; c < ce; ++c) {
    const int reg0 = (int)c * (FCHUNK / WREG) + RPW * warp;   // m < 2^31: 32-bit entry math
    float4 lbp = lb_params(p, (int64_t)reg0 * WREG);   // one map per 2^14 entries: both regions
    lbp.x *= binv;                                      // slope on the scaled stored lb~
    const bool staged = c < fe;
    const unsigned char* base = wsm + (size_t)st * FREG_BYTES;
    if (staged) mbar_wait(&s_bar[warp][st], phase);
    // block-weight runs of the kept points continue across the warp's regions
    int run_a = -1, run2_a = -1;
    RunW run_w = 0, run2_w = 0;
#pragma unroll 1
    for (int half = 0; half < RPW; ++half) {
      const int reg = reg0 + half;
      const int rbase = reg * WREG + 2 * lane;
      int a[FPER], q[FPER];
      float ub[FPER], lb[FPER];
      int nvalid = FPER;
      if (staged) {
        const int2* as = reinterpret_cast<const int2*>(base) + half * (WREG / 2);
        const uint2* bs = reinterpret_cast<const uint2*>(base + RPW * WREG * 4) + half * (WREG / 2);
#pragma unroll
        for (int h = 0; h < FPER / 2; ++h) {
          const int2 av = as[h * 32 + lane];
          const uint2 bw = bs[h * 32 + lane];
          // raw scaled values: the bound-map slopes below carry the 1/bound_scale factor
          const float2 b0 = bnd_raw(bw.x), b1 = bnd_raw(bw.y);
          a[2 * h] = av.x; a[2 * h + 1] = av.y;
          ub[2 * h] = b0.x; lb[2 * h] = b0.y;
          ub[2 * h + 1] = b1.x; lb[2 * h + 1] = b1.y;
          q[2 * h] = rbase + 64 * h;
          q[2 * h + 1] = rbase + 64 * h + 1;
        }
      } else {
        nvalid = 0;
#pragma unroll
        for (int e = 0; e < FPER; ++e) {
          const int li = rbase + 64 * (e >> 1) + (e & 1);
          q[e] = li < p.m ? (p.list ? p.list[li] : li) : -1;
          nvalid += q[e] >= 0;
          a[e] = q[e] >= 0 ? p.a[q[e]] : -1;
          const float2 v = q[e] >= 0 ? bnd_raw(reinterpret_cast<const unsigned*>(p.ublb)[q[e]])
                                     : make_float2(0.f, 0.f);
          ub[e] = v.x;
          lb[e] = v.y;
        }
      }
      // skip test + block weights of the kept points.  Fast path (most lanes): all 8
      // entries valid and in one block, so one parameter load and a branch-free skip
      // mask.  General path: run-length weights (at most two runs per lane are held; a
      // third, which needs three blocks among the lane's entries, goes to global memory).
      unsigned need = 0;
      bool same = staged && a[0] >= 0;
#pragma unroll
      for (int e = 1; e < FPER; ++e) same = same && a[e] == a[0];
      if (same) {
        float4 E = reinterpret_cast<const float4*>(p.ub_eval)[a[0]];
        E.x *= binv;   // exact: the stored ub~ carries bound_scale
        E.y *= binv;
        unsigned keep = 0;
#pragma unroll
        for (int e = 0; e < FPER; ++e) {
          // lb_evalf without its k == 1 test (A > 0 maps lb~ = inf to inf as well) and
          // without its floor at 0: the evaluated ub is a sound upper bound of a
          // distance, so it is >= 0 and "ub < lb" is unchanged by the floor
          const float lbv = __fmaf_rd(lbp.x, lb[e], -lbp.y);
          keep |= (unsigned)(ub_evalf(E, ub[e]) < lbv) << e;
        }
        need = keep ^ ((1u << FPER) - 1);
        if (keep) {
          RunW v = 0;
          if (WM == GP_W_UNIT) {
            v = (RunW)__popc(keep);
          } else {
#pragma unroll
            for (int e = 0; e < FPER; ++e)
              if (keep & (1u << e)) v += (RunW)weight_units<WM>(p.w, q[e], wshift);
          }
          if (a[0] == run_a) {
            run_w += v;
          } else {
            if (run_a >= 0) {
              if (run2_a >= 0)
                atomicAdd((unsigned long long*)&p.block_w[run2_a], (unsigned long long)run2_w);
              run2_a = run_a;
              run2_w = run_w;
            }
            run_a = a[0];
            run_w = v;
          }
        }
      } else {
        int ea = -1;          // block whose bound parameters E holds (runs share them)
        float4 E = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
        for (int e = 0; e < FPER; ++e) {
          const bool valid = staged || q[e] >= 0;
          const int ae = a[e];
          if (ae >= 0 && ae != ea) {
            E = reinterpret_cast<const float4*>(p.ub_eval)[ae];
            E.x *= binv;
            E.y *= binv;
            ea = ae;
          }
          const float lbv = fmaxf(__fmaf_rd(lbp.x, lb[e], -lbp.y), 0.f);
          const bool skip = valid && ae >= 0 && ub_evalf(E, ub[e]) < lbv;
          need |= (unsigned)(valid && !skip) << e;
          if (skip) {
            const RunW v = (RunW)weight_units<WM>(p.w, q[e], wshift);
            if (ae == run_a) {
              run_w += v;
            } else {
              if (run_a >= 0) {
                if (run2_a >= 0)
                  atomicAdd((unsigned long long*)&p.block_w[run2_a], (unsigned long long)run2_w);
                run2_a = run_a;
                run2_w = run_w;
              }
              run_a = ae;
              run_w = v;
            }
          }
        }
      }
      nskip += nvalid - __popc(need);
      if (!__any_sync(FULL, need)) {   // nothing to rescan in this region (the common case)
        if (lane == 0) runs[reg] = 0;
        continue;
      }
      // compaction of the points to scan into the region's own slots, in entry order
      // (entry 64h + 2l + b: ranks from two ballots per h)
      int2* dst = ent + (int64_t)reg * WREG;   // (position, old block): one 8-byte slot
      const unsigned lt = (1u << lane) - 1;
      int cnt = 0;
#pragma unroll
      for (int h = 0; h < FPER / 2; ++h) {
        const bool n0 = need & (1u << (2 * h)), n1 = need & (1u << (2 * h + 1));
        const unsigned b0 = __ballot_sync(FULL, n0), b1 = __ballot_sync(FULL, n1);
        int off = cnt + __popc(b0 & lt) + __popc(b1 & lt);
        if (n0) {
          dst[off] = make_int2(q[2 * h], a[2 * h]);  // the scan writes a only on a change
          ++off;
        }
        if (n1) dst[off] = make_int2(q[2 * h + 1], a[2 * h + 1]);
        cnt += __popc(b0) + __popc(b1);
      }
      if (lane == 0) runs[reg] = cnt;
    }
    if (staged) {
      __syncwarp();   // the stage is consumed: refill it
      if (lane == 0 && c + FSTAGES < fe) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        issue(c + FSTAGES, st);
      }
      if (++st == FSTAGES) {
        st = 0;
        phase ^= 1u;
      }
    }
    tab_add(tab, p.block_w, lane, run2_a >= 0, run2_a, run2_w);
    tab_add(tab, p.block_w, lane, run_a >= 0, run_a, run_w);
  }
  for (int o = 16; o; o >>= 1) nskip += __shfl_xor_sync(FULL, nskip, o);
  if (lane == 0 && nskip) atomicAdd(&p.counters[0], nskip);
  tab_flush(tab, p.block_w, lane);
}

// -------------------------------------------------------------- scan kernel
constexpr int STH = 256;           // 8 warps
#ifndef GP_SCAN_OCC
#define GP_SCAN_OCC 3              // resident scan CTAs per SM the register budget targets
#endif
constexpr int CAPW = 96;           // candidates staged per warp

template <int D>
struct WarpCand {
  double c[D][CAPW];
  double inf[CAPW];
  double i2[CAPW];
  double lsq[CAPW];   // box lower bound (squared) of the staged candidate
  int cid[CAPW];
  int order[CAPW];    // candidates by increasing lsq (index tie-break)
};

template <int D>
__device__ __forceinline__ void stage(WarpCand<D>& W, int slot, int c, const gp_assign_args& p) {
#pragma unroll
  for (int j = 0; j < D; ++j) W.c[j][slot] = p.centers[c * D + j];
  W.inf[slot] = p.infl[c];
  W.i2[slot] = p.inv2_hi[c];
  W.cid[slot] = c;
}

// keep the two smallest (q, idx) and the third smallest q when adding (t, it)
__device__ __forceinline__ void top3_add(double& q1, int& i1, double& q2, int& i2, double& q3,
                                         double t, int it) {
  const bool l1 = t < q1 || (t == q1 && it < i1);
  const bool l2 = !l1 && (t < q2 || (t == q2 && it < i2));
  q3 = (l1 || l2) ? q2 : fmin(q3, t);
  q2 = l1 ? q1 : (l2 ? t : q2);
  i2 = l1 ? i1 : (l2 ? it : i2);
  q1 = l1 ? t : q1;
  i1 = l1 ? it : i1;
}

// squared distance / infl^2 (prefilter only; any rounding)
template <int D>
__device__ __forceinline__ double qdist(const double* x, const WarpCand<D>& W, int i) {
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double t = x[j] - W.c[j][i];
    s = fma(t, t, s);
  }
  return s * W.i2[i];
}

__device__ unsigned long long g_scan_stats[8];  // gp_scan_stats (flags bit 0)

constexpr int UCH = 4;             // scan units per scheduler claim (large rounds)
constexpr int SREG = 32;           // max filter regions per scan unit (runtime sreg <= SREG)
constexpr double SEP = 1e-12;      // q separation above which no exact evaluation is needed
constexpr float AP_HI_F = 1.0f + 2.4e-7f;  // margins of the sqrt(q)-derived float bounds
constexpr float AP_LO_F = 1.0f - 2.4e-7f;

// Visit the grid cells at Chebyshev distance r from cell (c0,c1,c2).
template <int D, typename F>
__device__ __forceinline__ void for_ring(const gp_assign_args& p, const int* cc, int r, F&& fn) {
  const int G = p.grid_n;
  if (D == 2) {
    for (int i = cc[0] - r; i <= cc[0] + r; ++i) {
      if (i < 0 || i >= G) continue;
      const bool edge = i == cc[0] - r || i == cc[0] + r;
      for (int j = cc[1] - r; j <= cc[1] + r; j += (edge || r == 0) ? 1 : 2 * r) {
        if (j < 0 || j >= G) continue;
        fn(i * G + j);
      }
    }
  } else {
    for (int i = cc[0] - r; i <= cc[0] + r; ++i) {
      if (i < 0 || i >= G) continue;
      for (int j = cc[1] - r; j <= cc[1] + r; ++j) {
        if (j < 0 || j >= G) continue;
        const bool face = i == cc[0] - r || i == cc[0] + r || j == cc[1] - r || j == cc[1] + r;
        for (int l = cc[2] - r; l <= cc[2] + r; l += (face || r == 0) ? 1 : 2 * r) {
          if (l < 0 || l >= G) continue;
          fn((i * G + j) * G + l);
        }
      }
    }
  }
}

// Exact argmin (lowest index) and runner-up of one point by a ring walk over the
// center grid: approximate q = d^2/infl^2 with the two smallest kept; a ring is
// the last one once every farther cell is at least r*h away, i.e. q >= (r h)^2 *
// inv2_min > q2 (1 + tol).  Near ties fall back to the reference's arithmetic on
// every visited candidate within the tolerance.
template <int D>
__device__ void grid_point(const gp_assign_args& p, const double* x, int& bi, float& bestf,
                           float& secondf, unsigned long long& nq) {
  const int G = p.grid_n;
  int cc[3] = {0, 0, 0};
#pragma unroll
  for (int j = 0; j < D; ++j) {
    int c = (int)floor((x[j] - p.grid_lo[j]) / p.grid_h);
    cc[j] = c < 0 ? 0 : (c >= G ? G - 1 : c);
  }
  double q1 = INFINITY, q2 = INFINITY, q3 = INFINITY;
  int i1 = 0x7fffffff, i2 = 0x7fffffff;
  int rlast = 0;
  for (int r = 0;; ++r) {
    for_ring<D>(p, cc, r, [&](int cell) {
      for (int t = p.grid_start[cell]; t < p.grid_start[cell + 1]; ++t) {
        const int c = p.grid_items[t];
        double s2 = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const double dd = x[j] - p.centers[c * D + j];
          s2 = fma(dd, dd, s2);
        }
        top3_add(q1, i1, q2, i2, q3, s2 * p.inv2_hi[c], c);
        ++nq;
      }
    });
    rlast = r;
    bool covered = true;
#pragma unroll
    for (int j = 0; j < D; ++j) covered = covered && cc[j] - r <= 0 && cc[j] + r >= G - 1;
    if (covered) break;
    const double rh = (double)r * p.grid_h;
    const double bound = __dmul_rd(__dmul_rd(rh, rh), inv2_min_of(p)) * (1.0 - 1e-9);
    if (bound > fma(q2, Q_TOL, q2)) break;
  }
  const double thr = fma(q2, Q_TOL, q2);
  if (q3 > thr && q2 > fma(q1, SEP, q1)) {
    bi = i1;
    bestf = __fmul_ru(__fsqrt_ru(__double2float_ru(q1)), AP_HI_F);
    secondf = i2 != 0x7fffffff ? __fmul_rd(__fsqrt_rd(__double2float_rd(q2)), AP_LO_F) : INFINITY;
    return;
  }
  double best = INFINITY, second = INFINITY;
  bi = 0x7fffffff;
  for (int r = 0; r <= rlast; ++r) {
    for_ring<D>(p, cc, r, [&](int cell) {
      for (int t = p.grid_start[cell]; t < p.grid_start[cell + 1]; ++t) {
        const int c = p.grid_items[t];
        double s2 = 0.0;
#pragma unroll
        for (int j = 0; j < D; ++j) {
          const double dd = x[j] - p.centers[c * D + j];
          s2 = fma(dd, dd, s2);
        }
        if (s2 * p.inv2_hi[c] <= thr) {
          const double dist = effdist_rn<D>(x, p.centers + c * D, p.infl[c], p.order3);
          const bool win = dist < best || (dist == best && c < bi);
          second = win ? best : fmin(second, dist);
          best = win ? dist : best;
          bi = win ? c : bi;
        }
      }
    });
  }
  bestf = __double2float_ru(best);
  secondf = __double2float_rd(second);
}

// ------------------------------------------------------------ walk kernel
// Sparse warm-up rounds (flags bit 1: few active points per center): one warp per
// rescanned point walks the center grid ring by ring around it, the lanes sharing
// each ring's cells, until the ring's lower bound exceeds the point's runner-up
// (the per-lane walk of grid_point, made warp-parallel).  No candidate selection
// over all k per scan unit and no divergent per-lane rings.  Same decision rule
// as grid_point: the approximate top three (q, index) decide unless the best two
// are within SEP or the third within Q_TOL of the runner-up; then the reference's
// exact arithmetic over every visited candidate within the tolerance.
template <int D>
__device__ __forceinline__ int ring_size(int r) {
  if (r == 0) return 1;
  return D == 2 ? 8 * r : (2 * r + 1) * (2 * r + 1) * (2 * r + 1);
}
// cell e of the ring at Chebyshev distance r around cc (-1: outside the grid, or for
// 3D an interior cell of the enumerated cube)
template <int D>
__device__ __forceinline__ int ring_cell(const int* cc, int r, int e, int G) {
  int i[3] = {cc[0], cc[1], D == 3 ? cc[2] : 0};
  if (r > 0) {
    if (D == 2) {
      const int side = e / (2 * r), off = e - side * 2 * r;
      if (side == 0) { i[0] = cc[0] - r + off; i[1] = cc[1] - r; }
      else if (side == 1) { i[0] = cc[0] + r; i[1] = cc[1] - r + off; }
      else if (side == 2) { i[0] = cc[0] + r - off; i[1] = cc[1] + r; }
      else { i[0] = cc[0] - r; i[1] = cc[1] + r - off; }
    } else {
      const int n = 2 * r + 1;
      const int a = e / (n * n), b = (e / n) % n, c = e % n;
      if (a > 0 && a < n - 1 && b > 0 && b < n - 1 && c > 0 && c < n - 1) return -1;
      i[0] = cc[0] - r + a;
      i[1] = cc[1] - r + b;
      i[2] = cc[2] - r + c;
    }
  }
  int cell = 0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    if (i[j] < 0 || i[j] >= G) return -1;
    cell = cell * G + i[j];
  }
  return cell;
}

constexpr int WKT = 256;

template <int D, int WM>
__global__ void __launch_bounds__(WKT) walk_kernel(gp_assign_args p, int wshift, int64_t nregions,
                                                   const int2* __restrict__ ent,
                                                   const int32_t* __restrict__ runs) {
  typedef typename std::conditional<WM == GP_W_UNIT, int, long long>::type RunW;
  __shared__ WarpTab s_tab[WKT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  WarpTab& tab = s_tab[warp];
  tab_init(tab, lane);
  const int G = p.grid_n;
  unsigned long long nq = 0;
  const int64_t nitems = nregions * WREG;
  for (int64_t item = (int64_t)blockIdx.x * (WKT / 32) + warp; item < nitems;
       item += (int64_t)gridDim.x * (WKT / 32)) {
    const int64_t r = item / WREG;
    const int v = (int)(item - r * WREG);
    if (v >= runs[r]) continue;
    const int64_t slot = r * WREG + v;
    const int2 e = ent[slot];
    const int q = e.x;
    double x[D];
    load_point<D>(p.X, p.ldx, q, x);
    int cc[3] = {0, 0, 0};
#pragma unroll
    for (int j = 0; j < D; ++j) {
      const int c = (int)floor((x[j] - p.grid_lo[j]) / p.grid_h);
      cc[j] = c < 0 ? 0 : (c >= G ? G - 1 : c);
    }
    double q1 = INFINITY, q2 = INFINITY, q3 = INFINITY;
    int i1 = 0x7fffffff, i2 = 0x7fffffff;
    int rlast = 0;
    for (int rr = 0;; ++rr) {
      const int nc = ring_size<D>(rr);
      for (int e = lane; e < nc; e += 32) {
        const int cell = ring_cell<D>(cc, rr, e, G);
        if (cell < 0) continue;
        for (int t = p.grid_start[cell]; t < p.grid_start[cell + 1]; ++t) {
          const int c = p.grid_items[t];
          double s2 = 0.0;
#pragma unroll
          for (int j = 0; j < D; ++j) {
            const double dd = x[j] - p.centers[c * D + j];
            s2 = fma(dd, dd, s2);
          }
          top3_add(q1, i1, q2, i2, q3, s2 * p.inv2_hi[c], c);
          ++nq;
        }
      }
      double m1 = q1, m2 = q2;
      for (int o = 16; o; o >>= 1) {
        const double b1 = __shfl_xor_sync(FULL, m1, o);
        const double b2 = __shfl_xor_sync(FULL, m2, o);
        two_min_merge(m1, m2, b1, b2);
      }
      rlast = rr;
      bool covered = true;
#pragma unroll
      for (int j = 0; j < D; ++j) covered = covered && cc[j] - rr <= 0 && cc[j] + rr >= G - 1;
      if (covered) break;
      const double rh = (double)rr * p.grid_h;
      const double bound = __dmul_rd(__dmul_rd(rh, rh), inv2_min_of(p)) * (1.0 - 1e-9);
      if (bound > fma(m2, Q_TOL, m2)) break;
    }
    // union of the lanes' top-3 lists (every center was evaluated by one lane)
    for (int o = 16; o; o >>= 1) {
      const double b1 = __shfl_xor_sync(FULL, q1, o), b2 = __shfl_xor_sync(FULL, q2, o);
      const double b3 = __shfl_xor_sync(FULL, q3, o);
      const int j1 = __shfl_xor_sync(FULL, i1, o), j2 = __shfl_xor_sync(FULL, i2, o);
      top3_add(q1, i1, q2, i2, q3, b1, j1);
      top3_add(q1, i1, q2, i2, q3, b2, j2);
      q3 = fmin(q3, b3);
    }
    const double thr = fma(q2, Q_TOL, q2);
    int bi;
    float bestf, secondf;
    if (q3 > thr && q2 > fma(q1, SEP, q1)) {
      bi = i1;
      bestf = __fmul_ru(__fsqrt_ru(__double2float_ru(q1)), AP_HI_F);
      secondf = i2 != 0x7fffffff ? __fmul_rd(__fsqrt_rd(__double2float_rd(q2)), AP_LO_F)
                                 : INFINITY;
    } else {
      double best = INFINITY, second = INFINITY;
      int bix = 0x7fffffff;
      for (int rr = 0; rr <= rlast; ++rr) {
        const int nc = ring_size<D>(rr);
        for (int e = lane; e < nc; e += 32) {
          const int cell = ring_cell<D>(cc, rr, e, G);
          if (cell < 0) continue;
          for (int t = p.grid_start[cell]; t < p.grid_start[cell + 1]; ++t) {
            const int c = p.grid_items[t];
            double s2 = 0.0;
#pragma unroll
            for (int j = 0; j < D; ++j) {
              const double dd = x[j] - p.centers[c * D + j];
              s2 = fma(dd, dd, s2);
            }
            if (s2 * p.inv2_hi[c] <= thr) {
              const double dist = effdist_rn<D>(x, p.centers + c * D, p.infl[c], p.order3);
              const bool win = dist < best || (dist == best && c < bix);
              second = win ? best : fmin(second, dist);
              best = win ? dist : best;
              bix = win ? c : bix;
            }
          }
        }
      }
      for (int o = 16; o; o >>= 1) {
        const double ob = __shfl_xor_sync(FULL, best, o), os = __shfl_xor_sync(FULL, second, o);
        const int oi = __shfl_xor_sync(FULL, bix, o);
        const bool mine = best < ob || (best == ob && bix < oi);
        second = mine ? fmin(second, ob) : fmin(os, best);
        best = mine ? best : ob;
        bix = mine ? bix : oi;
      }
      bi = bix;
      bestf = __double2float_ru(best);
      secondf = __double2float_rd(second);
    }
    RunW wv = 0;
    if (lane == 0) {
      if (e.y != bi) p.a[q] = bi;
      store_bounds(p, lb_params(p, r * WREG), q, bi, bestf, secondf);
      wv = (RunW)weight_units<WM>(p.w, q, wshift);
    }
    tab_add(tab, p.block_w, lane, lane == 0, bi, wv);
  }
  for (int o = 16; o; o >>= 1) nq += __shfl_xor_sync(FULL, nq, o);
  if (lane == 0 && nq) atomicAdd(&p.counters[2], nq);
  tab_flush(tab, p.block_w, lane);
}

// near tie (or overflowed candidate set): the reference's exact arithmetic over every
// candidate within the tolerance, (dist, index) tie-break.  Out of line: it is the
// cold path, and keeping its IEEE div/sqrt sequences out of the scan loop keeps that
// loop's code small (instruction-cache misses were a fifth of the scan's stalls).
template <int D>
__device__ __forceinline__ void exact_argmin(const gp_assign_args& p, WarpCand<D>& W,
                                          const int32_t* src, int total, bool overflow,
                                          bool valid, const double* x, double thr, int lane,
                                          int& bi, float& bestf, float& secondf,
                                          unsigned long long& nexact) {
  double best = INFINITY, second = INFINITY;
  int b = 0x7fffffff;
  for (int c0 = 0; c0 < total; c0 += CAPW) {
    const int cn = min(CAPW, total - c0);
    if (overflow) {
      __syncwarp();
      for (int i = lane; i < cn; i += 32) stage<D>(W, i, src ? src[c0 + i] : c0 + i, p);
      __syncwarp();
    }
    for (int i = 0; i < cn; ++i) {
      if (valid && qdist<D>(x, W, i) <= thr) {
        double cc[D];
#pragma unroll
        for (int j = 0; j < D; ++j) cc[j] = W.c[j][i];
        const double dist = effdist_rn<D>(x, cc, W.inf[i], p.order3);
        const int cid = W.cid[i];
        const bool win = dist < best || (dist == best && cid < b);
        second = win ? best : fmin(second, dist);
        best = win ? dist : best;
        b = win ? cid : b;
        ++nexact;
      }
    }
  }
  bi = b;
  bestf = __double2float_ru(best);
  secondf = __double2float_rd(second);
}

template <int D, int WM>
__global__ void __launch_bounds__(STH, GP_SCAN_OCC) scan_kernel(gp_assign_args p, int wshift, int64_t nregions,
                                                   int sreg, const int2* __restrict__ ent,
                                                   const int32_t* __restrict__ runs,
                                                   unsigned long long* __restrict__ sched,
                                                   int uch, int pshift) {
  typedef typename std::conditional<WM == GP_W_UNIT, int, long long>::type RunW;
  __shared__ WarpCand<D> WCs[STH / 32];
  __shared__ WarpTab s_tab[STH / 32];
  __shared__ int s_rbeg[STH / 32][SREG];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  WarpCand<D>& W = WCs[warp];
  WarpTab& tab = s_tab[warp];
  tab_init(tab, lane);
  unsigned long long nq = 0, nexact = 0;
  const int64_t nunits = (nregions + sreg - 1) / sreg;
  // dynamic schedule: warps take chunks of UCH consecutive units from a counter (the
  // next chunk is claimed one chunk ahead), so no warp idles while others finish
  auto grab = [&]() -> int64_t {
    unsigned long long c = 0;
    if (lane == 0) c = atomicAdd(sched, 1ull);
    return (int64_t)__shfl_sync(FULL, c, 0) * uch;
  };
  // work items: unit u, passes sub, sub + 2^pshift, ... (pshift > 0 spreads the passes
  // of a small round's few units over more warps)
  const int64_t nitems = nunits << pshift;
  const int pstride = 32 << pshift;
  int64_t item = grab(), next_chunk = grab();
  // counts of the unit's regions (lane r < sreg holds region r's), prefetched one item ahead
  auto counts_of = [&](int64_t it) {
    const int64_t u = it >> pshift;
    return (it < nitems && lane < sreg && u * sreg + lane < nregions) ? runs[u * sreg + lane] : 0;
  };
  int my_cnt = counts_of(item);
  int64_t cur_g = -1;          // group whose candidate list src / nsrc hold
  const int32_t* src = nullptr;
  int nsrc = p.k;
  for (int64_t nxt; item < nitems; item = nxt) {
    const int cnt_here = my_cnt;
    const int64_t unit = item >> pshift;
    const int p0 = (int)(item & ((1 << pshift) - 1)) * 32;   // first pass of this item
    if ((item + 1) % uch != 0 && item + 1 < nitems) {
      nxt = item + 1;
    } else {
      nxt = next_chunk;
      if (nxt < nitems) next_chunk = grab();
    }
    my_cnt = counts_of(nxt);
    // prefix over the SREG region counts (lanes 0..SREG-1)
    int incl = cnt_here;
#pragma unroll
    for (int o = 1; o < SREG; o <<= 1) {
      const int t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    const int total_pts = __shfl_sync(FULL, incl, sreg - 1);
    if (total_pts <= p0) continue;
    // first scanned point of each region of the unit (shared memory, no registers)
    int* rbeg = s_rbeg[warp];
    __syncwarp();
    if (lane < sreg) rbeg[lane] = incl - cnt_here;
    __syncwarp();
    // v-th scanned point of the unit -> slot: the last region r with rbeg[r] <= v
    auto slot_of = [&](int v) {
      int lo = 0, hi = sreg - 1;
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (rbeg[mid] <= v) lo = mid;
        else hi = mid - 1;
      }
      return (unit * sreg + lo) * WREG + (v - rbeg[lo]);
    };
    auto pos_of = [&](int v) { return ent[slot_of(v)]; };   // (position, old block)
    // software pipeline of the passes: positions two passes ahead, coordinates one
    // pass ahead; the first pass's loads overlap the candidate selection below
    const int2 zero2 = make_int2(0, -1);
    int2 qA = p0 + lane < total_pts ? pos_of(p0 + lane) : zero2;
    int2 qB = p0 + pstride + lane < total_pts ? pos_of(p0 + pstride + lane) : zero2;
    // candidate source: the group's hierarchical list, or all k centers
    if (p.group_list) {
      const int64_t g = (unit * sreg * WREG) >> p.group_shift;
      if (g != cur_g) {   // consecutive units mostly share their group
        cur_g = g;
        const int gc = p.group_count[g];
        src = gc >= 0 ? p.group_list + g * (int64_t)p.group_cap : nullptr;
        nsrc = gc >= 0 ? gc : p.k;
      }
    }
    const float4 Lr = lb_params(p, unit * sreg * WREG);
    // ---- box: the unit's static box (all its active entries), or the box of the
    // unit's scanned points
    double lo[D], hi[D];
    if (p.unit_boxes) {
      const int64_t u = (unit * sreg * WREG) >> p.unit_shift;
#pragma unroll
      for (int j = 0; j < D; ++j) {
        lo[j] = p.unit_boxes[u * 2 * D + j];
        hi[j] = p.unit_boxes[u * 2 * D + D + j];
      }
    } else {
#pragma unroll
      for (int j = 0; j < D; ++j) {
        lo[j] = INFINITY;
        hi[j] = -INFINITY;
      }
      for (int v = lane; v < total_pts; v += 32) {
        const int q = pos_of(v).x;
        double xq[D];
        load_point<D>(p.X, p.ldx, q, xq);
#pragma unroll
        for (int j = 0; j < D; ++j) {
          lo[j] = fmin(lo[j], xq[j]);
          hi[j] = fmax(hi[j], xq[j]);
        }
      }
#pragma unroll
      for (int j = 0; j < D; ++j)
        for (int o = 16; o; o >>= 1) {
          lo[j] = fmin(lo[j], __shfl_xor_sync(FULL, lo[j], o));
          hi[j] = fmax(hi[j], __shfl_xor_sync(FULL, hi[j], o));
        }
    }
    // ---- candidates: lsq <= second smallest usq over the source
    double m1 = INFINITY, m2 = INFINITY;
    for (int i = lane; i < nsrc; i += 32) {
      const int c = src ? src[i] : i;
      two_min_merge(m1, m2, box_usq<D>(p.centers + c * D, lo, hi, p.inv2_hi[c]), INFINITY);
    }
    for (int o = 16; o; o >>= 1) {
      const double b1 = __shfl_xor_sync(FULL, m1, o);
      const double b2 = __shfl_xor_sync(FULL, m2, o);
      two_min_merge(m1, m2, b1, b2);
    }
    const double U = m2;  // +inf when only one center exists
    int ncand = 0;
    for (int b = 0; b < nsrc; b += 32) {
      const int i = b + lane;
      bool take = false;
      int c = 0;
      double take_lsq = 0.0;
      if (i < nsrc) {
        c = src ? src[i] : i;
        take_lsq = box_lsq<D>(p.centers + c * D, lo, hi, p.inv2_lo[c]);
        take = take_lsq <= U;
      }
      const unsigned bal = __ballot_sync(FULL, take);
      const int slot = ncand + __popc(bal & ((1u << lane) - 1));
      if (take && slot < CAPW) {
        stage<D>(W, slot, c, p);
        W.lsq[slot] = take_lsq;
      }
      ncand += __popc(bal);
    }
    const bool overflow = ncand > CAPW;  // then stream the whole source in chunks
    const int total = overflow ? nsrc : ncand;
    double xA[D];
    load_point<D>(p.X, p.ldx, qA.x, xA);  // first pass's coordinates (q = 0 when unused)
    if ((p.flags & 1) && lane == 0) {
      atomicAdd(&g_scan_stats[0], 1ull);
      atomicAdd(&g_scan_stats[1], (unsigned long long)total_pts);
      atomicAdd(&g_scan_stats[2], (unsigned long long)nsrc);
      atomicAdd(&g_scan_stats[3], (unsigned long long)ncand);
      atomicAdd(&g_scan_stats[4], overflow ? 1ull : 0ull);
      atomicAdd(&g_scan_stats[7], (unsigned long long)((total_pts + 31) / 32));
    }
    __syncwarp();
    if (!overflow) {
      // rank sort of the staged candidates by (lsq, slot): the per-point walk
      // below visits them in this order and stops once lsq exceeds its runner-up
      for (int i = lane; i < ncand; i += 32) {
        const double li = W.lsq[i];
        int r = 0;
        for (int j = 0; j < ncand; ++j) {
          const double lj = W.lsq[j];
          r += (lj < li) || (lj == li && j < i);
        }
        W.order[r] = i;
      }
      __syncwarp();
    }
    if (overflow && p.grid_n > 0) {
      // too many candidates for the staged set (sparse warm-up samples): every lane
      // walks the center grid around its own point, ring by ring, until the ring's
      // lower bound exceeds its runner-up
      for (int vb = p0; vb < total_pts; vb += pstride) {
        const int v = vb + lane;
        const bool valid = v < total_pts;
        int bi = -1, q = 0;
        int old = -1;
        if (valid) {
          const int2 e = pos_of(v);
          q = e.x;
          old = e.y;
          double x[D];
          load_point<D>(p.X, p.ldx, q, x);
          float bestf, secondf;
          unsigned long long nn = 0;
          grid_point<D>(p, x, bi, bestf, secondf, nn);
          nq += nn;
          if (old != bi) p.a[q] = bi;
          store_bounds(p, Lr, q, bi, bestf, secondf);
        }
        tab_add(tab, p.block_w, lane, valid, bi,
                valid ? (RunW)weight_units<WM>(p.w, q, wshift) : (RunW)0);
      }
      continue;
    }
    // ---- scan, one point per lane per pass
    for (int pb = p0; pb < total_pts; pb += pstride) {
      const int v = pb + lane;
      const bool valid = v < total_pts;
      const int q = valid ? qA.x : 0;
      const int oa = valid ? qA.y : -1;
      double x[D];
#pragma unroll
      for (int j = 0; j < D; ++j) x[j] = xA[j];
      if (pb + pstride < total_pts) {
        qA = qB;
        load_point<D>(p.X, p.ldx, qA.x, xA);
        qB = pb + 2 * pstride + lane < total_pts ? pos_of(pb + 2 * pstride + lane) : zero2;
      }
      // single pass: the two smallest q = d^2/infl^2 with their slots, and the third value
      double q1 = INFINITY, q2 = INFINITY, q3 = INFINITY;
      int i1 = -1, i2 = -1;
      if (!overflow) {
        // walk by increasing box lower bound; a lane is done once the next bound
        // exceeds its runner-up (+ tolerance): no later candidate can matter
        bool done = !valid;
        for (int t = 0; t < total; ++t) {
          const int i = W.order[t];
          done = done || W.lsq[i] > fma(q2, Q_TOL, q2);
          if (__all_sync(FULL, done)) break;
          if ((p.flags & 1) && lane == 0) atomicAdd(&g_scan_stats[6], 1ull);
          if (!done) {
            const double qq = qdist<D>(x, W, i);
            const bool l1 = qq < q1, l2 = qq < q2;
            q3 = l2 ? q2 : fmin(q3, qq);
            q2 = l1 ? q1 : (l2 ? qq : q2);
            i2 = l1 ? i1 : (l2 ? i : i2);
            q1 = l1 ? qq : q1;
            i1 = l1 ? i : i1;
            ++nq;
          }
        }
      } else {
        for (int c0 = 0; c0 < total; c0 += CAPW) {
          const int cn = min(CAPW, total - c0);
          __syncwarp();
          for (int i = lane; i < cn; i += 32) stage<D>(W, i, src ? src[c0 + i] : c0 + i, p);
          __syncwarp();
          for (int i = 0; i < cn; ++i) {
            const double t = qdist<D>(x, W, i);
            const bool l1 = t < q1, l2 = t < q2;
            q3 = l2 ? q2 : fmin(q3, t);
            q2 = l1 ? q1 : (l2 ? t : q2);
            q1 = l1 ? t : q1;
          }
          nq += valid ? cn : 0;
        }
      }
      const double thr = fma(q2, Q_TOL, q2);
      float bestf, secondf;
      int bi;
      const bool simple = q3 > thr;  // exactly the slots i1, i2 can hold the best two
      const bool clear = simple && q2 > fma(q1, SEP, q1);
      if (clear && !overflow) {
        // well separated: i1 is the exact argmin; sound float32 bounds straight from
        // sqrt(q) (relative error of q ~1e-15 << the 2^-22 margin)
        bi = W.cid[i1];
        bestf = __fmul_ru(__fsqrt_ru(__double2float_ru(q1)), AP_HI_F);
        secondf = i2 >= 0 ? __fmul_rd(__fsqrt_rd(__double2float_rd(q2)), AP_LO_F) : INFINITY;
      } else {
        exact_argmin<D>(p, W, src, total, overflow, valid, x, thr, lane, bi, bestf, secondf,
                        nexact);
      }
      // ---- write back + block weights of the scanned points
      RunW wv = 0;
      int c = -1;
      if (valid) {
        c = bi;
        if (oa != c) p.a[q] = c;   // most rescans keep their block
        store_bounds(p, Lr, q, c, bestf, secondf);
        wv = (RunW)weight_units<WM>(p.w, q, wshift);
      }
      tab_add(tab, p.block_w, lane, valid, c, wv);
    }
    __syncwarp();
  }
  for (int o = 16; o; o >>= 1) {
    nq += __shfl_xor_sync(FULL, nq, o);
    nexact += __shfl_xor_sync(FULL, nexact, o);
  }
  if (lane == 0 && nq) atomicAdd(&p.counters[2], nq);
  if ((p.flags & 1) && lane == 0) atomicAdd(&g_scan_stats[5], nexact);
  tab_flush(tab, p.block_w, lane);
}

// ------------------------------------------------------------------ audit
template <int D>
__global__ void audit_kernel(gp_assign_args p, unsigned long long* out) {
  unsigned long long aud = 0, viol = 0, bad = 0;
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < p.m;
       li += (int64_t)gridDim.x * blockDim.x) {
    const int q = p.list ? p.list[li] : (int)li;
    double x[D];
    load_point<D>(p.X, p.ldx, q, x);
    const int a = p.a[q];
    const float2 bnd =
        bnd_unpack(reinterpret_cast<const unsigned*>(p.ublb)[q], __frcp_rn(p.bound_scale));
    double m1 = INFINITY, m2 = INFINITY, own = 0.0;
    int arg = 0;
    for (int c = 0; c < p.k; ++c) {
      double cc[D];
#pragma unroll
      for (int j = 0; j < D; ++j) cc[j] = p.centers[c * D + j];
      const double dist = effdist_rn<D>(x, cc, p.infl[c], p.order3);
      if (c == (a >= 0 ? a : 0)) own = dist;
      if (dist < m1) {
        m2 = m1;
        m1 = dist;
        arg = c;
      } else {
        m2 = fmin(m2, dist);
      }
    }
    const double ub =
        a >= 0 ? ub_evalf(reinterpret_cast<const float4*>(p.ub_eval)[a], bnd.x) : INFINITY;
    const float4 L = lb_params(p, li);
    const double lb = lb_evalf(L.x, bnd.y, L.y);
    ++aud;
    if (a >= 0 && ub < own) ++viol;
    if (p.k > 1 && lb > m2) ++viol;
    if (a >= 0 && ub < lb && arg != a) ++bad;
  }
  atomicAdd(&out[0], aud);
  atomicAdd(&out[1], viol);
  atomicAdd(&out[2], bad);
}

// lower bounds of the active entries between the global map and region maps:
// mode 0: materialise under the global map (identity region maps follow);
// mode 1: region maps -> normalised under the global map again
__global__ void lb_remap_kernel(gp_assign_args p, int mode) {
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < p.m;
       li += (int64_t)gridDim.x * blockDim.x) {
    const int q = p.list ? p.list[li] : (int)li;
    float2 bnd =
        bnd_unpack(reinterpret_cast<const unsigned*>(p.ublb)[q], __frcp_rn(p.bound_scale));
    const float4 G = *reinterpret_cast<const float4*>(p.lb_par);
    if (mode == 0) {
      bnd.y = lb_evalf(G.x, bnd.y, G.y);
    } else {
      const float4 L = reinterpret_cast<const float4*>(p.lb_rpar)[li >> p.lb_rshift];
      bnd.y = lb_normf(G.z, G.w, lb_evalf(L.x, bnd.y, L.y));
    }
    reinterpret_cast<unsigned*>(p.ublb)[q] = bnd_pack(bnd.x, bnd.y, p.bound_scale);
  }
}

__global__ void rebase_kernel(gp_assign_args p) {
  for (int64_t li = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; li < p.m;
       li += (int64_t)gridDim.x * blockDim.x) {
    const int q = p.list ? p.list[li] : (int)li;
    const int a = p.a[q];
    const float2 bnd =
        bnd_unpack(reinterpret_cast<const unsigned*>(p.ublb)[q], __frcp_rn(p.bound_scale));
    // the host resets the maps to identity after this pass: store the values themselves
    const float ub = a >= 0 ? ub_evalf(reinterpret_cast<const float4*>(p.ub_eval)[a], bnd.x)
                            : bnd.x;
    const float4 L = lb_params(p, li);
    reinterpret_cast<unsigned*>(p.ublb)[q] = bnd_pack(ub, lb_evalf(L.x, bnd.y, L.y), p.bound_scale);
  }
}

// ----------------------------------------------------- hierarchical groups
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
    const int64_t q = list ? list[li] : li;
    double xq[D];
    load_point<D>(X, ldx, q, xq);
#pragma unroll
    for (int j = 0; j < D; ++j) {
      lo[j] = fmin(lo[j], xq[j]);
      hi[j] = fmax(hi[j], xq[j]);
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
    const int j = threadIdx.x;
    double v = s_red[j][0];
    for (int w = 1; w < (int)(blockDim.x / 32); ++w)
      v = j < D ? fmin(v, s_red[j][w]) : fmax(v, s_red[j][w]);
    boxes[g * 2 * D + j] = v;
  }
}

template <int D>
__global__ void __launch_bounds__(1024) group_candidates_kernel(
    const double* __restrict__ boxes, int k, const double* __restrict__ centers,
    const double* __restrict__ inv2_lo, const double* __restrict__ inv2_hi,
    const int32_t* __restrict__ parent_list, const int32_t* __restrict__ parent_count,
    int parent_cap, int ratio_log2, int32_t* __restrict__ list, int32_t* __restrict__ count,
    int cap) {
  __shared__ double s_two[2][32];
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
    const int64_t pg = g >> ratio_log2;
    const int pc = parent_count[pg];
    if (pc >= 0) {
      src = parent_list + pg * (int64_t)parent_cap;
      nsrc = pc;
    }
  }
  // four candidates per thread and step: their list entries, centers and 1/infl^2 bounds
  // are loaded together (the loops are bound by the latency of these dependent loads)
  constexpr int UN = 4;
  double m1 = INFINITY, m2 = INFINITY;
  for (int b = 0; b < nsrc; b += (int)blockDim.x * UN) {
    int c[UN];
    double cen[UN][D], iv[UN];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int i = b + (int)blockDim.x * u + (int)threadIdx.x;
      c[u] = i < nsrc ? (src ? src[i] : i) : -1;
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int cc = c[u] < 0 ? 0 : c[u];
#pragma unroll
      for (int j = 0; j < D; ++j) cen[u][j] = centers[cc * D + j];
      iv[u] = inv2_hi[cc];
    }
#pragma unroll
    for (int u = 0; u < UN; ++u)
      if (c[u] >= 0) two_min_merge(m1, m2, box_usq<D>(cen[u], lo, hi, iv[u]), INFINITY);
  }
  for (int o = 16; o; o >>= 1) {
    const double b1 = __shfl_xor_sync(FULL, m1, o);
    const double b2 = __shfl_xor_sync(FULL, m2, o);
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
  for (int b = 0; b < nsrc; b += (int)blockDim.x * UN) {
    int c[UN];
    double cen[UN][D], iv[UN];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int i = b + (int)blockDim.x * u + (int)threadIdx.x;
      c[u] = i < nsrc ? (src ? src[i] : i) : -1;
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int cc = c[u] < 0 ? 0 : c[u];
#pragma unroll
      for (int j = 0; j < D; ++j) cen[u][j] = centers[cc * D + j];
      iv[u] = inv2_lo[cc];
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      if (c[u] >= 0 && box_lsq<D>(cen[u], lo, hi, iv[u]) <= U) {
        const int slot = atomicAdd(&s_n, 1);
        if (slot < cap) out[slot] = c[u];
      }
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) count[g] = s_n <= cap ? s_n : -1;
}

// One warp per group (sources of at most a few thousand centers, e.g. super groups
// under a mega list): same candidate set as group_candidates_kernel, without a
// 256-thread block and two block barriers per group.
template <int D>
__global__ void __launch_bounds__(256) group_candidates_warp_kernel(
    const double* __restrict__ boxes, int64_t ngroups, int k, const double* __restrict__ centers,
    const double* __restrict__ inv2_lo, const double* __restrict__ inv2_hi,
    const int32_t* __restrict__ parent_list, const int32_t* __restrict__ parent_count,
    int parent_cap, int ratio_log2, int32_t* __restrict__ list, int32_t* __restrict__ count,
    int cap) {
  const int lane = threadIdx.x & 31;
  const int64_t g = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (g >= ngroups) return;
  double lo[D], hi[D];
#pragma unroll
  for (int j = 0; j < D; ++j) {
    lo[j] = boxes[g * 2 * D + j];
    hi[j] = boxes[g * 2 * D + D + j];
  }
  if (!(lo[0] <= hi[0])) {  // empty group
    if (lane == 0) count[g] = 0;
    return;
  }
  const int32_t* src = nullptr;
  int nsrc = k;
  if (parent_list) {
    const int64_t pg = g >> ratio_log2;
    const int pc = parent_count[pg];
    if (pc >= 0) {
      src = parent_list + pg * (int64_t)parent_cap;
      nsrc = pc;
    }
  }
  // four candidates per lane and step: their list entries, centers and 1/infl^2 bounds are
  // loaded together (the loop is bound by the latency of these dependent loads)
  constexpr int UN = 4;
  double m1 = INFINITY, m2 = INFINITY;
  for (int b = 0; b < nsrc; b += 32 * UN) {
    int c[UN];
    double cen[UN][D], iv[UN];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int i = b + 32 * u + lane;
      c[u] = i < nsrc ? (src ? src[i] : i) : -1;
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int cc = c[u] < 0 ? 0 : c[u];
#pragma unroll
      for (int j = 0; j < D; ++j) cen[u][j] = centers[cc * D + j];
      iv[u] = inv2_hi[cc];
    }
#pragma unroll
    for (int u = 0; u < UN; ++u)
      if (c[u] >= 0) two_min_merge(m1, m2, box_usq<D>(cen[u], lo, hi, iv[u]), INFINITY);
  }
  for (int o = 16; o; o >>= 1) {
    const double b1 = __shfl_xor_sync(FULL, m1, o);
    const double b2 = __shfl_xor_sync(FULL, m2, o);
    two_min_merge(m1, m2, b1, b2);
  }
  const double U = m2;
  int32_t* out = list + g * (int64_t)cap;
  int n = 0;
  for (int b = 0; b < nsrc; b += 32 * UN) {
    int c[UN];
    double cen[UN][D], iv[UN];
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int i = b + 32 * u + lane;
      c[u] = i < nsrc ? (src ? src[i] : i) : -1;
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) {
      const int cc = c[u] < 0 ? 0 : c[u];
#pragma unroll
      for (int j = 0; j < D; ++j) cen[u][j] = centers[cc * D + j];
      iv[u] = inv2_lo[cc];
    }
#pragma unroll
    for (int u = 0; u < UN; ++u) {   // entry order: sub-step u, then lane
      const bool take = c[u] >= 0 && box_lsq<D>(cen[u], lo, hi, iv[u]) <= U;
      const unsigned bal = __ballot_sync(FULL, take);
      const int slot = n + __popc(bal & ((1u << lane) - 1));
      if (take && slot < cap) out[slot] = c[u];
      n += __popc(bal);
    }
  }
  if (lane == 0) count[g] = n <= cap ? n : -1;
}

// ------------------------------------------------------------ bound maps
// Mirror of control.BoundMaps.relax + device_params for one CTA.
constexpr double UBS = 1.0 + 1e-12, LBS = 1.0 - 1e-12;

// gp_update_maps in three steps over many CTAs (it used to be one 1024-thread CTA,
// ~50 us per round at k = 16384):
//  1. maps_ratio_kernel: per cluster ratio = I_old/I_new and shift = move/I_new
//     (kept for gp_region_maps) and the global min ratio, max shift and "anything
//     changed" as order-preserving atomics (both are >= 0);
//  2. maps_global_kernel (one thread): the lower-bound map A, B, steps and lb_par;
//  3. maps_cluster_kernel: the per-cluster maps and parameters.
// state layout: S[k] | T[k] | A, B, steps | rmin, smax, any, max infl, inv2_min |
//               ratio[k] | shift[k]   (gp_map_state_size)
__global__ void maps_ratio_kernel(const double* __restrict__ old_infl,
                                  const double* __restrict__ new_infl,
                                  const double* __restrict__ moves, int k,
                                  double* __restrict__ st) {
  double* scr = st + 2 * k + 3;
  double* ratio = st + 2 * k + 8;
  double* shift = ratio + k;
  double rmin = INFINITY, smax = 0.0, imax = 0.0;
  int any = 0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) {
    const double mv = moves ? moves[c] : 0.0;
    any |= (mv != 0.0) || (old_infl[c] != new_infl[c]);
    imax = fmax(imax, new_infl[c]);
    const double r = old_infl[c] / new_infl[c];
    const double sh = mv / new_infl[c];
    ratio[c] = r;
    shift[c] = sh;
    rmin = fmin(rmin, r);
    smax = fmax(smax, sh);
  }
  for (int o = 16; o; o >>= 1) {
    rmin = fmin(rmin, __shfl_xor_sync(FULL, rmin, o));
    smax = fmax(smax, __shfl_xor_sync(FULL, smax, o));
    imax = fmax(imax, __shfl_xor_sync(FULL, imax, o));
    any |= __shfl_xor_sync(FULL, any, o);
  }
  if ((threadIdx.x & 31) == 0) {
    unsigned long long* u = reinterpret_cast<unsigned long long*>(scr);
    atomicMin(&u[0], (unsigned long long)__double_as_longlong(rmin));   // doubles >= 0
    atomicMax(&u[1], (unsigned long long)__double_as_longlong(smax));
    if (any) atomicOr(&u[2], 1ull);
    atomicMax(&u[3], (unsigned long long)__double_as_longlong(imax));
  }
}

__global__ void maps_global_kernel(int k, double* __restrict__ st, float* __restrict__ lb_par,
                                   int32_t* __restrict__ flags, int reset, double scale_hint) {
  double* ABs = st + 2 * k;
  const unsigned long long* u = reinterpret_cast<const unsigned long long*>(st + 2 * k + 3);
  const double rmin = __longlong_as_double((long long)u[0]);
  const double smax = __longlong_as_double((long long)u[1]);
  // the host's 1.0 / float(max(infl)) ** 2 * (1.0 - 1e-15), on the device
  const double imax = __longlong_as_double((long long)u[3]);
  st[2 * k + 7] = __dmul_rn(__ddiv_rn(1.0, __dmul_rn(imax, imax)), 1.0 - 1e-15);
  // relax_bounds' identity early return (kmeans.py:223-228)
  const bool compose = !reset && u[2] != 0;
  double A = reset ? 1.0 : ABs[0], B = reset ? 0.0 : ABs[1], steps = reset ? 0.0 : ABs[2];
  if (compose) {
    A = A * rmin * LBS;
    B = (B * rmin + smax) * LBS;
    steps += 1.0;
  }
  const double e = (4.0 * steps + 16.0) * 0x1p-52;
  ABs[0] = A;
  ABs[1] = B;
  ABs[2] = steps;
  lb_par[0] = __double2float_rd(__dmul_rd(A, 1.0 - e));
  lb_par[1] = __double2float_ru(__dmul_ru(B, 1.0 + e));
  lb_par[2] = __double2float_rd(__ddiv_rd(1.0, A));
  lb_par[3] = __double2float_rd(B);
  if (A < 1e-6 || A > 1e6 || B > 64.0 * scale_hint) flags[0] = 1;
}

__global__ void maps_cluster_kernel(const double* __restrict__ new_infl, int k,
                                    double* __restrict__ st, double* __restrict__ inv2_lo,
                                    double* __restrict__ inv2_hi, float4* __restrict__ ub_eval,
                                    float4* __restrict__ ub_norm, int32_t* __restrict__ flags,
                                    int reset, double scale_hint) {
  double* S = st;
  double* T = st + k;
  const double steps = st[2 * k + 2];   // already composed by maps_global_kernel
  const unsigned long long any = reinterpret_cast<const unsigned long long*>(st + 2 * k + 3)[2];
  const bool compose = !reset && any != 0;
  const double* ratio = st + 2 * k + 8;
  const double* shift = ratio + k;
  const double e = (4.0 * steps + 16.0) * 0x1p-52;
  int out_of_range = 0;
  for (int c = blockIdx.x * blockDim.x + threadIdx.x; c < k; c += gridDim.x * blockDim.x) {
    double Sc = reset ? 1.0 : S[c], Tc = reset ? 0.0 : T[c];
    if (compose) {
      const double r = ratio[c];
      Sc = Sc * r * UBS;
      Tc = (Tc * r + shift[c]) * UBS;
    }
    S[c] = Sc;
    T[c] = Tc;
    const double I = new_infl[c];
    inv2_lo[c] = __ddiv_rd(1.0, __dmul_ru(I, I));
    inv2_hi[c] = __ddiv_ru(1.0, __dmul_rd(I, I));
    ub_eval[c] = make_float4(__double2float_ru(__dmul_ru(Sc, 1.0 + e)),
                             __double2float_rd(__dmul_rd(Sc, 1.0 - e)),
                             __double2float_ru(__dmul_ru(Tc, 1.0 + e)), 0.f);
    ub_norm[c] = make_float4(__double2float_ru(__ddiv_ru(1.0, Sc)),
                             __double2float_rd(__ddiv_rd(1.0, Sc)), __double2float_rd(Tc), 0.f);
    out_of_range |= Sc < 1e-6 || Sc > 1e6 || Tc > 64.0 * scale_hint;
  }
  if (__any_sync(FULL, out_of_range) && (threadIdx.x & 31) == 0) flags[0] = 1;
}

// one warp per region: smallest ratio / largest shift over the region's candidate
// list (all k when the list overflowed), composed into its lower-bound map like
// update_maps_kernel composes the global one
__global__ void __launch_bounds__(256) region_maps_kernel(
    const double* __restrict__ ratio, const double* __restrict__ shift,
    const unsigned long long* __restrict__ any, int k, const int32_t* __restrict__ glist,
    const int32_t* __restrict__ gcount, int gcap, int64_t R, double* __restrict__ rst,
    float4* __restrict__ rpar, int32_t* __restrict__ flags, int reset, double scale_hint) {
  const int lane = threadIdx.x & 31;
  const int64_t r = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (r >= R) return;
  double A = 1.0, B = 0.0, steps = 0.0;
  if (!reset && any && *any == 0) {   // identity relaxation: keep the map
    A = rst[3 * r];
    B = rst[3 * r + 1];
    steps = rst[3 * r + 2];
  } else if (!reset) {
    const int gc = gcount[r];
    const int32_t* lst = gc >= 0 ? glist + r * (int64_t)gcap : nullptr;
    const int ns = gc >= 0 ? gc : k;
    double rmin = INFINITY, smax = 0.0;
    for (int i = lane; i < ns; i += 32) {
      const int c = lst ? lst[i] : i;
      rmin = fmin(rmin, ratio[c]);
      smax = fmax(smax, shift[c]);
    }
    for (int o = 16; o; o >>= 1) {
      rmin = fmin(rmin, __shfl_xor_sync(FULL, rmin, o));
      smax = fmax(smax, __shfl_xor_sync(FULL, smax, o));
    }
    if (!(rmin < INFINITY)) rmin = 1.0;
    A = rst[3 * r];
    B = rst[3 * r + 1];
    steps = rst[3 * r + 2];
    A = A * rmin * LBS;
    B = (B * rmin + smax) * LBS;
    steps += 1.0;
  }
  if (lane == 0) {
    const double e = (4.0 * steps + 16.0) * 0x1p-52;
    rst[3 * r] = A;
    rst[3 * r + 1] = B;
    rst[3 * r + 2] = steps;
    rpar[r] = make_float4(__double2float_rd(__dmul_rd(A, 1.0 - e)),
                          __double2float_ru(__dmul_ru(B, 1.0 + e)),
                          __double2float_rd(__ddiv_rd(1.0, A)), __double2float_rd(B));
    if (A < 1e-6 || A > 1e6 || B > 64.0 * scale_hint) flags[0] = 1;
  }
}

static int validate(const gp_assign_args* a) {
  GP_REQUIRE(a != nullptr, "null args");
  GP_REQUIRE(a->d == 2 || a->d == 3, "d must be 2 or 3");
  GP_REQUIRE(a->k >= 1, "k must be >= 1");
  GP_REQUIRE(a->m >= 0 && a->m < (1ll << 31), "m out of range");
  GP_REQUIRE(a->wmode == GP_W_UNIT || a->w != nullptr, "weights missing");
  GP_REQUIRE(a->inv2_lo && a->inv2_hi, "inv2 bounds missing");
  GP_REQUIRE(a->ub_eval && a->ub_norm && a->lb_par, "bound maps missing");
  GP_REQUIRE(a->bound_scale > 0.f, "bound_scale must be a positive power of two");
  return GP_OK;
}

static unsigned persistent_grid(const void* fn, int threads, int64_t work, size_t dsmem = 0) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, dsmem);
  int64_t g = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  if (work < g) g = work;
  return (unsigned)(g < 1 ? 1 : g);
}

static int g_sreg = 0;  // 0: automatic (GP_SCAN_REGIONS overrides)

template <int WM>
static void launch_round(const gp_assign_args* a, int wshift, const AssignLayout& L,
                         int2* ent, int32_t* runs,
                         unsigned long long* sched, cudaStream_t s) {
  static bool attr_set[3] = {false, false, false};
  const size_t fsm = (size_t)(FTH / 32) * FSTAGES * FREG_BYTES;
  if (!attr_set[WM]) {
    cudaFuncSetAttribute(filter_kernel<WM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)fsm);
    attr_set[WM] = true;
  }
  unsigned gf = persistent_grid((const void*)filter_kernel<WM>, FTH, L.nchunks, fsm);
  filter_kernel<WM><<<gf, FTH, fsm, s>>>(*a, wshift, L.nchunks, ent, runs, sched);
  if (a->split_event) cudaEventRecord((cudaEvent_t)a->split_event, s);
  if (g_sreg == 0) {
    const char* e = getenv("GP_SCAN_REGIONS");
    g_sreg = e ? atoi(e) : -1;
  }
  // dense (full-phase) lists: 4 regions per scan unit; sparse sample lists: 1
  int sreg = a->scan_regions > 0 ? a->scan_regions : (a->list ? 1 : SREG);
  // the tuning override may only change the unit when no per-unit boxes (sized for
  // scan_regions) or group lists (sized for at least one unit) depend on it
  if (g_sreg > 0 && !a->unit_boxes &&
      (!a->group_list || (int64_t)g_sreg * WREG <= (1ll << a->group_shift)))
    sreg = g_sreg;
  if (sreg > SREG) sreg = SREG;
  // consecutive units per claim only when there are many more units than warps (few,
  // heavy units of a small warm-up sample go one per warp)
  const int64_t nunits = (L.nregions + sreg - 1) / sreg;
  // and a small round's units split into per-pass items, so more warps share them
  auto plan = [&](const void* fn, unsigned& gs, int& uch, int& pshift) {
    const unsigned gmax = persistent_grid(fn, STH, INT64_MAX);
    const int64_t warps = (int64_t)gmax * (STH / 32);
    int pmax = 0;
    while ((1 << (pmax + 1)) <= 8 * sreg) ++pmax;   // a unit has at most 8 * sreg passes
    pshift = 0;
    while (pshift < pmax && (nunits << (pshift + 1)) <= 2 * warps) ++pshift;
    uch = nunits >= 16 * warps ? UCH : 1;
    const int64_t items = ((nunits << pshift) + (STH / 32) - 1) / (STH / 32);
    gs = (unsigned)std::max<int64_t>(1, std::min<int64_t>(gmax, items));
  };
  if (a->flags & 2) {   // sparse warm-up round: warp-per-point grid walks
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int64_t items = L.nregions * WREG;
    const unsigned gw = (unsigned)std::max<int64_t>(
        1, std::min<int64_t>((items + (WKT / 32) * 4 - 1) / ((WKT / 32) * 4), (int64_t)sms * 8));
    if (a->d == 2)
      walk_kernel<2, WM><<<gw, WKT, 0, s>>>(*a, wshift, L.nregions, ent, runs);
    else
      walk_kernel<3, WM><<<gw, WKT, 0, s>>>(*a, wshift, L.nregions, ent, runs);
    return;
  }
  unsigned gs;
  int uch, pshift;
  if (a->d == 2) {
    plan((const void*)scan_kernel<2, WM>, gs, uch, pshift);
    scan_kernel<2, WM><<<gs, STH, 0, s>>>(*a, wshift, L.nregions, sreg, ent, runs, sched,
                                          uch, pshift);
  } else {
    plan((const void*)scan_kernel<3, WM>, gs, uch, pshift);
    scan_kernel<3, WM><<<gs, STH, 0, s>>>(*a, wshift, L.nregions, sreg, ent, runs, sched,
                                          uch, pshift);
  }
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
    GP_REQUIRE((int64_t)(args->scan_regions > 0 ? args->scan_regions : SREG) * WREG <= (1ll << args->group_shift),
               "group_shift smaller than a scan unit");
  if (args->unit_boxes)
    GP_REQUIRE(args->scan_regions >= 1 && (1ll << args->unit_shift) == args->scan_regions * WREG,
               "unit_shift must equal log2(scan_regions * 256)");
  int wshift = 0;
  frexp(args->wscale, &wshift);
  wshift -= 1;
  GP_REQUIRE(ldexp(1.0, wshift) == args->wscale, "gp_assign_round: wscale must be a power of 2");
  cudaStream_t s = (cudaStream_t)stream;
  char* ws = (char*)args->workspace;
  int2* ent = (int2*)(ws + L.off_list);
  int32_t* runs = (int32_t*)(ws + L.off_runs);
  unsigned long long* sched = (unsigned long long*)(ws + L.off_sched);
  if (args->wmode == GP_W_UNIT) launch_round<GP_W_UNIT>(args, wshift, L, ent, runs, sched, s);
  else if (args->wmode == GP_W_F32)
    launch_round<GP_W_F32>(args, wshift, L, ent, runs, sched, s);
  else launch_round<GP_W_F64>(args, wshift, L, ent, runs, sched, s);
  return check_launch("assign_round");
}

int gp_update_maps(const double* old_infl, const double* new_infl, const double* moves, int k,
                   double* state, double* inv2_lo, double* inv2_hi, float* ub_eval,
                   float* ub_norm, float* lb_par, int32_t* flags, int reset, double scale_hint,
                   void* stream) {
  GP_REQUIRE(k >= 1 && old_infl && new_infl && state, "gp_update_maps: bad args");
  cudaStream_t s = (cudaStream_t)stream;
  double* scr = state + 2 * k + 3;
  GP_CUDA(cudaMemsetAsync(scr, 0xff, sizeof(double), s));            // rmin: +max key
  GP_CUDA(cudaMemsetAsync(scr + 1, 0, 3 * sizeof(double), s));       // smax, any, max infl
  const unsigned g = grid_for(k, 256, 148);
  maps_ratio_kernel<<<g, 256, 0, s>>>(old_infl, new_infl, moves, k, state);
  maps_global_kernel<<<1, 1, 0, s>>>(k, state, lb_par, flags, reset, scale_hint);
  maps_cluster_kernel<<<g, 256, 0, s>>>(new_infl, k, state, inv2_lo, inv2_hi, (float4*)ub_eval,
                                        (float4*)ub_norm, flags, reset, scale_hint);
  return check_launch("update_maps");
}

int gp_region_maps(const double* map_state, int k, const int32_t* group_list,
                   const int32_t* group_count, int group_cap, int64_t nregions, double* rstate,
                   float* rpar, int32_t* flags, int reset, double scale_hint, void* stream) {
  GP_REQUIRE(k >= 1 && rstate && rpar && flags && nregions >= 1, "gp_region_maps: bad args");
  GP_REQUIRE(reset || (map_state && group_list && group_count),
             "gp_region_maps: inputs missing");
  const double* ratio = map_state ? map_state + 2 * k + 8 : nullptr;
  // the reference's identity early return (nothing moved or changed) holds here too
  const unsigned long long* any =
      map_state ? reinterpret_cast<const unsigned long long*>(map_state + 2 * k + 5) : nullptr;
  region_maps_kernel<<<grid_for(nregions * 32, 256), 256, 0, (cudaStream_t)stream>>>(
      ratio, ratio ? ratio + k : nullptr, any, k, group_list, group_count, group_cap, nregions,
      rstate, (float4*)rpar, flags, reset, scale_hint);
  return check_launch("region_maps");
}

int gp_lb_remap(const gp_assign_args* args, int mode, void* stream) {
  int rc = validate(args);
  if (rc) return rc;
  GP_REQUIRE(mode == 0 || (mode == 1 && args->lb_rpar), "gp_lb_remap: bad mode");
  if (args->m == 0) return GP_OK;
  lb_remap_kernel<<<grid_for(args->m, 256, 148 * 16), 256, 0, (cudaStream_t)stream>>>(*args, mode);
  return check_launch("lb_remap");
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

int gp_scan_stats(uint64_t* out, int reset) {
  GP_CUDA(cudaDeviceSynchronize());
  GP_CUDA(cudaMemcpyFromSymbol(out, g_scan_stats, sizeof(g_scan_stats)));
  if (reset) {
    unsigned long long z[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    GP_CUDA(cudaMemcpyToSymbol(g_scan_stats, z, sizeof(z)));
  }
  return GP_OK;
}

int gp_group_boxes(const double* X, int64_t ldx, int d, const int32_t* list, int64_t m, int shift,
                   double* boxes, void* stream) {
  GP_REQUIRE(d == 2 || d == 3, "gp_group_boxes: bad d");
  GP_REQUIRE(shift >= 5 && shift < 31, "gp_group_boxes: bad shift");
  if (m <= 0) return GP_OK;
  const int64_t ng = (m + (1ll << shift) - 1) >> shift;
  cudaStream_t s = (cudaStream_t)stream;
  if (d == 2) group_boxes_kernel<2><<<(unsigned)ng, 256, 0, s>>>(X, ldx, list, m, shift, boxes);
  else group_boxes_kernel<3><<<(unsigned)ng, 256, 0, s>>>(X, ldx, list, m, shift, boxes);
  return check_launch("group_boxes");
}

int gp_group_candidates(const double* boxes, int64_t ngroups, int d, int k,
                        const double* centers, const double* inv2_lo, const double* inv2_hi,
                        const int32_t* parent_list, const int32_t* parent_count, int parent_cap,
                        int parent_ratio_log2, int32_t* list, int32_t* count, int cap,
                        void* stream) {
  GP_REQUIRE(d == 2 || d == 3, "gp_group_candidates: bad d");
  GP_REQUIRE(cap >= 1 && k >= 1, "gp_group_candidates: bad sizes");
  if (ngroups <= 0) return GP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  // short parent lists (super groups under mega / giga lists): one warp per group, when
  // there are enough groups to fill the GPU with warps; a few hundred groups (warm-up
  // samples) take a CTA each, so that the walk over the parent list is 8x shorter
  if (parent_list && parent_cap <= 4096 && ngroups >= 4096) {
    const unsigned gw = (unsigned)((ngroups * 32 + 255) / 256);
    if (d == 2)
      group_candidates_warp_kernel<2><<<gw, 256, 0, s>>>(
          boxes, ngroups, k, centers, inv2_lo, inv2_hi, parent_list, parent_count, parent_cap,
          parent_ratio_log2, list, count, cap);
    else
      group_candidates_warp_kernel<3><<<gw, 256, 0, s>>>(
          boxes, ngroups, k, centers, inv2_lo, inv2_hi, parent_list, parent_count, parent_cap,
          parent_ratio_log2, list, count, cap);
    return check_launch("group_candidates");
  }
  // a few groups walking long sources (the top level over all k centers, warm-up samples):
  // 1024 threads per group, so that the walk is four times shorter
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int threads = ngroups <= 2 * sms ? 1024 : 256;
  if (d == 2)
    group_candidates_kernel<2><<<(unsigned)ngroups, threads, 0, s>>>(
        boxes, k, centers, inv2_lo, inv2_hi, parent_list, parent_count, parent_cap,
        parent_ratio_log2, list, count, cap);
  else
    group_candidates_kernel<3><<<(unsigned)ngroups, threads, 0, s>>>(
        boxes, k, centers, inv2_lo, inv2_hi, parent_list, parent_count, parent_cap,
        parent_ratio_log2, list, count, cap);
  return check_launch("group_candidates");
}

}  // extern "C"
