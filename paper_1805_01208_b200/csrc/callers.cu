// Callers of the partition path:
//
//  * gp_sfc_cut      — the cut step of the SFC baseline sfc_labels
//                      (baselines.py:62-89): prefix weight along the Hilbert
//                      order, block = min(floor(before*k/total), k-1), written
//                      back by original vertex id.
//  * gp_predict      — GeographerPartitioner.predict (estimators.py:107-114):
//                      argmin over centers of norm(x - c) / influence.
//
// Both are bit-exact restatements of the numpy expressions they replace.
#include <cub/cub.cuh>

#include "common.cuh"

namespace gp {

// ---------------------------------------------------------------- SFC cut
// Exact mode: every weight is an integer number of units of 2^-s and the total
// stays below 2^53 units (gp_weight_probe), so numpy's sequential cumsum, the
// subtraction cumsum - w and the pairwise w.sum() are all exact and equal the
// integer prefix sums computed here.
__global__ void sfc_units_kernel(const uint32_t* __restrict__ gids, const double* __restrict__ w,
                                 int64_t n, double scale, int64_t* __restrict__ units) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    units[i] = w ? (int64_t)__dmul_rn(w[gids[i]], scale) : 1;
}

// block of SFC position i from its exact prefix (before) and the total:
// numpy (before * k / total).astype(int64), then minimum(., k-1)
__device__ __forceinline__ int64_t cut_block(double before, double total, int k) {
  const double q = __ddiv_rn(__dmul_rn(before, (double)k), total);
  int64_t b = (int64_t)q;  // astype(int64) truncates toward zero
  return b < (int64_t)(k - 1) ? b : (int64_t)(k - 1);
}

__global__ void sfc_label_exact_kernel(const uint32_t* __restrict__ gids,
                                       const int64_t* __restrict__ prefix,
                                       const int64_t* __restrict__ units, int64_t n, int k,
                                       double inv_scale, int64_t* __restrict__ labels) {
  const double total = __dmul_rn((double)(prefix[n - 1] + units[n - 1]), inv_scale);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double before = __dmul_rn((double)prefix[i], inv_scale);
    labels[gids[i]] = cut_block(before, total, k);
  }
}

// Inexact mode (weights with no common exact fixed point): the reference's
// bits depend on the summation order, so the cut restates it literally.
//  * total = w.sum(): numpy's pairwise summation (8 accumulators below 128
//    elements, halving splits rounded to multiples of 8 above) over the
//    contiguous curve-ordered copy.
//  * before = cumsum(w) - w: a sequential fold, one dependent add per point.
__global__ void sfc_gather_w_kernel(const uint32_t* __restrict__ gids, const double* __restrict__ w,
                                    int64_t n, double* __restrict__ wo) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    wo[i] = w[gids[i]];
}

__device__ double pairwise_leaf(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int64_t i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  }
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

// numpy pairwise_sum split: n2 = n/2 rounded down to a multiple of 8
__device__ __forceinline__ int64_t pw_split(int64_t n) {
  int64_t n2 = n / 2;
  return n2 - n2 % 8;
}

// pairwise sum of a[0, n) without recursion: an explicit stack of pending
// right halves and partial left results (depth <= 64)
__device__ double pairwise_sum(const double* a, int64_t n) {
  struct Frame { int64_t lo, n; int state; double left; };
  Frame st[64];
  int sp = 0;
  st[0] = {0, n, 0, 0.0};
  double ret = 0.0;
  while (true) {
    Frame& f = st[sp];
    if (f.n <= 128) {
      ret = pairwise_leaf(a + f.lo, f.n);
    } else if (f.state == 0) {
      f.state = 1;
      st[++sp] = {f.lo, pw_split(f.n), 0, 0.0};
      continue;
    } else if (f.state == 1) {
      f.state = 2;
      f.left = ret;
      const int64_t n2 = pw_split(f.n);
      st[++sp] = {f.lo + n2, f.n - n2, 0, 0.0};
      continue;
    } else {
      ret = __dadd_rn(f.left, ret);
    }
    if (sp == 0) return ret;
    --sp;
  }
}

// Subtrees at a fixed depth L of the pairwise tree: thread t walks the bits of t
// from the root to find its subtree (every node above depth L has n > 128 by the
// choice of L) and sums it; the top L levels are combined by one thread.
__global__ void pairwise_subtrees_kernel(const double* __restrict__ a, int64_t n, int L,
                                         double* __restrict__ part) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= (1ll << L)) return;
  int64_t lo = 0, len = n;
  for (int l = L - 1; l >= 0; --l) {
    const int64_t n2 = pw_split(len);
    if ((t >> l) & 1) { lo += n2; len -= n2; }
    else len = n2;
  }
  part[t] = pairwise_sum(a + lo, len);
}

__global__ void pairwise_top_kernel(const double* __restrict__ part, int L,
                                    double* __restrict__ total) {
  // combine bottom-up: level L has 2^L partials in tree order
  extern __shared__ double s[];
  const int m = 1 << L;
  for (int i = threadIdx.x; i < m; i += blockDim.x) s[i] = part[i];
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = m; w > 1; w >>= 1)
      for (int i = 0; i < w / 2; ++i) s[i] = __dadd_rn(s[2 * i], s[2 * i + 1]);
    *total = s[0];
  }
}

__global__ void sequential_before_kernel(const double* __restrict__ wo, int64_t n,
                                         double* __restrict__ before) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double c = 0.0;
  int64_t i = 0;
  for (; i + 8 <= n; i += 8) {
    double v[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) v[j] = wo[i + j];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      c = (i + j == 0) ? v[j] : __dadd_rn(c, v[j]);
      before[i + j] = __dsub_rn(c, v[j]);
    }
  }
  for (; i < n; ++i) {
    const double v = wo[i];
    c = (i == 0) ? v : __dadd_rn(c, v);
    before[i] = __dsub_rn(c, v);
  }
}

__global__ void sfc_label_inexact_kernel(const uint32_t* __restrict__ gids,
                                         const double* __restrict__ before, int64_t n, int k,
                                         const double* __restrict__ total,
                                         int64_t* __restrict__ labels) {
  const double t = *total;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    labels[gids[i]] = cut_block(before[i], t, k);
}

static int pairwise_depth(int64_t n) {
  // deepest L <= 12 with every node above depth L still split (n/2^L > 256)
  int L = 0;
  while (L < 12 && (n >> (L + 1)) > 256) ++L;
  return L;
}

// numpy's pairwise sum of a[0, n) into *total (part: 4096 doubles of scratch); shared with
// graphs.cu (the weighted edge cut)
int pairwise_sum_async(const double* a, int64_t n, double* part, double* total, cudaStream_t s) {
  const int L = pairwise_depth(n);
  const int m = 1 << L;
  pairwise_subtrees_kernel<<<(m + 127) / 128, 128, 0, s>>>(a, n, L, part);
  pairwise_top_kernel<<<1, 256, m * sizeof(double), s>>>(part, L, total);
  return check_launch("pairwise_sum");
}

static unsigned sm_grid(int64_t n, int per) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int64_t want = (n + per - 1) / per;
  int64_t cap = (int64_t)sms * 8;
  return (unsigned)(want < 1 ? 1 : (want < cap ? want : cap));
}

// ---------------------------------------------------------------- predict
// norm(x - c) with numpy's linalg.norm reduction over the last axis:
// sqrt((dx^2 + dy^2) + dz^2), every operation separately rounded.
template <int D>
__device__ __forceinline__ double norm_dist_rn(const double* p, const double* c) {
  double s = 0.0;
#pragma unroll
  for (int j = 0; j < D; ++j) {
    const double t = __dsub_rn(p[j], c[j]);
    s = j == 0 ? __dmul_rn(t, t) : __dadd_rn(s, __dmul_rn(t, t));
  }
  return __dsqrt_rn(s);
}

// numpy argmin: first index of the minimum; a NaN is the minimum (first NaN wins)
__device__ __forceinline__ bool argmin_better(double v, int c, double best, int bi) {
  if (isnan(best)) return false;
  if (isnan(v)) return true;
  return v < best || (v == best && c < bi);
}

// the reference arithmetic over all k centers (near ties and non-finite input)
template <int D>
__device__ __noinline__ int predict_exact(double x, double y, double z, const double* C,
                                          const double* infl, int k) {
  const double pt[3] = {x, y, z};
  double bd = 0.0;
  int best = -1;
  for (int c = 0; c < k; ++c) {
    double cc[3];
#pragma unroll
    for (int j = 0; j < D; ++j) cc[j] = C[(int64_t)c * D + j];
    const double dv = __ddiv_rn(norm_dist_rn<D>(pt, cc), infl[c]);
    if (best < 0 || argmin_better(dv, c, bd, best)) {
      bd = dv;
      best = c;
    }
  }
  return best;
}

constexpr int PRED_TILE = 1024;  // centers per shared-memory tile
constexpr int PRED_THREADS = 256;
constexpr int PRED_P = 4;        // points per thread

// Pass 1 ranks every center by the approximate key q = s * (1/infl^2) (fp64,
// a few ulps from dist^2) and keeps the best and the runner-up keys.  When the
// runner-up is clearly separated the approximate winner is the exact argmin;
// otherwise (near ties, duplicates, non-finite values) the point re-scans all
// centers with the reference arithmetic.
template <int D>
__global__ void __launch_bounds__(PRED_THREADS) predict_kernel(
    const double* __restrict__ X, int64_t n, const double* __restrict__ C,
    const double* __restrict__ infl, int k, int safe_infl, int64_t* __restrict__ labels) {
  __shared__ double4 tile[PRED_TILE];
  const int64_t base = (int64_t)blockIdx.x * PRED_THREADS * PRED_P + threadIdx.x;
  double p[PRED_P][D];
  double q1[PRED_P], q2[PRED_P];
  int i1[PRED_P];
#pragma unroll
  for (int r = 0; r < PRED_P; ++r) {
    const int64_t i = base + (int64_t)r * PRED_THREADS;
#pragma unroll
    for (int j = 0; j < D; ++j) p[r][j] = i < n ? X[i * D + j] : 0.0;
    q1[r] = q2[r] = __longlong_as_double(0x7ff0000000000000ll);
    i1[r] = 0;
  }
  for (int c0 = 0; c0 < k; c0 += PRED_TILE) {
    const int m = min(PRED_TILE, k - c0);
    __syncthreads();
    for (int t = threadIdx.x; t < m; t += PRED_THREADS) {
      const int c = c0 + t;
      const double f = infl[c];
      double4 v;
      v.x = C[(int64_t)c * D];
      v.y = C[(int64_t)c * D + 1];
      v.z = D == 3 ? C[(int64_t)c * D + 2] : 0.0;
      v.w = 1.0 / (f * f);
      tile[t] = v;
    }
    __syncthreads();
#pragma unroll 2
    for (int t = 0; t < m; ++t) {
      const double4 v = tile[t];
#pragma unroll
      for (int r = 0; r < PRED_P; ++r) {
        const double dx = p[r][0] - v.x, dy = p[r][1] - v.y;
        double s = dx * dx + dy * dy;
        if (D == 3) {
          const double dz = p[r][2] - v.z;
          s += dz * dz;
        }
        const double q = s * v.w;
        const bool win = q < q1[r];
        q2[r] = fmin(q2[r], fmax(q, q1[r]));
        i1[r] = win ? c0 + t : i1[r];
        q1[r] = fmin(q1[r], q);
      }
    }
  }
#pragma unroll
  for (int r = 0; r < PRED_P; ++r) {
    const int64_t i = base + (int64_t)r * PRED_THREADS;
    if (i >= n) continue;
    // relative error of q against dist^2 is below ~16 ulp; 1e-12 is a wide margin
    const bool sure = safe_infl && isfinite(q1[r]) && isfinite(q2[r]) &&
                      q2[r] > q1[r] * (1.0 + 1e-12) + 1e-300;
    labels[i] = sure ? i1[r] : predict_exact<D>(p[r][0], p[r][1], D == 3 ? p[r][D - 1] : 0.0,
                                                C, infl, k);
  }
}

}  // namespace gp

using namespace gp;

extern "C" {

int gp_sfc_cut_workspace_bytes(int64_t n, size_t* bytes) {
  GP_REQUIRE(n >= 0 && n < (1ll << 31), "gp_sfc_cut: n out of range");
  size_t scan = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, scan, (const int64_t*)nullptr,
                                                (int64_t*)nullptr, (int)(n > 0 ? n : 1));
  if (e != cudaSuccess) {
    set_error("sfc_cut scan workspace query failed: %s", cudaGetErrorString(e));
    return GP_ERR_CUDA;
  }
  const size_t arrays = 2 * (size_t)n * sizeof(int64_t);
  const size_t top = ((size_t)1 << 12) * sizeof(double) + 64;
  *bytes = arrays + ((scan + 255) & ~(size_t)255) + top;
  return GP_OK;
}

int gp_sfc_cut(const uint32_t* gids, const double* w, int64_t n, int k, double scale,
               int64_t* labels, void* workspace, size_t workspace_bytes, void* stream) {
  GP_REQUIRE(n >= 1 && n < (1ll << 31), "gp_sfc_cut: n out of range");
  GP_REQUIRE(k >= 1 && (int64_t)k <= n, "gp_sfc_cut: k=%d out of range 1..%lld", k,
             (long long)n);
  GP_REQUIRE(scale >= 0.0, "gp_sfc_cut: scale must be >= 0");
  GP_REQUIRE(w || scale == 1.0, "gp_sfc_cut: unit weights need scale 1");
  size_t need = 0;
  int rc = gp_sfc_cut_workspace_bytes(n, &need);
  if (rc) return rc;
  GP_REQUIRE(workspace_bytes >= need, "gp_sfc_cut: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  char* ws = (char*)workspace;
  int64_t* A = (int64_t*)ws;            // units | curve-ordered weights
  int64_t* B = A + n;                   // prefix | before
  char* rest = (char*)(B + n);
  double* top = (double*)rest;          // 2^12 partials + total
  void* scan_ws = rest + ((size_t)1 << 12) * sizeof(double) + 64;
  size_t scan_bytes = workspace_bytes - ((char*)scan_ws - ws);
  const unsigned g = sm_grid(n, 256);
  if (scale > 0.0) {
    sfc_units_kernel<<<g, 256, 0, s>>>(gids, w, n, scale, A);
    GP_CUDA(cub::DeviceScan::ExclusiveSum(scan_ws, scan_bytes, A, B, (int)n, s));
    sfc_label_exact_kernel<<<g, 256, 0, s>>>(gids, B, A, n, k, 1.0 / scale, labels);
    return check_launch("sfc_cut");
  }
  double* wo = (double*)A;
  double* before = (double*)B;
  double* total = top + (1 << 12);
  sfc_gather_w_kernel<<<g, 256, 0, s>>>(gids, w, n, wo);
  const int L = pairwise_depth(n);
  const int m = 1 << L;
  pairwise_subtrees_kernel<<<(m + 127) / 128, 128, 0, s>>>(wo, n, L, top);
  pairwise_top_kernel<<<1, 256, m * sizeof(double), s>>>(top, L, total);
  sequential_before_kernel<<<1, 32, 0, s>>>(wo, n, before);
  sfc_label_inexact_kernel<<<g, 256, 0, s>>>(gids, before, n, k, total, labels);
  return check_launch("sfc_cut");
}

int gp_predict(const double* X, int64_t n, int d, const double* centers, const double* influence,
               int k, int safe_influence, int64_t* labels, void* stream) {
  GP_REQUIRE(d == 2 || d == 3, "gp_predict: unsupported dimension %d", d);
  GP_REQUIRE(k >= 1, "gp_predict: k must be >= 1");
  GP_REQUIRE(n >= 0, "gp_predict: n must be >= 0");
  if (n == 0) return GP_OK;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t per = (int64_t)PRED_THREADS * PRED_P;
  const unsigned g = (unsigned)((n + per - 1) / per);
  if (d == 2)
    predict_kernel<2><<<g, PRED_THREADS, 0, s>>>(X, n, centers, influence, k, safe_influence,
                                                 labels);
  else
    predict_kernel<3><<<g, PRED_THREADS, 0, s>>>(X, n, centers, influence, k, safe_influence,
                                                 labels);
  return check_launch("predict");
}

}  // extern "C"
