// gp_balance_decide: one balance-round decision of assign_and_balance
// (kmeans.py:425-443) on the device, so the host loop reads back a six-double
// record per round instead of doing the k-sized control math itself
// (d = 2 with exact block weights).
#include <cmath>

#include "common.cuh"

namespace gp {

// gp_balance_decide: one block; the block-weight sums are exact (integer units of
// 1/wscale below 2^53), so any summation order gives numpy's bits.
__global__ void __launch_bounds__(1024) balance_decide_kernel(
    const long long* __restrict__ red, int k, double wscale, double eps, int max_rounds,
    double* __restrict__ bal, const double* __restrict__ cur, double* __restrict__ next) {
  __shared__ double s_sum[32], s_max[32];
  __shared__ double s_tgt, s_cap;
  __shared__ int s_stop;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // wscale is a power of two (the exact weight scale 2^s), so multiplying by its inverse
  // gives the bits of blk_int.astype(float64) / scale
  const double winv = 1.0 / wscale;
  double sum = 0.0, mx = -INFINITY;
#pragma unroll 8
  for (int c = tid; c < k; c += blockDim.x) {
    const double w = (double)red[c] * winv;
    sum += w;
    mx = fmax(mx, w);
  }
  for (int o = 16; o; o >>= 1) {
    sum += __shfl_xor_sync(FULL, sum, o);
    mx = fmax(mx, __shfl_xor_sync(FULL, mx, o));
  }
  if (lane == 0) {
    s_sum[warp] = sum;
    s_max[warp] = mx;
  }
  __syncthreads();
  if (tid == 0) {
    double total = 0.0, bmax = -INFINITY;
    for (int w = 0; w < (int)(blockDim.x / 32); ++w) {
      total += s_sum[w];
      bmax = fmax(bmax, s_max[w]);
    }
    const int r = (int)bal[3];
    int stop = 0;
    double tgt = 0.0, cap = bal[0];
    if (!(total > 0.0)) {                       // imbalance(): total weight must be positive
      bal[4] = 1.0;
      stop = 1;
    } else {
      // balance_target (metrics.py:26-30): integer ceil when the total is integral
      double tb;
      if (total == floor(total)) {
        const long long t = (long long)total;
        tb = (double)((t + k - 1) / k);
      } else {
        tb = ceil(total / (double)k);
      }
      const double imb = bmax / tb - 1.0;
      bal[8 + r] = imb;
      bal[8 + max_rounds + r] = (double)red[k];
      bal[8 + 2 * max_rounds + r] = (double)red[k + 2];
      stop = imb <= eps || r == max_rounds - 1;
      if (!stop) {
        if (imb > bal[2]) {                     // step halving from the second regression
          bal[1] += 1.0;
          if (bal[1] >= 2.0) cap *= 0.5;
        }
        bal[2] = fmin(bal[2], imb);
        bal[0] = cap;
        tgt = total / (double)k;                // float(block_w.sum()) / k
        if (!(tgt > 0.0)) {
          bal[4] = 2.0;
          stop = 1;
        }
      }
    }
    bal[3] = (double)(r + 1);
    bal[5] = stop ? 1.0 : 0.0;
    s_stop = stop;
    s_tgt = tgt;
    s_cap = cap;
  }
  __syncthreads();
  if (!s_stop) {
    const double lo = 1.0 - s_cap, hi = 1.0 + s_cap, tgt = s_tgt;
#pragma unroll 4
    for (int c = tid; c < k; c += blockDim.x) {
      const double w = (double)red[c] * winv;
      const double gamma = w > 0.0 ? tgt / w : INFINITY;
      const double f = fmin(fmax(__dsqrt_rn(gamma), lo), hi);   // clip(gamma ** 0.5)
      next[c] = cur[c] * f;
    }
  }
}

}  // namespace gp

extern "C" int gp_balance_decide(const long long* red, int k, double wscale, double eps,
                                 int max_rounds, double* bal, const double* infl_cur,
                                 double* infl_next, void* stream) {
  GP_REQUIRE(red && bal && infl_cur && infl_next && k >= 1 && max_rounds >= 1 && wscale > 0,
             "gp_balance_decide: bad args");
  {
    int e = 0;
    GP_REQUIRE(frexp(wscale, &e) == 0.5, "gp_balance_decide: wscale must be a power of two");
  }
  gp::balance_decide_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(
      red, k, wscale, eps, max_rounds, bal, infl_cur, infl_next);
  return gp::check_launch("balance_decide");
}
