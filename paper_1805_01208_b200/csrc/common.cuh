// Shared helpers for the geopart-b200 sm_100a kernels.
//
// Every fp64 operation whose bits must equal the reference's numpy result is
// written with an explicit round-to-nearest intrinsic (__dsub_rn, __dmul_rn,
// __dadd_rn, __dsqrt_rn, __ddiv_rn): those are never contracted into FMA,
// whatever -fmad says, so the kernels reproduce numpy's separately rounded
// ufunc arithmetic.  Pruning bounds use directed rounding (_ru / _rd) so that
// they stay rigorous.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/geopart_b200.h"

namespace gp {

void set_error(const char* fmt, ...);
int check_launch(const char* what);

#define GP_REQUIRE(cond, ...)            \
  do {                                   \
    if (!(cond)) {                       \
      ::gp::set_error(__VA_ARGS__);      \
      return GP_ERR_INVALID;             \
    }                                    \
  } while (0)

#define GP_CUDA(call)                                                              \
  do {                                                                             \
    cudaError_t _e = (call);                                                       \
    if (_e != cudaSuccess) {                                                       \
      ::gp::set_error("%s failed: %s", #call, cudaGetErrorString(_e));             \
      return GP_ERR_CUDA;                                                          \
    }                                                                              \
  } while (0)

constexpr unsigned FULL = 0xffffffffu;

// Squared Euclidean norm of a difference vector in the summation order the
// host numpy einsum('ij,ij->i') uses (probed at import).
//   2D: dx^2 + dy^2
//   3D: order 0: (x+y)+z   1: (x+z)+y   2: (y+z)+x
__device__ __forceinline__ double sqnorm_rn(const double* v, int d, int order3) {
  double xx = __dmul_rn(v[0], v[0]);
  double yy = __dmul_rn(v[1], v[1]);
  if (d == 2) return __dadd_rn(xx, yy);
  double zz = __dmul_rn(v[2], v[2]);
  if (order3 == 1) return __dadd_rn(__dadd_rn(xx, zz), yy);
  if (order3 == 2) return __dadd_rn(__dadd_rn(yy, zz), xx);
  return __dadd_rn(__dadd_rn(xx, yy), zz);
}

// Reference effective distance sqrt(einsum(diff, diff)) / influence
// (kmeans.py:157-159), bit for bit.
template <int D>
__device__ __forceinline__ double effdist_rn(const double* p, const double* c, double infl,
                                             int order3) {
  double diff[3];
#pragma unroll
  for (int j = 0; j < D; ++j) diff[j] = __dsub_rn(p[j], c[j]);
  return __ddiv_rn(__dsqrt_rn(sqnorm_rn(diff, D, order3)), infl);
}

// Order-preserving map from doubles to unsigned 64-bit keys (for atomic min/max).
__device__ __forceinline__ unsigned long long dkey(double x) {
  unsigned long long b = (unsigned long long)__double_as_longlong(x);
  return (b & 0x8000000000000000ull) ? ~b : (b | 0x8000000000000000ull);
}
__device__ __forceinline__ double dkey_inv(unsigned long long k) {
  unsigned long long b = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)b);
}
__host__ __device__ __forceinline__ unsigned long long dkey_host_min() { return ~0ull; }

// Lazily relaxed Hamerly bounds, evaluated in float32 with
// outward rounding from host parameters that already include the composition
// error margin (control.BoundMaps.device_params).
__device__ __forceinline__ float ub_evalf(float4 E, float u) {
  return __fmaf_ru(u >= 0.f ? E.x : E.y, u, E.z);
}
__device__ __forceinline__ float lb_evalf(float A, float l, float B) {
  if (isinf(l)) return l;  // k == 1: no runner-up
  return fmaxf(__fmaf_rd(A, l, -B), 0.f);
}
// normalise fresh bounds (b rounded up, s rounded down) under the current maps
__device__ __forceinline__ float ub_normf(float4 N, float b_up) {
  const float num = __fsub_ru(b_up, N.z);
  return __fmul_ru(num, num >= 0.f ? N.x : N.y);
}
__device__ __forceinline__ float lb_normf(float inva, float blo, float s_dn) {
  if (isinf(s_dn)) return s_dn;
  return __fmul_rd(__fadd_rd(s_dn, blo), inva);
}

// Stored bounds: (ub~, lb~) times the power of two `scale` as an fp16 pair, ub~
// rounded up and lb~ rounded down (4 bytes per point).  Unpacking
// multiplies by 1/scale, exact for a power of two.
__device__ __forceinline__ unsigned bnd_pack(float u, float l, float scale) {
  const __half hu = __float2half_ru(u * scale);
  const __half hl = __float2half_rd(l * scale);
  return (unsigned)__half_as_ushort(hu) | ((unsigned)__half_as_ushort(hl) << 16);
}
__device__ __forceinline__ float2 bnd_unpack(unsigned w, float inv_scale) {
  const float u = __half2float(__ushort_as_half((unsigned short)(w & 0xffffu)));
  const float l = __half2float(__ushort_as_half((unsigned short)(w >> 16)));
  return make_float2(u * inv_scale, l * inv_scale);
}

// the stored pair as floats, still multiplied by the scale (the filter folds
// 1/scale into the bound-map slopes: exact for a power of two)
__device__ __forceinline__ float2 bnd_raw(unsigned w) {
  return __half22float2(*reinterpret_cast<const __half2*>(&w));
}

// point i of an AoS coordinate array with point stride ldx
template <int D>
__device__ __forceinline__ void load_point(const double* X, int64_t ldx, int64_t i, double* out) {
  if (D == 2 && ldx == 2) {
    const double2 v = reinterpret_cast<const double2*>(X)[i];
    out[0] = v.x;
    out[1] = v.y;
  } else {
#pragma unroll
    for (int j = 0; j < D; ++j) out[j] = X[i * ldx + j];
  }
}

__device__ __forceinline__ double load_weight(const void* w, int wmode, int64_t i) {
  if (wmode == GP_W_UNIT) return 1.0;
  if (wmode == GP_W_F32) return (double)((const float*)w)[i];
  return ((const double*)w)[i];
}

// Segment (of GP_SEGMENTS equal position ranges, ranksim.py:74-75) of a global
// position: the largest s with floor(s*n/S) <= pos.  S is a power of two, so
// the boundaries are (s*n) >> 8; a floating-point estimate is corrected with
// exact integer checks (no 64-bit division).
__device__ __forceinline__ int segment_of(int64_t pos, int64_t n) {
  int s = (int)((double)pos * ((double)GP_SEGMENTS / (double)n));
  s = s < 0 ? 0 : (s > GP_SEGMENTS - 1 ? GP_SEGMENTS - 1 : s);
  while (s > 0 && (((int64_t)s * n) >> 8) > pos) --s;
  while (s < GP_SEGMENTS - 1 && (((int64_t)(s + 1) * n) >> 8) <= pos) ++s;
  return s;
}

inline unsigned grid_for(int64_t work, int per_block, int cap = 1 << 30) {
  int64_t g = (work + per_block - 1) / per_block;
  if (g < 1) g = 1;
  if (g > cap) g = cap;
  return (unsigned)g;
}

}  // namespace gp
