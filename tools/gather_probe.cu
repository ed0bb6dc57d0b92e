// Random gather / scatter rates vs array size: is the bootstrap's random access
// TLB-bound (cost grows with the span) or sector-bound (flat)?
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o gather_probe tools/gather_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__global__ void fill_idx(uint32_t* idx, int64_t m, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + seed) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    z ^= z >> 31;
    idx[i] = (uint32_t)(z % (uint64_t)n);
  }
}

// idx confined to windows of w consecutive targets, windows in order
__global__ void fill_win(uint32_t* idx, int64_t m, int64_t w, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    uint64_t z = (i + seed) * 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z ^= z >> 31;
    idx[i] = (uint32_t)((i / w) * w + (int64_t)(z % (uint64_t)w));
  }
}

__global__ void gather(const double2* __restrict__ X, const uint32_t* __restrict__ idx,
                       double2* __restrict__ out, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    out[i] = X[idx[i]];
}

__global__ void scatter(const int32_t* __restrict__ a, const uint32_t* __restrict__ idx,
                        int64_t* __restrict__ out, int64_t m) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    out[idx[i]] = a[i];
}

int main() {
  const int64_t m = 1ll << 27;   // accesses per test
  uint32_t* idx;
  double2* out;
  int32_t* a;
  cudaMalloc(&idx, m * 4);
  cudaMalloc(&out, m * 16);
  cudaMalloc(&a, m * 4);
  cudaMemset(a, 1, m * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  size_t gran = 0;
  cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity);
  printf("default cudaLimitMaxL2FetchGranularity = %zu\n", gran);
  for (size_t g : {(size_t)32, (size_t)64, (size_t)128}) {
  cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g);
  cudaDeviceGetLimit(&gran, cudaLimitMaxL2FetchGranularity);
  printf("L2 fetch granularity %zu (set %zu)\n", gran, g);
  printf("span_GiB gather16B_ms Ggather/s  scatter8B_ms Gscatter/s  (2^27 random accesses)\n");
  for (double gib : {0.125, 2.0, 16.0}) {
    const int64_t n = (int64_t)(gib * (1ll << 30) / 16);
    double2* X;
    if (cudaMalloc(&X, n * 16) != cudaSuccess) break;
    cudaMemset(X, 0, n * 16);
    fill_idx<<<148 * 16, 256>>>(idx, m, n, 12345);
    float tg = 1e30f, ts = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(e0);
      gather<<<148 * 16, 256>>>(X, idx, out, m);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r) tg = ms < tg ? ms : tg;
      cudaEventRecord(e0);
      scatter<<<148 * 16, 256>>>(a, idx, (int64_t*)X, m);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      if (r) ts = ms < ts ? ms : ts;
    }
    printf("%7.3f %10.3f %8.2f %12.3f %8.2f\n", gib, tg, m / tg / 1e6, ts, m / ts / 1e6);
    cudaFree(X);
  }
  }
  printf("windowed scatter of 2^27 8-byte writes (targets random inside consecutive windows)\n");
  int64_t* O;
  cudaMalloc(&O, m * 8);
  for (int64_t w : {1ll << 14, 1ll << 17, 1ll << 19, 1ll << 21, 1ll << 23}) {
    fill_win<<<148 * 16, 256>>>(idx, m, w, 777);
    float best = 1e30f;
    for (int r = 0; r < 4; ++r) {
      cudaEventRecord(e0);
      scatter<<<148 * 16, 256>>>(a, idx, O, m);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r) best = ms < best ? ms : best;
    }
    printf("window %8lld entries (%6.1f MiB): %8.3f ms  %8.2f G/s\n", (long long)w,
           w * 8 / 1048576.0, best, m / best / 1e6);
  }
  return 0;
}
