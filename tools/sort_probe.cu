// CUB device radix sort rates for the SFC-sort shapes (is the 2^30 x (u64 key, u32
// gid) sort near the copy bandwidth per pass?).
//   nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -o sort_probe tools/sort_probe.cu
#include <cub/device/device_radix_sort.cuh>
#include <cstdio>
#include <cstdint>

template <typename K, typename V>
static void run(const char* name, int64_t n, int bits) {
  K *k0, *k1;
  V *v0, *v1;
  cudaMalloc(&k0, n * sizeof(K));
  cudaMalloc(&k1, n * sizeof(K));
  cudaMalloc(&v0, n * sizeof(V));
  cudaMalloc(&v1, n * sizeof(V));
  cudaMemset(k0, 0x5a, n * sizeof(K));
  cudaMemset(v0, 0, n * sizeof(V));
  size_t tb = 0;
  cub::DoubleBuffer<K> kb(k0, k1);
  cub::DoubleBuffer<V> vb(v0, v1);
  cub::DeviceRadixSort::SortPairs(nullptr, tb, kb, vb, (int)n, 0, bits);
  void* tmp;
  cudaMalloc(&tmp, tb);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cub::DoubleBuffer<K> kb2(k0, k1);
    cub::DoubleBuffer<V> vb2(v0, v1);
    cudaEventRecord(e0);
    cub::DeviceRadixSort::SortPairs(tmp, tb, kb2, vb2, (int)n, 0, bits);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r) best = ms < best ? ms : best;
  }
  const int passes = (bits + 7) / 8;
  const double bytes = (double)n * (sizeof(K) + sizeof(V)) * 2 * passes;
  printf("%-22s n=%lld bits=%d: %8.2f ms  (%d passes, %.2f TB/s of pass traffic)\n", name,
         (long long)n, bits, best, passes, bytes / (best * 1e-3) / 1e12);
  cudaFree(k0);
  cudaFree(k1);
  cudaFree(v0);
  cudaFree(v1);
  cudaFree(tmp);
}

int main() {
  const int64_t n = 1ll << 30;
  run<uint64_t, uint32_t>("u64 key, u32 val", n, 62);
  run<uint64_t, uint64_t>("u64 key, u64 val", n, 62);
  run<uint32_t, uint32_t>("u32 key, u32 val", n, 30);
  run<uint32_t, uint32_t>("u32 key, u32 val", n, 32);
  run<uint64_t, uint32_t>("u64 key, u32 val 2^28", n / 4, 62);
  return 0;
}
