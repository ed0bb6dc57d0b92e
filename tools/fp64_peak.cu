// FP64 peak of this GPU: dependent-free DFMA chains on every SM (the FP64 term of
// north_star's roofline; MEASURED_PEAKS.json has no FP64 figure).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o fp64_peak tools/fp64_peak.cu
//   ./fp64_peak            -> one JSON line {"tflops": ..., "how": ...}
#include <cstdio>
#include <cuda_runtime.h>

constexpr int CHAINS = 8;
constexpr int ITERS = 4096;

__global__ void dfma_kernel(double* out, double a, double b) {
  double x[CHAINS];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) x[c] = threadIdx.x * 1e-3 + c;
  for (int i = 0; i < ITERS; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c) x[c] = fma(x[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += x[c];
  if (s == 12345.678) out[0] = s;   // never true; keeps the chains alive
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int threads = 512, blocks = sms * 4;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);   // warm-up
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 10; ++rep) {
    cudaEventRecord(e0);
    dfma_kernel<<<blocks, threads>>>(out, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double flops = 2.0 * CHAINS * ITERS * (double)threads * blocks;
  printf("{\"tflops\": %.3f, \"ms\": %.4f, \"sms\": %d, \"how\": \"tools/fp64_peak.cu: %d blocks x %d "
         "threads x %d independent DFMA chains x %d iterations (2 flops each), best of 10, CUDA "
         "events\"}\n",
         flops / (best * 1e-3) / 1e12, best, sms, blocks, threads, CHAINS, ITERS);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}
