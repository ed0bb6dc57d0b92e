// Device-resident loops: a CUDA graph holding one conditional WHILE node whose body
// is captured from the work issued on a stream (the balance rounds of one
// movement iteration).  A kernel of the body decides whether the
// loop runs again (cudaGraphSetConditional), so the host issues the whole loop
// once and synchronises once, instead of once per round.
#include "common.cuh"

namespace gp {

struct LoopGraph {
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaGraphConditionalHandle handle = 0;
  cudaStream_t stream = nullptr;
};

__global__ void countdown_kernel(int* counter, cudaGraphConditionalHandle h) {
  const int left = --(*counter);
  cudaGraphSetConditional(h, left > 0 ? 1u : 0u);
}

}  // namespace gp

using namespace gp;

extern "C" {

int gp_loop_graph_begin(void* stream, void** ctx_out) {
  GP_REQUIRE(ctx_out != nullptr, "gp_loop_graph_begin: ctx_out is NULL");
  LoopGraph* g = new LoopGraph();
  g->stream = (cudaStream_t)stream;
  GP_CUDA(cudaGraphCreate(&g->graph, 0));
  GP_CUDA(cudaGraphConditionalHandleCreate(&g->handle, g->graph, 1, cudaGraphCondAssignDefault));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = g->handle;
  p.conditional.type = cudaGraphCondTypeWhile;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  GP_CUDA(cudaGraphAddNode(&node, g->graph, nullptr, 0, &p));
  cudaGraph_t body = p.conditional.phGraph_out[0];
  GP_CUDA(cudaStreamBeginCaptureToGraph(g->stream, body, nullptr, nullptr, 0,
                                        cudaStreamCaptureModeRelaxed));
  *ctx_out = g;
  return GP_OK;
}

unsigned long long gp_loop_graph_handle(void* ctx) {
  return ctx ? (unsigned long long)((LoopGraph*)ctx)->handle : 0ull;
}

int gp_loop_graph_end(void* ctx) {
  GP_REQUIRE(ctx != nullptr, "gp_loop_graph_end: no graph");
  LoopGraph* g = (LoopGraph*)ctx;
  cudaGraph_t body = nullptr;
  GP_CUDA(cudaStreamEndCapture(g->stream, &body));
  GP_CUDA(cudaGraphInstantiate(&g->exec, g->graph, 0));
  return GP_OK;
}

int gp_loop_graph_launch(void* ctx, void* stream) {
  GP_REQUIRE(ctx != nullptr && ((LoopGraph*)ctx)->exec, "gp_loop_graph_launch: not built");
  GP_CUDA(cudaGraphLaunch(((LoopGraph*)ctx)->exec, (cudaStream_t)stream));
  return GP_OK;
}

int gp_loop_graph_destroy(void* ctx) {
  if (!ctx) return GP_OK;
  LoopGraph* g = (LoopGraph*)ctx;
  if (g->exec) cudaGraphExecDestroy(g->exec);
  if (g->graph) cudaGraphDestroy(g->graph);
  delete g;
  return GP_OK;
}

int gp_loop_test_countdown(int* counter, unsigned long long handle, void* stream) {
  countdown_kernel<<<1, 1, 0, (cudaStream_t)stream>>>(counter,
                                                       (cudaGraphConditionalHandle)handle);
  return check_launch("loop_test_countdown");
}

}  // extern "C"

namespace gp {

// gp_balance_decide: one block; the block-weight sums are exact (integer units of
// 1/wscale below 2^53), so any summation order gives numpy's bits.
__global__ void __launch_bounds__(1024) balance_decide_kernel(
    const long long* __restrict__ red, int k, double wscale, double eps, int max_rounds,
    double* __restrict__ bal, const double* __restrict__ cur, double* __restrict__ next,
    cudaGraphConditionalHandle handle, int use_handle) {
  __shared__ double s_sum[32], s_max[32];
  __shared__ double s_tgt, s_cap;
  __shared__ int s_stop;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double sum = 0.0, mx = -INFINITY;
  for (int c = tid; c < k; c += blockDim.x) {
    const double w = (double)red[c] / wscale;   // blk_int.astype(float64) / scale
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
    for (int c = tid; c < k; c += blockDim.x) {
      const double w = (double)red[c] / wscale;
      const double gamma = w > 0.0 ? tgt / w : INFINITY;
      const double f = fmin(fmax(__dsqrt_rn(gamma), lo), hi);   // clip(gamma ** 0.5)
      next[c] = cur[c] * f;
    }
  }
  if (tid == 0 && use_handle) cudaGraphSetConditional(handle, s_stop ? 0u : 1u);
}

}  // namespace gp

extern "C" int gp_balance_decide(const long long* red, int k, double wscale, double eps,
                                 int max_rounds, double* bal, const double* infl_cur,
                                 double* infl_next, unsigned long long handle, void* stream) {
  GP_REQUIRE(red && bal && infl_cur && infl_next && k >= 1 && max_rounds >= 1 && wscale > 0,
             "gp_balance_decide: bad args");
  gp::balance_decide_kernel<<<1, 1024, 0, (cudaStream_t)stream>>>(
      red, k, wscale, eps, max_rounds, bal, infl_cur, infl_next,
      (cudaGraphConditionalHandle)handle, handle != 0);
  return gp::check_launch("balance_decide");
}
