// The step after the partition path: structural checks of a CSR
// graph and the partition quality metrics of the reference's metrics.py, on the device.
//
//   gp_graph_check     graph.py:85-128 and fileio.py:173-187: neighbor range, self loops,
//                      parallel edges, symmetry (sorted directed-edge keys u*n+v against
//                      v*n+u, the reference's own test, with the hand-written radix sort)
//   gp_edge_cut        metrics.py:48-60
//   gp_comm_volumes    metrics.py:63-77: distinct foreign blocks among each vertex's
//                      neighbors, accumulated per block
//   gp_block_weights   graph.py:165-166 (np.bincount with weights): exact int64 units,
//                      or the sequential per-block fold in vertex order
//   gp_block_bfs,      metrics.py:121-168: the per-block BFS sweeps run for ALL blocks at
//   gp_block_level_top once (edges leaving a block are ignored), one CTA per block
#include <cub/device/device_scan.cuh>

#include "common.cuh"
#include "radix.cuh"

namespace gp {

// callers.cu: numpy's pairwise sum of a[0, n) into *total (part: 4096 doubles scratch)
int pairwise_sum_async(const double* a, int64_t n, double* part, double* total, cudaStream_t s);

namespace {

unsigned sm_grid(long long work, int per) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  long long want = (work + per - 1) / per;
  const long long cap = (long long)sms * 16;
  return (unsigned)(want < 1 ? 1 : (want < cap ? want : cap));
}
size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }
size_t scan_bytes(long long n) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, (const long long*)nullptr, (long long*)nullptr,
                                (int)(n > 0 ? n : 1));
  return align256(b);
}

#define VERTEX_LOOP(u, n)                                                       \
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < (n); \
       u += (long long)gridDim.x * blockDim.x)

// ---------------------------------------------------------------- structure check
// result[0] bit flags, result[1] = smallest directed-edge key u*n+v missing its reverse
enum : long long {
  CHK_RANGE = 1, CHK_SELF = 2, CHK_PARALLEL = 4, CHK_ASYM = 8, CHK_EW_ASYM = 16,
  CHK_EW_NONPOS = 32, CHK_OFFSETS = 64,
};

__global__ void check_offsets(const long long* __restrict__ off, long long n, long long nnz,
                              long long* __restrict__ result) {
  long long bad = 0;
  VERTEX_LOOP(u, n) if (off[u + 1] < off[u]) bad = CHK_OFFSETS;
  if (blockIdx.x == 0 && threadIdx.x == 0 && (off[0] != 0 || off[n] != nnz)) bad = CHK_OFFSETS;
  if (bad) atomicOr((unsigned long long*)result, (unsigned long long)bad);
}

__global__ void edge_keys(const long long* __restrict__ off, const long long* __restrict__ nbr,
                          const double* __restrict__ ew, long long n, long long nnz,
                          unsigned long long* __restrict__ fwd, unsigned long long* __restrict__ rev,
                          long long* __restrict__ result) {
  long long bad = 0;
  VERTEX_LOOP(u, n) {
    // malformed offsets (reported by check_offsets) must not index outside the arrays
    const long long j0 = off[u] < 0 ? 0 : off[u], j1 = off[u + 1] > nnz ? nnz : off[u + 1];
    for (long long j = j0; j < j1; ++j) {
      long long v = nbr[j];
      if (v < 0 || v >= n) { bad |= CHK_RANGE; v = u; }
      else if (v == u) bad |= CHK_SELF;
      if (ew && !(ew[j] > 0.0)) bad |= CHK_EW_NONPOS;
      fwd[j] = (unsigned long long)u * (unsigned long long)n + (unsigned long long)v;
      rev[j] = (unsigned long long)v * (unsigned long long)n + (unsigned long long)u;
    }
  }
  if (bad) atomicOr((unsigned long long*)result, (unsigned long long)bad);
}

__global__ void compare_sorted(const unsigned long long* __restrict__ fs,
                               const unsigned long long* __restrict__ rs,
                               const unsigned* __restrict__ fo, const unsigned* __restrict__ ro,
                               const double* __restrict__ ew, long long nnz, long long n,
                               unsigned char* __restrict__ vertex_flags,
                               long long* __restrict__ result) {
  long long bad = 0;
  VERTEX_LOOP(i, nnz) {
    const unsigned long long f = fs[i];
    if (f != rs[i]) bad |= CHK_ASYM;
    if (i > 0 && fs[i - 1] == f) {
      bad |= CHK_PARALLEL;
      if (vertex_flags) vertex_flags[f / (unsigned long long)n] = 1;
    }
    if (ew && ew[fo[i]] != ew[ro[i]]) bad |= CHK_EW_ASYM;
  }
  if (bad) atomicOr((unsigned long long*)result, (unsigned long long)bad);
}

// np.setdiff1d(fwd, rev)[0] (fileio.py:178-183): only when the sorted sequences differ
__global__ void first_missing(const unsigned long long* __restrict__ fs,
                              const unsigned long long* __restrict__ rs, long long nnz,
                              long long* __restrict__ result) {
  if (!(result[0] & CHK_ASYM)) return;
  unsigned long long best = ~0ull;
  VERTEX_LOOP(i, nnz) {
    const unsigned long long f = fs[i];
    long long lo = 0, hi = nnz;
    while (lo < hi) {
      const long long mid = (lo + hi) >> 1;
      if (rs[mid] < f) lo = mid + 1; else hi = mid;
    }
    if ((lo >= nnz || rs[lo] != f) && f < best) best = f;
  }
  if (best != ~0ull) atomicMin((unsigned long long*)&result[1], best);
}

// ---------------------------------------------------------------- edge cut
__global__ void cut_count(const long long* __restrict__ off, const long long* __restrict__ nbr,
                          const int* __restrict__ a, long long n, long long* __restrict__ per_vertex,
                          unsigned long long* __restrict__ total) {
  unsigned long long mine = 0;
  VERTEX_LOOP(u, n) {
    const int au = a[u];
    long long c = 0;
    for (long long j = off[u]; j < off[u + 1]; ++j) {
      const long long v = nbr[j];
      c += (u < v && a[v] != au) ? 1 : 0;
    }
    if (per_vertex) per_vertex[u] = c;
    mine += (unsigned long long)c;
  }
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(FULL, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(total, mine);
}

// exact integer units of the cut weights (every weight * scale is an integer)
__global__ void cut_units(const long long* __restrict__ off, const long long* __restrict__ nbr,
                          const double* __restrict__ ew, const int* __restrict__ a, long long n,
                          double scale, unsigned long long* __restrict__ total) {
  long long mine = 0;
  VERTEX_LOOP(u, n) {
    const int au = a[u];
    for (long long j = off[u]; j < off[u + 1]; ++j) {
      const long long v = nbr[j];
      if (u < v && a[v] != au) mine += (long long)(ew[j] * scale);
    }
  }
  for (int o = 16; o; o >>= 1) mine += __shfl_xor_sync(FULL, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(total, (unsigned long long)mine);
}

// the cut weights in CSR order, compacted (graph.edge_weights[mask])
__global__ void cut_gather(const long long* __restrict__ off, const long long* __restrict__ nbr,
                           const double* __restrict__ ew, const int* __restrict__ a, long long n,
                           const long long* __restrict__ pos, double* __restrict__ out) {
  VERTEX_LOOP(u, n) {
    const int au = a[u];
    long long p = pos[u];
    for (long long j = off[u]; j < off[u + 1]; ++j) {
      const long long v = nbr[j];
      if (u < v && a[v] != au) out[p++] = ew[j];
    }
  }
}

__global__ void units_to_double(const unsigned long long* __restrict__ units, double inv_scale,
                                double* __restrict__ out) {
  if (threadIdx.x == 0 && blockIdx.x == 0) out[0] = (double)(long long)units[0] * inv_scale;
}

// ---------------------------------------------------------------- communication volume
constexpr int CV_LOCAL = 48;  // neighbor blocks a single thread dedupes

__device__ __forceinline__ void add_block(long long* per_block, int* s_hist, int k_s, int b,
                                          int c) {
  if (c == 0) return;
  if (b < k_s) atomicAdd(&s_hist[b], c);
  else atomicAdd((unsigned long long*)&per_block[b], (unsigned long long)c);
}

__global__ void comm_light(const long long* __restrict__ off, const long long* __restrict__ nbr,
                           const int* __restrict__ a, long long n, int k,
                           long long* __restrict__ per_block, long long* __restrict__ heavy,
                           unsigned long long* __restrict__ n_heavy) {
  extern __shared__ int s_hist[];
  const int k_s = k < 4096 ? k : 4096;
  for (int i = threadIdx.x; i < k_s; i += blockDim.x) s_hist[i] = 0;
  __syncthreads();
  VERTEX_LOOP(u, n) {
    const long long o0 = off[u], deg = off[u + 1] - o0;
    if (deg > CV_LOCAL) {
      heavy[atomicAdd(n_heavy, 1ull)] = u;
      continue;
    }
    const int au = a[u];
    int seen[CV_LOCAL];
    int ns = 0;
    for (long long j = 0; j < deg; ++j) {
      const int b = a[nbr[o0 + j]];
      if (b == au) continue;
      bool dup = false;
      for (int i = 0; i < ns; ++i) dup |= seen[i] == b;
      if (!dup) seen[ns++] = b;
    }
    add_block(per_block, s_hist, k_s, au, ns);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < k_s; i += blockDim.x)
    if (s_hist[i]) atomicAdd((unsigned long long*)&per_block[i], (unsigned long long)s_hist[i]);
}

// one warp per high-degree vertex: neighbor j counts when no earlier neighbor has its block
__global__ void comm_heavy(const long long* __restrict__ off, const long long* __restrict__ nbr,
                           const int* __restrict__ a, const long long* __restrict__ heavy,
                           const unsigned long long* __restrict__ n_heavy,
                           long long* __restrict__ per_block) {
  const int lane = threadIdx.x & 31;
  const long long warps = ((long long)gridDim.x * blockDim.x) >> 5;
  for (long long h = (blockIdx.x * (long long)blockDim.x + threadIdx.x) >> 5;
       h < (long long)*n_heavy; h += warps) {
    const long long u = heavy[h];
    const long long o0 = off[u], deg = off[u + 1] - o0;
    const int au = a[u];
    int count = 0;
    for (long long j = lane; j < ((deg + 31) & ~31ll); j += 32) {
      const int b = j < deg ? a[nbr[o0 + j]] : au;
      bool fresh = b != au;
      // earlier chunks: every lane scans all of them (cached reads)
      for (long long i = 0; fresh && i < (j & ~31ll); ++i) fresh = a[nbr[o0 + i]] != b;
      // this chunk: lower lanes
      for (int l = 0; l < 32; ++l) {
        const int bl = __shfl_sync(FULL, b, l);
        if (l < lane && bl == b) fresh = false;
      }
      count += fresh ? 1 : 0;
    }
    for (int o = 16; o; o >>= 1) count += __shfl_xor_sync(FULL, count, o);
    if (lane == 0 && count) atomicAdd((unsigned long long*)&per_block[au], (unsigned long long)count);
  }
}

// ---------------------------------------------------------------- block weights
// warp-uniform vertex loop: every lane of a warp runs the same iterations
#define WARP_VERTEX_LOOP(u, valid, n)                                                         \
  for (long long _b = blockIdx.x * (long long)blockDim.x + (threadIdx.x & ~31); _b < (n);    \
       _b += (long long)gridDim.x * blockDim.x)                                               \
    if (long long u = _b + (threadIdx.x & 31); true)                                          \
      if (const bool valid = u < (n); true)

__global__ void block_units(const double* __restrict__ w, const int* __restrict__ a, long long n,
                            double scale, long long* __restrict__ units) {
  const int lane = threadIdx.x & 31;
  WARP_VERTEX_LOOP(u, valid, n) {
    const int b = valid ? a[u] : -1;
    long long x = !valid ? 0 : (w ? (long long)(w[u] * scale) : 1);
    // consecutive vertices mostly share a block: one atomic per warp then
    if (__match_any_sync(FULL, b) == FULL) {
      for (int o = 16; o; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
      if (lane == 0 && b >= 0) atomicAdd((unsigned long long*)&units[b], (unsigned long long)x);
    } else if (valid) {
      atomicAdd((unsigned long long*)&units[b], (unsigned long long)x);
    }
  }
}

__global__ void units_to_weights(const long long* __restrict__ units, int k, double inv_scale,
                                 double* __restrict__ out) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < k; b += gridDim.x * blockDim.x)
    out[b] = (double)units[b] * inv_scale;
}

__global__ void block_keys(const int* __restrict__ a, long long n, unsigned long long* __restrict__ keys) {
  VERTEX_LOOP(u, n) keys[u] = (unsigned long long)(unsigned)a[u];
}
__global__ void block_starts(const unsigned long long* __restrict__ ks, long long n, int k,
                             long long* __restrict__ start) {
  // start[b] = first sorted position of block >= b; start[k] = n
  VERTEX_LOOP(i, n) {
    const long long b = (long long)ks[i];
    const long long prev = i == 0 ? -1 : (long long)ks[i - 1];
    for (long long x = prev + 1; x <= b; ++x) start[x] = i;
    if (i == n - 1) for (long long x = b + 1; x <= k; ++x) start[x] = n;
  }
}
// np.bincount(a, weights): sequential fold per block, in vertex order
__global__ void block_fold(const unsigned* __restrict__ order, const long long* __restrict__ start,
                           const double* __restrict__ w, int k, double* __restrict__ out) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < k; b += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (long long i = start[b]; i < start[b + 1]; ++i) s = __dadd_rn(s, w[order[i]]);
    out[b] = s;
  }
}

// ---------------------------------------------------------------- per-block BFS
// One CTA per block (blocks are independent: edges leaving a block are ignored), so a
// sweep of ALL blocks is one launch with no grid-wide step per level.  The CTA keeps the
// block's frontier queue in global memory (a block's vertices enter it exactly once, so
// block b owns queue[qbase[b], qbase[b + 1])), claims unvisited neighbors with an
// atomicCAS on their level and synchronises its own levels with __syncthreads.
constexpr int BFS_THREADS = 256;   // frontiers are small; 8 CTAs per SM hide the per-level latency

__global__ void __launch_bounds__(BFS_THREADS) bfs_blocks(
    const long long* __restrict__ off, const long long* __restrict__ nbr,
    const int* __restrict__ a, int k, const long long* __restrict__ roots,
    const long long* __restrict__ qbase, long long* __restrict__ queue, int* __restrict__ level,
    int* __restrict__ depth, long long* __restrict__ far, long long* __restrict__ reached) {
  __shared__ long long s_head, s_tail, s_next;
  __shared__ unsigned long long s_far;
  for (int b = blockIdx.x; b < k; b += gridDim.x) {
    const long long root = roots[b];
    if (root < 0) {
      if (threadIdx.x == 0) { depth[b] = -1; far[b] = -1; reached[b] = 0; }
      continue;
    }
    long long* q = queue + qbase[b];
    __syncthreads();  // the previous block's reads of the shared cursors are done
    if (threadIdx.x == 0) {
      q[0] = root;
      level[root] = 0;
      s_head = 0; s_tail = 1; s_next = 1;
    }
    __syncthreads();
    int d = 0;
    long long head = 0, tail = 1;
    for (;;) {
      for (long long i = head + threadIdx.x; i < tail; i += BFS_THREADS) {
        const long long u = q[i];
        for (long long j = off[u]; j < off[u + 1]; ++j) {
          const long long v = nbr[j];
          if (a[v] != b || level[v] >= 0) continue;
          if (atomicCAS(&level[v], -1, d + 1) == -1)
            q[atomicAdd((unsigned long long*)&s_next, 1ull)] = v;
        }
      }
      __syncthreads();
      const long long next = s_next;
      if (next == tail) break;  // no deeper level: [head, tail) is the deepest one
      head = tail;
      tail = next;
      ++d;
      __syncthreads();
    }
    // deepest level: its lowest vertex id (metrics.py:115-118)
    if (threadIdx.x == 0) s_far = ~0ull;
    __syncthreads();
    unsigned long long mine = ~0ull;
    for (long long i = head + threadIdx.x; i < tail; i += BFS_THREADS)
      mine = (unsigned long long)q[i] < mine ? (unsigned long long)q[i] : mine;
    for (int o = 16; o; o >>= 1) {
      const unsigned long long other = __shfl_xor_sync(FULL, mine, o);
      mine = other < mine ? other : mine;
    }
    if ((threadIdx.x & 31) == 0 && mine != ~0ull) atomicMin(&s_far, mine);
    __syncthreads();
    if (threadIdx.x == 0) { depth[b] = d; far[b] = (long long)s_far; reached[b] = tail; }
  }
}

// per block: the largest key (level + 1) << 32 | (2^32 - 1 - vertex) over its vertices
// v != exclude[b] with key < below[b]; unreached vertices have key < 2^32.
__global__ void level_top(const int* __restrict__ level, const int* __restrict__ a, long long n,
                          const long long* __restrict__ exclude,
                          const unsigned long long* __restrict__ below,
                          unsigned long long* __restrict__ out,
                          unsigned long long* __restrict__ unreached) {
  const int lane = threadIdx.x & 31;
  WARP_VERTEX_LOOP(u, valid, n) {
    const int b = valid ? a[u] : -1;
    const int lv = valid ? level[u] : 0;
    unsigned long long key =
        ((unsigned long long)(lv + 1) << 32) | (0xffffffffull - (unsigned long long)u);
    if (!valid || (exclude && exclude[b] == u) || (below && key >= below[b])) key = 0;
    unsigned long long miss = valid && lv < 0 ? 1 : 0;
    if (__match_any_sync(FULL, b) == FULL) {
      for (int o = 16; o; o >>= 1) {
        const unsigned long long other = __shfl_xor_sync(FULL, key, o);
        key = other > key ? other : key;
        miss += __shfl_xor_sync(FULL, miss, o);
      }
      if (lane != 0) { key = 0; miss = 0; }
    }
    if (b >= 0 && key) atomicMax(&out[b], key);
    if (b >= 0 && unreached && miss) atomicAdd(&unreached[b], miss);
  }
}

}  // namespace
}  // namespace gp

using namespace gp;

extern "C" {

int gp_graph_check_workspace_bytes(int64_t nnz, size_t* bytes) {
  GP_REQUIRE(nnz >= 0 && nnz < (1ll << 31), "gp_graph_check: more than 2^31 directed edges");
  size_t sort = 0;
  int rc = gp_sort_workspace_bytes(nnz, &sort);
  if (rc) return rc;
  *bytes = 4 * align256((size_t)nnz * 8) + 2 * align256((size_t)nnz * 4) + align256(sort) + 256;
  return GP_OK;
}

int gp_graph_check(const int64_t* offsets, const int64_t* neighbors, const double* edge_weights,
                   int64_t n, int64_t nnz, uint8_t* vertex_flags, int64_t* result,
                   void* workspace, size_t workspace_bytes, void* stream) {
  GP_REQUIRE(n >= 1 && n <= (1ll << 31), "gp_graph_check: n out of range");
  size_t need = 0;
  int rc = gp_graph_check_workspace_bytes(nnz, &need);
  if (rc) return rc;
  GP_REQUIRE(workspace_bytes >= need, "gp_graph_check: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  GP_CUDA(cudaMemsetAsync(result, 0, sizeof(int64_t), s));
  GP_CUDA(cudaMemsetAsync(result + 1, 0xff, sizeof(int64_t), s));
  check_offsets<<<sm_grid(n, 256), 256, 0, s>>>((const long long*)offsets, n, nnz,
                                                 (long long*)result);
  if (nnz == 0) return check_launch("gp_graph_check");
  char* p = (char*)workspace;
  // entries no vertex owns (malformed offsets) keep key 0 on both sides
  GP_CUDA(cudaMemsetAsync(p, 0, 2 * align256((size_t)nnz * 8), s));
  const size_t a8 = align256((size_t)nnz * 8), a4 = align256((size_t)nnz * 4);
  unsigned long long* fwd = (unsigned long long*)p; p += a8;
  unsigned long long* rev = (unsigned long long*)p; p += a8;
  unsigned long long* fs = (unsigned long long*)p; p += a8;
  unsigned long long* rs = (unsigned long long*)p; p += a8;
  unsigned* fo = (unsigned*)p; p += a4;
  unsigned* ro = (unsigned*)p; p += a4;
  size_t sort = 0;
  gp_sort_workspace_bytes(nnz, &sort);
  edge_keys<<<sm_grid(n, 128), 128, 0, s>>>((const long long*)offsets, (const long long*)neighbors,
                                            edge_weights, n, nnz, fwd, rev, (long long*)result);
  int bits = 1;
  while (bits < 64 && ((unsigned long long)n * (unsigned long long)n - 1) >> bits) ++bits;
  rc = gp_sort_pairs((const uint64_t*)fwd, nullptr, (uint64_t*)fs, fo, nnz, bits, p, sort, stream);
  if (rc) return rc;
  rc = gp_sort_pairs((const uint64_t*)rev, nullptr, (uint64_t*)rs, ro, nnz, bits, p, sort, stream);
  if (rc) return rc;
  compare_sorted<<<sm_grid(nnz, 256), 256, 0, s>>>(fs, rs, fo, ro, edge_weights, nnz, n,
                                                    vertex_flags, (long long*)result);
  first_missing<<<sm_grid(nnz, 256), 256, 0, s>>>(fs, rs, nnz, (long long*)result);
  return check_launch("gp_graph_check");
}

int gp_edge_cut_workspace_bytes(int64_t n, int64_t nnz, size_t* bytes) {
  GP_REQUIRE(n >= 1 && n < (1ll << 31) - 1 && nnz >= 0, "gp_edge_cut: sizes out of range");
  *bytes = 2 * align256((size_t)(n + 1) * 8) + scan_bytes(n + 1) + align256((size_t)nnz / 2 * 8 + 8) +
           align256(4097 * 8) + 256;
  return GP_OK;
}

int gp_edge_cut(const int64_t* offsets, const int64_t* neighbors, const double* edge_weights,
                double scale, const int32_t* assignment, int64_t n, int64_t nnz, double* out,
                void* workspace, size_t workspace_bytes, void* stream) {
  size_t need = 0;
  int rc = gp_edge_cut_workspace_bytes(n, nnz, &need);
  if (rc) return rc;
  GP_REQUIRE(workspace_bytes >= need, "gp_edge_cut: workspace too small");
  GP_REQUIRE(scale >= 0.0, "gp_edge_cut: scale must be >= 0");
  cudaStream_t s = (cudaStream_t)stream;
  char* p = (char*)workspace;
  const size_t an = align256((size_t)(n + 1) * 8);
  long long* cnt = (long long*)p; p += an;
  long long* pos = (long long*)p; p += an;
  void* sws = p;
  size_t sb = scan_bytes(n + 1);
  p += sb;
  double* cutw = (double*)p; p += align256((size_t)nnz / 2 * 8 + 8);
  double* part = (double*)p; p += align256(4097 * 8);
  unsigned long long* total = (unsigned long long*)p;
  GP_CUDA(cudaMemsetAsync(total, 0, 8, s));
  const unsigned g = sm_grid(n, 128);
  const long long* off = (const long long*)offsets;
  const long long* nb = (const long long*)neighbors;
  if (!edge_weights) {
    cut_count<<<g, 128, 0, s>>>(off, nb, assignment, n, nullptr, total);
    units_to_double<<<1, 32, 0, s>>>(total, 1.0, out);
    return check_launch("gp_edge_cut");
  }
  if (scale > 0.0) {
    cut_units<<<g, 128, 0, s>>>(off, nb, edge_weights, assignment, n, scale, total);
    units_to_double<<<1, 32, 0, s>>>(total, 1.0 / scale, out);
    return check_launch("gp_edge_cut");
  }
  // weights that are not exactly summable: numpy's pairwise sum of the masked weights
  GP_CUDA(cudaMemsetAsync(cnt + n, 0, 8, s));
  cut_count<<<g, 128, 0, s>>>(off, nb, assignment, n, cnt, total);
  GP_CUDA(cub::DeviceScan::ExclusiveSum(sws, sb, cnt, pos, (int)(n + 1), s));
  cut_gather<<<g, 128, 0, s>>>(off, nb, edge_weights, assignment, n, pos, cutw);
  long long m_cut = 0;
  GP_CUDA(cudaMemcpyAsync(&m_cut, pos + n, 8, cudaMemcpyDeviceToHost, s));
  GP_CUDA(cudaStreamSynchronize(s));
  if (m_cut == 0) {
    GP_CUDA(cudaMemsetAsync(out, 0, 8, s));
    return GP_OK;
  }
  return pairwise_sum_async(cutw, m_cut, part, out, s);
}

int gp_comm_volumes(const int64_t* offsets, const int64_t* neighbors, const int32_t* assignment,
                    int64_t n, int k, int64_t* per_block, int64_t* heavy_scratch, void* stream) {
  GP_REQUIRE(n >= 1 && k >= 1, "gp_comm_volumes: sizes out of range");
  cudaStream_t s = (cudaStream_t)stream;
  // heavy_scratch: n + 1 int64 (the count lives in the last slot)
  unsigned long long* n_heavy = (unsigned long long*)(heavy_scratch + n);
  GP_CUDA(cudaMemsetAsync(per_block, 0, (size_t)k * 8, s));
  GP_CUDA(cudaMemsetAsync(n_heavy, 0, 8, s));
  const int k_s = k < 4096 ? k : 4096;
  comm_light<<<sm_grid(n, 128), 128, (size_t)k_s * sizeof(int), s>>>(
      (const long long*)offsets, (const long long*)neighbors, assignment, n, k,
      (long long*)per_block, (long long*)heavy_scratch, n_heavy);
  comm_heavy<<<592, 256, 0, s>>>(
      (const long long*)offsets, (const long long*)neighbors, assignment,
      (const long long*)heavy_scratch, n_heavy, (long long*)per_block);
  return check_launch("gp_comm_volumes");
}

int gp_block_weights_workspace_bytes(int64_t n, int k, size_t* bytes) {
  GP_REQUIRE(n >= 1 && n < (1ll << 31) && k >= 1, "gp_block_weights: sizes out of range");
  size_t sort = 0;
  int rc = gp_sort_workspace_bytes(n, &sort);
  if (rc) return rc;
  *bytes = 2 * align256((size_t)n * 8) + align256((size_t)n * 4) + align256((size_t)(k + 1) * 8) +
           align256(sort) + 256;
  return GP_OK;
}

int gp_block_weights(const double* weights, const int32_t* assignment, int64_t n, int k,
                     double scale, double* out, void* workspace, size_t workspace_bytes,
                     void* stream) {
  size_t need = 0;
  int rc = gp_block_weights_workspace_bytes(n, k, &need);
  if (rc) return rc;
  GP_REQUIRE(workspace_bytes >= need, "gp_block_weights: workspace too small");
  GP_REQUIRE(weights || scale == 1.0, "gp_block_weights: unit weights need scale 1");
  cudaStream_t s = (cudaStream_t)stream;
  char* p = (char*)workspace;
  if (scale > 0.0) {
    long long* units = (long long*)p;
    GP_CUDA(cudaMemsetAsync(units, 0, (size_t)k * 8, s));
    block_units<<<sm_grid(n, 256), 256, 0, s>>>(weights, assignment, n, scale, units);
    units_to_weights<<<grid_for(k, 256), 256, 0, s>>>(units, k, 1.0 / scale, out);
    return check_launch("gp_block_weights");
  }
  unsigned long long* keys = (unsigned long long*)p; p += align256((size_t)n * 8);
  unsigned long long* ks = (unsigned long long*)p; p += align256((size_t)n * 8);
  unsigned* order = (unsigned*)p; p += align256((size_t)n * 4);
  long long* start = (long long*)p; p += align256((size_t)(k + 1) * 8);
  size_t sort = 0;
  gp_sort_workspace_bytes(n, &sort);
  block_keys<<<sm_grid(n, 256), 256, 0, s>>>(assignment, n, keys);
  int bits = 1;
  while (bits < 32 && ((unsigned)(k - 1) >> bits)) ++bits;
  rc = radix::sort_pairs<uint64_t, uint32_t>((const uint64_t*)keys, nullptr, (uint64_t*)ks, order,
                                             n, 0, bits, p, sort, s, false);
  if (rc) return rc;
  block_starts<<<sm_grid(n, 256), 256, 0, s>>>(ks, n, k, start);
  block_fold<<<grid_for(k, 64), 64, 0, s>>>(order, start, weights, k, out);
  return check_launch("gp_block_weights");
}

int gp_block_bfs(const int64_t* offsets, const int64_t* neighbors, const int32_t* assignment,
                 int64_t n, int k, const int64_t* roots, const int64_t* qbase, int64_t* queue,
                 int32_t* level, int32_t* depth, int64_t* far, int64_t* reached, void* stream) {
  GP_REQUIRE(n >= 1 && k >= 1, "gp_block_bfs: sizes out of range");
  cudaStream_t s = (cudaStream_t)stream;
  GP_CUDA(cudaMemsetAsync(level, 0xff, (size_t)n * 4, s));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int grid = k < sms * 8 ? k : sms * 8;
  bfs_blocks<<<grid, BFS_THREADS, 0, s>>>((const long long*)offsets, (const long long*)neighbors,
                                          assignment, k, (const long long*)roots,
                                          (const long long*)qbase, (long long*)queue, level,
                                          depth, (long long*)far, (long long*)reached);
  return check_launch("gp_block_bfs");
}

int gp_block_level_top(const int32_t* level, const int32_t* assignment, int64_t n, int k,
                       const int64_t* exclude, const uint64_t* below, uint64_t* out,
                       uint64_t* unreached, void* stream) {
  GP_REQUIRE(n >= 1 && n <= (1ll << 32) - 1 && k >= 1, "gp_block_level_top: sizes out of range");
  cudaStream_t s = (cudaStream_t)stream;
  GP_CUDA(cudaMemsetAsync(out, 0, (size_t)k * 8, s));
  if (unreached) GP_CUDA(cudaMemsetAsync(unreached, 0, (size_t)k * 8, s));
  level_top<<<sm_grid(n, 256), 256, 0, s>>>(level, assignment, n, (const long long*)exclude,
                                            (const unsigned long long*)below,
                                            (unsigned long long*)out,
                                            (unsigned long long*)unreached);
  return check_launch("gp_block_level_top");
}

}  // extern "C"
