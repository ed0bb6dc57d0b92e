// Hand-written device radix sort (see radix.cuh for the design).
//
// Replaces the reference's np.lexsort((gids, keys)) (ranksim.py:158) for the SFC
// stage and the library sorts of the internal passes (fold run sort, warm-up
// permutation, center grid).
#include "common.cuh"
#include "radix.cuh"

namespace gp {
namespace radix {

namespace {

constexpr uint64_t kFlagAgg = 1ull << 62;
constexpr uint64_t kFlagIncl = 2ull << 62;
constexpr uint64_t kValMask = (1ull << 56) - 1;

__device__ __forceinline__ uint64_t pack(uint64_t flag, uint32_t epoch, uint64_t v) {
  return flag | ((uint64_t)epoch << 56) | v;
}

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

template <typename K>
__device__ __forceinline__ unsigned digit_of(K k, int shift, unsigned mask) {
  return (unsigned)(k >> shift) & mask;
}

// exclusive scan of one value per thread over the 256 threads of the block
template <typename T>
__device__ __forceinline__ T block_excl_scan(T v, T* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  T x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T y = __shfl_up_sync(FULL, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_tot[warp] = x;
  __syncthreads();
  T before = 0;
  for (int w = 0; w < warp; ++w) before += warp_tot[w];
  __syncthreads();
  return before + x - v;
}

// Digit counts of npass consecutive 8-bit digits starting at shift0 (< end_bit),
// one read of the keys.  gate: run only when *gate != 0 (nullptr: always).
template <typename K>
__global__ void __launch_bounds__(kThreads) hist_kernel(const K* __restrict__ keys, int64_t n,
                                                         int shift0, int end_bit, int npass,
                                                         unsigned long long* counts,
                                                         const int* gate) {
  if (gate && *(volatile const int*)gate == 0) return;
  __shared__ unsigned sh[kMaxPasses * kRadix];
  for (int i = threadIdx.x; i < npass * kRadix; i += kThreads) sh[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * kThreads;
  constexpr int HU = 4;   // keys in flight per thread
  for (int64_t i0 = (int64_t)blockIdx.x * kThreads + threadIdx.x; i0 < n; i0 += HU * stride) {
    K k[HU];
#pragma unroll
    for (int u = 0; u < HU; ++u) k[u] = i0 + u * stride < n ? keys[i0 + u * stride] : (K)0;
#pragma unroll
    for (int u = 0; u < HU; ++u) {
      if (i0 + u * stride >= n) break;
      for (int p = 0; p < npass; ++p) {
        const int sft = shift0 + 8 * p;
        const int nb = end_bit - sft < 8 ? end_bit - sft : 8;
        atomicAdd(&sh[p * kRadix + digit_of(k[u], sft, (1u << nb) - 1)], 1u);
      }
    }
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * kRadix; i += kThreads)
    if (sh[i]) atomicAdd(&counts[i], (unsigned long long)sh[i]);
}

// One stable LSD pass on digit [shift, shift+nb).  Persistent; tiles in counter order.
template <typename K, typename V>
__global__ void __launch_bounds__(kThreads, 2)
    onesweep_kernel(const K* __restrict__ kin, const V* __restrict__ vin, K* __restrict__ kout,
                    V* __restrict__ vout, int64_t n, int shift, int nb,
                    const unsigned long long* __restrict__ counts, unsigned long long* status,
                    unsigned* tile_ctr, uint32_t epoch, const int* gate) {
  if (gate && *(volatile const int*)gate == 0) return;
  extern __shared__ __align__(16) unsigned char dyn[];
  K* sk = reinterpret_cast<K*>(dyn);
  V* sv = reinterpret_cast<V*>(dyn + sizeof(K) * kTile);
  __shared__ unsigned whist[kWarps][kRadix];
  __shared__ long long dbase[kRadix];  // first output position of each digit
  __shared__ long long gofs[kRadix];   // per tile: output position - local position
  __shared__ unsigned toff[kRadix];    // per tile: first local position of each digit
  __shared__ long long wtot[kWarps];
  __shared__ int s_tile;

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const unsigned mask = (1u << nb) - 1;
  const int64_t ntiles = (n + kTile - 1) / kTile;
  {
    const long long c = (long long)counts[t];
    dbase[t] = block_excl_scan<long long>(c, wtot);
  }
  for (;;) {
    if (t == 0) s_tile = (int)atomicAdd(tile_ctr, 1u);
    for (int i = t; i < kWarps * kRadix; i += kThreads) (&whist[0][0])[i] = 0;
    __syncthreads();
    const int tile = s_tile;
    if (tile >= ntiles) break;
    const int64_t t0 = (int64_t)tile * kTile;
    const int64_t wbase = t0 + warp * (32 * kItems);

    K key[kItems];
    V val[kItems];
    unsigned rank[kItems];
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int64_t idx = wbase + i * 32 + lane;
      if (idx < n) {
        key[i] = kin[idx];
        val[i] = vin ? vin[idx] : (V)idx;
      } else {
        key[i] = 0;
        val[i] = 0;
      }
    }
    // warp ranking: items in (i, lane) order = position order within the warp
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int64_t idx = wbase + i * 32 + lane;
      const unsigned d = idx < n ? digit_of(key[i], shift, mask) : (unsigned)kRadix;
      const unsigned peers = __match_any_sync(FULL, d);
      const int leader = __ffs(peers) - 1;
      unsigned b = 0;
      if (lane == leader && d < kRadix) {
        b = whist[warp][d];
        whist[warp][d] = b + __popc(peers);
      }
      b = __shfl_sync(FULL, b, leader);
      rank[i] = b + __popc(peers & lanemask_lt());
      __syncwarp();
    }
    __syncthreads();
    // thread t = digit t: warp offsets and the tile's count
    unsigned cnt = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      const unsigned c = whist[w][t];
      whist[w][t] = cnt;
      cnt += c;
    }
    // decoupled look-back over the earlier tiles' counts of digit t
    unsigned long long* st = status + (int64_t)tile * kRadix + t;
    long long excl = 0;
    if (tile == 0) {
      *(volatile unsigned long long*)st = pack(kFlagIncl, epoch, cnt);
    } else {
      *(volatile unsigned long long*)st = pack(kFlagAgg, epoch, cnt);
      int64_t p = tile - 1;
      for (;;) {
        const unsigned long long s =
            *(volatile const unsigned long long*)(status + p * kRadix + t);
        if ((uint32_t)((s >> 56) & 63) != epoch || (s >> 62) == 0) continue;
        excl += (long long)(s & kValMask);
        if ((s >> 62) == 2) break;
        --p;
      }
      *(volatile unsigned long long*)st = pack(kFlagIncl, epoch, (uint64_t)(excl + cnt));
    }
    const unsigned lo = block_excl_scan<unsigned>(cnt, reinterpret_cast<unsigned*>(wtot));
    toff[t] = lo;
    gofs[t] = dbase[t] + excl - (long long)lo;
    __syncthreads();
    // reorder by digit in shared memory
#pragma unroll
    for (int i = 0; i < kItems; ++i) {
      const int64_t idx = wbase + i * 32 + lane;
      if (idx < n) {
        const unsigned d = digit_of(key[i], shift, mask);
        const unsigned pos = toff[d] + whist[warp][d] + rank[i];
        sk[pos] = key[i];
        sv[pos] = val[i];
      }
    }
    __syncthreads();
    const int valid = (int)(n - t0 < kTile ? n - t0 : kTile);
    for (int j = t; j < valid; j += kThreads) {
      const K k = sk[j];
      const int64_t g = gofs[digit_of(k, shift, mask)] + j;
      kout[g] = k;
      vout[g] = sv[j];
    }
    __syncthreads();
  }
}

// Final pass of the hybrid: the input is stably sorted by the key bits above
// `lowbits`; every bucket of equal high bits is ordered by the full key, ties in
// position order.  CTA b owns the buckets that START in positions
// [b*kSegTile, (b+1)*kSegTile).  A bucket larger than kSegMax sets *overflow.
template <typename K, typename V>
__global__ void __launch_bounds__(kThreads) bucket_rank_kernel(
    const K* __restrict__ kin, const V* __restrict__ vin, K* __restrict__ kout,
    V* __restrict__ vout, int64_t n, int lowbits, K kmask, int* overflow) {
  constexpr int CAP = kSegTile + kSegMax + 256 + 1;
  __shared__ K sk[CAP];  // sk[r + 1] = key at position lo + r
  __shared__ int s_first, s_found;
  const int t = threadIdx.x;
  const int64_t lo = (int64_t)blockIdx.x * kSegTile;
  if (lo >= n) return;
  const int span = (int)(n - lo < kSegTile ? n - lo : kSegTile);
  for (int r = t - 1; r < span; r += kThreads)
    if (lo + r >= 0) sk[r + 1] = kin[lo + r];
  if (t == 0) {
    s_first = INT32_MAX;
    s_found = INT32_MAX;
  }
  __syncthreads();
  for (int r = t; r < span; r += kThreads) {
    const bool start =
        (lo + r == 0) || (((sk[r + 1] & kmask) >> lowbits) != ((sk[r] & kmask) >> lowbits));
    if (start) atomicMin(&s_first, r);
  }
  __syncthreads();
  const int r0 = s_first;
  if (r0 == INT32_MAX) return;  // every position continues a bucket owned earlier
  // end of the last owned bucket: the first bucket start at or after span
  int re;
  if (lo + span >= n) {
    re = span;
  } else {
    int c = span;  // positions [span, c) are loaded
    for (;;) {
      const int cnt = (int)(n - (lo + c) < 256 ? n - (lo + c) : 256);
      if (t < cnt) sk[c + t + 1] = kin[lo + c + t];
      __syncthreads();
      if (t < cnt && ((sk[c + t + 1] & kmask) >> lowbits) != ((sk[c + t] & kmask) >> lowbits))
        atomicMin(&s_found, c + t);
      __syncthreads();
      const int f = s_found;
      __syncthreads();  // every thread has read s_found before it is reset
      if (t == 0) s_found = INT32_MAX;
      if (f != INT32_MAX) {
        re = f;
        break;
      }
      c += cnt;
      if (lo + c >= n) {
        re = c;
        break;
      }
      if (c + 256 + 1 > CAP) {  // the bucket is longer than kSegMax
        if (t == 0) atomicExch(overflow, 1);
        return;
      }
    }
  }
  for (int r = r0 + t; r < re; r += kThreads) {
    const K full = sk[r + 1];
    const K key = full & kmask;  // the sort bits (bits outside [begin, end) are carried)
    const K h = key >> lowbits;
    int a = r, b = r + 1;
    while (a > r0 && ((sk[a] & kmask) >> lowbits) == h) --a;
    while (b < re && ((sk[b + 1] & kmask) >> lowbits) == h) ++b;
    if (b - a > kSegMax) {
      atomicExch(overflow, 1);
      continue;
    }
    int rank = 0;
    for (int j = a; j < b; ++j) {
      const K kj = sk[j + 1] & kmask;
      rank += (kj < key) | ((kj == key) & (j < r));
    }
    const int64_t dst = lo + a + rank;
    kout[dst] = full;
    vout[dst] = vin[lo + r];
  }
}

struct Layout {
  size_t tmpk, tmpv, counts, ctr, flag, status, total;
};

Layout layout(int64_t n, int kb, int vb) {
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  Layout L;
  size_t o = 0;
  L.tmpk = o;
  o += al((size_t)n * kb);
  L.tmpv = o;
  o += al((size_t)n * vb);
  L.counts = o;  // zeroed region starts here
  o += al(sizeof(unsigned long long) * kMaxPasses * kRadix);
  L.ctr = o;
  o += al(sizeof(unsigned) * kMaxPasses);
  L.flag = o;
  o += al(sizeof(int));
  L.status = o;
  const int64_t ntiles = (n + kTile - 1) / kTile;
  o += al(sizeof(unsigned long long) * kRadix * (size_t)(ntiles > 0 ? ntiles : 1));
  L.total = o;
  return L;
}

int top_passes(int64_t n, int width) {
  int lg = 0;
  while ((1ll << lg) < n) ++lg;
  int p = (lg - 3 + 7) / 8;
  if (p < 1) p = 1;
  return p;
}

template <typename K, typename V>
int grid_onesweep() {
  static int g = 0;
  if (!g) {
    int dev = 0, sms = 148, occ = 1;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int dyn = (int)((sizeof(K) + sizeof(V)) * kTile);
    cudaFuncSetAttribute(onesweep_kernel<K, V>, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, onesweep_kernel<K, V>, kThreads, dyn);
    g = sms * (occ > 0 ? occ : 1);
  }
  return g;
}

int grid_hist() {
  static int g = 0;
  if (!g) {
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    g = sms * 8;
  }
  return g;
}

// npass LSD passes on digits starting at shift0 (histogram first), ping-pong
// ending in (kout, vout).
template <typename K, typename V>
int lsd(const K* kin, const V* vin, K* kout, V* vout, K* tk, V* tv, int64_t n, int shift0,
        int end_bit, int npass, unsigned long long* counts, unsigned* ctr, uint32_t& epoch,
        unsigned long long* status, const int* gate, cudaStream_t s) {
  const int dyn = (int)((sizeof(K) + sizeof(V)) * kTile);
  const int64_t hb = (n + kThreads - 1) / kThreads;
  const int hg = (int)(hb < grid_hist() ? hb : grid_hist());
  hist_kernel<K><<<hg, kThreads, 0, s>>>(kin, n, shift0, end_bit, npass, counts, gate);
  const int og = grid_onesweep<K, V>();
  const K* sk = kin;
  const V* sv = vin;
  K* dk = (npass & 1) ? kout : tk;
  V* dv = (npass & 1) ? vout : tv;
  for (int p = 0; p < npass; ++p) {
    const int sft = shift0 + 8 * p;
    const int nb = end_bit - sft < 8 ? end_bit - sft : 8;
    onesweep_kernel<K, V><<<og, kThreads, dyn, s>>>(sk, sv, dk, dv, n, sft, nb,
                                                    counts + p * kRadix, status, ctr + p,
                                                    epoch++, gate);
    sk = dk;
    sv = dv;
    dk = (dk == kout) ? tk : kout;
    dv = (dv == vout) ? tv : vout;
  }
  return GP_OK;
}

}  // namespace

size_t workspace_bytes(int64_t n, int key_bytes, int val_bytes) {
  return layout(n, key_bytes, val_bytes).total;
}

int launches(int64_t n, int begin_bit, int end_bit, bool hybrid, int key_bytes) {
  const int width = end_bit - begin_bit;
  const int nfull = (width + 7) / 8;
  const int P = top_passes(n, width);
  if (hybrid && key_bytes == 8 && 8 * P < width) return 1 + P + 1 + 1 + nfull;
  return 1 + nfull;
}

template <typename K, typename V>
int sort_pairs(const K* kin, const V* vin, K* kout, V* vout, int64_t n, int begin_bit,
               int end_bit, void* ws, size_t ws_bytes, cudaStream_t s, bool hybrid) {
  GP_REQUIRE(n >= 0 && n < (1ll << 31), "radix sort: n out of range");
  GP_REQUIRE(begin_bit >= 0 && end_bit > begin_bit && end_bit <= (int)(8 * sizeof(K)),
             "radix sort: bit range [%d, %d) out of range", begin_bit, end_bit);
  GP_REQUIRE((const void*)kin != (const void*)kout, "radix sort: keys_out must not alias keys_in");
  if (n == 0) return GP_OK;
  const Layout L = layout(n, (int)sizeof(K), (int)sizeof(V));
  GP_REQUIRE(ws && ws_bytes >= L.total, "radix sort: workspace too small (%zu < %zu)", ws_bytes,
             L.total);
  unsigned char* w = (unsigned char*)ws;
  K* tk = (K*)(w + L.tmpk);
  V* tv = (V*)(w + L.tmpv);
  unsigned long long* counts = (unsigned long long*)(w + L.counts);
  unsigned* ctr = (unsigned*)(w + L.ctr);
  int* flag = (int*)(w + L.flag);
  unsigned long long* status = (unsigned long long*)(w + L.status);
  GP_CUDA(cudaMemsetAsync(w + L.counts, 0, L.total - L.counts, s));
  const int width = end_bit - begin_bit;
  const int nfull = (width + 7) / 8;
  const int P = top_passes(n, width);
  uint32_t epoch = 1;
  if (hybrid && sizeof(K) == 8 && 8 * P < width) {
    const int top0 = end_bit - 8 * P;
    // P passes ending in the scratch buffers: lsd() ends in its "out" argument
    lsd<K, V>(kin, vin, tk, tv, kout, vout, n, top0, end_bit, P, counts, ctr, epoch, status,
              nullptr, s);
    const int64_t nb = (n + kSegTile - 1) / kSegTile;
    const K kmask = (end_bit >= (int)(8 * sizeof(K)) ? ~(K)0 : (((K)1 << end_bit) - 1)) &
                    ~(((K)1 << begin_bit) - 1);
    bucket_rank_kernel<K, V><<<(unsigned)nb, kThreads, 0, s>>>(tk, tv, kout, vout, n, top0,
                                                               kmask, flag);
    // only when a bucket overflowed: the full sort from the untouched input
    lsd<K, V>(kin, vin, kout, vout, tk, tv, n, begin_bit, end_bit, nfull,
              counts + P * kRadix, ctr + P, epoch, status, flag, s);
  } else {
    lsd<K, V>(kin, vin, kout, vout, tk, tv, n, begin_bit, end_bit, nfull, counts, ctr, epoch,
              status, nullptr, s);
  }
  return check_launch("radix sort");
}

template int sort_pairs<uint64_t, uint32_t>(const uint64_t*, const uint32_t*, uint64_t*,
                                            uint32_t*, int64_t, int, int, void*, size_t,
                                            cudaStream_t, bool);
template int sort_pairs<uint32_t, int32_t>(const uint32_t*, const int32_t*, uint32_t*, int32_t*,
                                           int64_t, int, int, void*, size_t, cudaStream_t, bool);
template int sort_pairs<uint32_t, uint32_t>(const uint32_t*, const uint32_t*, uint32_t*,
                                            uint32_t*, int64_t, int, int, void*, size_t,
                                            cudaStream_t, bool);

}  // namespace radix
}  // namespace gp
