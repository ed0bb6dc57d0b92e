// K7 movement reduction, bit-exact with the reference.
//
// The reference sums w*x and w per (segment, block) with sequential bincount
// folds in SFC order (ranksim.py:173-197), then folds the 256 segment partials
// sequentially (np.add.reduce(axis=0), ranksim.py:218-222 / kmeans.py:374).
// A sequential fold cannot be parallelised, but the folds of different
// (segment, block) pairs are independent.  SFC order keeps a block in a few
// runs of consecutive positions, so:
//   runs     : every maximal run of positions with the same (segment, block)
//              key (stable compaction of the key-change positions);
//   group    : stable radix sort of the runs by key -> each pair's runs in
//              position order; pair boundaries -> work list;
//   fold     : one warp per pair walks its runs in order, stages each chunk's
//              values in shared memory and lets lane j fold column j in
//              position order (the exact bincount order); extents (max
//              distance to the old center, kmeans.py:474-487) and the
//              objective terms (kmeans.py:490-499) are computed in parallel
//              by all lanes of the chunk;
//   combine  : per block, fold the pair partials in segment order.
#include <cub/block/block_scan.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "radix.cuh"

namespace gp {

constexpr int FT = 128;     // threads per fold CTA (4 warps; ~34 KB of staging)

constexpr int MAXCOL = 5;   // d wx columns + w + objective (d <= 3)

// Pair keys are (local segment << bb) | block with bb = bit length of k, so that the
// run sort needs only the block bits (runs are in entry order, hence segment order
// within a block) and the invalid key 0xffffffff still sorts last.
__host__ __device__ __forceinline__ int block_bits(int k) {
  int bb = 1;
  while ((1 << bb) <= k) ++bb;
  return bb;
}

// counters[]: 0 runs, 1 work cursor, 2 valid runs, 3 pairs
struct FoldLayout {
  int64_t s0, nseg, cells, cap, pcap, ntiles;
  size_t off_flags, off_starts, off_rkey, off_skey, off_sidx, off_ridx, off_pbeg, off_slot,
      off_out, off_counters, off_cub, cub_bytes, off_tiles, off_mask, off_skey_final, total;
};

constexpr int RT = 256;             // run extraction: threads per tile
constexpr int RPER = 16;            // entries per thread (16 words of 32 per warp)
constexpr int RTILE = RT * RPER;    // positions per tile

static FoldLayout layout(int64_t n_local, int64_t pos0, int64_t n_global, int k) {
  FoldLayout L;
  auto seg = [&](int64_t pos) { return ((pos + 1) * (int64_t)GP_SEGMENTS - 1) / n_global; };
  L.s0 = n_local > 0 ? seg(pos0) : 0;
  int64_t s1 = n_local > 0 ? seg(pos0 + n_local - 1) : 0;
  L.nseg = n_local > 0 ? s1 - L.s0 + 1 : 1;
  L.cells = L.nseg << block_bits(k);   // key space (segment, block)
  L.cap = n_local > 0 ? n_local : 1;
  L.pcap = L.cells < L.cap ? L.cells : L.cap;  // pairs <= min(segments x blocks, runs)
  L.ntiles = (L.cap + RTILE - 1) / RTILE;
  size_t b1 = 0, b2 = 0, b3 = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b3, (const int32_t*)nullptr, (int32_t*)nullptr,
                                (int)L.ntiles + 1);
  cub::DeviceSelect::Flagged(nullptr, b1, cub::CountingInputIterator<int32_t>(0),
                             (const uint8_t*)nullptr, (int32_t*)nullptr, (int64_t*)nullptr,
                             (int)L.cap);
  b2 = radix::workspace_bytes(L.cap, 4, 4);   // the run sort's scratch (hand-written, radix.cu)
  L.cub_bytes = b1 > b2 ? b1 : b2;
  if (b3 > L.cub_bytes) L.cub_bytes = b3;
  auto al = [](size_t x) { return (x + 255) & ~(size_t)255; };
  size_t o = 0;
  L.off_flags = o; o = al(o + L.cap);
  L.off_starts = o; o = al(o + (L.cap + 1) * 4);
  L.off_rkey = o; o = al(o + L.cap * 4);
  L.off_skey = o; o = al(o + L.cap * 4);
  L.off_skey_final = L.off_skey;
  L.off_sidx = o; o = al(o + L.cap * 4);
  L.off_ridx = o; o = al(o + L.cap * 4);
  L.off_pbeg = o; o = al(o + (L.pcap + 1) * 4);
  L.off_slot = o; o = al(o + L.cells * 4);
  L.off_out = o; o = al(o + L.pcap * (MAXCOL + 1) * sizeof(double));
  L.off_counters = o; o = al(o + 8 * sizeof(int64_t));
  L.off_cub = o; o = al(o + L.cub_bytes);
  L.off_tiles = o; o = al(o + (L.ntiles + 1) * 4);
  L.off_mask = o; o = al(o + L.ntiles * (RTILE / 8));
  L.total = o;
  return L;
}

// key of entry i (segment of its position, block); -1: unassigned / inactive
__device__ __forceinline__ int32_t entry_key(const gp_fold_args& f, int64_t i, int c, int64_t s0,
                                             int bb) {
  if (c < 0) return -1;
  const int sg = segment_of(f.pos0 + (f.list ? f.list[i] : i), f.n_global);
  return (int32_t)(((sg - s0) << bb) | c);
}

// Pass 1 (streams a once): bit i of mask = entry i starts a run (its key differs from
// its predecessor's), tiles[t] = run starts in tile t (RTILE entries).  Warp w of a
// tile owns 512 consecutive entries as 16 words of 32: lane l takes entry 32 t + l of
// word t (coalesced 128-byte loads, all 16 issued first), so a word's run-start bits
// are one ballot in entry order.  A warp whose entries all lie in one segment (all
// but the few at the 256 segment boundaries) compares blocks directly: its keys
// differ exactly where the blocks differ.
__global__ void __launch_bounds__(RT) run_mark(gp_fold_args f, int64_t cnt, int64_t s0, int bb,
                                               uint32_t* __restrict__ mask,
                                               int32_t* __restrict__ tiles) {
  __shared__ int s_warp[RT / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int WE = RTILE / (RT / 32);        // entries per warp (512)
  constexpr int NW = WE / 32;                  // words per warp (16)
  const int64_t wbase = (int64_t)blockIdx.x * RTILE + (int64_t)warp * WE;
  // every load first (the key computations below would otherwise keep them from
  // being issued until their own loads return)
  int av[NW];
  const bool whole = wbase + WE <= cnt;
  if (whole) {
    const int* ap = f.a + wbase + lane;
#pragma unroll
    for (int t = 0; t < NW; ++t) av[t] = __ldcs(ap + 32 * t);
  } else {
#pragma unroll
    for (int t = 0; t < NW; ++t) {
      const int64_t i = wbase + 32 * t + lane;
      av[t] = i < cnt ? __ldcs(f.a + i) : -1;
    }
  }
  int total = 0;
  if (wbase < cnt) {
    // segment of the warp's first entry, and whether every entry shares it
    const int64_t last = min(cnt, wbase + (int64_t)WE) - 1;
    const int64_t p0 = f.list ? f.list[wbase] : wbase;
    const int64_t p1 = f.list ? f.list[last] : last;
    const int wseg = segment_of(f.pos0 + p0, f.n_global);
    const int64_t wnext =
        wseg + 1 < GP_SEGMENTS ? ((int64_t)(wseg + 1) * f.n_global >> 8) - f.pos0 : INT64_MAX;
    const bool uni = p1 < wnext;
    // carry: key of the entry before the current word (lane 0's predecessor); inside
    // the warp's segment it is hi | a (no segment search)
    int32_t carry = -2;
    const int32_t hi = (int32_t)((wseg - s0) << bb);
    if (lane == 0 && wbase > 0) {
      const int ap = f.a[wbase - 1];
      const int64_t pp = f.list ? f.list[wbase - 1] : wbase - 1;
      const int64_t sstart = ((int64_t)wseg * f.n_global >> 8) - f.pos0;
      carry = pp >= sstart ? (ap < 0 ? -1 : (hi | ap)) : entry_key(f, wbase - 1, ap, s0, bb);
    }
    if (uni && whole) {
      // keys = hi | a for a >= 0, -1 for a < 0: compare blocks, first word against carry;
      // lane t keeps word t, and the warp stores its 16 words at once
      unsigned mine = 0;
#pragma unroll
      for (int t = 0; t < NW; ++t) {
        const int32_t key = av[t] < 0 ? -1 : (hi | av[t]);
        int32_t prev = __shfl_up_sync(FULL, key, 1);
        if (lane == 0) prev = carry;
        carry = __shfl_sync(FULL, key, 31);
        const unsigned word = __ballot_sync(FULL, key != prev);
        if (lane == t) mine = word;
      }
      if (lane < NW) mask[(wbase >> 5) + lane] = mine;
      total = __reduce_add_sync(FULL, lane < NW ? __popc(mine) : 0u);
    } else if (uni) {
#pragma unroll
      for (int t = 0; t < NW; ++t) {
        const int32_t key = av[t] < 0 ? -1 : (hi | av[t]);
        int32_t prev = __shfl_up_sync(FULL, key, 1);
        if (lane == 0) prev = carry;
        carry = __shfl_sync(FULL, key, 31);
        const bool in = wbase + 32 * t + lane < cnt;
        const unsigned word = __ballot_sync(FULL, in && key != prev);
        total += __popc(word);
        if (lane == 0 && wbase + 32 * t < cnt) mask[(wbase >> 5) + t] = word;
      }
    } else {
      for (int t = 0; t < NW; ++t) {
        const int64_t i = wbase + 32 * t + lane;
        const int32_t key = i < cnt ? entry_key(f, i, av[t], s0, bb) : -1;
        int32_t prev = __shfl_up_sync(FULL, key, 1);
        if (lane == 0) prev = carry;
        carry = __shfl_sync(FULL, key, 31);
        const unsigned word = __ballot_sync(FULL, i < cnt && key != prev);
        total += __popc(word);
        if (lane == 0 && wbase + 32 * t < cnt) mask[(wbase >> 5) + t] = word;
      }
    }
  }
  if (lane == 0) s_warp[warp] = total;
  __syncthreads();
  if (threadIdx.x == 0) {
    int t = 0;
    for (int w = 0; w < RT / 32; ++w) t += s_warp[w];
    tiles[blockIdx.x] = t;
  }
}

// Pass 2 (reads only the mask and the run-start entries): run r in entry order ->
// starts[r], (key, r) for the sort; one thread per 32-entry mask word.
constexpr int WT2 = RTILE / 32;   // mask words per tile (128)
__global__ void __launch_bounds__(WT2) run_emit(gp_fold_args f, int64_t cnt, int64_t s0,
                                                const uint32_t* __restrict__ mask,
                                                const int32_t* __restrict__ tile_off,
                                                int64_t ntiles, int32_t* __restrict__ starts,
                                                uint32_t* __restrict__ rkey,
                                                int32_t* __restrict__ ridx, int64_t* counters) {
  typedef cub::BlockScan<int, WT2> Scan;
  __shared__ typename Scan::TempStorage tmp;
  const int bb = block_bits(f.k);
  const int64_t wi = (int64_t)blockIdx.x * WT2 + threadIdx.x;   // mask word
  const int64_t e0 = wi * 32;
  unsigned w = e0 < cnt ? mask[wi] : 0u;
  int excl;
  Scan(tmp).ExclusiveSum(__popc(w), excl);
  int r = tile_off[blockIdx.x] + excl;
  int valid = 0;
  while (w) {
    const int t = __ffs(w) - 1;
    w &= w - 1;
    const int64_t i = e0 + t;
    const int32_t key = entry_key(f, i, f.a[i], s0, bb);
    starts[r] = (int32_t)i;
    rkey[r] = (uint32_t)key;
    ridx[r] = r;
    valid += key >= 0;
    ++r;
  }
  for (int o = 16; o; o >>= 1) valid += __shfl_xor_sync(FULL, valid, o);
  if ((threadIdx.x & 31) == 0 && valid)
    atomicAdd((unsigned long long*)&counters[2], (unsigned long long)valid);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int R = tile_off[ntiles];
    starts[R] = (int32_t)cnt;  // sentinel end
    counters[0] = R;
  }
}

// first sorted run of every pair (valid runs occupy the first counters[2] slots)
__global__ void fold_pair_flags(const uint32_t* __restrict__ skey, int64_t R,
                                const int64_t* counters, uint8_t* __restrict__ flags) {
  const int64_t V = counters[2];
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < R;
       j += (int64_t)gridDim.x * blockDim.x)
    flags[j] = j < V && (j == 0 || skey[j] != skey[j - 1]);
}

__global__ void fold_slots(const uint32_t* __restrict__ skey, int32_t* __restrict__ pbeg,
                           const int64_t* counters, int32_t* __restrict__ slot) {
  const int64_t P = counters[3];
  if (blockIdx.x == 0 && threadIdx.x == 0) pbeg[P] = (int32_t)counters[2];  // sentinel end
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x)
    slot[skey[pbeg[p]]] = (int32_t)p;
}

// Pair folds, G pairs per warp (G * NC <= 32), B batches of 32 entries per step.
// Lane g < G owns group g's cursor (pair, sorted run j, entry cur, run end re);
// each step the whole warp loads up to 32 B consecutive entries of every group's
// current run (all loads issued together), computes w*x, w, w*|x-c|^2 (and the
// max |x-c|^2 for the extent) and stages them in shared memory; then lane
// (g, col) folds column col of group g in entry order, which is the bincount
// order of the reference.  A group whose pair ends writes the pair's partials and
// takes the next pair from the work counter.  Many pairs: G = 32 / NC, B = 1 (lane
// utilisation); few pairs: G = 1, B = 8 (fewer, longer steps on the critical path).
template <int D, int NC, int G, int B>
__global__ void __launch_bounds__(FT) fold_groups(gp_fold_args f, const int32_t* __restrict__ starts,
                                                  const int32_t* __restrict__ sidx,
                                                  const uint32_t* __restrict__ skey,
                                                  const int32_t* __restrict__ pbeg,
                                                  int64_t* counters, double* __restrict__ out) {
  static_assert(G * NC <= 32 && G * B <= 32, "fold_groups shape");
  constexpr int W = FT / 32;
  constexpr int T = 32 * B;        // entries per group step
  __shared__ double st[W][G * NC][T + 1];
  __shared__ double scen[W][G][D];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t P = counters[3];
  // (ns, ne): bounds of run j + 1 and rn2 = sidx[j + 2], prefetched one run ahead so
  // that a run change needs no dependent loads on the step's critical path
  int pair = -1, j = 0, j1 = 0, cur = 0, re = 0, ns = 0, ne = 0, rn2 = 0;
  auto fetch = [&]() {
    const int64_t pi = (int64_t)atomicAdd((unsigned long long*)&counters[1], 1ull);
    if (pi >= P) {
      pair = -1;
      return;
    }
    pair = (int)pi;
    j = pbeg[pi];
    j1 = pbeg[pi + 1];
    const int r = sidx[j];
    cur = starts[r];
    re = starts[r + 1];
    if (j + 1 < j1) {
      const int r1 = sidx[j + 1];
      ns = starts[r1];
      ne = starts[r1 + 1];
    }
    if (j + 2 < j1) rn2 = sidx[j + 2];
    if (NC > 1) {
      const int c = (int)(skey[j] & ((1u << block_bits(f.k)) - 1));
#pragma unroll
      for (int q = 0; q < D; ++q) scen[warp][lane][q] = f.centers[c * D + q];
    }
  };
  if (lane < G) fetch();
  __syncwarp();
  const int mg = lane / NC, col = lane - mg * NC;
  double acc = 0.0;  // bincount starts from 0.0
  double extg[G];
#pragma unroll
  for (int g = 0; g < G; ++g) extg[g] = 0.0;
  for (;;) {
    const bool live = lane < G && pair >= 0;
    const int cnt = live ? min(T, re - cur) : 0;
    if (!__any_sync(FULL, live)) break;
    // all groups' loads first (clamped to a valid entry), so they are in flight together
    int ngs[G];
    double xr[G][B][D], wr[G][B];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int cg = __shfl_sync(FULL, cur, g);
      ngs[g] = __shfl_sync(FULL, cnt, g);
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int t = b * 32 + lane;
        const int i = ngs[g] > 0 ? cg + min(t, ngs[g] - 1) : 0;
        wr[g][b] = load_weight(f.w, f.wmode, i);
        if (NC > 1) load_point<D>(f.X, f.ldx, i, xr[g][b]);
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int t = b * 32 + lane;
        if (t < ngs[g]) {
          const double w = wr[g][b];
          if (NC == 1) {
            st[warp][g][t] = w;
          } else {
            double diff[D];
#pragma unroll
            for (int q = 0; q < D; ++q) {
              st[warp][g * NC + q][t] = __dmul_rn(xr[g][b][q], w);  // wx = points * weights[:, None]
              diff[q] = __dsub_rn(xr[g][b][q], scen[warp][g][q]);
            }
            const double sq = sqnorm_rn(diff, D, f.order3);
            st[warp][g * NC + D][t] = w;
            st[warp][g * NC + D + 1][t] = __dmul_rn(sq, w);
            extg[g] = fmax(extg[g], sq);  // sqrt is monotone: max of sqrt = sqrt of max
          }
        }
      }
    }
    __syncwarp();
    const int nmine = __shfl_sync(FULL, cnt, mg < G ? mg : 0);
    if (mg < G) {
      const double* colp = st[warp][mg * NC + col];
      if (nmine == T) {
#pragma unroll 32
        for (int t = 0; t < T; ++t) acc = __dadd_rn(acc, colp[t]);
      } else {
        for (int t = 0; t < nmine; ++t) acc = __dadd_rn(acc, colp[t]);
      }
    }
    __syncwarp();
    bool done = false;
    if (live) {
      cur += cnt;
      if (cur >= re) {
        ++j;
        if (j < j1) {
          cur = ns;
          re = ne;
          if (j + 1 < j1) {
            ns = starts[rn2];
            ne = starts[rn2 + 1];
            if (j + 2 < j1) rn2 = sidx[j + 2];
          }
        } else {
          done = true;
        }
      }
    }
    const unsigned dm = __ballot_sync(FULL, done);
    if (dm) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (!(dm & (1u << g))) continue;
        const int pg = __shfl_sync(FULL, pair, g);
        double* po = out + (int64_t)pg * (MAXCOL + 1);
        if (mg == g) {
          po[col] = acc;
          acc = 0.0;
        }
        if (NC > 1) {
          double e = extg[g];
          for (int o = 16; o; o >>= 1) e = fmax(e, __shfl_xor_sync(FULL, e, o));
          if (lane == 0) po[MAXCOL] = __dsqrt_rn(e);
          extg[g] = 0.0;
        }
      }
      if (done) fetch();
      __syncwarp();
    }
  }
}

// fold_groups with the next step's loads issued before the current step is staged
// and folded (register double buffer), so a group's chain of steps no longer waits
// for a full load latency per step.  A group whose current batch ends its pair
// issues no load for the next step (the next pair is fetched after the fold writes
// the partials), so it idles one step per pair.  UNIT: unit weights (no weight
// loads or registers).
template <int D, int NC, int G, int B, bool UNIT>
__global__ void __launch_bounds__(FT) fold_pipe(gp_fold_args f, const int32_t* __restrict__ starts,
                                                const int32_t* __restrict__ sidx,
                                                const uint32_t* __restrict__ skey,
                                                const int32_t* __restrict__ pbeg,
                                                int64_t* counters, double* __restrict__ out) {
  static_assert(G * NC <= 32 && G * B <= 32, "fold_pipe shape");
  constexpr int W = FT / 32;
  constexpr int T = 32 * B;
  __shared__ double st[W][G * NC][T + 1];
  __shared__ double scen[W][G][D];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t P = counters[3];
  int pair = -1, j = 0, j1 = 0, cur = 0, re = 0, ns = 0, ne = 0, rn2 = 0;
  auto fetch = [&]() {
    const int64_t pi = (int64_t)atomicAdd((unsigned long long*)&counters[1], 1ull);
    if (pi >= P) {
      pair = -1;
      return;
    }
    pair = (int)pi;
    j = pbeg[pi];
    j1 = pbeg[pi + 1];
    const int r = sidx[j];
    cur = starts[r];
    re = starts[r + 1];
    if (j + 1 < j1) {
      const int r1 = sidx[j + 1];
      ns = starts[r1];
      ne = starts[r1 + 1];
    }
    if (j + 2 < j1) rn2 = sidx[j + 2];
    if (NC > 1) {
      const int c = (int)(skey[j] & ((1u << block_bits(f.k)) - 1));
#pragma unroll
      for (int q = 0; q < D; ++q) scen[warp][lane][q] = f.centers[c * D + q];
    }
  };
  // next batch of group lane g: its first entry and count, then the cursor moves on;
  // last = the batch ends the pair
  auto next_batch = [&](int& c0, int& cnt, bool& last) {
    c0 = cur;
    cnt = 0;
    last = false;
    if (lane >= G || pair < 0) return;
    cnt = min(T, re - cur);
    cur += cnt;
    if (cur >= re) {
      ++j;
      if (j < j1) {
        cur = ns;
        re = ne;
        if (j + 1 < j1) {
          ns = starts[rn2];
          ne = starts[rn2 + 1];
          if (j + 2 < j1) rn2 = sidx[j + 2];
        }
      } else {
        last = true;
      }
    }
  };
  auto load = [&](int c0, int cnt, double (&xr)[G][B][D], double (&wr)[G][B], int (&ngs)[G]) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      const int cg = __shfl_sync(FULL, c0, g);
      ngs[g] = __shfl_sync(FULL, cnt, g);
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int t = b * 32 + lane;
        const int i = ngs[g] > 0 ? cg + min(t, ngs[g] - 1) : 0;
        wr[g][b] = UNIT ? 1.0 : load_weight(f.w, f.wmode, i);
        if (NC > 1) load_point<D>(f.X, f.ldx, i, xr[g][b]);
      }
    }
  };
  if (lane < G) fetch();
  __syncwarp();
  const int mg = lane / NC, col = lane - mg * NC;
  double acc = 0.0;  // bincount starts from 0.0
  double extg[G];
#pragma unroll
  for (int g = 0; g < G; ++g) extg[g] = 0.0;
  double xa[G][B][D], wa[G][B], xb[G][B][D], wb[G][B];
  int na[G], nb[G];
  int c0, cnt_c;
  bool last_c;
  next_batch(c0, cnt_c, last_c);
  load(c0, cnt_c, xa, wa, na);
  for (;;) {
    if (!__any_sync(FULL, lane < G && (pair >= 0 || cnt_c > 0))) break;
    // the next step's loads first
    int c1 = 0, cnt_n = 0;
    bool last_n = false;
    if (!last_c) next_batch(c1, cnt_n, last_n);
    load(c1, cnt_n, xb, wb, nb);
    // stage and fold the current step
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int b = 0; b < B; ++b) {
        const int t = b * 32 + lane;
        if (t < na[g]) {
          const double w = wa[g][b];
          if (NC == 1) {
            st[warp][g][t] = w;
          } else {
            double diff[D];
#pragma unroll
            for (int q = 0; q < D; ++q) {
              st[warp][g * NC + q][t] = __dmul_rn(xa[g][b][q], w);  // wx = points * weights[:, None]
              diff[q] = __dsub_rn(xa[g][b][q], scen[warp][g][q]);
            }
            const double sq = sqnorm_rn(diff, D, f.order3);
            st[warp][g * NC + D][t] = w;
            st[warp][g * NC + D + 1][t] = __dmul_rn(sq, w);
            extg[g] = fmax(extg[g], sq);  // sqrt is monotone: max of sqrt = sqrt of max
          }
        }
      }
    }
    __syncwarp();
    const int nmine = __shfl_sync(FULL, cnt_c, mg < G ? mg : 0);
    if (mg < G) {
      const double* colp = st[warp][mg * NC + col];
      if (nmine == T) {
#pragma unroll 32
        for (int t = 0; t < T; ++t) acc = __dadd_rn(acc, colp[t]);
      } else {
        for (int t = 0; t < nmine; ++t) acc = __dadd_rn(acc, colp[t]);
      }
    }
    __syncwarp();
    const unsigned dm = __ballot_sync(FULL, lane < G && last_c);
    if (dm) {
#pragma unroll
      for (int g = 0; g < G; ++g) {
        if (!(dm & (1u << g))) continue;
        const int pg = __shfl_sync(FULL, pair, g);
        double* po = out + (int64_t)pg * (MAXCOL + 1);
        if (mg == g) {
          po[col] = acc;
          acc = 0.0;
        }
        if (NC > 1) {
          double e = extg[g];
          for (int o = 16; o; o >>= 1) e = fmax(e, __shfl_xor_sync(FULL, e, o));
          if (lane == 0) po[MAXCOL] = __dsqrt_rn(e);
          extg[g] = 0.0;
        }
      }
      if (lane < G && last_c) fetch();
      __syncwarp();
    }
    // the prefetched step becomes the current one
#pragma unroll
    for (int g = 0; g < G; ++g) {
      na[g] = nb[g];
#pragma unroll
      for (int b = 0; b < B; ++b) {
        wa[g][b] = wb[g][b];
#pragma unroll
        for (int q = 0; q < D; ++q) xa[g][b][q] = xb[g][b][q];
      }
    }
    cnt_c = cnt_n;
    last_c = last_n;
  }
}

// GP_FOLD_PIPE=1: the prefetching fold for every many-pair shape (tuning switch)
static bool pipe_all() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("GP_FOLD_PIPE");
    v = e && atoi(e) == 1;
  }
  return v == 1;
}

template <int D, int NC, int G, int B, bool UNIT>
static void launch_fold_pipe(const gp_fold_args* f, int sms, const int32_t* starts,
                             const int32_t* sidx, const uint32_t* skey, const int32_t* pbeg,
                             int64_t* counters, double* out, cudaStream_t s) {
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fold_pipe<D, NC, G, B, UNIT>, FT, 0);
  fold_pipe<D, NC, G, B, UNIT><<<sms * (per_sm > 0 ? per_sm : 1), FT, 0, s>>>(
      *f, starts, sidx, skey, pbeg, counters, out);
}

template <int D, int NC, int G, int B>
static void launch_fold_groups(const gp_fold_args* f, int sms, const int32_t* starts,
                               const int32_t* sidx, const uint32_t* skey, const int32_t* pbeg,
                               int64_t* counters, double* out, cudaStream_t s) {
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fold_groups<D, NC, G, B>, FT, 0);
  fold_groups<D, NC, G, B><<<sms * (per_sm > 0 ? per_sm : 1), FT, 0, s>>>(
      *f, starts, sidx, skey, pbeg, counters, out);
}

// One warp per block: gather the block's pair partials over the segments
// (independent loads), then fold them in segment order (np.add.reduce(axis=0)).
template <int D>
// slot[] index of (segment s, block c): (s << bb) | c for the local pair keys (bb > 0),
// s * k + c for the gathered global keys of gp_fold_combine (bb = 0)
__global__ void fold_combine(gp_fold_args f, const int32_t* __restrict__ slot, int64_t nseg,
                             const double* __restrict__ out, int bb) {
  __shared__ int32_t s_slot[4][GP_SEGMENTS];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int c = blockIdx.x * 4 + warp;
  if (c >= f.k) return;
  int base = 0;
  for (int64_t s0 = 0; s0 < nseg; s0 += 32) {
    int64_t s = s0 + lane;
    int32_t p = s < nseg ? slot[bb ? ((s << bb) | c) : s * f.k + c] : -1;
    unsigned m = __ballot_sync(FULL, p >= 0);
    if (p >= 0) s_slot[warp][base + __popc(m & ((1u << lane) - 1))] = p;
    base += __popc(m);
  }
  __syncwarp();
  const int np = base;
  const int ncols = f.weights_only ? 1 : D + 2;
  if (lane < ncols) {
    double acc = 0.0;
    for (int i = 0; i < np; ++i)
      acc = __dadd_rn(acc, out[(int64_t)s_slot[warp][i] * (MAXCOL + 1) + lane]);
    if (f.weights_only) f.wsum[c] = acc;
    else if (lane < D) f.sums[c * D + lane] = acc;
    else if (lane == D) f.wsum[c] = acc;
    else f.objective[c] = acc;
  }
  if (!f.weights_only) {
    double ext = 0.0;
    for (int i = lane; i < np; i += 32)
      ext = fmax(ext, out[(int64_t)s_slot[warp][i] * (MAXCOL + 1) + MAXCOL]);
    for (int o = 16; o; o >>= 1) ext = fmax(ext, __shfl_xor_sync(FULL, ext, o));
    if (lane == 0) f.extent[c] = ext;
  }
}

__global__ void fold_export_kernel(const uint32_t* __restrict__ skey,
                                   const int32_t* __restrict__ pbeg,
                                   const int64_t* __restrict__ counters,
                                   const double* __restrict__ out, int64_t s0, int k,
                                   int64_t* __restrict__ keys, double* __restrict__ vals,
                                   int64_t* npairs) {
  const int64_t P = counters[3];
  if (blockIdx.x == 0 && threadIdx.x == 0) *npairs = P;
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P;
       p += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t key = skey[pbeg[p]];
    const int bb = block_bits(k);
    const int64_t seg = (key >> bb) + s0, c = key & ((1u << bb) - 1);
    keys[p] = seg * k + c;
#pragma unroll
    for (int j = 0; j < MAXCOL + 1; ++j) vals[p * (MAXCOL + 1) + j] = out[p * (MAXCOL + 1) + j];
  }
}

__global__ void combine_slots(const int64_t* __restrict__ keys, int64_t npairs,
                              int32_t* __restrict__ slot) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < npairs;
       p += (int64_t)gridDim.x * blockDim.x)
    slot[keys[p]] = (int32_t)p;
}

}  // namespace gp

using namespace gp;

static int64_t* g_last_counters = nullptr;

extern "C" {

int gp_fold_stats(int64_t* out) {
  // debugging aid: {runs, cursor, valid runs, pairs} of the last gp_movement_fold (syncs)
  if (!g_last_counters) return GP_ERR_INVALID;
  GP_CUDA(cudaDeviceSynchronize());
  GP_CUDA(cudaMemcpy(out, g_last_counters, 4 * sizeof(int64_t), cudaMemcpyDeviceToHost));
  return GP_OK;
}

int gp_fold_export(const gp_fold_args* f, int64_t* keys, double* vals, int64_t* npairs,
                   void* stream) {
  GP_REQUIRE(f && keys && vals && npairs, "gp_fold_export: bad args");
  FoldLayout L = layout(f->n_local, f->pos0, f->n_global, f->k);
  char* ws = (char*)f->workspace;
  fold_export_kernel<<<grid_for(L.pcap, 256, 148 * 8), 256, 0, (cudaStream_t)stream>>>(
      (const uint32_t*)(ws + L.off_skey_final), (const int32_t*)(ws + L.off_pbeg),
      (const int64_t*)(ws + L.off_counters), (const double*)(ws + L.off_out), L.s0, f->k, keys,
      vals, npairs);
  return check_launch("fold_export");
}

int gp_fold_combine_bytes(int k, size_t* bytes) {
  GP_REQUIRE(k >= 1, "gp_fold_combine_bytes: bad k");
  *bytes = (size_t)GP_SEGMENTS * k * sizeof(int32_t);
  return GP_OK;
}

int gp_fold_combine(const int64_t* keys, const double* vals, int64_t npairs, int k, int d,
                    int weights_only, double* sums, double* wsum, double* extent,
                    double* objective, void* workspace, size_t workspace_bytes, void* stream) {
  GP_REQUIRE(d == 2 || d == 3, "gp_fold_combine: bad d");
  GP_REQUIRE(workspace_bytes >= (size_t)GP_SEGMENTS * k * sizeof(int32_t),
             "gp_fold_combine: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  int32_t* slot = (int32_t*)workspace;
  GP_CUDA(cudaMemsetAsync(slot, 0xff, (size_t)GP_SEGMENTS * k * sizeof(int32_t), s));
  if (npairs > 0)
    combine_slots<<<grid_for(npairs, 256, 148 * 8), 256, 0, s>>>(keys, npairs, slot);
  gp_fold_args f{};
  f.d = d;
  f.k = k;
  f.weights_only = weights_only;
  f.sums = sums;
  f.wsum = wsum;
  f.extent = extent;
  f.objective = objective;
  if (d == 2) fold_combine<2><<<grid_for(k, 4), 128, 0, s>>>(f, slot, GP_SEGMENTS, vals, 0);
  else fold_combine<3><<<grid_for(k, 4), 128, 0, s>>>(f, slot, GP_SEGMENTS, vals, 0);
  return check_launch("fold_combine");
}

int gp_fold_workspace_bytes(int64_t n_local, int64_t pos0, int64_t n_global, int k,
                            size_t* bytes) {
  GP_REQUIRE(n_global >= 1 && k >= 1, "gp_fold_workspace_bytes: bad sizes");
  *bytes = layout(n_local, pos0, n_global, k).total;
  return GP_OK;
}

int gp_movement_fold(const gp_fold_args* f, void* stream) {
  GP_REQUIRE(f && (f->d == 2 || f->d == 3) && f->k >= 1, "gp_movement_fold: bad args");
  GP_REQUIRE(f->n_local >= 0 && f->n_local < (1ll << 31), "gp_movement_fold: n out of range");
  GP_REQUIRE(!f->list || (f->m >= 0 && f->m <= f->n_local), "gp_movement_fold: m out of range");
  GP_REQUIRE(f->wmode == GP_W_UNIT || f->w != nullptr, "gp_movement_fold: weights missing");
  GP_REQUIRE(f->wsum != nullptr, "gp_movement_fold: wsum missing");
  GP_REQUIRE(f->weights_only || (f->sums && f->extent && f->objective && f->centers),
             "gp_movement_fold: outputs missing");
  FoldLayout L = layout(f->n_local, f->pos0, f->n_global, f->k);
  GP_REQUIRE(f->workspace_bytes >= L.total, "gp_movement_fold: workspace too small (%zu < %zu)",
             f->workspace_bytes, L.total);
  GP_REQUIRE(L.cells < (1ll << 31), "gp_movement_fold: segment x block table too large");
  cudaStream_t s = (cudaStream_t)stream;
  char* ws = (char*)f->workspace;
  uint8_t* flags = (uint8_t*)(ws + L.off_flags);
  int32_t* starts = (int32_t*)(ws + L.off_starts);
  uint32_t* rkey = (uint32_t*)(ws + L.off_rkey);
  uint32_t* skey = (uint32_t*)(ws + L.off_skey);
  int32_t* sidx = (int32_t*)(ws + L.off_sidx);
  int32_t* ridx = (int32_t*)(ws + L.off_ridx);
  int32_t* pbeg = (int32_t*)(ws + L.off_pbeg);
  int32_t* slot = (int32_t*)(ws + L.off_slot);
  double* out = (double*)(ws + L.off_out);
  int64_t* counters = (int64_t*)(ws + L.off_counters);
  g_last_counters = counters;
  void* cub_tmp = ws + L.off_cub;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t cnt = f->list ? f->m : f->n_local;   // entries

  GP_CUDA(cudaMemsetAsync(counters, 0, 8 * sizeof(int64_t), s));
  GP_CUDA(cudaMemsetAsync(slot, 0xff, L.cells * sizeof(int32_t), s));
  if (cnt > 0) {
    const int64_t nt = (cnt + RTILE - 1) / RTILE;
    int32_t* tiles = (int32_t*)(ws + L.off_tiles);
    uint32_t* mask = (uint32_t*)(ws + L.off_mask);
    run_mark<<<(unsigned)nt, RT, 0, s>>>(*f, cnt, L.s0, block_bits(f->k), mask, tiles);
    GP_CUDA(cudaMemsetAsync(tiles + nt, 0, sizeof(int32_t), s));
    size_t sb = L.cub_bytes;
    GP_CUDA(cub::DeviceScan::ExclusiveSum(cub_tmp, sb, tiles, tiles, (int)nt + 1, s));
    run_emit<<<(unsigned)nt, WT2, 0, s>>>(*f, cnt, L.s0, mask, tiles, nt, starts, rkey, ridx,
                                         counters);
    int64_t R = 0;
    GP_CUDA(cudaMemcpyAsync(&R, counters, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    GP_CUDA(cudaStreamSynchronize(s));
    // stable sort by the block bits only: valid blocks are < k < 2^bb - 1 and the
    // invalid key is all-ones there, so the invalid runs stay last (hand-written onesweep
    // LSD passes, radix.cu; the sorted keys land where gp_fold_export expects them)
    size_t b = L.cub_bytes;
    if (R > 0) {
      const int rc = radix::sort_pairs<uint32_t, int32_t>(rkey, ridx, skey, sidx, R, 0,
                                                          block_bits(f->k), cub_tmp, b, s, false);
      if (rc) return rc;
    }
    fold_pair_flags<<<grid_for(R, 256, sms * 16), 256, 0, s>>>(skey, R, counters, flags);
    b = L.cub_bytes;
    GP_CUDA(cub::DeviceSelect::Flagged(cub_tmp, b, cub::CountingInputIterator<int32_t>(0), flags,
                                       pbeg, counters + 3, (int)R, s));
    fold_slots<<<grid_for(R, 256, sms * 8), 256, 0, s>>>(skey, pbeg, counters, slot);
  }
  // pairs per warp G and batches per step B (G * B = 8 register sets): enough groups
  // to fill every resident warp, and otherwise longer steps for the critical path
  int64_t P_host = 0;
  if (cnt > 0) {
    GP_CUDA(cudaMemcpyAsync(&P_host, counters + 3, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    GP_CUDA(cudaStreamSynchronize(s));
  }
  const int64_t warps = (int64_t)sms * 16;   // ~resident fold warps
  const int64_t per = P_host / warps;        // pairs per warp if every warp is busy
#define GP_FOLD(Dd, NCc, Gg, Bb) \
  launch_fold_groups<Dd, NCc, Gg, Bb>(f, sms, starts, sidx, skey, pbeg, counters, out, s)
  if (f->weights_only) {
    if (f->d == 2) {
      if (per >= 32) GP_FOLD(2, 1, 32, 1);
      else if (per >= 4) GP_FOLD(2, 1, 4, 8);
      else GP_FOLD(2, 1, 1, 8);
    } else {
      if (per >= 32) GP_FOLD(3, 1, 32, 1);
      else if (per >= 4) GP_FOLD(3, 1, 4, 8);
      else GP_FOLD(3, 1, 1, 8);
    }
  } else if (f->d == 2) {
    static int shape = -1;   // GP_FOLD_SHAPE=G (1, 2, 4, 8) overrides the choice (tuning)
    if (shape < 0) {
      const char* e = getenv("GP_FOLD_SHAPE");
      shape = e ? atoi(e) : 0;
    }
    if (shape == 9) {   // GP_FOLD_SHAPE=9: the prefetching 8 x 1 fold for any weights
      if (f->wmode == GP_W_UNIT)
        launch_fold_pipe<2, 4, 8, 1, true>(f, sms, starts, sidx, skey, pbeg, counters, out, s);
      else
        launch_fold_pipe<2, 4, 8, 1, false>(f, sms, starts, sidx, skey, pbeg, counters, out, s);
    } else if (shape == 8) GP_FOLD(2, 4, 8, 1);
    else if (shape == 0 && per >= 8 && (f->wmode == GP_W_UNIT || pipe_all()))
      // measured 18% faster at C5
      if (f->wmode == GP_W_UNIT)
        launch_fold_pipe<2, 4, 8, 1, true>(f, sms, starts, sidx, skey, pbeg, counters, out, s);
      else
        launch_fold_pipe<2, 4, 8, 1, false>(f, sms, starts, sidx, skey, pbeg, counters, out, s);
    else if (shape == 4) GP_FOLD(2, 4, 4, 2);
    else if (shape == 2) GP_FOLD(2, 4, 2, 4);
    else if (shape == 1) GP_FOLD(2, 4, 1, 8);
    else if (per >= 8) GP_FOLD(2, 4, 8, 1);
    else if (per >= 4) GP_FOLD(2, 4, 4, 2);
    else if (per >= 2) GP_FOLD(2, 4, 2, 4);
    else GP_FOLD(2, 4, 1, 8);
  } else {
    if (per >= 6 && pipe_all()) {
      if (f->wmode == GP_W_UNIT)
        launch_fold_pipe<3, 5, 6, 1, true>(f, sms, starts, sidx, skey, pbeg, counters, out, s);
      else
        launch_fold_pipe<3, 5, 6, 1, false>(f, sms, starts, sidx, skey, pbeg, counters, out, s);
    } else if (per >= 6) GP_FOLD(3, 5, 6, 1);
    else if (per >= 4) GP_FOLD(3, 5, 4, 2);
    else if (per >= 2) GP_FOLD(3, 5, 2, 4);
    else GP_FOLD(3, 5, 1, 8);
  }
#undef GP_FOLD
  const int bbk = block_bits(f->k);
  if (f->d == 2) fold_combine<2><<<grid_for(f->k, 4), 128, 0, s>>>(*f, slot, L.nseg, out, bbk);
  else fold_combine<3><<<grid_for(f->k, 4), 128, 0, s>>>(*f, slot, L.nseg, out, bbk);
  return check_launch("movement_fold");
}

}  // extern "C"
