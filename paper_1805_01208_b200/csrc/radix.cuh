// Hand-written device radix sort (K3 and the internal sorts), sm_100a.
//
// Stable LSD "onesweep" passes: one read and one write of the (key, value) pairs
// per 8-bit digit.  A persistent grid takes 4096-pair tiles in order from an
// atomic counter; each tile ranks its pairs per warp (match.any on the digit,
// warp-private digit counters), publishes its per-digit counts, and finds the
// pairs of the same digit in all earlier tiles by a decoupled look-back over
// those published counts (one 64-bit status word per (tile, digit): flag,
// pass epoch and count in one word, so no fence is needed).  The tile is then
// reordered by digit in shared memory and written out in runs of consecutive
// addresses.
//
// For the SFC sort (ranksim.py:158, n up to 2^30 pairs of a 62-bit key and a
// 32-bit gid) a hybrid needs fewer passes: LSD passes over only the TOP 8P key
// bits (P chosen so a top-bits bucket holds a handful of pairs), then one pass
// that orders every bucket by the full key.  Buckets arrive in input (gid) order,
// so a pair's place in its bucket is the number of bucket pairs with a smaller
// key, or an equal key and a smaller position: the pass counts that in shared
// memory.  A bucket larger than kSegMax (heavily duplicated or clustered keys)
// raises a device flag, and full-width LSD passes -- launched every time, but
// gated on that flag -- redo the sort from the untouched input.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace gp {
namespace radix {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kRadix = 256;
constexpr int kItems = 16;
constexpr int kTile = kThreads * kItems;  // pairs per onesweep tile
constexpr int kSegTile = 2048;            // positions per bucket-rank CTA
constexpr int kSegMax = 512;              // largest bucket the rank pass handles
constexpr int kMaxPasses = 16;

// workspace for sorting n pairs of (key_bytes, val_bytes)
size_t workspace_bytes(int64_t n, int key_bytes, int val_bytes);

// Stable sort of (kin, vin) by key bits [begin_bit, end_bit) into (kout, vout).
// vin == nullptr means value = input position.  kin/vin are left intact; kout
// must not alias kin.  hybrid: top-bits passes + bucket rank (64-bit keys only).
template <typename K, typename V>
int sort_pairs(const K* kin, const V* vin, K* kout, V* vout, int64_t n, int begin_bit,
               int end_bit, void* ws, size_t ws_bytes, cudaStream_t s, bool hybrid);

// number of kernels sort_pairs launches (for the bench's launch count)
int launches(int64_t n, int begin_bit, int end_bit, bool hybrid, int key_bytes);

}  // namespace radix
}  // namespace gp
