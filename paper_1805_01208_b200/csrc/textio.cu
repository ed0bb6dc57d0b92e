// Text formats either side of the partition path, parsed and
// written on the device: the METIS adjacency file, the coordinate file and the
// partition file of the reference's fileio.py:70-278.
//
// The file bytes are uploaded once.  Two streaming passes over the text build a line
// and token index and convert every token in place:
//
//   text_count   one CTA per 8 KiB tile: line starts, token starts (split at the
//                tile's first line break so that a '#' comment entering from the
//                previous tile can void the leading tokens), comment carry-out
//   text_tiles   one CTA: prefix sums of the tile counts and the comment carry
//   text_emit    the same tiles again, now with global line / token numbers: writes
//                the byte offset and first token of every line, and parses every token
//                where it starts (decimal integers exactly; decimal reals with the
//                Eisel-Lemire algorithm, correctly rounded or flagged)
//
// Every token gets a value (int64 or the bits of a double) and a kind.  Tokens outside
// the plain decimal grammar (nan, inf, 1_000, more than 19 significant digits, the rare
// inconclusive Eisel-Lemire product) are kind SUSPECT: the host arbitrates those lines
// with Python's own int()/float() (fileio.py), so results equal the reference's for
// every input the reference accepts.
//
// The assembly kernels below turn the token stream of a METIS file into CSR arrays
// (fileio.py:126-170) and flag every vertex line the reference would reject; a table
// file (np.loadtxt in fileio.py:219-268) is the token values in order once every
// non-blank line is known to have the same number of columns.
#include <cub/device/device_reduce.cuh>
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace gp {
namespace {

struct Pow5 { unsigned long long hi, lo; };
__device__ const Pow5 g_pow5[] = {
#include "pow5_table.inc"
};
const Pow5 h_pow5[] = {
#include "pow5_table.inc"
};

constexpr int TILE = 8192;       // bytes per CTA tile
constexpr int TPB = 256;         // threads per CTA
constexpr int PER = TILE / TPB;  // 32 bytes per thread
constexpr int MAX_TOKEN = 96;    // longer tokens are SUSPECT

__host__ __device__ __forceinline__ bool is_break(unsigned c, unsigned next) {
  // '\n', or a '\r' that is not the first half of "\r\n" (universal newlines)
  return c == '\n' || (c == '\r' && next != '\n');
}
// blank: every byte <= ' ' (the host rejects a file holding control bytes other than
// \t \n \r before any token is used, so those never separate tokens in practice)
__host__ __device__ __forceinline__ bool is_space(unsigned c) { return c <= ' '; }

// ---------------------------------------------------------------- number parsing
__host__ __device__ inline unsigned long long mulhi64(unsigned long long a, unsigned long long b,
                                                      unsigned long long* lo) {
#ifdef __CUDA_ARCH__
  *lo = a * b;
  return __umul64hi(a, b);
#else
  unsigned __int128 p = (unsigned __int128)a * b;
  *lo = (unsigned long long)p;
  return (unsigned long long)(p >> 64);
#endif
}
__host__ __device__ inline int clz64(unsigned long long x) {
#ifdef __CUDA_ARCH__
  return __clzll((long long)x);
#else
  return __builtin_clzll(x);
#endif
}

// Eisel-Lemire: w * 10^q (w != 0, at most 19 digits) to the nearest binary64, ties to
// even.  Returns false when the 128-bit product cannot decide the rounding.
__host__ __device__ inline bool decimal_to_double(unsigned long long w, long long q, bool neg,
                                                  unsigned long long* bits) {
  const unsigned long long sign = neg ? 0x8000000000000000ull : 0ull;
  if (w == 0 || q < -342) { *bits = sign; return true; }
  if (q > 308) { *bits = sign | 0x7ff0000000000000ull; return true; }
  int lz = clz64(w);
  w <<= lz;
#ifdef __CUDA_ARCH__
  const Pow5 p5 = g_pow5[q + 342];
#else
  const Pow5 p5 = h_pow5[q + 342];
#endif
  unsigned long long lower, upper = mulhi64(w, p5.hi, &lower);
  if ((upper & 0x1ffull) == 0x1ffull) {
    unsigned long long slo, shi = mulhi64(w, p5.lo, &slo);
    (void)slo;
    lower += shi;
    if (shi > lower) ++upper;
  }
  if (lower == 0xffffffffffffffffull && (q < -27 || q > 55)) return false;
  const int upperbit = (int)(upper >> 63);
  unsigned long long mant = upper >> (upperbit + 9);
  long long power2 = (((152170ll + 65536ll) * q) >> 16) + 63 + upperbit - lz + 1023;
  if (power2 <= 0) {  // subnormal or zero
    if (-power2 + 1 >= 64) { *bits = sign; return true; }
    mant >>= (-power2 + 1);
    mant += (mant & 1);
    mant >>= 1;
    const unsigned long long e = mant < (1ull << 52) ? 0ull : 1ull;
    *bits = sign | (e << 52) | (mant & ((1ull << 52) - 1));
    return true;
  }
  if (lower <= 1 && q >= -4 && q <= 23 && (mant & 3) == 1 &&
      (mant << (upperbit + 9)) == upper)
    mant &= ~1ull;  // exactly halfway: round to even
  mant += (mant & 1);
  mant >>= 1;
  if (mant >= (2ull << 52)) { mant = 1ull << 52; ++power2; }
  mant &= ~(1ull << 52);
  if (power2 >= 0x7ff) { *bits = sign | 0x7ff0000000000000ull; return true; }
  *bits = sign | ((unsigned long long)power2 << 52) | mant;
  return true;
}

// One token: text[0, len).  kind GP_TOK_INT: *val = the integer; GP_TOK_REAL: *val =
// the bits of the correctly rounded double; GP_TOK_PERCENT: starts with '%';
// GP_TOK_SUSPECT: not plain decimal (the host decides).
__host__ __device__ inline int parse_number(const unsigned char* t, int len, long long* val) {
  *val = 0;
  if (len <= 0 || len > MAX_TOKEN) return GP_TOK_SUSPECT;
  if (t[0] == '%') return GP_TOK_PERCENT;
  int i = 0;
  bool neg = false;
  if (t[0] == '+' || t[0] == '-') { neg = t[0] == '-'; i = 1; }
  unsigned long long w = 0;
  int sig = 0;        // significant digits accumulated into w
  int digits = 0;     // digits seen (integer + fraction)
  long long q = 0;    // decimal exponent of w
  bool dropped = false;
  const int i0 = i;
  while (i < len && t[i] >= '0' && t[i] <= '9') {
    const unsigned d = t[i] - '0';
    if (sig > 0 || d) {
      if (sig < 19) { w = w * 10 + d; ++sig; } else { ++q; dropped |= d != 0; }
    }
    ++digits; ++i;
  }
  const int int_digits = i - i0;
  if (i == len) {  // integer grammar
    if (int_digits == 0) return GP_TOK_SUSPECT;
    if (sig <= 18) { *val = neg ? -(long long)w : (long long)w; return GP_TOK_INT; }
    // 19 digits or more: not an int64 this parser vouches for; as a real it is
    // converted below (an integer role then sends the token to the host)
  }
  if (i < len && t[i] == '.') {
    ++i;
    while (i < len && t[i] >= '0' && t[i] <= '9') {
      const unsigned d = t[i] - '0';
      if (sig > 0 || d) {
        if (sig < 19) { w = w * 10 + d; ++sig; --q; } else { dropped |= d != 0; }
      } else {
        --q;
      }
      ++digits; ++i;
    }
  }
  if (digits == 0) return GP_TOK_SUSPECT;
  if (i < len && (t[i] == 'e' || t[i] == 'E')) {
    ++i;
    bool eneg = false;
    if (i < len && (t[i] == '+' || t[i] == '-')) { eneg = t[i] == '-'; ++i; }
    if (i >= len) return GP_TOK_SUSPECT;
    long long e = 0;
    while (i < len && t[i] >= '0' && t[i] <= '9') {
      if (e < 100000) e = e * 10 + (t[i] - '0');
      ++i;
    }
    q += eneg ? -e : e;
  }
  if (i != len) return GP_TOK_SUSPECT;  // trailing junk
  unsigned long long bits;
  if (!decimal_to_double(w, q, neg, &bits)) return GP_TOK_SUSPECT;
  if (dropped) {
    // more than 19 significant digits: the value lies strictly between w and w + 1 units
    // of 10^q; when both round to the same double, so does the value
    unsigned long long above;
    if (!decimal_to_double(w + 1, q, neg, &above) || above != bits) return GP_TOK_SUSPECT;
  }
  *val = (long long)bits;
  return GP_TOK_REAL;
}

// ---------------------------------------------------------------- tokenizer
struct TileSum {
  int lines;      // line starts in the tile
  int tok_pre;    // token starts before the tile's first break (void if entering in a comment)
  int tok_post;   // token starts after it
  int nonascii;   // bytes >= 0x7f and control bytes other than \t \n \r
  unsigned char has_break, ends_cmt, pad[2];
};
struct TileBase {
  long long line0, tok0;
  int enter_cmt, pad;
};

// comment-carry monoid over (has_break, ends_in_comment-if-not-entered-in-one)
__device__ __forceinline__ unsigned cmt_combine(unsigned a, unsigned b) {
  const unsigned hb = (a | b) & 1u;
  const unsigned en = (b & 1u) ? (b & 2u) : ((a | b) & 2u);
  return hb | en;
}

// Per-thread view of its PER bytes: bit j of the masks describes byte j.
struct Chunk {
  unsigned brk, spc, hash, hi;  // break, whitespace, comment char, non-ASCII or control byte
};

// Word-wise byte tests: bit 7 of every byte of the result is set where the test holds.
__device__ __forceinline__ unsigned bytes_ge(unsigned w, unsigned c) {   // byte >= c, c in 1..0x80
  return (((w & 0x7f7f7f7fu) + (0x80u - c) * 0x01010101u) | w) & 0x80808080u;
}
__device__ __forceinline__ unsigned bytes_eq(unsigned w, unsigned c) {   // byte == c, c < 0x80
  const unsigned x = w ^ (c * 0x01010101u);
  return ~(((x & 0x7f7f7f7fu) + 0x7f7f7f7fu) | x) & 0x80808080u;
}
// bits 7, 15, 23, 31 -> bits 0..3 (the four partial products do not overlap)
__device__ __forceinline__ unsigned pack4(unsigned m) { return ((m >> 7) * 0x01020408u) >> 24; }

__device__ __forceinline__ Chunk load_chunk(const unsigned char* __restrict__ text, long long len,
                                            long long base, int cmt_char) {
  Chunk c{0u, 0u, 0u, 0u};
  if (base + PER + 1 <= len && ((uintptr_t)(text + base) & 15) == 0) {
    // four bytes per operation: classify each 32-bit word, pack the per-byte flags
    const uint4* p = reinterpret_cast<const uint4*>(text + base);
    unsigned nl = 0, cr = 0;
#pragma unroll
    for (int v = 0; v < PER / 16; ++v) {
      const uint4 x = p[v];
      const unsigned wds[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const unsigned w = wds[k];
        const int sh = 16 * v + 4 * k;
        const unsigned e_nl = bytes_eq(w, '\n'), e_cr = bytes_eq(w, '\r');
        const unsigned ctl = (bytes_ge(w, 0x20) ^ 0x80808080u) & ~(e_nl | e_cr | bytes_eq(w, '\t'));
        c.spc |= pack4(bytes_ge(w, 0x21) ^ 0x80808080u) << sh;
        nl |= pack4(e_nl) << sh;
        cr |= pack4(e_cr) << sh;
        c.hi |= pack4(bytes_ge(w, 0x7f) | ctl) << sh;
        if (cmt_char) c.hash |= pack4(bytes_eq(w, (unsigned)cmt_char)) << sh;
      }
    }
    // a '\r' directly before a '\n' is not a break of its own
    const unsigned next_nl = (nl >> 1) | (text[base + PER] == '\n' ? 0x80000000u : 0u);
    c.brk = nl | (cr & ~next_nl);
    return c;
  }
#pragma unroll 1
  for (int j = 0; j < PER; ++j) {   // the last chunks of the text
    if (base + j >= len) { c.spc |= 1u << j; continue; }  // past the end: padding
    const unsigned ch = text[base + j];
    const unsigned nx = base + j + 1 < len ? text[base + j + 1] : 0u;
    if (is_break(ch, nx)) c.brk |= 1u << j;
    if (is_space(ch)) c.spc |= 1u << j;
    if (cmt_char && ch == (unsigned)cmt_char) c.hash |= 1u << j;
    if (ch >= 0x7fu || (ch < 0x20u && ch != '\t' && ch != '\n' && ch != '\r')) c.hi |= 1u << j;
  }
  return c;
}

// bits of the chunk that lie inside a '#' comment, given the state at its first byte
__device__ __forceinline__ unsigned comment_mask(const Chunk& c, bool entering) {
  if (!c.hash)   // no comment starts here: an entering one runs up to the first break
    return !entering ? 0u : (c.brk ? (c.brk & (0u - c.brk)) - 1u : 0xffffffffu);
  unsigned m = 0;
  bool in = entering;
#pragma unroll
  for (int j = 0; j < PER; ++j) {
    if (c.brk >> j & 1u) in = false;
    else if (c.hash >> j & 1u) in = true;
    if (in) m |= 1u << j;
  }
  return m;
}
__device__ __forceinline__ unsigned chunk_carry(const Chunk& c) {
  // (has_break, ends in comment assuming it was not entered in one)
  if (!c.brk) return c.hash ? 2u : 0u;
  const int last = 31 - __clz(c.brk);
  const unsigned after = last == 31 ? 0u : (c.hash >> (last + 1));
  return 1u | (after ? 2u : 0u);
}

// Exclusive scan of the comment carry over the CTA's threads; returns whether thread t
// starts inside a comment, given the tile's entry state.
__device__ bool block_comment_entry(unsigned carry, bool tile_enter, unsigned* tile_carry) {
  __shared__ unsigned warp_c[TPB / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned inc = carry;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned up = __shfl_up_sync(FULL, inc, o);
    if (lane >= o) inc = cmt_combine(up, inc);
  }
  if (lane == 31) warp_c[wid] = inc;
  __syncthreads();
  unsigned pre = 0;  // carry of all earlier warps
  for (int w2 = 0; w2 < wid; ++w2) pre = cmt_combine(pre, warp_c[w2]);
  unsigned exc = __shfl_up_sync(FULL, inc, 1);
  if (lane == 0) exc = 0;
  const unsigned before = cmt_combine(pre, exc);
  if (tile_carry && threadIdx.x == TPB - 1) *tile_carry = cmt_combine(pre, inc);
  __syncthreads();
  return (before & 1u) ? (before & 2u) != 0 : (tile_enter || (before & 2u) != 0);
}

// line starts and token starts of a chunk; `prev_*` describe the byte before it
__device__ __forceinline__ void chunk_starts(const Chunk& c, unsigned cmt, bool prev_break,
                                             bool prev_blank, unsigned valid, unsigned* line_start,
                                             unsigned* tok_start) {
  const unsigned blank = c.spc | cmt;
  *line_start = ((c.brk << 1) | (prev_break ? 1u : 0u)) & valid;
  *tok_start = ~blank & ((blank << 1) | (prev_blank ? 1u : 0u)) & valid;
}

__device__ __forceinline__ unsigned valid_mask(long long base, long long len) {
  const long long left = len - base;
  return left >= PER ? 0xffffffffu : (left <= 0 ? 0u : ((1u << left) - 1u));
}

// state of the byte just before `base` (the previous thread's last byte)
__device__ __forceinline__ void prev_byte(const unsigned char* text, long long len, long long base,
                                          bool* is_brk, bool* is_spc) {
  if (base == 0 || base > len) { *is_brk = base == 0; *is_spc = true; return; }
  const unsigned p = text[base - 1];
  const unsigned cur = base < len ? text[base] : 0u;
  *is_brk = is_break(p, cur);
  *is_spc = is_space(p);
}

__global__ void __launch_bounds__(TPB) text_count(const unsigned char* __restrict__ text,
                                                  long long len, int cmt_char,
                                                  TileSum* __restrict__ sums) {
  const long long base = (long long)blockIdx.x * TILE + (long long)threadIdx.x * PER;
  const Chunk c = load_chunk(text, len, base, cmt_char);
  __shared__ unsigned tile_carry;
  __shared__ int s_first_break;  // byte index (in tile) of the first break, TILE if none
  __shared__ int s_cnt[4];
  if (threadIdx.x == 0) { s_first_break = TILE; s_cnt[0] = s_cnt[1] = s_cnt[2] = s_cnt[3] = 0; }
  __syncthreads();
  const bool enter = cmt_char ? block_comment_entry(chunk_carry(c), false, &tile_carry) : false;
  const unsigned cmt = cmt_char ? comment_mask(c, enter) : 0u;
  bool pb, ps;
  prev_byte(text, len, base, &pb, &ps);
  // the previous byte counts as blank when it is whitespace or inside a comment: a byte
  // inside a comment is followed either by more comment or by a break, so only the
  // whitespace test matters for a token start (a token cannot start inside a comment)
  unsigned ls, ts;
  chunk_starts(c, cmt, pb, ps || enter, valid_mask(base, len), &ls, &ts);
  if (c.brk) atomicMin(&s_first_break, threadIdx.x * PER + (__ffs(c.brk) - 1));
  __syncthreads();
  const int fb = s_first_break - threadIdx.x * PER;  // first break relative to this chunk
  const unsigned pre_mask = fb >= PER ? 0xffffffffu : (fb <= 0 ? 0u : ((1u << fb) - 1u));
  const int n_ls = __popc(ls), n_pre = __popc(ts & pre_mask), n_post = __popc(ts & ~pre_mask);
  const int n_hi = __popc(c.hi);
  // warp totals, then one atomic per warp
  int v0 = n_ls, v1 = n_pre, v2 = n_post, v3 = n_hi;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    v0 += __shfl_xor_sync(FULL, v0, o);
    v1 += __shfl_xor_sync(FULL, v1, o);
    v2 += __shfl_xor_sync(FULL, v2, o);
    v3 += __shfl_xor_sync(FULL, v3, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(&s_cnt[0], v0); atomicAdd(&s_cnt[1], v1);
    atomicAdd(&s_cnt[2], v2); atomicAdd(&s_cnt[3], v3);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    TileSum s;
    s.lines = s_cnt[0]; s.tok_pre = s_cnt[1]; s.tok_post = s_cnt[2]; s.nonascii = s_cnt[3];
    const unsigned tc = cmt_char ? tile_carry : (s_first_break < TILE ? 1u : 0u);
    s.has_break = tc & 1u; s.ends_cmt = (tc >> 1) & 1u; s.pad[0] = s.pad[1] = 0;
    sums[blockIdx.x] = s;
  }
}

// One CTA: tile prefix sums.  Thread t owns a contiguous range of tiles; three walks
// (comment carry, counts, write) around two serial scans over the 1024 thread totals.
__global__ void __launch_bounds__(1024) text_tiles(const TileSum* __restrict__ sums,
                                                   long long n_tiles, TileBase* __restrict__ bases,
                                                   long long* __restrict__ totals) {
  __shared__ unsigned s_carry[1024];
  __shared__ long long s_lines[1024], s_toks[1024], s_hi[1024];
  const long long per = (n_tiles + 1023) / 1024;
  const long long lo = threadIdx.x * per, hi = lo + per < n_tiles ? lo + per : n_tiles;
  unsigned carry = 0;
  for (long long t = lo; t < hi; ++t)
    carry = cmt_combine(carry, (unsigned)sums[t].has_break | ((unsigned)sums[t].ends_cmt << 1));
  s_carry[threadIdx.x] = carry;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned run = 0;
    for (int i = 0; i < 1024; ++i) { const unsigned c = s_carry[i]; s_carry[i] = run; run = cmt_combine(run, c); }
  }
  __syncthreads();
  bool in_cmt = (s_carry[threadIdx.x] & 2u) != 0;
  const bool enter0 = in_cmt;
  long long nl = 0, nt = 0, nh = 0;
  for (long long t = lo; t < hi; ++t) {
    const TileSum s = sums[t];
    nl += s.lines; nt += (in_cmt ? 0 : s.tok_pre) + s.tok_post; nh += s.nonascii;
    in_cmt = s.has_break ? s.ends_cmt != 0 : (in_cmt || s.ends_cmt != 0);
  }
  s_lines[threadIdx.x] = nl; s_toks[threadIdx.x] = nt; s_hi[threadIdx.x] = nh;
  __syncthreads();
  if (threadIdx.x == 0) {
    long long a = 0, b = 0, h = 0;
    for (int i = 0; i < 1024; ++i) {
      const long long x = s_lines[i], y = s_toks[i];
      s_lines[i] = a; s_toks[i] = b; a += x; b += y; h += s_hi[i];
    }
    totals[0] = a; totals[1] = b; totals[2] = h;
  }
  __syncthreads();
  long long l0 = s_lines[threadIdx.x], t0 = s_toks[threadIdx.x];
  in_cmt = enter0;
  for (long long t = lo; t < hi; ++t) {
    const TileSum s = sums[t];
    bases[t] = TileBase{l0, t0, in_cmt ? 1 : 0, 0};
    l0 += s.lines; t0 += (in_cmt ? 0 : s.tok_pre) + s.tok_post;
    in_cmt = s.has_break ? s.ends_cmt != 0 : (in_cmt || s.ends_cmt != 0);
  }
}

__global__ void __launch_bounds__(TPB) text_emit(const unsigned char* __restrict__ text,
                                                 long long len, int cmt_char,
                                                 const TileBase* __restrict__ bases,
                                                 long long n_lines, long long n_tokens,
                                                 long long* __restrict__ line_off,
                                                 long long* __restrict__ line_tok0,
                                                 long long* __restrict__ tok_val,
                                                 unsigned char* __restrict__ tok_kind) {
  const long long base = (long long)blockIdx.x * TILE + (long long)threadIdx.x * PER;
  const Chunk c = load_chunk(text, len, base, cmt_char);
  const TileBase tb = bases[blockIdx.x];
  const bool enter = cmt_char ? block_comment_entry(chunk_carry(c), tb.enter_cmt != 0, nullptr)
                              : false;
  const unsigned cmt = cmt_char ? comment_mask(c, enter) : 0u;
  bool pb, ps;
  prev_byte(text, len, base, &pb, &ps);
  unsigned ls, ts;
  chunk_starts(c, cmt, pb, ps || enter, valid_mask(base, len), &ls, &ts);
  // exclusive scan of (line starts, token starts) over the CTA
  __shared__ int w_l[TPB / 32], w_t[TPB / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int il = __popc(ls), it = __popc(ts);
  const int ml = il, mt = it;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int a = __shfl_up_sync(FULL, il, o), b = __shfl_up_sync(FULL, it, o);
    if (lane >= o) { il += a; it += b; }
  }
  if (lane == 31) { w_l[wid] = il; w_t[wid] = it; }
  __syncthreads();
  long long l_id = tb.line0 + il - ml, t_id = tb.tok0 + it - mt;
  for (int w2 = 0; w2 < wid; ++w2) { l_id += w_l[w2]; t_id += w_t[w2]; }
  // walk the chunk in byte order
  unsigned any = ls | ts;
  while (any) {
    const int j = __ffs(any) - 1;
    any &= any - 1;
    if (ls >> j & 1u) {
      line_off[l_id] = base + j;
      line_tok0[l_id] = t_id;
      ++l_id;
    }
    if (ts >> j & 1u) {
      const unsigned char* t = text + base + j;
      const long long left = len - (base + j);
      // the token ends at the next blank or comment byte: inside this chunk by the masks
      const unsigned rest = (c.spc | cmt) >> j;
      int tl;
      if (rest) {
        tl = __ffs(rest) - 1;
      } else {
        tl = PER - j;
        while (tl < left && tl <= MAX_TOKEN && !is_space(t[tl]) &&
               !(cmt_char && t[tl] == (unsigned char)cmt_char))
          ++tl;
      }
      long long v;
      const int kind = parse_number(t, tl, &v);
      tok_val[t_id] = v;
      tok_kind[t_id] = (unsigned char)kind;
      ++t_id;
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {  // sentinels
    line_off[n_lines] = len;
    line_tok0[n_lines] = n_tokens;
  }
}

// ---------------------------------------------------------------- METIS assembly
// body flag per line: 1 unless its first token starts with '%' (fileio.py:85-93)
__global__ void metis_line_kind(const long long* __restrict__ line_tok0,
                                const unsigned char* __restrict__ tok_kind, long long n_lines,
                                long long* __restrict__ body_flag) {
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < n_lines;
       l += (long long)gridDim.x * blockDim.x) {
    const long long t0 = line_tok0[l], t1 = line_tok0[l + 1];
    body_flag[l] = (t1 > t0 && tok_kind[t0] == GP_TOK_PERCENT) ? 0 : 1;
  }
}

// rank r among the non-comment lines: r = 0 is the header, r - 1 the vertex.  Writes
// the line of every vertex, the header line, and the last vertex line holding a token.
__global__ void metis_body_lines(const long long* __restrict__ rank_excl,
                                 const long long* __restrict__ body_flag,
                                 const long long* __restrict__ line_tok0, long long n_lines,
                                 long long* __restrict__ body_line, long long body_cap,
                                 long long* __restrict__ info) {
  unsigned long long last = 0;  // 1 + largest vertex index whose line holds a token
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < n_lines;
       l += (long long)gridDim.x * blockDim.x) {
    if (!body_flag[l]) continue;
    const long long r = rank_excl[l];
    if (r == 0) { info[1] = l; continue; }
    if (r - 1 < body_cap) body_line[r - 1] = l;
    if (line_tok0[l + 1] > line_tok0[l] && (unsigned long long)r > last) last = r;
  }
  __shared__ unsigned long long s_last;
  if (threadIdx.x == 0) s_last = 0;
  __syncthreads();
  for (int o = 16; o; o >>= 1) {
    const unsigned long long other = __shfl_xor_sync(FULL, last, o);
    last = other > last ? other : last;
  }
  if ((threadIdx.x & 31) == 0 && last) atomicMax(&s_last, last);
  __syncthreads();
  if (threadIdx.x == 0 && s_last) atomicMax((unsigned long long*)&info[2], s_last);
}

// degrees (fileio.py:131-149): tokens minus the optional weight, halved with edge weights
__global__ void metis_degrees(const long long* __restrict__ line_tok0,
                              const long long* __restrict__ body_line, long long n, int has_vw,
                              int has_ew, long long* __restrict__ deg,
                              unsigned char* __restrict__ flags) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n;
       u += (long long)gridDim.x * blockDim.x) {
    const long long l = body_line[u];
    const long long nt = line_tok0[l + 1] - line_tok0[l];
    unsigned char f = 0;
    long long rest = nt - (has_vw ? 1 : 0);
    if (rest < 0) { f = 1; rest = 0; }           // missing vertex weight
    if (has_ew && (rest & 1)) f = 1;             // dangling neighbor
    deg[u] = has_ew ? rest / 2 : rest;
    flags[u] = f;
  }
}

__device__ __forceinline__ bool token_real(long long v, int kind, double* out) {
  if (kind == GP_TOK_INT) { *out = (double)v; return true; }
  if (kind == GP_TOK_REAL) { *out = __longlong_as_double(v); return true; }
  return false;
}

// adjacency, weights and per-line checks (fileio.py:131-160); the duplicate test is left
// to gp_graph_check (sorted directed edges)
__global__ void metis_fill(const long long* __restrict__ line_tok0,
                           const long long* __restrict__ body_line,
                           const long long* __restrict__ tok_val,
                           const unsigned char* __restrict__ tok_kind, long long n, int has_vw,
                           int has_ew, const long long* __restrict__ offsets,
                           long long* __restrict__ nbrs, double* __restrict__ ew,
                           double* __restrict__ vw, unsigned char* __restrict__ flags) {
  for (long long u = blockIdx.x * (long long)blockDim.x + threadIdx.x; u < n;
       u += (long long)gridDim.x * blockDim.x) {
    const long long l = body_line[u];
    long long t = line_tok0[l];
    const long long t1 = line_tok0[l + 1];
    bool bad = flags[u] != 0;
    if (has_vw) {
      double w = 1.0;
      if (t < t1) {
        if (!token_real(tok_val[t], tok_kind[t], &w) || !(w > 0.0) || isinf(w)) bad = true;
        ++t;
      }
      vw[u] = w;
    }
    const long long o0 = offsets[u], o1 = offsets[u + 1];
    for (long long j = o0; j < o1; ++j) {
      const long long v = tok_val[t];
      if (tok_kind[t] != GP_TOK_INT || v < 1 || v > n || v == u + 1) bad = true;
      nbrs[j] = v - 1;
      ++t;
      if (has_ew) {
        double w = 1.0;
        if (!token_real(tok_val[t], tok_kind[t], &w) || !(w > 0.0) || isinf(w)) bad = true;
        ew[j] = w;
        ++t;
      }
    }
    flags[u] = bad ? 1 : 0;
  }
}

// ---------------------------------------------------------------- tables (np.loadtxt)
// values of a whitespace table in row-major order = the token values in order, once
// every non-blank line has `ncols` tokens.  info[0] = rows, info[1] = first line whose
// token count differs (or -1), info[2] = first token that is not a plain number (or -1).
__global__ void table_first_row(const long long* __restrict__ line_tok0, long long n_lines,
                                long long* __restrict__ info) {
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < n_lines;
       l += (long long)gridDim.x * blockDim.x)
    if (line_tok0[l] == 0 && line_tok0[l + 1] > 0) info[3] = line_tok0[l + 1];
}

__global__ void table_lines(const long long* __restrict__ line_tok0, long long n_lines,
                            long long* __restrict__ info) {
  const long long ncols = info[3];
  long long rows = 0;
  unsigned long long bad = ~0ull;
  for (long long l = blockIdx.x * (long long)blockDim.x + threadIdx.x; l < n_lines;
       l += (long long)gridDim.x * blockDim.x) {
    const long long nt = line_tok0[l + 1] - line_tok0[l];
    if (nt == 0) continue;
    ++rows;
    if (nt != ncols && (unsigned long long)l < bad) bad = (unsigned long long)l;
  }
  for (int o = 16; o; o >>= 1) {
    rows += __shfl_xor_sync(FULL, rows, o);
    const unsigned long long b2 = __shfl_xor_sync(FULL, bad, o);
    bad = b2 < bad ? b2 : bad;
  }
  if ((threadIdx.x & 31) == 0) {
    if (rows) atomicAdd((unsigned long long*)&info[0], (unsigned long long)rows);
    if (bad != ~0ull) atomicMin((unsigned long long*)&info[1], bad);
  }
}

__global__ void table_values(const long long* __restrict__ tok_val,
                             const unsigned char* __restrict__ tok_kind, long long n_tokens,
                             int want_int, void* __restrict__ out, long long* __restrict__ info) {
  unsigned long long bad = ~0ull;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < n_tokens;
       t += (long long)gridDim.x * blockDim.x) {
    const long long v = tok_val[t];
    const int kind = tok_kind[t];
    if (want_int) {
      ((long long*)out)[t] = v;
      if (kind != GP_TOK_INT && (unsigned long long)t < bad) bad = (unsigned long long)t;
    } else {
      double x = 0.0;
      if (!token_real(v, kind, &x) && (unsigned long long)t < bad) bad = (unsigned long long)t;
      ((double*)out)[t] = x;
    }
  }
  for (int o = 16; o; o >>= 1) {
    const unsigned long long b2 = __shfl_xor_sync(FULL, bad, o);
    bad = b2 < bad ? b2 : bad;
  }
  if ((threadIdx.x & 31) == 0 && bad != ~0ull) atomicMin((unsigned long long*)&info[2], bad);
}

// ---------------------------------------------------------------- integer writer
__device__ __forceinline__ int dec_len(long long v) {
  unsigned long long a = v < 0 ? 0ull - (unsigned long long)v : (unsigned long long)v;
  int n = v < 0 ? 2 : 1;
  while (a >= 10) { a /= 10; ++n; }
  return n;
}
__global__ void format_lengths(const long long* __restrict__ v, long long n,
                               long long* __restrict__ lens) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x)
    lens[i] = dec_len(v[i]) + 1;  // + the '\n'
}
__global__ void format_write(const long long* __restrict__ v, long long n,
                             const long long* __restrict__ pos, unsigned char* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n;
       i += (long long)gridDim.x * blockDim.x) {
    const long long x = v[i];
    unsigned long long a = x < 0 ? 0ull - (unsigned long long)x : (unsigned long long)x;
    const int L = dec_len(x);
    unsigned char* p = out + pos[i];
    p[L] = '\n';
    for (int j = L - 1; j >= (x < 0 ? 1 : 0); --j) { p[j] = (unsigned char)('0' + a % 10); a /= 10; }
    if (x < 0) p[0] = '-';
  }
}

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

}  // namespace
}  // namespace gp

using namespace gp;

extern "C" {

int gp_parse_number_host(const char* text, int len, int64_t* value) {
  long long v = 0;
  const int kind = parse_number((const unsigned char*)text, len, &v);
  *value = v;
  return kind;
}

int gp_text_index_workspace_bytes(int64_t len, size_t* bytes) {
  GP_REQUIRE(len >= 0, "gp_text_index: negative length");
  const long long tiles = (len + TILE - 1) / TILE;
  *bytes = align256((size_t)(tiles + 1) * sizeof(TileSum)) +
           align256((size_t)(tiles + 1) * sizeof(TileBase)) + 256;
  return GP_OK;
}

int gp_text_index(const uint8_t* text, int64_t len, int comment_char, int64_t* counts,
                  void* workspace, size_t workspace_bytes, void* stream) {
  GP_REQUIRE(len >= 1, "gp_text_index: empty text");
  size_t need = 0;
  gp_text_index_workspace_bytes(len, &need);
  GP_REQUIRE(workspace_bytes >= need, "gp_text_index: workspace too small");
  GP_REQUIRE(comment_char >= 0 && comment_char < 128, "gp_text_index: bad comment char");
  cudaStream_t s = (cudaStream_t)stream;
  const long long tiles = (len + TILE - 1) / TILE;
  GP_REQUIRE(tiles < (1ll << 31), "gp_text_index: text too long");
  TileSum* sums = (TileSum*)workspace;
  TileBase* bases = (TileBase*)((char*)workspace + align256((size_t)(tiles + 1) * sizeof(TileSum)));
  text_count<<<(unsigned)tiles, TPB, 0, s>>>(text, len, comment_char, sums);
  text_tiles<<<1, 1024, 0, s>>>(sums, tiles, bases, (long long*)counts);
  return check_launch("gp_text_index");
}

int gp_text_tokens(const uint8_t* text, int64_t len, int comment_char, const void* workspace,
                   int64_t n_lines, int64_t n_tokens, int64_t* line_off, int64_t* line_tok0,
                   int64_t* tok_val, uint8_t* tok_kind, void* stream) {
  GP_REQUIRE(len >= 1, "gp_text_tokens: empty text");
  cudaStream_t s = (cudaStream_t)stream;
  const long long tiles = (len + TILE - 1) / TILE;
  const TileBase* bases =
      (const TileBase*)((const char*)workspace + align256((size_t)(tiles + 1) * sizeof(TileSum)));
  text_emit<<<(unsigned)tiles, TPB, 0, s>>>(text, len, comment_char, bases, n_lines, n_tokens,
                                            (long long*)line_off, (long long*)line_tok0,
                                            (long long*)tok_val, tok_kind);
  return check_launch("gp_text_tokens");
}

int gp_metis_workspace_bytes(int64_t n_lines, size_t* bytes) {
  GP_REQUIRE(n_lines >= 0 && n_lines < (1ll << 31), "gp_metis: line count out of range");
  *bytes = 2 * align256((size_t)(n_lines + 1) * sizeof(long long)) + scan_bytes(n_lines + 1);
  return GP_OK;
}

int gp_metis_lines(const int64_t* line_tok0, const uint8_t* tok_kind, int64_t n_lines,
                   int64_t* body_line, int64_t body_cap, int64_t* info, void* workspace,
                   size_t workspace_bytes, void* stream) {
  size_t need = 0;
  int rc = gp_metis_workspace_bytes(n_lines, &need);
  if (rc) return rc;
  GP_REQUIRE(n_lines >= 1, "gp_metis_lines: no lines");
  GP_REQUIRE(workspace_bytes >= need, "gp_metis_lines: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t arr = align256((size_t)(n_lines + 1) * sizeof(long long));
  long long* flag = (long long*)workspace;
  long long* rank = (long long*)((char*)workspace + arr);
  void* sws = (char*)workspace + 2 * arr;
  size_t sb = workspace_bytes - 2 * arr;
  const unsigned g = sm_grid(n_lines, 256);
  // info: [non-comment lines, header line, 1 + last vertex index with a token]
  GP_CUDA(cudaMemsetAsync(info, 0, 3 * sizeof(int64_t), s));
  GP_CUDA(cudaMemsetAsync(flag + n_lines, 0, sizeof(long long), s));
  metis_line_kind<<<g, 256, 0, s>>>((const long long*)line_tok0, tok_kind, n_lines, flag);
  GP_CUDA(cub::DeviceScan::ExclusiveSum(sws, sb, flag, rank, (int)(n_lines + 1), s));
  GP_CUDA(cudaMemcpyAsync(info, rank + n_lines, sizeof(long long), cudaMemcpyDeviceToDevice, s));
  metis_body_lines<<<g, 256, 0, s>>>(rank, flag, (const long long*)line_tok0, n_lines,
                                     (long long*)body_line, body_cap, (long long*)info);
  return check_launch("gp_metis_lines");
}

int gp_metis_offsets(const int64_t* line_tok0, const int64_t* body_line, int64_t n, int has_vw,
                     int has_ew, int64_t* offsets, uint8_t* flags, void* workspace,
                     size_t workspace_bytes, void* stream) {
  GP_REQUIRE(n >= 1 && n < (1ll << 31) - 1, "gp_metis_offsets: n out of range");
  size_t need = 0;
  gp_metis_workspace_bytes(n, &need);
  GP_REQUIRE(workspace_bytes >= need, "gp_metis_offsets: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t arr = align256((size_t)(n + 1) * sizeof(long long));
  long long* deg = (long long*)workspace;
  void* sws = (char*)workspace + 2 * arr;
  size_t sb = workspace_bytes - 2 * arr;
  GP_CUDA(cudaMemsetAsync(deg + n, 0, sizeof(long long), s));
  metis_degrees<<<sm_grid(n, 256), 256, 0, s>>>((const long long*)line_tok0,
                                                 (const long long*)body_line, n, has_vw, has_ew,
                                                 deg, flags);
  GP_CUDA(cub::DeviceScan::ExclusiveSum(sws, sb, deg, (long long*)offsets, (int)(n + 1), s));
  return check_launch("gp_metis_offsets");
}

int gp_metis_fill(const int64_t* line_tok0, const int64_t* body_line, const int64_t* tok_val,
                  const uint8_t* tok_kind, int64_t n, int has_vw, int has_ew,
                  const int64_t* offsets, int64_t* neighbors, double* edge_weights,
                  double* vertex_weights, uint8_t* flags, void* stream) {
  GP_REQUIRE(n >= 1, "gp_metis_fill: n out of range");
  GP_REQUIRE(!has_ew || edge_weights, "gp_metis_fill: edge weights wanted but no buffer");
  GP_REQUIRE(!has_vw || vertex_weights, "gp_metis_fill: vertex weights wanted but no buffer");
  metis_fill<<<sm_grid(n, 128), 128, 0, (cudaStream_t)stream>>>(
      (const long long*)line_tok0, (const long long*)body_line, (const long long*)tok_val,
      tok_kind, n, has_vw, has_ew, (const long long*)offsets, (long long*)neighbors,
      edge_weights, vertex_weights, flags);
  return check_launch("gp_metis_fill");
}

int gp_table_values(const int64_t* line_tok0, int64_t n_lines, const int64_t* tok_val,
                    const uint8_t* tok_kind, int64_t n_tokens, int want_int, void* out,
                    int64_t* info, void* stream) {
  GP_REQUIRE(n_lines >= 1 && n_tokens >= 0, "gp_table_values: bad sizes");
  cudaStream_t s = (cudaStream_t)stream;
  GP_CUDA(cudaMemsetAsync(info, 0, 4 * sizeof(int64_t), s));
  GP_CUDA(cudaMemsetAsync(info + 1, 0xff, 2 * sizeof(int64_t), s));
  const unsigned g = sm_grid(n_lines, 256);
  table_first_row<<<g, 256, 0, s>>>((const long long*)line_tok0, n_lines, (long long*)info);
  table_lines<<<g, 256, 0, s>>>((const long long*)line_tok0, n_lines, (long long*)info);
  if (n_tokens > 0)
    table_values<<<sm_grid(n_tokens, 256), 256, 0, s>>>((const long long*)tok_val, tok_kind,
                                                        n_tokens, want_int, out,
                                                        (long long*)info);
  return check_launch("gp_table_values");
}

int gp_format_ints_workspace_bytes(int64_t n, size_t* bytes) {
  GP_REQUIRE(n >= 0 && n < (1ll << 31) - 1, "gp_format_ints: n out of range");
  *bytes = 2 * align256((size_t)(n + 1) * sizeof(long long)) + scan_bytes(n + 1);
  return GP_OK;
}

int gp_format_ints_plan(const int64_t* values, int64_t n, int64_t* out_len, void* workspace,
                        size_t workspace_bytes, void* stream) {
  size_t need = 0;
  int rc = gp_format_ints_workspace_bytes(n, &need);
  if (rc) return rc;
  GP_REQUIRE(n >= 1, "gp_format_ints: nothing to write");
  GP_REQUIRE(workspace_bytes >= need, "gp_format_ints: workspace too small");
  cudaStream_t s = (cudaStream_t)stream;
  const size_t arr = align256((size_t)(n + 1) * sizeof(long long));
  long long* lens = (long long*)workspace;
  long long* pos = (long long*)((char*)workspace + arr);
  void* sws = (char*)workspace + 2 * arr;
  size_t sb = workspace_bytes - 2 * arr;
  GP_CUDA(cudaMemsetAsync(lens + n, 0, sizeof(long long), s));
  format_lengths<<<sm_grid(n, 256), 256, 0, s>>>((const long long*)values, n, lens);
  GP_CUDA(cub::DeviceScan::ExclusiveSum(sws, sb, lens, pos, (int)(n + 1), s));
  GP_CUDA(cudaMemcpyAsync(out_len, pos + n, sizeof(long long), cudaMemcpyDeviceToDevice, s));
  return check_launch("gp_format_ints_plan");
}

int gp_format_ints_write(const int64_t* values, int64_t n, uint8_t* out, const void* workspace,
                         void* stream) {
  GP_REQUIRE(n >= 1, "gp_format_ints: nothing to write");
  const size_t arr = align256((size_t)(n + 1) * sizeof(long long));
  const long long* pos = (const long long*)((const char*)workspace + arr);
  format_write<<<sm_grid(n, 256), 256, 0, (cudaStream_t)stream>>>((const long long*)values, n, pos,
                                                                  out);
  return check_launch("gp_format_ints_write");
}

}  // extern "C"
