// kernels.cuh -- launch-shape constants and kernel declarations.
#pragma once
#include <cuda.h>

#include "actc_internal.cuh"

namespace actc {

// K1: 256 threads x 16 elements per tile
constexpr int K1_THREADS = 256;
constexpr int K1_EPT = 16;
constexpr int K1_TILE = K1_THREADS * K1_EPT;
constexpr uint32_t K1_WIN = 8192;  // shared-memory histogram window (bins)

// K2: one CTA
constexpr int K2_THREADS = 1024;
constexpr uint32_t K2_SMEM_SORT_MAX = 8192;  // keys sorted in shared memory

// K3 segment encoder: one warp per segment of 32 lanes x 32 symbols; codes
// of up to K3_SHORT_MAXLEN bits take the shared-window path, longer ones
// (<= 56 bits) the u64 path
constexpr int K3_SHORT_MAXLEN = 26;
constexpr int K3L_THREADS = 256;
constexpr int K3L_EPT = 32;
constexpr int K3L_SEG = 32 * K3L_EPT;                                     // symbols per segment
constexpr uint32_t K3L_WIN = 16384;                                       // u32 code-table window
constexpr int K3L_WORDS = (K3L_SEG * K3_SHORT_MAXLEN + 31) / 32 + 2;      // packed words per segment (max)

// K4 (scan variant, streams without a lattice index): one thread per chunk
constexpr int K4_THREADS = 128;
// K4 (warp variant, indexed streams): one warp per 32 chunks
// K4L (indexed streams): one CTA of up to 768 threads per SM, lane per chunk; the
// canonical deltas in the shared memory the warps leave (all of them, or the
// leading canonical indices of a wide alphabet)
constexpr int K4L_THREADS = 768;  // at most; small streams launch fewer warps per CTA
constexpr int K4_TILE = K4_THREADS * ACTC_CHUNK;

// lookback status for the encoder (per K3 tile)
struct EncStatus {
  unsigned *flag;
  unsigned long long *agg_bits, *agg_nz, *inc_bits, *inc_nz;
  unsigned *tail;
};
// lookback status for the decoder (per K4 tile)
struct DecStatus {
  unsigned *flag;
  int *agg_r;
  long long *agg_v, *inc_v;
};

template <typename SymT>
__global__ void k1_quant_lorenzo_hist(const float *__restrict__ x, uint64_t n, QParams P,
                                      uint32_t radius, SymT *__restrict__ sym,
                                      unsigned long long *__restrict__ ghist,
                                      unsigned long long *__restrict__ n_outliers, uint32_t win_lo,
                                      uint32_t win_n, unsigned *__restrict__ nonfinite,
                                      long long *__restrict__ chunk_lat);
__global__ void k_hist_u32(const uint32_t *__restrict__ s, uint64_t n, uint64_t alphabet,
                           unsigned long long *__restrict__ ghist, unsigned *__restrict__ bad,
                           uint32_t win_n);
__global__ void k_quant_check(uint64_t lo, uint64_t count, QParams P, unsigned long long *__restrict__ out);
__global__ void k_prequantize(const void *__restrict__ x, int dtype, uint64_t n, double eb,
                              long long *__restrict__ q);
__global__ void k_lorenzo_encode(const long long *__restrict__ lat, uint64_t n, uint32_t radius,
                                 const uint8_t *__restrict__ force, uint32_t *__restrict__ sym,
                                 unsigned long long *__restrict__ n_out);

// K2 codebook.  Scratch layout is owned by the host side (CodebookScratch).
struct CodebookArgs {
  const unsigned long long *hist;  // [A]
  uint64_t A;
  const uint16_t *in_lengths;      // if non-null: skip Huffman, use these lengths
  // outputs
  unsigned long long *ctab;        // [A] (code << 8) | len, live entries only
  uint8_t *len8;                   // [A] code length per symbol, live entries only (may be null)
  uint32_t *canon;                 // [L] canonical order
  uint32_t *len_counts;            // [64]
  uint16_t *out_lengths;           // optional [A] full length table
  actc_plan_t *plan;               // device plan (fields n / n_outliers preset)
  const unsigned long long *n_outliers;  // optional counter from K1
  const unsigned *nonfinite;             // optional flag from K1 -> ACTC_EDATA
  // scratch (global, used when L exceeds the shared-memory capacity)
  uint32_t *live_sym;              // [A]
  unsigned long long *live_freq;   // [A]
  unsigned long long *keys, *keys2;  // [A] radix ping-pong
  uint32_t *vals, *vals2;            // [A]
  unsigned long long *nf;          // [A]
  uint32_t *lpar, *npar;           // [A], [A]
  uint8_t *llen, *ndepth;          // [A], [A]
  uint64_t n_symbols;              // total symbol count (for entropy)
  uint32_t sym_bytes;
  unsigned long long *dbg;         // optional stage timestamps (clock64)
  uint16_t *cls16;                 // [A] class id per symbol (k2r scratch)
  unsigned *fallback;              // k2r: 1 = caps exceeded, run k2_codebook
  const unsigned *gate;            // k2_codebook: if non-null and *gate == 0, do nothing
  uint16_t *rank_tab;              // [1024 x 34] k2r -> k2s starting canonical ranks
};
__global__ void k2_codebook(CodebookArgs a);
// K2r (frequency-class codebook) capacities; dynamic shared memory size
constexpr int K2R_NL = 32;            // k2r: max distinct code lengths
constexpr int K2R_TS = K2R_NL + 2;     // k2r: per-thread length-counter stride (u16, odd word count)

// Canonical-code emission for the symbols of k2r's per-thread segments
// (huffman.py:78-94 rule: code = first[len] + rank among the symbols of that
// length in symbol order).  Thread t (0..K2_THREADS-1) replays k2r thread t's
// segment from the starting ranks k2r left in rank_tab.  Run by k2s_emit, or
// -- on the batched path -- folded into the first warps of k3_seg_count.
struct EmitArgs {
  const unsigned *fallback;  // nonzero: k2_codebook built the tables, nothing to emit
  const uint16_t *rank_tab;  // [K2_THREADS][K2R_TS]; null = no emission pending
  const uint32_t *len_counts;
  const uint8_t *len8;
  const actc_plan_t *plan;
  uint32_t *canon;
  unsigned long long *ctab;
};
// one warp emits k2r threads 32*wblk .. 32*wblk+31; s_row holds 32*K2R_TS u16
__device__ __forceinline__ void k2s_emit_warp(const EmitArgs &e, uint32_t wblk, uint16_t *s_row,
                                              unsigned long long *s_first, uint32_t *s_base) {
  const int lane = threadIdx.x & 31;
  const uint32_t t = wblk * 32 + lane;
  // the per-length counts: two parallel loads per lane (not 64 dependent
  // loads by one thread), staged through s_base, then the canonical firsts
  const uint32_t c0 = __ldg(e.len_counts + lane), c1 = __ldg(e.len_counts + 32 + lane);
  const unsigned b0 = __ballot_sync(0xffffffffu, c0 != 0 && lane > 0), b1 = __ballot_sync(0xffffffffu, c1 != 0);
  const uint32_t minlen = b0 ? (uint32_t)(__ffs(b0) - 1) : b1 ? (uint32_t)(32 + __ffs(b1) - 1) : 64u;
  s_base[lane] = c0;
  s_base[32 + lane] = c1;
  __syncwarp();
  if (lane == 0) {
    unsigned long long code = 0;
    uint32_t idx = 0;
    for (int l = 0; l < 64; l++) {
      const uint32_t c = s_base[l];
      code <<= 1;
      s_first[l] = code;
      s_base[l] = idx;
      code += c;
      idx += c;
    }
  }
  {
    const uint32_t *src = reinterpret_cast<const uint32_t *>(e.rank_tab + (size_t)t * K2R_TS);
    uint32_t *dst = reinterpret_cast<uint32_t *>(s_row + lane * K2R_TS);
#pragma unroll
    for (int u = 0; u < K2R_TS / 2; u++) dst[u] = src[u];
  }
  __syncwarp();
  const uint32_t lo = e.plan->sym_lo, hi = e.plan->sym_hi;
  const uint32_t p0 = lo & ~15u;
  const uint32_t SEG = ((((hi + 1 - p0) + K2_THREADS - 1) / K2_THREADS) + 15) & ~15u;
  const uint32_t q0 = p0 + t * SEG, q1 = min(hi + 1, q0 + SEG);
  uint16_t *row = s_row + lane * K2R_TS;
  for (uint32_t c0 = q0; c0 < q1; c0 += 16) {
    const uint4 lv = *reinterpret_cast<const uint4 *>(e.len8 + c0);
    const uint32_t wv[4] = {lv.x, lv.y, lv.z, lv.w};
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const uint32_t s = c0 + u;
      const uint32_t len = (wv[u >> 2] >> (8 * (u & 3))) & 0xFFu;
      if (len && s < q1) {
        const uint32_t ci = row[len - minlen];
        row[len - minlen] = (uint16_t)(ci + 1);
        e.canon[ci] = s;
        if (len <= 56) e.ctab[s] = ((s_first[len] + (ci - s_base[len])) << 8) | len;
      }
    }
  }
  __syncwarp();
}

constexpr uint32_t kRCap = 6144;
constexpr uint32_t kICap = 11264;
constexpr size_t kK2rSmem = (size_t)(3 * (kRCap + 1) + 3 * (kICap + 1)) * 4;
__global__ void k2r_codebook(CodebookArgs a);
__global__ void k2s_emit(CodebookArgs a);

// segment encoder (codes <= 26 bits): per-CTA ranges of segments
struct SegArgs {
  uint64_t n;
  const unsigned long long *ctab;  // [A] (code << 8) | len
  const uint8_t *len8;             // [A] lengths
  uint32_t lo, span;               // live symbol range (len8 window)
  uint32_t win_lo, win_n;          // (code, len) window for the pack pass
  uint64_t spc;                    // segments per count CTA
  uint32_t *seg_bits, *seg_nz;     // [nseg]
  uint8_t *seg_long;               // [nseg] segment holds a code longer than K3_SHORT_MAXLEN
  unsigned long long *cta_bits, *cta_nz;  // [ncta] totals, then exclusive prefixes (in place)
  uint32_t ncta;
  unsigned *ticket;                // count CTAs done (zero before the launch; the last CTA resets it)
  const float *x;
  uint32_t *payload;
  unsigned long long *out_idx;
  float *out_val;
  unsigned long long *chunk_off;
  int extract;
  // device-planned launch (actc_compress_async): when dplan is set the kernels
  // take the live range / window from the device plan, skip everything when
  // the stream does not fit the caps (the host redoes it synchronously), the
  // count pass zeroes the payload and the scan copies the canonical table
  const actc_plan_t *dplan;
  uint64_t k;  // outlier count (from the plan); 0 skips the marker scan
  uint32_t radius;
  uint64_t cap_bits, k_cap;
  const uint32_t *canon_src, *lencnt_src;
  uint32_t *canon_out, *lencnt_out;
  EmitArgs emit;  // deferred k2s emission (rank_tab null: none)
  void *table;    // decode table built by the first pack CTAs (null: none)
  actc_plan_t *plan_host;  // mapped pinned plan mailbox the pack's last CTA fills (null: none)
  unsigned *pack_ticket;   // pack CTAs done (zero, reset by the last)
  int sw16;       // 16-bit symbols
};
// resolve a device-planned SegArgs; false = this stream takes the host path
__device__ __forceinline__ bool seg_resolve(SegArgs &a) {
  if (!a.dplan) return true;
  const actc_plan_t &p = *a.dplan;
  if (p.status != ACTC_OK || p.max_len > 56u || p.payload_bits > a.cap_bits ||
      p.n_outliers > a.k_cap)
    return false;
  const uint32_t lo = p.sym_lo, hi = p.sym_hi;
  const uint32_t span = hi >= lo ? hi - lo + 1 : 1;
  a.k = p.n_outliers;
  a.lo = lo;
  a.span = span;
  a.win_lo = lo;
  a.win_n = min(span, K3L_WIN);
  if (span > K3L_WIN) {
    const uint32_t centre = a.radius ? a.radius : (lo + hi) / 2;
    uint32_t wl = centre > K3L_WIN / 2 ? centre - K3L_WIN / 2 : 0;
    if (wl < lo) wl = lo;
    if (wl + K3L_WIN > hi + 1) wl = hi + 1 - K3L_WIN;
    a.win_lo = wl;
  }
  return true;
}
template <typename SymT>
__global__ void k3_seg_count(const SymT *__restrict__ sym, SegArgs a);
template <typename SymT>
__global__ void k3_seg_pack(const SymT *__restrict__ sym, SegArgs a);

// mode bit0: short-code entries carry the canonical index instead of the
// symbol; bit1: long prefixes with a single code length get "exact" entries
// (length field 63, length above it)
__global__ void k_build_lut(const uint32_t *__restrict__ canon, const uint32_t *__restrict__ len_counts,
                            uint32_t *__restrict__ lut, int mode);

// decoder LUT: kLutSize entries + a header word (bit0: fast long-code path
// valid, i.e. prefix-free code with max length <= 32)
constexpr int kLutWords = kLutSize + 4;

struct DecodeArgs {
  uint64_t n;
  double eb, two_eb;
  uint32_t radius;
  int preserve;
  uint64_t k;
  const unsigned long long *out_idx;
  const float *out_val;
  const uint32_t *canon;
  const uint32_t *len_counts;
  const uint32_t *lut;
  const uint32_t *payload;
  uint64_t payload_bits;
  const unsigned long long *chunk_off;
  const long long *chunk_lat;  // lattice value before every chunk (warp decoder)
  uint32_t live;               // number of codes (canon length)
  void *out;  // f32 / f64 values or u32 symbols
  DecStatus st;
  unsigned *ticket;
  uint64_t ntiles;
  unsigned long long *nonzero;
  unsigned long long *markers;
  unsigned *status;
  unsigned long long *mcount;  // K4L: markers of this launch (null: no stored outliers), self-resetting
  uint32_t cd_lim;             // K4L wide alphabets: leading canonical indices whose deltas are in shared memory
};
// a decode fault: the call's status word and, right after it, the context's
// sticky word (collected by actc_ctx_take_status at the caller's next sync --
// decoders launched without a result mailbox are checked that way)
__device__ __forceinline__ void report_format_error(const DecodeArgs &a) {
  atomicOr(a.status, (unsigned)ACTC_EFORMAT);
  atomicOr(a.status + 1, (unsigned)ACTC_EFORMAT);
}

// MODE: 0 = fp32 recon, 1 = fp64 recon, 2 = raw u32 symbols
// SW: staging width of decoded symbols in shared memory (16 or 32 bits)
template <int MODE, int SW>
__global__ void k4_decode(DecodeArgs a);
// K4L decode table (ACTC_TABLE_BYTES): T1[p] (4 bytes) for every 12-bit
// prefix p of the left-aligned 32-bit window, then two header words.
// Entry: bits 0-4 the code length len (0: slow path), bits 16-31 the payload:
//  * every code under p of one length len <= 31, canonical indices < 2^16:
//    payload = (base[len] - first[len]) mod 2^16 -- the canonical index of
//    the code under W is (payload + (W >> (32 - len))) mod 2^16;
//  * otherwise len 0 and payload l0, the shortest length a code under p can
//    have (0: no code, or an over-subscribed table, whose first-match rule
//    the scan from length 1 reproduces; 33: past every code of <= 32 bits).
// Header: word kLutSize = 1 if the code table is prefix-free (Kraft <= 1),
// word kLutSize + 1 = the longest code length.
constexpr size_t kK4lTableBytes = (size_t)kLutSize * 4 + 16;
static_assert(kK4lTableBytes == ACTC_TABLE_BYTES, "include/actc.h ACTC_TABLE_BYTES");
__global__ void k4l_build_table(const uint32_t *__restrict__ len_counts, const uint32_t *__restrict__ canon,
                                uint32_t radius, uint32_t *__restrict__ table);
// MODE: 0 = fp32 recon, 1 = fp64 recon, 2 = raw u32 symbols;
// GCANON: canonical symbols read from global memory (wide alphabets);
// NZ: count the nonzero reconstructed values (R, training.py:351-352).
// tm: the output as a 2-D tensor [n / ACTC_CHUNK rows][ACTC_CHUNK values],
// box 32 rows x 64 B, 64-B swizzle (TMA stores of full tiles).
template <int MODE, bool GCANON, bool NZ>
__global__ void k4l_decode(DecodeArgs a, const __grid_constant__ CUtensorMap tm);
size_t k4l_smem_bytes(uint32_t cd_entries, int warps);
int k4l_max_warps(uint32_t cd_entries, size_t dyn_max);
__global__ void k_excl_scan_u64(const unsigned long long *__restrict__ in, uint64_t m,
                                unsigned long long *__restrict__ out, unsigned long long *__restrict__ total);

__global__ void k_lorenzo_decode_seq(const uint32_t *__restrict__ sym, uint64_t n,
                                     const long long *__restrict__ olat, uint64_t k,
                                     uint32_t radius, long long *__restrict__ out,
                                     unsigned *__restrict__ status);

// index rebuild for streams without chunk offsets
__global__ void k_sync_pass(const uint32_t *__restrict__ payload, uint64_t payload_bits,
                            const uint32_t *__restrict__ lut, const uint32_t *__restrict__ len_counts,
                            uint64_t seg_bits, uint64_t nseg, unsigned long long *__restrict__ start,
                            unsigned long long *__restrict__ end_pos,
                            unsigned long long *__restrict__ count, unsigned *__restrict__ changed,
                            unsigned *__restrict__ status, int first);
__global__ void k_index_emit(const uint32_t *__restrict__ payload, uint64_t payload_bits,
                             const uint32_t *__restrict__ lut, const uint32_t *__restrict__ len_counts,
                             uint64_t seg_bits, uint64_t nseg,
                             const unsigned long long *__restrict__ start,
                             const unsigned long long *__restrict__ sym_base, uint64_t n,
                             unsigned long long *__restrict__ chunk_off);

// statistics
__global__ void k_count_nonzero(const void *__restrict__ x, int dtype, uint64_t n,
                                unsigned long long *__restrict__ out);
__global__ void k_pairwise_partials(const void *__restrict__ x, int dtype, uint64_t n, int depth,
                                    double *__restrict__ partial);
__global__ void k_pairwise_finish(const double *__restrict__ partial, int dtype, uint64_t n,
                                  int depth, double *__restrict__ out);
__global__ void k_sample_max(const void *__restrict__ g, int dtype, uint64_t N, uint64_t per,
                             unsigned long long *__restrict__ bits);
__global__ void k_lbar_finish(const unsigned long long *__restrict__ bits, int dtype, uint64_t N,
                              void *__restrict__ per_sample_max, double *__restrict__ out);

// K6 CRC-32 (k6_crc.cu)
uint64_t crc32_blocks(uint64_t len);
int crc32_launch(const uint8_t *data, uint64_t len, uint32_t crc_in, uint32_t *part, unsigned *ticket,
                 uint32_t *out_dev, cudaStream_t s);

// canonical code tables from the per-length counts (huffman.py:97-117)
struct CodeTables {
  unsigned long long first[64];
  unsigned long long lim[64];  // (first + count) << (32 - l), l <= 32 (left-aligned limit)
  uint32_t count[64];
  uint32_t base[64];
  uint32_t maxlen;
};

// the 64 per-length code counts into shared memory by the first two warps
// (parallel loads: a serial per-length loop by one thread would wait on 64
// dependent-latency global loads); callers __syncthreads() before use
__device__ __forceinline__ void stage_len_counts(uint32_t *dst, const uint32_t *__restrict__ len_counts) {
  if (threadIdx.x < 64) dst[threadIdx.x] = __ldg(len_counts + threadIdx.x);
}

__device__ __forceinline__ void build_tables(CodeTables &t, const uint32_t *len_counts) {
  __shared__ uint32_t s_cnt[64];
  stage_len_counts(s_cnt, len_counts);
  __syncthreads();
  len_counts = s_cnt;
  if (threadIdx.x == 0) {
    unsigned long long code = 0;
    uint32_t idx = 0, mx = 0;
    for (int l = 0; l < 64; l++) {
      code <<= 1;
      uint32_t c = len_counts[l];
      t.first[l] = code;
      t.count[l] = c;
      t.base[l] = idx;
      t.lim[l] = l <= 32 ? (code + c) << (32 - l) : 0;
      code += c;
      idx += c;
      if (c && l > 0) mx = l;
    }
    t.maxlen = mx;
  }
}

// LUT entry for every 12-bit prefix: (symbol << 6) | length for a code of
// length <= 12 (same first-match rule as the reference's bit loop); for a
// prefix of longer codes, (l0 << 6) with l0 the first length whose
// left-aligned limit exceeds the prefix (decoding continues from l0 on the
// register window); 0 if no code starts with the prefix.  lut[kLutSize]
// holds the fast-path flag: 1 if the code is prefix-free (Kraft <= 1) and
// max length <= 32.
__device__ __forceinline__ void lut32_body(const uint32_t *__restrict__ canon, const uint32_t *__restrict__ len_counts,
                                           uint32_t *__restrict__ lut, int mode, uint32_t blk) {
  __shared__ CodeTables t;
  __shared__ unsigned s_ok;
  build_tables(t, len_counts);
  __syncthreads();
  const int ci_mode = mode & 1;
  uint32_t p = blk * blockDim.x + threadIdx.x;
  if (threadIdx.x == 0) {
    // Kraft sum in units of 2^-63
    unsigned long long k = 0;
    bool over = false;
    for (int l = 1; l < 64 && !over; l++) {
      unsigned long long add = (unsigned long long)t.count[l] << (63 - l);
      if (t.count[l] >> l) over = true;  // count >= 2^l alone exceeds the budget
      if (k + add < k) over = true;
      k += add;
      if (k > (1ull << 63)) over = true;
    }
    s_ok = (!over && t.maxlen <= 32) ? 1u : 0u;
    if (p == 0) lut[kLutSize] = s_ok;
  }
  __syncthreads();
  if (p >= (uint32_t)kLutSize) return;
  uint32_t e = 0;
  int lim = t.maxlen < (uint32_t)kLutBits ? (int)t.maxlen : kLutBits;
  for (int l = 1; l <= lim; l++) {
    unsigned long long code = p >> (kLutBits - l);
    unsigned long long off = code - t.first[l];
    if (off < t.count[l]) {
      e = ((ci_mode ? (uint32_t)(t.base[l] + off) : canon[t.base[l] + off]) << 6) | (uint32_t)l;
      break;
    }
  }
  if (!e && t.maxlen > (uint32_t)kLutBits && t.maxlen <= 32) {
    const unsigned long long w = (unsigned long long)p << (32 - kLutBits);
    const unsigned long long w1 = w | ((1ull << (32 - kLutBits)) - 1);
    int l0 = 0, l1 = 0;
    for (int l = kLutBits + 1; l <= (int)t.maxlen; l++) {
      unsigned long long limit = (t.first[l] + t.count[l]) << (32 - l);
      if (!l0 && limit > w) l0 = l;
      if (!l1 && limit > w1) l1 = l;
    }
    if (l0) e = (uint32_t)l0 << 6;
    // mode bit1: every code behind the prefix has the same length -> "exact
    // long" entry (length field 63): the decoder skips the limit probes
    if ((mode & 2) && s_ok && l0 && l1 == l0) e |= 63u;
  }
  lut[p] = e;
}

// decode table rows [blk*blockDim, (blk+1)*blockDim) (layout above)
__device__ __forceinline__ void k4l_table_rows(const uint32_t *__restrict__ len_counts, const uint32_t *__restrict__ canon,
                                               uint32_t radius, uint32_t *__restrict__ table, uint32_t blk) {
  __shared__ unsigned long long s_first[33], s_lim[33];
  __shared__ uint32_t s_base[33], s_cnt[64];
  __shared__ unsigned s_ok, s_max;
  stage_len_counts(s_cnt, len_counts);
  __syncthreads();
  len_counts = s_cnt;
  if (threadIdx.x == 0) {
    unsigned long long code = 0, kraft = 0;
    uint32_t idx = 0, mx = 0;
    bool over = false;
    for (int l = 0; l < 64; l++) {
      code <<= 1;
      const uint32_t c = len_counts[l];
      if (l <= 32) {
        s_first[l] = code;
        s_lim[l] = (code + c) << (32 - l);
        s_base[l] = idx;
      }
      if (l >= 1) {
        // Kraft sum in units of 2^-63: an over-subscribed table has no
        // canonical order (the reference's first-match rule decides)
        const unsigned long long add = (unsigned long long)c << (63 - l);
        if ((unsigned long long)c >> l) over = true;
        if (kraft + add < kraft) over = true;
        kraft += add;
        if (kraft > (1ull << 63)) over = true;
      }
      code += c;
      idx += c;
      if (c && l > 0) mx = l;
    }
    s_ok = over ? 0u : 1u;
    s_max = mx;
  }
  __syncthreads();
  const uint32_t p = blk * blockDim.x + threadIdx.x;
  if (p >= (uint32_t)kLutSize) return;
  uint32_t e = 0;
  if (s_ok) {
    const unsigned long long w0 = (unsigned long long)p << (32 - kLutBits);
    const unsigned long long w1 = w0 | ((1ull << (32 - kLutBits)) - 1);
    const int top = s_max < 32u ? (int)s_max : 32;
    int l0 = 0, l1 = 0;
    for (int l = 1; l <= top; l++) {
      if (!l0 && s_lim[l] > w0) l0 = l;
      if (!l1 && s_lim[l] > w1) l1 = l;
    }
    bool done = false;
    if (l0 && l0 == l1 && l0 <= 31) {
      // every code under p has length l0: canonical indices up to ci1
      const uint32_t ci1 = s_base[l0] + (uint32_t)((w1 >> (32 - l0)) - s_first[l0]);
      if (ci1 < 65536u) {
        e = ((s_base[l0] - (uint32_t)s_first[l0]) << 16) | (uint32_t)l0;
        done = true;
      }
    }
    if (!done) {
      if (l0) e = (uint32_t)l0 << 16;  // mixed lengths, 32-bit codes, wide index: the scan starts at l0
      else if (s_max > 32) e = 33u << 16;  // past every code of <= 32 bits: longer codes only
    }
  }
  table[p] = e;
  if (p == 0) {
    table[kLutSize] = s_ok;
    table[kLutSize + 1] = s_max;
  }
}

// decode table rows [256*b, 256*b + 256) of a stream compressed by the
// async chain (the pack kernel's first CTAs run it): the K4L table
__device__ __forceinline__ void table_rows_plan(const uint32_t *canon, const uint32_t *len_counts, uint32_t radius,
                                                void *table, uint32_t blk) {
  k4l_table_rows(len_counts, canon, radius, (uint32_t *)table, blk);
}

// K7 uniform error injection (k7_inject.cu); state = {st_hi, st_lo, inc_hi, inc_lo}
int inject_launch(const void *x, int dtype, uint64_t n, double eb, int preserve, const uint64_t state[4],
                  double *out, cudaStream_t s);

}  // namespace actc
