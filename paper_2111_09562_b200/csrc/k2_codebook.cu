// K2: Huffman codebook on one CTA (1024 threads).
//
// Replaces build_code_lengths (huffman.py:37-75), canonical_codes
// (huffman.py:78-94), the RLE record count of _rle_encode_lengths
// (codec.py:201-226) and stream_entropy_bits (huffman.py:239-246).
//
// Bit-exactness.  heapq pops items in (freq, tiebreak) order with leaf
// tiebreak = symbol and internal tiebreak = creation counter >= alphabet,
// i.e. the two-queue algorithm in which a leaf wins a frequency tie and an
// older internal node beats a newer one.  We run that algorithm in
// *phases*: with m the smallest remaining frequency, every item of
// frequency < 2m is popped in merged (freq, class, index) order and paired
// consecutively before any node created in the phase can be popped (new
// nodes are >= 2m); an odd leftover pairs with the smallest remaining item.
// Each phase at least doubles m, so there are <= log2(n)+1 phases, each a
// merge-path parallel merge.  Code lengths are depths, computed by walking
// the phases backwards.
//
// Sorting uses a stable block-wide LSD radix sort (8-bit digits, warp
// match_any ranking), so (freq, symbol) order comes from stability.  Arrays
// live in shared memory when the live alphabet is small, else in global
// scratch (L2-resident).
#include "kernels.cuh"

namespace actc {

namespace {

constexpr int NWARP = K2_THREADS / 32;
constexpr uint32_t kSmemL = 4096;
constexpr int kMaxPhases = 128;
constexpr uint32_t kWin = 22528;  // merged positions per staged window (180 KB of u64)

struct RadixSmem {
  uint32_t hist[NWARP][257];
  uint32_t tot[256];
};

// One stable LSD pass on digit (key >> shift) & 0xFF, src -> dst.
__device__ void radix_pass(const unsigned long long *__restrict__ sk, const uint32_t *__restrict__ sv,
                           unsigned long long *__restrict__ dk, uint32_t *__restrict__ dv, uint32_t L,
                           int shift, RadixSmem &rs) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t seg = ((L + NWARP - 1) / NWARP + 127) & ~127u;  // multiple of the 4x32 batch
  const uint32_t b0 = min(L, w * seg), b1 = min(L, b0 + seg);
  for (int d = lane; d < 257; d += 32) rs.hist[w][d] = 0;
  __syncwarp();
  for (uint32_t base = b0; base < b1; base += 128) {
    // four independent loads in flight per lane
    uint32_t d[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const uint32_t i = base + 32 * u + lane;
      d[u] = i < b1 ? (uint32_t)((sk[i] >> shift) & 0xFF) : 256u;
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      unsigned peers = __match_any_sync(0xffffffffu, d[u]);
      if (lane == __ffs(peers) - 1) rs.hist[w][d[u]] += __popc(peers);
      __syncwarp();
    }
  }
  __syncthreads();
  // per digit: exclusive prefix over warps, totals
  if (threadIdx.x < 256) {
    const int d = threadIdx.x;
    uint32_t run = 0;
    for (int ww = 0; ww < NWARP; ww++) {
      uint32_t c = rs.hist[ww][d];
      rs.hist[ww][d] = run;
      run += c;
    }
    rs.tot[d] = run;
  }
  __syncthreads();
  if (w == 0) {
    // exclusive scan of 256 digit totals (8 per lane)
    uint32_t v[8], s = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      v[k] = rs.tot[lane * 8 + k];
      s += v[k];
    }
    uint32_t inc = warp_incl_sum(s);
    uint32_t run = inc - s;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      rs.tot[lane * 8 + k] = run;
      run += v[k];
    }
  }
  __syncthreads();
  for (int d = lane; d < 256; d += 32) rs.hist[w][d] += rs.tot[d];
  __syncwarp();
  for (uint32_t base = b0; base < b1; base += 128) {
    unsigned long long kk[4];
    uint32_t vv[4], dd[4];
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const uint32_t i = base + 32 * u + lane;
      kk[u] = 0;
      vv[u] = 0;
      dd[u] = 256u;
      if (i < b1) {
        kk[u] = sk[i];
        vv[u] = sv[i];
        dd[u] = (uint32_t)((kk[u] >> shift) & 0xFF);
      }
    }
#pragma unroll
    for (int u = 0; u < 4; u++) {
      const uint32_t dg = dd[u];
      unsigned peers = __match_any_sync(0xffffffffu, dg);
      unsigned lower = peers & ((1u << lane) - 1u);
      if (dg < 256) {
        uint32_t pos = rs.hist[w][dg] + __popc(lower);
        dk[pos] = kk[u];
        dv[pos] = vv[u];
      }
      __syncwarp();
      if (dg < 256 && lane == __ffs(peers) - 1) rs.hist[w][dg] += __popc(peers);
      __syncwarp();
    }
  }
  __syncthreads();
}

// Stable LSD pass on keys only (digit (key >> shift) & 0xFF), src -> dst,
// with 16 loads in flight per lane: a warp walks its segment in batches of
// 512 keys (lane owns every 32nd), so one L2 round trip covers 512 keys.
constexpr int KB = 16;
__device__ void radix_pass_keys(const unsigned long long *__restrict__ sk, unsigned long long *__restrict__ dk,
                                uint32_t L, int shift, RadixSmem &rs) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t seg = ((L + NWARP - 1) / NWARP + 32 * KB - 1) & ~uint32_t(32 * KB - 1);
  const uint32_t b0 = min(L, w * seg), b1 = min(L, b0 + seg);
  for (int d = lane; d < 257; d += 32) rs.hist[w][d] = 0;
  __syncwarp();
  for (uint32_t base = b0; base < b1; base += 32 * KB) {
    uint32_t d[KB];
#pragma unroll
    for (int u = 0; u < KB; u++) {
      const uint32_t i = base + 32 * u + lane;
      d[u] = i < b1 ? (uint32_t)((sk[i] >> shift) & 0xFF) : 256u;
    }
#pragma unroll
    for (int u = 0; u < KB; u++) {
      const unsigned peers = __match_any_sync(0xffffffffu, d[u]);
      if (lane == __ffs(peers) - 1) rs.hist[w][d[u]] += __popc(peers);
      __syncwarp();
    }
  }
  __syncthreads();
  if (threadIdx.x < 256) {
    const int d = threadIdx.x;
    uint32_t run = 0;
    for (int ww = 0; ww < NWARP; ww++) {
      const uint32_t c = rs.hist[ww][d];
      rs.hist[ww][d] = run;
      run += c;
    }
    rs.tot[d] = run;
  }
  __syncthreads();
  if (w == 0) {
    uint32_t v[8], t = 0;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      v[k] = rs.tot[lane * 8 + k];
      t += v[k];
    }
    const uint32_t inc = warp_incl_sum(t);
    uint32_t run = inc - t;
#pragma unroll
    for (int k = 0; k < 8; k++) {
      rs.tot[lane * 8 + k] = run;
      run += v[k];
    }
  }
  __syncthreads();
  for (int d = lane; d < 256; d += 32) rs.hist[w][d] += rs.tot[d];
  __syncwarp();
  for (uint32_t base = b0; base < b1; base += 32 * (KB / 2)) {
    unsigned long long kk[KB / 2];
#pragma unroll
    for (int u = 0; u < KB / 2; u++) {
      const uint32_t i = base + 32 * u + lane;
      kk[u] = i < b1 ? sk[i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < KB / 2; u++) {
      const uint32_t i = base + 32 * u + lane;
      const uint32_t dg = i < b1 ? (uint32_t)((kk[u] >> shift) & 0xFF) : 256u;
      const unsigned peers = __match_any_sync(0xffffffffu, dg);
      if (dg < 256) dk[rs.hist[w][dg] + __popc(peers & ((1u << lane) - 1u))] = kk[u];
      __syncwarp();
      if (dg < 256 && lane == __ffs(peers) - 1) rs.hist[w][dg] += __popc(peers);
      __syncwarp();
    }
  }
  __syncthreads();
}

// first index in sorted v[lo, hi) with v[i] >= T (block-wide, all threads
// get the result).  1024-way probing, repeated on the bracketing interval.
__device__ uint32_t block_lower_bound(const unsigned long long *v, uint32_t lo, uint32_t hi,
                                      unsigned long long T) {
  while (hi > lo) {
    uint32_t len = hi - lo;
    uint32_t step = (len + K2_THREADS - 1) / K2_THREADS;
    uint32_t idx = lo + threadIdx.x * step;
    bool below = idx < hi && v[idx] < T;
    uint32_t k = (uint32_t)__syncthreads_count(below);  // probes < T form a prefix
    if (step == 1) return lo + k;
    if (k == 0) return lo;
    uint32_t nlo = lo + (k - 1) * step + 1;  // probe k-1 is < T
    uint32_t nhi = min(hi, lo + k * step);
    lo = nlo;
    hi = nhi;
  }
  return lo;
}

// Both lower bounds of a phase at once: threads [0, 512) probe v1[lo1, hi1),
// threads [512, 1024) probe v2[lo2, hi2) -- one memory round trip per
// refinement step for the pair.  Results: first index with v >= T.
__device__ void block_lower_bound2(const unsigned long long *v1, uint32_t lo1, uint32_t hi1,
                                   const unsigned long long *v2, uint32_t lo2, uint32_t hi2,
                                   unsigned long long T, uint32_t &r1, uint32_t &r2) {
  constexpr uint32_t H = K2_THREADS / 2;
  const bool second = threadIdx.x >= H;
  const uint32_t t = threadIdx.x & (H - 1);
  bool d1 = hi1 <= lo1, d2 = hi2 <= lo2;
  r1 = lo1;
  r2 = lo2;
  while (!(d1 && d2)) {
    const uint32_t s1 = d1 ? 1 : (hi1 - lo1 + H - 1) / H, s2 = d2 ? 1 : (hi2 - lo2 + H - 1) / H;
    bool below = false;
    if (!second && !d1) {
      const uint32_t idx = lo1 + t * s1;
      below = idx < hi1 && v1[idx] < T;
    } else if (second && !d2) {
      const uint32_t idx = lo2 + t * s2;
      below = idx < hi2 && v2[idx] < T;
    }
    const uint32_t k1 = (uint32_t)__syncthreads_count(below && !second);
    const uint32_t k2 = (uint32_t)__syncthreads_count(below && second);
    if (!d1) {
      if (s1 == 1 || k1 == 0) {
        r1 = lo1 + (s1 == 1 ? k1 : 0);
        d1 = true;
      } else {
        const uint32_t nlo = lo1 + (k1 - 1) * s1 + 1, nhi = min(hi1, lo1 + k1 * s1);
        lo1 = nlo;
        hi1 = nhi;
        if (hi1 <= lo1) {
          r1 = lo1;
          d1 = true;
        }
      }
    }
    if (!d2) {
      if (s2 == 1 || k2 == 0) {
        r2 = lo2 + (s2 == 1 ? k2 : 0);
        d2 = true;
      } else {
        const uint32_t nlo = lo2 + (k2 - 1) * s2 + 1, nhi = min(hi2, lo2 + k2 * s2);
        lo2 = nlo;
        hi2 = nhi;
        if (hi2 <= lo2) {
          r2 = lo2;
          d2 = true;
        }
      }
    }
  }
}

// number of leaves among the first d merged items of (leaves lf[0,na),
// internals nf[0,nb)), leaf wins ties -- block-wide 1024-way probing
__device__ uint32_t merge_split_block(const unsigned long long *lf, const unsigned long long *nf, uint32_t na,
                                      uint32_t nb, uint32_t d) {
  uint32_t lo = d > nb ? d - nb : 0, hi = min(d, na);  // answer in [lo, hi]
  while (lo < hi) {
    const uint32_t len = hi - lo;
    const uint32_t step = (len + K2_THREADS - 1) / K2_THREADS;
    // candidate i = lo + 1 + t*step: predicate "leaf i-1 precedes internal d-i"
    const uint32_t i = lo + 1 + threadIdx.x * step;
    bool p = false;
    if (i <= hi) {
      const uint32_t j = d - i;
      p = j >= nb || lf[i - 1] <= nf[j];
    }
    const uint32_t k = (uint32_t)__syncthreads_count(p);  // true probes form a prefix
    if (step == 1) return lo + k;
    // answer in [c_{k-1}, c_k - 1] with c_t = lo + 1 + t*step, c_{-1} = lo
    const uint32_t nlo = k ? lo + 1 + (k - 1) * step : lo;
    const uint32_t nhi = min(hi, lo + k * step);
    lo = nlo;
    hi = nhi;
  }
  return lo;
}

// Sequentially merge merged positions [d0, d1) of (a[0,na), b[0,nb)) (leaf
// wins ties), creating pair nodes nn + p/2 for p < 2*pairs (positions are
// relative to the window) and recording the odd leftover.
__device__ __forceinline__ void merge_range(const unsigned long long *a, const unsigned long long *b, uint32_t na,
                                            uint32_t nb, uint32_t d0, uint32_t d1, uint32_t abase, uint32_t bbase,
                                            uint32_t nn, uint32_t pairs, uint32_t *lpar, uint32_t *npar,
                                            unsigned long long *nf, uint32_t &odd_item) {
  uint32_t lo = d0 > nb ? d0 - nb : 0, hi = min(d0, na);
  while (lo < hi) {
    const uint32_t mid = (lo + hi + 1) >> 1;
    const uint32_t j = d0 - mid;
    if (j >= nb || a[mid - 1] <= b[j])
      lo = mid;
    else
      hi = mid - 1;
  }
  uint32_t i = lo, j = d0 - lo;
  unsigned long long fprev = 0;
  for (uint32_t p = d0; p < d1; p++) {
    const bool leaf = j >= nb || (i < na && a[i] <= b[j]);
    unsigned long long f;
    uint32_t item;
    if (leaf) {
      f = a[i];
      item = abase + i;
      i++;
    } else {
      f = b[j];
      item = 0x80000000u | (bbase + j);
      j++;
    }
    if (p < 2 * pairs) {
      const uint32_t node = nn + (p >> 1);
      if (item & 0x80000000u) npar[item & 0x7FFFFFFFu] = node; else lpar[item] = node;
      if (p & 1) nf[node] = fprev + f;
      fprev = f;
    } else {
      odd_item = item;  // the single leftover (tot odd)
    }
  }
}

}  // namespace

__global__ void __launch_bounds__(K2_THREADS) k2_codebook(CodebookArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ RadixSmem rs;
  __shared__ unsigned long long wbuf[33];
  __shared__ unsigned long long wbuf2[33];
  __shared__ uint32_t s_lp, s_np, s_nn, s_nph;
  __shared__ uint32_t ph_begin[kMaxPhases], ph_pairs[kMaxPhases];
  __shared__ uint8_t ph_odd[kMaxPhases];
  __shared__ uint32_t s_cnt[64];
  __shared__ unsigned long long s_first[64];
  __shared__ uint32_t s_base[64];
  __shared__ unsigned s_err, s_maxlen;
  __shared__ unsigned long long s_maxf;
  __shared__ uint32_t s_odd_item;
  __shared__ double dbuf[33];

  if (a.gate && *a.gate == 0u) return;  // k2r produced the codebook
  const int tid = threadIdx.x;
  const uint64_t A = a.A;
#define K2_STAMP(i) \
  if (a.dbg && tid == 0) a.dbg[i] = clock64();
  K2_STAMP(0)

  if (tid == 0) {
    s_err = 0;
    s_maxlen = 0;
    s_maxf = 0;
  }
  if (tid < 64) s_cnt[tid] = 0;
  __syncthreads();

  // ---- 1. compact live symbols (symbol order) ----
  // warp w owns a contiguous segment of bins, read coalesced 8 rounds at a
  // time (all loads in flight); ballot + popc ranks live bins inside a
  // round.  Pass 1 counts, one scan over the 32 warp counts, pass 2 writes.
  uint64_t L = 0;
  unsigned long long maxf = 0;
  {
    const int lane = tid & 31, w = tid >> 5;
    const uint64_t per_w = (((A + NWARP - 1) / NWARP) + 255) & ~uint64_t(255);
    const uint64_t wb0 = min(A, (uint64_t)w * per_w), wb1 = min(A, wb0 + per_w);
    const unsigned lt = (1u << lane) - 1u;
    unsigned cnt = 0;
    for (uint64_t base = wb0; base < wb1; base += 256) {
      unsigned long long v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const uint64_t sidx = base + 32 * u + lane;
        v[u] = sidx < wb1 ? (a.in_lengths ? (unsigned long long)a.in_lengths[sidx] : a.hist[sidx]) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 8; u++) {
        cnt += __popc(__ballot_sync(0xffffffffu, v[u] != 0));
        maxf = v[u] > maxf ? v[u] : maxf;
      }
    }
    __shared__ unsigned s_wcnt[NWARP + 1];
    if (lane == 0) s_wcnt[w] = cnt;
    __syncthreads();
    if (w == 0) {
      const unsigned c = s_wcnt[lane];
      const unsigned inc = warp_incl_sum(c);
      s_wcnt[lane] = inc - c;
      if (lane == 31) s_wcnt[NWARP] = inc;
    }
    __syncthreads();
    unsigned long long off = s_wcnt[w];
    L = s_wcnt[NWARP];
    for (uint64_t base = wb0; base < wb1 && cnt; base += 256) {
      unsigned long long v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const uint64_t sidx = base + 32 * u + lane;
        v[u] = sidx < wb1 ? (a.in_lengths ? (unsigned long long)a.in_lengths[sidx] : a.hist[sidx]) : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const unsigned m = __ballot_sync(0xffffffffu, v[u] != 0);
        if (v[u]) {
          const unsigned long long pos = off + __popc(m & lt);
          a.live_sym[pos] = (uint32_t)(base + 32 * u + lane);
          a.live_freq[pos] = v[u];
        }
        off += __popc(m);
      }
    }
  }
  atomicMax(&s_maxf, maxf);
  __syncthreads();
  maxf = s_maxf;
  K2_STAMP(1)

  // generic pointers: shared memory for small L, global scratch otherwise
  unsigned long long *k0 = a.keys, *k1 = a.keys2, *nf = a.nf;
  uint32_t *v0 = a.vals, *v1 = a.vals2, *lpar = a.lpar, *npar = a.npar;
  uint32_t *ndepth = (uint32_t *)a.ndepth;
  uint8_t *llen = a.llen;
  const bool big = L > kSmemL;
  if (!big) {
    unsigned char *p = smem;
    k0 = (unsigned long long *)p; p += 8 * (size_t)kSmemL;
    k1 = (unsigned long long *)p; p += 8 * (size_t)kSmemL;
    nf = (unsigned long long *)p; p += 8 * (size_t)kSmemL;
    v0 = (uint32_t *)p; p += 4 * (size_t)kSmemL;
    v1 = (uint32_t *)p; p += 4 * (size_t)kSmemL;
    lpar = (uint32_t *)p; p += 4 * (size_t)kSmemL;
    npar = (uint32_t *)p; p += 4 * (size_t)kSmemL;
    ndepth = (uint32_t *)p; p += 4 * (size_t)kSmemL;
    llen = (uint8_t *)p;
  }

  if (a.in_lengths) {
    for (uint32_t j = tid; j < L; j += K2_THREADS) {
      unsigned l = (unsigned)a.live_freq[j];
      if (l > ACTC_MAX_CODE_LENGTH) atomicOr(&s_err, 1u);
      llen[j] = (uint8_t)(l > 255 ? 255 : l);
    }
  } else if (L == 1) {
    if (tid == 0) llen[0] = 1;  // huffman.py:50-52
  } else if (L > 1) {
    // ---- 2. sort leaves by (freq, symbol): stable radix on freq ----
    int passes = 0;
    while (passes < 8 && (maxf >> (8 * passes)) != 0) passes++;
    if (big && (maxf >> 38) == 0) {
      // packed keys (freq << 26 | live index), unique, sorted on the freq
      // digits only (stability keeps the index order); then split
#pragma unroll 8
      for (uint32_t i = tid; i < L; i += K2_THREADS) k0[i] = (a.live_freq[i] << kSymKeyBits) | i;
      __syncthreads();
      K2_STAMP(10)
      for (int p = 0; p < passes; p++) {
        radix_pass_keys(k0, k1, (uint32_t)L, kSymKeyBits + 8 * p, rs);
        unsigned long long *tk = k0; k0 = k1; k1 = tk;
        if (p < 3) { K2_STAMP(11 + p) }
      }
#pragma unroll 8
      for (uint32_t i = tid; i < L; i += K2_THREADS) {
        const unsigned long long key = k0[i];
        k0[i] = key >> kSymKeyBits;
        v0[i] = (uint32_t)(key & (kMaxAlphabet - 1));
      }
      __syncthreads();
    } else {
      for (uint32_t i = tid; i < L; i += K2_THREADS) {
        k0[i] = a.live_freq[i];
        v0[i] = i;
      }
      __syncthreads();
      for (int p = 0; p < passes; p++) {
        radix_pass(k0, v0, k1, v1, (uint32_t)L, 8 * p, rs);
        unsigned long long *tk = k0; k0 = k1; k1 = tk;
        uint32_t *tv = v0; v0 = v1; v1 = tv;
      }
    }
    // sorted leaf i: freq k0[i], live index v0[i]
    const unsigned long long *lf = k0;
    K2_STAMP(2)

    // ---- 3. phase-parallel two-queue merge ----
    if (tid == 0) {
      s_lp = 0; s_np = 0; s_nn = 0; s_nph = 0;
    }
    __syncthreads();
    const unsigned long long INF = ~0ull;
    unsigned long long t_lb = 0, t_merge = 0, t_book = 0, t_c0 = 0;
    while (true) {
      if (a.dbg && tid == 0) t_c0 = clock64();
      const uint32_t lp = s_lp, np = s_np, nn = s_nn;
      if ((L - lp) + (nn - np) <= 1) break;
      unsigned long long m = INF;
      if (lp < L) m = lf[lp];
      if (np < nn && nf[np] < m) m = nf[np];
      const unsigned long long T = 2 * m;
      uint32_t ea, eb2;
      block_lower_bound2(lf, lp, (uint32_t)L, nf, np, nn, T, ea, eb2);
      const uint32_t na = ea - lp, nb = eb2 - np;
      if (a.dbg && tid == 0) { const unsigned long long c = clock64(); t_lb += c - t_c0; t_c0 = c; }
      const uint32_t tot = na + nb, pairs = tot >> 1;
      if (!big) {
        // merge path on the (shared-memory) arrays: thread t owns merged
        // positions [t*q, t*q+q), q even so pairs never straddle threads
        uint32_t q = (tot + K2_THREADS - 1) / K2_THREADS;
        q = (q + 1) & ~1u;
        const uint32_t d0 = tid * q;
        if (d0 < tot)
          merge_range(lf + lp, nf + np, na, nb, d0, min(tot, d0 + q), lp, np, nn, pairs, lpar, npar, nf, s_odd_item);
      } else {
        // global arrays: stage the phase's inputs through shared memory in
        // windows of kWin merged positions
        for (uint32_t wa = 0; wa < tot; wa += kWin) {
          const uint32_t wb = min(tot, wa + kWin);
          // a phase that fits one window needs no merge-path split
          const uint32_t ia = wa == 0 ? 0u : merge_split_block(lf + lp, nf + np, na, nb, wa);
          const uint32_t ib = wb == tot ? na : merge_split_block(lf + lp, nf + np, na, nb, wb);
          const uint32_t ja = wa - ia, jb = wb - ib;
          unsigned long long *sl = reinterpret_cast<unsigned long long *>(smem);
          unsigned long long *sn = sl + (ib - ia);
          for (uint32_t i = tid; i < ib - ia; i += K2_THREADS) sl[i] = lf[lp + ia + i];
          for (uint32_t j = tid; j < jb - ja; j += K2_THREADS) sn[j] = nf[np + ja + j];
          __syncthreads();
          const uint32_t wt = wb - wa;
          uint32_t q = (wt + K2_THREADS - 1) / K2_THREADS;
          q = (q + 1) & ~1u;  // wa is even (kWin even), so pairs stay inside a thread
          const uint32_t d0 = tid * q;
          if (d0 < wt)
            merge_range(sl, sn, ib - ia, jb - ja, d0, min(wt, d0 + q), lp + ia, np + ja, nn + wa / 2,
                        pairs > wa / 2 ? pairs - wa / 2 : 0, lpar, npar, nf, s_odd_item);
          __syncthreads();
        }
      }
      __syncthreads();
      if (a.dbg && tid == 0) { const unsigned long long c = clock64(); t_merge += c - t_c0; t_c0 = c; }
      if (tid == 0) {
        uint32_t ph = s_nph;
        ph_begin[ph] = nn;
        ph_pairs[ph] = pairs;
        ph_odd[ph] = tot & 1;
        uint32_t nlp = lp + na, nnp = np + nb, nnn = nn + pairs;
        if (tot & 1) {
          uint32_t z = s_odd_item;
          unsigned long long fz = (z & 0x80000000u) ? nf[z & 0x7FFFFFFFu] : lf[z];
          unsigned long long fl = nlp < L ? lf[nlp] : INF;
          unsigned long long fi = nnp < nnn ? nf[nnp] : INF;
          uint32_t y;
          unsigned long long fy;
          if (nlp < L && fl <= fi) {
            y = nlp; fy = fl; nlp++;
          } else {
            y = 0x80000000u | nnp; fy = fi; nnp++;
          }
          uint32_t node = nnn;
          nf[node] = fz + fy;
          if (z & 0x80000000u) npar[z & 0x7FFFFFFFu] = node; else lpar[z] = node;
          if (y & 0x80000000u) npar[y & 0x7FFFFFFFu] = node; else lpar[y] = node;
          nnn++;
        }
        s_lp = nlp; s_np = nnp; s_nn = nnn;
        s_nph = ph + 1;
        if (ph + 1 >= kMaxPhases) s_err |= 2u;  // cannot happen for n < 2^38
      }
      __syncthreads();
      if (a.dbg && tid == 0) { const unsigned long long c = clock64(); t_book += c - t_c0; t_c0 = c; }
      if (s_err & 2u) break;
    }
    if (a.dbg && tid == 0) {
      a.dbg[16] = t_lb;
      a.dbg[17] = t_merge;
      a.dbg[18] = t_book;
    }
    // ---- 4. depths, walking phases backwards ----
    // internal-node depths as bytes in shared memory (saturating at 255;
    // anything > 63 is an error anyway)
    K2_STAMP(3)
    if (a.dbg && tid == 0) a.dbg[8] = s_nph;
    const uint32_t nn = s_nn, root = nn - 1, nph = s_nph;
    uint8_t *dep = big ? reinterpret_cast<uint8_t *>(smem) : reinterpret_cast<uint8_t *>(ndepth);
    __syncthreads();
    if (tid == 0) dep[root] = 0;
    __syncthreads();
    for (int ph = (int)nph - 1; ph >= 0; ph--) {
      const uint32_t b = ph_begin[ph], pr = ph_pairs[ph];
      if (ph_odd[ph]) {
        if (tid == 0) {
          const uint32_t o = b + pr;
          if (o != root) dep[o] = (uint8_t)min(255, dep[npar[o]] + 1);
        }
        __syncthreads();
      }
      // parents of this phase's nodes are all newer: gather 8 at a time
      for (uint32_t t0 = b + tid; t0 < b + pr; t0 += 8 * K2_THREADS) {
        uint32_t par[8];
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const uint32_t t = t0 + u * K2_THREADS;
          par[u] = (t < b + pr && t != root) ? npar[t] : 0xFFFFFFFFu;
        }
#pragma unroll
        for (int u = 0; u < 8; u++) {
          const uint32_t t = t0 + u * K2_THREADS;
          if (par[u] != 0xFFFFFFFFu) dep[t] = (uint8_t)min(255, dep[par[u]] + 1);
        }
      }
      __syncthreads();
    }
    for (uint32_t i0 = tid; i0 < L; i0 += 8 * K2_THREADS) {
      uint32_t lp8[8], vv[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const uint32_t i = i0 + u * K2_THREADS;
        lp8[u] = i < L ? lpar[i] : 0u;
        vv[u] = i < L ? v0[i] : 0u;
      }
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const uint32_t i = i0 + u * K2_THREADS;
        if (i < L) {
          const uint32_t d = (uint32_t)dep[lp8[u]] + 1;
          if (d > ACTC_MAX_CODE_LENGTH) atomicOr(&s_err, 1u);
          llen[vv[u]] = (uint8_t)(d > 255 ? 255 : d);
        }
      }
    }
  }
  __syncthreads();

  K2_STAMP(4)
  // ---- 5. canonical order: stable radix pass on length (input in symbol order) ----
  // keys (len << 26 | live index): one keys-only pass on the length digit
#pragma unroll 8
  for (uint32_t i = tid; i < L; i += K2_THREADS) k1[i] = ((unsigned long long)llen[i] << kSymKeyBits) | i;
  __syncthreads();
  unsigned long long *ck = k1;
  if (L > 1) {
    if (big)
      radix_pass_keys(k1, k0, (uint32_t)L, kSymKeyBits, rs);
    else {
      for (uint32_t i = tid; i < L; i += K2_THREADS) v1[i] = i;
      __syncthreads();
      radix_pass(k1, v1, k0, v0, (uint32_t)L, kSymKeyBits, rs);
    }
    ck = k0;
  }
  if (big && L > 1) {
    // per-length counts = the digit totals of the pass (exclusive prefix in rs.tot)
    if (tid < 64) {
      const uint32_t hi = tid + 1 < 256 ? rs.tot[tid + 1] : (uint32_t)L;
      s_cnt[tid] = hi - rs.tot[tid];
    }
    __syncthreads();
    if (tid == 0) {
      unsigned mx = 0;
      for (int l = 0; l < 64; l++)
        if (s_cnt[l]) mx = l;
      // lengths >= 64 (saturated depths) only occur with an error already flagged
      s_maxlen = (rs.tot[64] < (uint32_t)L) ? 255u : mx;
    }
  } else {
    unsigned lmax = 0;
    for (uint32_t i = tid; i < L; i += K2_THREADS) {
      unsigned l = (unsigned)(ck[i] >> kSymKeyBits);
      atomicAdd(&s_cnt[l & 63], 1u);
      lmax = max(lmax, l);
    }
    atomicMax(&s_maxlen, lmax);
  }
  __syncthreads();
  if (tid == 0) {
    // huffman.py:97-117 (first_code per length, base index per length)
    unsigned long long code = 0;
    uint32_t idx = 0;
    for (int l = 0; l < 64; l++) {
      code <<= 1;
      s_first[l] = code;
      s_base[l] = idx;
      code += s_cnt[l];
      idx += s_cnt[l];
    }
  }
  __syncthreads();
  for (uint32_t i0 = tid; i0 < L; i0 += 8 * K2_THREADS) {
    unsigned long long kk[8];
    uint32_t sy[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const uint32_t i = i0 + u * K2_THREADS;
      kk[u] = i < L ? ck[i] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const uint32_t i = i0 + u * K2_THREADS;
      sy[u] = i < L ? a.live_sym[kk[u] & (kMaxAlphabet - 1)] : 0u;
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const uint32_t i = i0 + u * K2_THREADS;
      if (i < L) {
        const uint32_t l = (uint32_t)(kk[u] >> kSymKeyBits), s = sy[u];
        a.canon[i] = s;
        if (a.ctab && l <= 56) a.ctab[s] = ((s_first[l] + (i - s_base[l])) << 8) | l;
        if (a.len8) a.len8[s] = (uint8_t)l;
      }
    }
  }
  if (tid < 64) a.len_counts[tid] = s_cnt[tid];
  if (a.out_lengths) {
    for (uint64_t s = tid; s < A; s += K2_THREADS) a.out_lengths[s] = 0;
    __syncthreads();
    for (uint32_t j = tid; j < L; j += K2_THREADS) a.out_lengths[a.live_sym[j]] = llen[j];
  }

  K2_STAMP(5)
  // ---- 6. plan: payload bits, RLE record count, entropy, live range ----
  // p*log2(p) = (f/T) * (log2 f - log2 T) with log2 f from a shared table for
  // f < kLgTab (the shared arrays of stages 2-5 are dead here); the
  // summation order differs from numpy's anyway (report value, rel. 1e-12)
  constexpr uint32_t kLgTab = 4096;
  double *lgtab = reinterpret_cast<double *>(smem);
  const double total = (double)a.n_symbols;
  if (!a.in_lengths) {
    for (uint32_t f = tid; f < kLgTab; f += K2_THREADS) lgtab[f] = f ? log2((double)f) : 0.0;
  }
  __syncthreads();
  const double lgT = log2(total), invT = 1.0 / total;
  unsigned long long bits = 0, recs = 0;
  double ent = 0.0;
  for (uint32_t j0 = tid; j0 < L; j0 += 8 * K2_THREADS) {
    uint32_t sy[8], pe[8];
    unsigned long long fr[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const uint32_t j = j0 + u * K2_THREADS;
      sy[u] = j < L ? a.live_sym[j] : 0u;
      pe[u] = (j < L && j) ? a.live_sym[j - 1] + 1 : 0u;
      fr[u] = j < L ? a.live_freq[j] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const uint32_t j = j0 + u * K2_THREADS;
      if (j >= L) continue;
      const unsigned long long f = fr[u];
      const uint32_t lj = llen[j];
      if (!a.in_lengths) {
        bits += f * lj;
        const double pp = (double)f * invT;
        ent += pp * (f < kLgTab ? lgtab[f] - lgT : log2(pp));
      }
      const uint64_t g = sy[u] - pe[u];
      if (g) recs += (g + 65534) / 65535;
      if (j == 0 || g || lj != llen[j - 1]) recs += 1;
    }
  }
  unsigned long long tb;
  block_excl_sum<unsigned long long>(bits, wbuf, &tb);
  unsigned long long tr;
  block_excl_sum<unsigned long long>(recs, wbuf2, &tr);
  double te;
  block_excl_sum<double>(ent, dbuf, &te);
  if (tid == 0) {
    uint64_t tail = L ? A - ((uint64_t)a.live_sym[L - 1] + 1) : A;
    tr += (tail + 65534) / 65535;
    if (L > 65535) {
      // exact record count when a live run could exceed 65535 symbols
      tr = 0;
      uint64_t run = 0;
      unsigned cur = 0xFFFFFFFFu;
      uint64_t prev = 0;
      for (uint32_t j = 0; j < L; j++) {
        uint32_t s = a.live_sym[j];
        uint64_t g = s - prev;
        if (g) {
          if (run) tr += (run + 65534) / 65535;
          tr += (g + 65534) / 65535;
          run = 0;
          cur = 0;
        }
        if (llen[j] != cur) {
          if (run) tr += (run + 65534) / 65535;
          run = 0;
          cur = llen[j];
        }
        run++;
        prev = (uint64_t)s + 1;
      }
      if (run) tr += (run + 65534) / 65535;
      tr += (tail + 65534) / 65535;
    }
    actc_plan_t *pl = a.plan;
    pl->n = a.n_symbols;
    pl->sym_bytes = a.sym_bytes;
    pl->live_symbols = (uint32_t)L;
    pl->max_len = s_maxlen;
    pl->payload_bits = tb;
    pl->rle_runs = tr;
    pl->entropy_bits = L > 1 ? -te : 0.0;
    if (pl->entropy_bits == 0.0) pl->entropy_bits = 0.0;
    pl->status = (s_err & 1u) ? ACTC_EPARAM : ((s_err & 2u) ? ACTC_ECUDA : ACTC_OK);
    if (s_maxlen > 56 && !a.in_lengths) pl->status = ACTC_EPARAM;
    if (a.n_outliers) pl->n_outliers = *a.n_outliers;
    if (a.nonfinite && *a.nonfinite) pl->status = ACTC_EDATA;
    pl->sym_lo = L ? a.live_sym[0] : 0;
    pl->sym_hi = L ? a.live_sym[L - 1] : 0;
    if (a.dbg) {
      a.dbg[6] = clock64();
      a.dbg[9] = L;
    }
  }
}

}  // namespace actc
