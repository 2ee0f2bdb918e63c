// K2: Huffman codebook on one CTA.
//
// Replaces build_code_lengths (huffman.py:37-75), canonical_codes
// (huffman.py:78-94), the RLE record count of _rle_encode_lengths
// (codec.py:201-226) and stream_entropy_bits (huffman.py:239-246).
//
// Bit-exactness.  heapq pops items in (freq, tiebreak) order with leaf
// tiebreak = symbol and internal tiebreak = creation counter >= alphabet,
// i.e. the classic two-queue algorithm where a leaf wins a frequency tie
// and older internal nodes beat newer ones.  We run that algorithm in
// *phases*: with m the smallest remaining frequency, every item of
// frequency < 2m is popped in merged (freq, class, index) order and paired
// consecutively before any node created in the phase can be popped (new
// nodes are >= 2m); an odd leftover pairs with the smallest remaining item.
// Each phase at least doubles m, so there are <= log2(n)+1 phases, each a
// parallel merge.  Code lengths are depths (max(1, depth)), computed by
// walking the phases backwards.
#include "kernels.cuh"

namespace actc {

namespace {

// Bitonic sort of (key, val) pairs, lexicographic, in place; P is a power
// of two, all threads of the CTA participate.
__device__ __forceinline__ void bitonic_sort(unsigned long long *keys, uint32_t *vals, uint32_t P) {
  for (uint32_t k = 2; k <= P; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t p = threadIdx.x; p < P / 2; p += blockDim.x) {
        uint32_t i = (p / j) * 2 * j + (p % j);
        uint32_t ixj = i + j;
        unsigned long long x = keys[i], y = keys[ixj];
        uint32_t xv = vals[i], yv = vals[ixj];
        bool gt = x > y || (x == y && xv > yv);
        bool up = (i & k) == 0;
        if (gt == up) {
          keys[i] = y; keys[ixj] = x;
          vals[i] = yv; vals[ixj] = xv;
        }
      }
      __syncthreads();
    }
  }
}

// number of elements in sorted v[0..len) strictly below t
__device__ __forceinline__ uint32_t lower_bound_u64(const unsigned long long *v, uint32_t len,
                                                    unsigned long long t) {
  uint32_t lo = 0, hi = len;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (v[mid] < t)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}
// number of elements in sorted v[0..len) <= t
__device__ __forceinline__ uint32_t upper_bound_u64(const unsigned long long *v, uint32_t len,
                                                    unsigned long long t) {
  uint32_t lo = 0, hi = len;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (v[mid] <= t)
      lo = mid + 1;
    else
      hi = mid;
  }
  return lo;
}

constexpr uint32_t kIntBit = 0x80000000u;
constexpr uint32_t kSmemL = 4096;
constexpr int kMaxPhases = 128;

}  // namespace

__global__ void __launch_bounds__(K2_THREADS) k2_codebook(CodebookArgs a) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long wbuf[33];
  __shared__ unsigned long long wbuf2[33];
  __shared__ uint32_t s_lp, s_np, s_nn, s_a, s_b, s_nph;
  __shared__ uint32_t ph_begin[kMaxPhases], ph_pairs[kMaxPhases];
  __shared__ uint8_t ph_odd[kMaxPhases];
  __shared__ uint32_t s_cnt[64];
  __shared__ unsigned long long s_first[64];
  __shared__ uint32_t s_base[64];
  __shared__ unsigned s_err, s_maxlen;
  __shared__ double dbuf[33];

  const int tid = threadIdx.x;
  const uint64_t A = a.A;

  // ---- 1. compact live symbols (symbol order) ----
  uint64_t L = 0;
  for (uint64_t c = 0; c < A; c += (uint64_t)K2_THREADS * 8) {
    uint64_t b0 = c + (uint64_t)tid * 8;
    unsigned long long f[8];
    unsigned cnt = 0;
#pragma unroll
    for (int j = 0; j < 8; j++) {
      uint64_t s = b0 + j;
      unsigned long long v = 0;
      if (s < A) v = a.in_lengths ? (unsigned long long)a.in_lengths[s] : a.hist[s];
      f[j] = v;
      cnt += v != 0;
    }
    unsigned long long tot;
    unsigned long long off = block_excl_sum<unsigned long long>(cnt, wbuf, &tot);
#pragma unroll
    for (int j = 0; j < 8; j++) {
      if (f[j]) {
        a.live_sym[L + off] = (uint32_t)(b0 + j);
        a.live_freq[L + off] = f[j];
        off++;
      }
    }
    L += tot;
  }
  __syncthreads();

  if (tid == 0) {
    s_err = 0;
    s_maxlen = 0;
  }
  if (tid < 64) s_cnt[tid] = 0;

  // generic pointers: shared memory for small L, global scratch otherwise
  uint32_t P = 1;
  while (P < L) P <<= 1;
  unsigned long long *keys = a.keys;
  uint32_t *vals = a.vals;
  unsigned long long *nf = a.nf;
  uint32_t *lpar = a.lpar, *npar = a.npar, *S = a.S;
  uint32_t *ndepth = (uint32_t *)a.ndepth;
  uint8_t *llen = a.llen;
  if (L <= kSmemL) {
    unsigned char *p = smem;
    keys = (unsigned long long *)p; p += 8 * (size_t)kSmemL;
    nf = (unsigned long long *)p; p += 8 * (size_t)kSmemL;
    vals = (uint32_t *)p; p += 4 * (size_t)kSmemL;
    lpar = (uint32_t *)p; p += 4 * (size_t)kSmemL;
    npar = (uint32_t *)p; p += 4 * (size_t)kSmemL;
    S = (uint32_t *)p; p += 8 * (size_t)kSmemL;
    ndepth = (uint32_t *)p; p += 4 * (size_t)kSmemL;
    llen = (uint8_t *)p;
  }
  __syncthreads();

  if (a.in_lengths) {
    // lengths given (codebook_from_lengths): clamp display, check range
    for (uint32_t j = tid; j < L; j += K2_THREADS) {
      unsigned l = (unsigned)a.live_freq[j];
      if (l > ACTC_MAX_CODE_LENGTH) atomicOr(&s_err, 1u);
      llen[j] = (uint8_t)(l > 255 ? 255 : l);
    }
  } else if (L == 1) {
    if (tid == 0) llen[0] = 1;  // huffman.py:50-52
  } else if (L > 1) {
    // ---- 2. sort leaves by (freq, symbol) ----
    for (uint32_t i = tid; i < P; i += K2_THREADS) {
      keys[i] = i < L ? a.live_freq[i] : ~0ull;
      vals[i] = i < L ? i : 0xFFFFFFFFu;
    }
    __syncthreads();
    bitonic_sort(keys, vals, P);
    // leaf i: freq = keys[i], live index = vals[i]

    // ---- 3. phase-parallel two-queue merge ----
    if (tid == 0) {
      s_lp = 0; s_np = 0; s_nn = 0; s_nph = 0;
    }
    __syncthreads();
    const unsigned long long INF = ~0ull;
    while (true) {
      uint32_t lp = s_lp, np = s_np, nn = s_nn;
      if ((L - lp) + (nn - np) <= 1) break;
      if (tid == 0) {
        unsigned long long m = INF;
        if (lp < L) m = keys[lp];
        if (np < nn && nf[np] < m) m = nf[np];
        unsigned long long T = 2 * m;
        s_a = lower_bound_u64(keys + lp, (uint32_t)(L - lp), T);
        s_b = lower_bound_u64(nf + np, nn - np, T);
      }
      __syncthreads();
      const uint32_t na = s_a, nb = s_b;
      for (uint32_t i = tid; i < na; i += K2_THREADS) {
        unsigned long long f = keys[lp + i];
        uint32_t pos = i + lower_bound_u64(nf + np, nb, f);  // internals strictly below
        S[pos] = lp + i;
      }
      for (uint32_t j = tid; j < nb; j += K2_THREADS) {
        unsigned long long f = nf[np + j];
        uint32_t pos = j + upper_bound_u64(keys + lp, na, f);  // leaves <= win ties
        S[pos] = kIntBit | (np + j);
      }
      __syncthreads();
      const uint32_t tot = na + nb, pairs = tot >> 1;
      for (uint32_t t = tid; t < pairs; t += K2_THREADS) {
        uint32_t x = S[2 * t], y = S[2 * t + 1];
        unsigned long long fx = (x & kIntBit) ? nf[x & ~kIntBit] : keys[x];
        unsigned long long fy = (y & kIntBit) ? nf[y & ~kIntBit] : keys[y];
        nf[nn + t] = fx + fy;
        if (x & kIntBit) npar[x & ~kIntBit] = nn + t; else lpar[x] = nn + t;
        if (y & kIntBit) npar[y & ~kIntBit] = nn + t; else lpar[y] = nn + t;
      }
      __syncthreads();
      if (tid == 0) {
        uint32_t ph = s_nph;
        ph_begin[ph] = nn;
        ph_pairs[ph] = pairs;
        ph_odd[ph] = tot & 1;
        uint32_t nlp = lp + na, nnp = np + nb, nnn = nn + pairs;
        if (tot & 1) {
          uint32_t z = S[tot - 1];
          unsigned long long fz = (z & kIntBit) ? nf[z & ~kIntBit] : keys[z];
          // candidates: next leaf, next internal (old or the first new one);
          // leaf wins ties, and among internals the lower index wins
          unsigned long long fl = nlp < L ? keys[nlp] : INF;
          unsigned long long fi = nnp < nnn ? nf[nnp] : INF;
          uint32_t y;
          unsigned long long fy;
          if (nlp < L && fl <= fi) {
            y = nlp; fy = fl; nlp++;
          } else {
            y = kIntBit | nnp; fy = fi; nnp++;
          }
          uint32_t node = nnn;
          nf[node] = fz + fy;
          if (z & kIntBit) npar[z & ~kIntBit] = node; else lpar[z] = node;
          if (y & kIntBit) npar[y & ~kIntBit] = node; else lpar[y] = node;
          nnn++;
        }
        s_lp = nlp; s_np = nnp; s_nn = nnn;
        s_nph = ph + 1;
        if (ph + 1 >= kMaxPhases) s_err |= 2u;  // cannot happen for n < 2^38
      }
      __syncthreads();
      if (s_err & 2u) break;
    }
    // ---- 4. depths, walking phases backwards ----
    const uint32_t nn = s_nn, root = nn - 1, nph = s_nph;
    if (tid == 0) ndepth[root] = 0;
    __syncthreads();
    for (int ph = (int)nph - 1; ph >= 0; ph--) {
      const uint32_t b = ph_begin[ph], pr = ph_pairs[ph];
      if (ph_odd[ph]) {
        if (tid == 0) {
          uint32_t o = b + pr;
          if (o != root) ndepth[o] = ndepth[npar[o]] + 1;
        }
        __syncthreads();
      }
      for (uint32_t t = b + tid; t < b + pr; t += K2_THREADS)
        if (t != root) ndepth[t] = ndepth[npar[t]] + 1;
      __syncthreads();
    }
    for (uint32_t i = tid; i < L; i += K2_THREADS) {
      uint32_t d = ndepth[lpar[i]] + 1;
      if (d > ACTC_MAX_CODE_LENGTH) atomicOr(&s_err, 1u);
      llen[vals[i]] = (uint8_t)(d > 255 ? 255 : d);
    }
  }
  __syncthreads();

  // ---- 5. canonical order: sort live symbols by (length, symbol) ----
  for (uint32_t i = tid; i < P; i += K2_THREADS) {
    keys[i] = i < L ? (unsigned long long)llen[i] : ~0ull;
    vals[i] = i < L ? a.live_sym[i] : 0xFFFFFFFFu;
  }
  __syncthreads();
  if (L > 1) bitonic_sort(keys, vals, P);
  unsigned lmax = 0;
  for (uint32_t i = tid; i < L; i += K2_THREADS) {
    unsigned l = (unsigned)keys[i];
    atomicAdd(&s_cnt[l & 63], 1u);
    lmax = max(lmax, l);
  }
  atomicMax(&s_maxlen, lmax);
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
  for (uint32_t i = tid; i < L; i += K2_THREADS) {
    uint32_t l = (uint32_t)keys[i], s = vals[i];
    a.canon[i] = s;
    if (a.ctab && l <= 56) a.ctab[s] = ((s_first[l] + (i - s_base[l])) << 8) | l;
  }
  if (tid < 64) a.len_counts[tid] = s_cnt[tid];
  if (a.out_lengths) {
    for (uint64_t s = tid; s < A; s += K2_THREADS) a.out_lengths[s] = 0;
    __syncthreads();
    for (uint32_t j = tid; j < L; j += K2_THREADS) a.out_lengths[a.live_sym[j]] = llen[j];
  }

  // ---- 6. plan: payload bits, RLE record count, entropy ----
  unsigned long long bits = 0, recs = 0;
  double ent = 0.0;
  const double total = (double)a.n_symbols;
  for (uint32_t j = tid; j < L; j += K2_THREADS) {
    uint32_t s = a.live_sym[j];
    unsigned long long f = a.live_freq[j];
    if (!a.in_lengths) {
      bits += f * llen[j];
      double p = (double)f / total;
      ent += p * log2(p);
    }
    uint32_t prev_end = j ? a.live_sym[j - 1] + 1 : 0;
    uint64_t g = s - prev_end;
    if (g) recs += (g + 65534) / 65535;
    if (j == 0 || g || llen[j] != llen[j - 1]) recs += 1;
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
    if (pl->entropy_bits == -0.0) pl->entropy_bits = 0.0;
    pl->status = (s_err & 1u) ? ACTC_EPARAM : ((s_err & 2u) ? ACTC_ECUDA : ACTC_OK);
    if (s_maxlen > 56 && !a.in_lengths) pl->status = ACTC_EPARAM;
    if (a.n_outliers) pl->n_outliers = *a.n_outliers;
    if (a.nonfinite && *a.nonfinite) pl->status = ACTC_EDATA;
  }
}

}  // namespace actc
