// K2r: Huffman codebook on frequency classes (one CTA, 1024 threads).
//
// Same outputs as k2_codebook (build_code_lengths huffman.py:37-75,
// canonical_codes huffman.py:78-94, the RLE record count of
// _rle_encode_lengths codec.py:201-226, stream_entropy_bits
// huffman.py:239-246), computed on *runs* instead of symbols.
//
// heapq with (freq, tiebreak) is the two-queue algorithm (leaf wins a
// frequency tie, older internal node wins among internals).  Its pop order
// M is the merge of the leaves sorted by (freq, symbol) with the internal
// nodes in creation order, and internal node j is the pair (M[2j],
// M[2j+1]).  Equal-frequency leaves form one run (a frequency class);
// internal nodes created from the pairs inside one merged run share a
// weight and form one run too.  The phase schedule of k2_codebook (with m
// the smallest remaining weight, every item lighter than 2m is popped
// before any node made in the phase) is run over runs: a phase merges the
// leaf runs and internal runs lighter than 2m (merge path), scans their
// counts into merge positions, and each merged run emits <= 2 new runs (a
// pair straddling the previous run, then its inner pairs); an odd leftover
// pairs with the lightest remaining item ("carry").  The activation
// alphabets of the bench have 0.5-5 K classes for 12-64 K live symbols.
//
// Depths need no tree walk: depth is non-increasing in creation order
// (internals) and in sorted order (leaves), so with B_0 = root and
// B_d = min{ j : pos(j) >= 2 B_{d-1} } (pos = merge position), the nodes of
// depth <= d are exactly those popped at positions >= 2 B_{d-1}.  One
// search per level over the run arrays gives the level boundaries; a
// frequency class then has one depth, or (if a boundary cuts it) the first
// t symbols in symbol order are one level deeper.
//
// Symbol passes (warp per contiguous symbol range): class id per symbol ->
// code length -> canonical rank by (length, symbol) via per-warp counters.
//
// Limits of this fast path (else the host-launched k2_codebook runs: the
// kernel leaves *fallback = 1): alphabet <= 65536, n < 2^32, <= kRCap
// classes, <= kICap internal runs, <= kBigCap symbols with freq >= 2^18.
#include "kernels.cuh"

namespace actc {

namespace {

constexpr int NT = K2_THREADS;
constexpr int NW = NT / 32;
constexpr uint32_t kFTBits = 18;
constexpr uint32_t kFT = 1u << kFTBits;   // frequencies below: bitmap classes
constexpr uint32_t kBMW = kFT / 32;       // bitmap words
constexpr uint32_t kBigCap = 2048;
constexpr uint32_t kHT = 0x80000000u;     // head-taken flag on a run's position
constexpr int kMaxLv = 64;
constexpr int kMaxSide = 96;
constexpr uint32_t kInf32 = 0xFFFFFFFFu;

struct Side {
  uint32_t run, pos, leaf;
};

// first k in [0, nr) with pred(k) (monotone), warp-cooperative 32-ary search
template <typename Pred>
__device__ __forceinline__ uint32_t warp_first(uint32_t nr, Pred pred) {
  const int lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = nr;
  while (hi - lo > 32) {
    const uint32_t step = (hi - lo + 31) / 32;
    const uint32_t c = min(hi - 1, lo + (lane + 1) * step - 1);
    const unsigned b = __ballot_sync(0xffffffffu, pred(c));
    if (!b) return hi;
    const uint32_t f = __ffs(b) - 1;
    const uint32_t nlo = lo + f * step;
    hi = min(hi, lo + (f + 1) * step);
    lo = nlo;
  }
  const uint32_t c = lo + lane;
  const unsigned b = __ballot_sync(0xffffffffu, c < hi && pred(c));
  return b ? lo + __ffs(b) - 1 : hi;
}

// in-place exclusive prefix of v[0..n), v[n] = total
__device__ void prefix_inplace(uint32_t *v, uint32_t n, uint32_t *wb) {
  const uint32_t per = (n + NT - 1) / NT;
  const uint32_t b0 = min(n, threadIdx.x * per), b1 = min(n, b0 + per);
  uint32_t s = 0;
  for (uint32_t i = b0; i < b1; i++) s += v[i];
  uint32_t tot;
  uint32_t ex = block_excl_sum<uint32_t>(s, wb, &tot);
  for (uint32_t i = b0; i < b1; i++) {
    const uint32_t t = v[i];
    v[i] = ex;
    ex += t;
  }
  if (threadIdx.x == 0) v[n] = tot;
  __syncthreads();
}

}  // namespace

__global__ void __launch_bounds__(NT, 1) k2r_codebook(CodebookArgs a) {
  extern __shared__ __align__(16) uint32_t sm[];
  // run arrays: leaf (class) runs and internal runs: weight, count, position
  uint32_t *LW = sm, *LC = LW + (kRCap + 1), *LM = LC + (kRCap + 1);
  uint32_t *IW = LM + (kRCap + 1), *IC = IW + (kICap + 1), *IM = IC + (kICap + 1);
  // class-building scratch aliases the internal-run region (dead until the phases)
  uint32_t *bm = IW, *bpre = bm + kBMW, *BL = bpre + kBMW, *SB = BL + kBigCap;
  // symbol-pass counters alias it again after the depth stage
  uint32_t *cntA = IW, *cntL = IW + NW * 64;

  __shared__ uint32_t s_wb[NW + 1], s_wb2[NW + 1];
  __shared__ unsigned long long s_wbl[NW + 1];
  __shared__ double s_wbd[NW + 1];
  __shared__ uint32_t s_lastw_t[NT];
  __shared__ unsigned s_fail, s_err;
  __shared__ uint32_t s_L, s_lo, s_hi, s_nbig, s_lastw;
  __shared__ unsigned long long s_sum;
  __shared__ uint32_t s_li, s_lh, s_ii, s_ih, s_ni, s_P, s_le, s_ie, s_nph;
  __shared__ Side s_side[kMaxSide];
  __shared__ uint32_t s_nside;
  __shared__ uint32_t s_thr[kMaxLv + 1], s_LB[kMaxLv + 1], s_nlv;
  __shared__ uint32_t s_lencnt[64], s_base[64];
  __shared__ unsigned long long s_first[64];
  __shared__ uint32_t sc_s0[64], sc_da[64], sc_db[64], sc_dl[64], s_nsc;
  __shared__ uint32_t w_first[NW], w_last[NW], w_starts[NW], w_has[NW];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const uint32_t A = (uint32_t)a.A;
#define K2R_STAMP(i) \
  if (a.dbg && tid == 0) a.dbg[i] = clock64();
  K2R_STAMP(0)

  if (tid == 0) {
    s_fail = 0;
    s_err = 0;
    s_L = 0;
    s_lo = kInf32;
    s_hi = 0;
    s_nbig = 0;
    s_sum = 0;
    s_nside = 0;
    s_nsc = 0;
    s_nlv = 0;
  }
  if (tid < 64) s_lencnt[tid] = 0;
  for (uint32_t i = tid; i < kBMW; i += NT) bm[i] = 0;
  __syncthreads();

  // ---- S1: live range, frequency bitmap, heavy frequencies ----
  {
    const uint32_t WS = (((A + NW - 1) / NW) + 31) & ~31u;
    const uint32_t w0 = min(A, warp * WS), w1 = min(A, w0 + WS);
    uint32_t myL = 0, mylo = kInf32, myhi = 0;
    unsigned long long mysum = 0;
    for (uint32_t base = w0; base < w1; base += 256) {
      unsigned long long v[8];
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const uint32_t s = base + 32 * u + lane;
        v[u] = s < w1 ? a.hist[s] : 0ull;
      }
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const uint32_t s = base + 32 * u + lane;
        if (a.out_lengths && s < w1) a.out_lengths[s] = 0;
        if (v[u]) {
          const uint32_t f = (uint32_t)v[u];
          mysum += v[u] >> 32 ? (1ull << 32) : v[u];  // weights must fit u32
          myL++;
          mylo = min(mylo, s);
          myhi = max(myhi, s);
          if (f < kFT) {
            atomicOr(&bm[f >> 5], 1u << (f & 31));
          } else {
            const uint32_t p = atomicAdd(&s_nbig, 1u);
            if (p < kBigCap) BL[p] = f;
          }
        }
      }
    }
    myL = warp_sum(myL);
    mysum = warp_sum(mysum);
    mylo = __reduce_min_sync(0xffffffffu, mylo);
    myhi = __reduce_max_sync(0xffffffffu, myhi);
    if (lane == 0) {
      if (myL) atomicAdd(&s_L, myL);
      if (mysum) atomicAdd(&s_sum, mysum);
      atomicMin(&s_lo, mylo);
      atomicMax(&s_hi, myhi);
    }
  }
  __syncthreads();
  const uint32_t L = s_L;
  const uint32_t nbig = s_nbig;
  if (L == 0 || nbig > kBigCap || s_sum >= (1ull << 32)) {
    if (tid == 0) *a.fallback = 1u;
    return;
  }
  const uint32_t lo = s_lo, hi = s_hi;

  // bitmap rank prefix (8 words per thread)
  uint32_t Rs;
  {
    constexpr int PW = kBMW / NT;
    uint32_t pc[PW], tot = 0;
#pragma unroll
    for (int u = 0; u < PW; u++) {
      pc[u] = __popc(bm[tid * PW + u]);
      tot += pc[u];
    }
    uint32_t ex = block_excl_sum<uint32_t>(tot, s_wb, &Rs);
#pragma unroll
    for (int u = 0; u < PW; u++) {
      bpre[tid * PW + u] = ex;
      ex += pc[u];
    }
  }
  // heavy frequencies: rank sort, then unique
  for (uint32_t i = tid; i < nbig; i += NT) {
    const uint32_t v = BL[i];
    uint32_t r = 0;
    for (uint32_t j = 0; j < nbig; j++) {
      const uint32_t w = BL[j];
      r += (w < v) || (w == v && j < i);
    }
    SB[r] = v;
  }
  __syncthreads();
  uint32_t nu;
  {
    const uint32_t i0 = 2 * tid, i1 = i0 + 1;
    const uint32_t f0 = i0 < nbig && (i0 == 0 || SB[i0] != SB[i0 - 1]);
    const uint32_t f1 = i1 < nbig && SB[i1] != SB[i1 - 1];
    const uint32_t v0 = i0 < nbig ? SB[i0] : 0, v1 = i1 < nbig ? SB[i1] : 0;
    const uint32_t ex = block_excl_sum<uint32_t>(f0 + f1, s_wb, &nu);
    if (f0) BL[ex] = v0;
    if (f1) BL[ex + f0] = v1;
  }
  const uint32_t R = Rs + nu;
  if (R > kRCap) {
    if (tid == 0) *a.fallback = 1u;
    return;
  }
  for (uint32_t i = tid; i < R; i += NT) LC[i] = 0;
  __syncthreads();
  K2R_STAMP(1)

  // ---- S2: class id per live symbol, class sizes and weights ----
  const uint32_t span = hi - lo + 1;
  const uint32_t WS2 = (((span + NW - 1) / NW) + 31) & ~31u;
  const uint32_t v0 = min(hi + 1, lo + warp * WS2), v1 = min(hi + 1, v0 + WS2);
  for (uint32_t base = v0; base < v1; base += 256) {
    unsigned long long v[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const uint32_t s = base + 32 * u + lane;
      v[u] = s < v1 ? a.hist[s] : 0ull;
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const uint32_t s = base + 32 * u + lane;
      const uint32_t f = (uint32_t)v[u];
      uint32_t k = kInf32;
      if (f) {
        if (f < kFT) {
          const uint32_t wd = f >> 5;
          k = bpre[wd] + __popc(bm[wd] & ((1u << (f & 31)) - 1u));
        } else {
          uint32_t l2 = 0, h2 = nu;
          while (l2 < h2) {
            const uint32_t m = (l2 + h2) >> 1;
            if (BL[m] < f) l2 = m + 1; else h2 = m;
          }
          k = Rs + l2;
        }
      }
      const unsigned peers = __match_any_sync(0xffffffffu, k);
      if (f && lane == __ffs(peers) - 1) {
        atomicAdd(&LC[k], (uint32_t)__popc(peers));
        LW[k] = f;
      }
      if (s < v1) a.cls16[s] = f ? (uint16_t)k : (uint16_t)0xFFFF;
    }
  }
  __syncthreads();
  K2R_STAMP(2)

  // ---- phases over runs ----
  if (tid == 0) {
    s_li = 0;
    s_lh = 0;
    s_ii = 0;
    s_ih = 0;
    s_ni = 0;
    s_P = 0;
    s_nph = 0;
  }
  __syncthreads();
  const uint32_t target = 2 * (L - 1);
  while (true) {
    const uint32_t P = s_P;
    if (P >= target || s_fail) break;
    if (tid == 0) {
      const uint32_t li = s_li, ii = s_ii, ni = s_ni;
      const unsigned long long wl = li < R ? LW[li] : ~0ull, wi = ii < ni ? IW[ii] : ~0ull;
      const unsigned long long lim = 2ull * min(wl, wi);
      uint32_t l2 = li, h2 = R;
      while (l2 < h2) {
        const uint32_t m = (l2 + h2) >> 1;
        if (LW[m] < lim) l2 = m + 1; else h2 = m;
      }
      s_le = l2;
      l2 = ii;
      h2 = ni;
      while (l2 < h2) {
        const uint32_t m = (l2 + h2) >> 1;
        if (IW[m] < lim) l2 = m + 1; else h2 = m;
      }
      s_ie = l2;
      if (++s_nph > 96) s_fail = 1;
    }
    __syncthreads();
    if (s_fail) break;
    const uint32_t li = s_li, lh = s_lh, ii = s_ii, ih = s_ih, ni = s_ni, le = s_le, ie = s_ie;
    const uint32_t nL = le - li, nI = ie - ii, T = nL + nI;
    const uint32_t K = (T + NT - 1) / NT;
    const uint32_t j0 = min(T, tid * K), j1 = min(T, j0 + K);
    uint32_t a0;
    {
      uint32_t l2 = j0 > nI ? j0 - nI : 0, h2 = min(j0, nL);
      while (l2 < h2) {
        const uint32_t m = (l2 + h2) >> 1;
        if (LW[li + m] <= IW[ii + j0 - 1 - m]) l2 = m + 1; else h2 = m;
      }
      a0 = l2;
    }
#define K2R_NEXT                                                        \
  const bool tl = ax < nL && (bx >= nI || LW[li + ax] <= IW[ii + bx]);  \
  uint32_t w, c;                                                        \
  if (tl) {                                                             \
    w = LW[li + ax];                                                    \
    c = LC[li + ax] - (ax == 0 ? lh : 0u);                              \
  } else {                                                              \
    w = IW[ii + bx];                                                    \
    c = IC[ii + bx] - (bx == 0 ? ih : 0u);                              \
  }
    uint32_t sumc = 0, lastw = 0;
    {
      uint32_t ax = a0, bx = j0 - a0;
      for (uint32_t j = j0; j < j1; j++) {
        K2R_NEXT
        if (tl) ax++; else bx++;
        sumc += c;
        lastw = w;
      }
    }
    s_lastw_t[tid] = lastw;
    if (j0 < j1 && j1 == T) s_lastw = lastw;
    uint32_t C;
    const uint32_t cex = block_excl_sum<uint32_t>(sumc, s_wb, &C);
    const uint32_t pw0 = (tid > 0 && j0 < j1) ? s_lastw_t[tid - 1] : 0u;
    uint32_t e = 0;
    {
      uint32_t ax = a0, bx = j0 - a0, p = P + cex;
      for (uint32_t j = j0; j < j1; j++) {
        K2R_NEXT
        if (tl) {
          LM[li + ax] = p | ((ax == 0 && lh) ? kHT : 0u);
          ax++;
        } else {
          IM[ii + bx] = p | ((bx == 0 && ih) ? kHT : 0u);
          bx++;
        }
        const uint32_t bnd = p & 1u;
        e += bnd + ((c - bnd) >= 2u);
        p += c;
      }
    }
    uint32_t E;
    const uint32_t eex = block_excl_sum<uint32_t>(e, s_wb2, &E);
    if (ni + E + 1 > kICap) {
      if (tid == 0) s_fail = 1;
      __syncthreads();
      break;
    }
    {
      uint32_t ax = a0, bx = j0 - a0, p = P + cex, o = ni + eex, prevw = pw0;
      for (uint32_t j = j0; j < j1; j++) {
        K2R_NEXT
        if (tl) ax++; else bx++;
        const uint32_t bnd = p & 1u;
        if (bnd) {
          IW[o] = prevw + w;
          IC[o] = 1;
          o++;
        }
        const uint32_t rem = c - bnd;
        if (rem >= 2u) {
          IW[o] = 2u * w;
          IC[o] = rem >> 1;
          o++;
        }
        p += c;
        prevw = w;
      }
    }
#undef K2R_NEXT
    __syncthreads();
    if (tid == 0) {
      uint32_t Pn = P + C, nli = le, nlh = le == li ? lh : 0u, nii = ie, nih = ie == ii ? ih : 0u, nni = ni + E;
      if (C & 1u) {
        // the odd leftover pairs with the lightest remaining item (leaf on ties)
        const unsigned long long wl = le < R ? LW[le] : ~0ull;
        const uint32_t icand = ie < ni ? ie : ni;
        const unsigned long long wi = icand < nni ? IW[icand] : ~0ull;
        uint32_t wp;
        const uint32_t ns = s_nside;
        if (ns >= kMaxSide) s_fail = 1;
        if (wl <= wi) {
          wp = LW[le];
          if (ns < kMaxSide) s_side[ns] = Side{le, Pn, 1u};
          if (LC[le] == 1u) {
            LM[le] = Pn | kHT;
            nli = le + 1;
            nlh = 0;
          } else {
            nli = le;
            nlh = 1;
          }
        } else {
          wp = IW[icand];
          if (ns < kMaxSide) s_side[ns] = Side{icand, Pn, 0u};
          if (IC[icand] == 1u) {
            IM[icand] = Pn | kHT;
            nii = icand + 1;
            nih = 0;
          } else {
            nii = icand;
            nih = 1;
          }
        }
        s_nside = ns + 1;
        IW[nni] = s_lastw + wp;
        IC[nni] = 1;
        nni++;
        Pn++;
      }
      s_li = nli;
      s_lh = nlh;
      s_ii = nii;
      s_ih = nih;
      s_ni = nni;
      s_P = Pn;
    }
    __syncthreads();
  }
  if (s_fail) {
    if (tid == 0) *a.fallback = 1u;
    return;
  }
  K2R_STAMP(3)

  // ---- depth levels ----
  const uint32_t ni = s_ni, nside = s_nside;
  prefix_inplace(LC, R, s_wb);  // LC -> first sorted-leaf index of each class (LC[R] = L)
  if (L >= 2) prefix_inplace(IC, ni, s_wb);  // IC -> first internal index of each run
  // position of the first / last item of a run; head-taken runs keep their
  // first item's position in the side table
  auto first_pos = [&](const uint32_t *M, const uint32_t *S, uint32_t k, uint32_t leaf) -> uint32_t {
    const uint32_t m = M[k];
    if (!(m & kHT)) return m;
    if (S[k + 1] - S[k] == 1u) return m & ~kHT;
    for (uint32_t q = 0; q < nside; q++)
      if (s_side[q].run == k && s_side[q].leaf == leaf) return s_side[q].pos;
    return 0u;
  };
  auto last_pos = [&](const uint32_t *M, const uint32_t *S, uint32_t k) -> uint32_t {
    const uint32_t m = M[k], ht = m >> 31, cnt = S[k + 1] - S[k];
    return cnt - ht >= 1u ? (m & ~kHT) + (cnt - ht - 1u) : (m & ~kHT);
  };
  // first item index (in run order) popped at a position >= thr, or `none`
  auto first_at = [&](const uint32_t *M, const uint32_t *S, uint32_t nr, uint32_t leaf, uint32_t thr,
                      uint32_t none) -> uint32_t {
    const uint32_t k = warp_first(nr, [&](uint32_t kk) { return last_pos(M, S, kk) >= thr; });
    if (k >= nr) return none;
    const uint32_t m = M[k], mr = m & ~kHT;
    if (m & kHT) {
      if (first_pos(M, S, k, leaf) >= thr) return S[k];
      return S[k] + 1u + (thr > mr ? thr - mr : 0u);
    }
    return S[k] + (thr > mr ? thr - mr : 0u);
  };
  if (L >= 2 && warp == 0) {
    // internal runs [0, ni-1): the last run is the root alone
    uint32_t Bp = L - 2, nlv = 0;
    while (true) {
      const uint32_t thr = 2u * Bp;
      if (lane == 0) s_thr[nlv] = thr;
      nlv++;
      if (Bp == 0 || nlv > kMaxLv - 1) break;
      Bp = first_at(IM, IC, ni - 1, 0u, thr, L - 2);
    }
    if (lane == 0) {
      s_nlv = nlv;
      if (Bp != 0) s_err |= 1u;  // deeper than 63 levels
    }
  }
  __syncthreads();
  const uint32_t nlv = s_nlv;
  for (uint32_t d = warp; d < nlv; d += NW) {
    const uint32_t lb = first_at(LM, LC, R, 1u, s_thr[d], L);
    if (lane == 0) s_LB[d] = lb;
  }
  __syncthreads();
  K2R_STAMP(4)

  // ---- per class: depth, split points, bits, entropy, length counts ----
  unsigned long long bits = 0;
  double ent = 0.0;
  const double total = (double)a.n_symbols;
  for (uint32_t k = tid; k < R; k += NT) {
    const uint32_t s0 = LC[k], s1 = LC[k + 1], cnt = s1 - s0, f = LW[k];
    // depth(i) = 1 + #{levels with LB > i}; LB decreasing over levels
    auto depth_of = [&](uint32_t i) -> uint32_t {
      uint32_t l2 = 0, h2 = nlv;
      while (l2 < h2) {
        const uint32_t m = (l2 + h2) >> 1;
        if (s_LB[m] > i) l2 = m + 1; else h2 = m;
      }
      return 1u + l2;
    };
    const uint32_t dl = depth_of(s1 - 1), df = depth_of(s0);
    uint32_t ci = dl;
    unsigned long long sumt = 0;
    if (df != dl) {
      // level indices x in [dl-1, df-1) have s0 < LB[x] <= s1-1: they cut the
      // class at rank t = LB[x] - s0 (t decreasing in x)
      const uint32_t da = dl - 1, db = df - 1;
      const uint32_t sc = atomicAdd(&s_nsc, 1u);
      if (sc < 64) {
        sc_s0[sc] = s0;
        sc_da[sc] = da;
        sc_db[sc] = db;
        sc_dl[sc] = dl;
      } else {
        atomicOr(&s_err, 2u);
      }
      ci = dl | 0x100u | (sc << 9);
      // ranks [t, prev) are j levels deeper than the class's last symbol
      uint32_t prev = cnt, j = 0;
      for (uint32_t x = da; x < db; x++) {
        const uint32_t t = s_LB[x] - s0;
        sumt += t;
        atomicAdd(&s_lencnt[min(63u, dl + j)], prev - t);
        prev = t;
        j++;
      }
      atomicAdd(&s_lencnt[min(63u, dl + j)], prev);
    } else {
      atomicAdd(&s_lencnt[min(63u, dl)], cnt);
    }
    bits += (unsigned long long)f * ((unsigned long long)cnt * dl + sumt);
    const double p = (double)f / total;
    ent += (double)cnt * (p * log2(p));
    LW[k] = ci;
  }
  unsigned long long tb;
  block_excl_sum<unsigned long long>(bits, s_wbl, &tb);
  double te;
  block_excl_sum<double>(ent, s_wbd, &te);
  if (tid == 0) {
    unsigned long long code = 0;
    uint32_t idx = 0, mx = 0;
    for (int l = 0; l < 64; l++) {
      code <<= 1;
      s_first[l] = code;
      s_base[l] = idx;
      code += s_lencnt[l];
      idx += s_lencnt[l];
      if (s_lencnt[l]) mx = l;
    }
    s_lencnt[0] = mx;  // stash: max length (length 0 never counted)
  }
  for (uint32_t i = tid; i < 2 * NW * 64; i += NT) cntA[i] = 0;
  __syncthreads();
  const uint32_t maxlen = s_lencnt[0], nsc = min(64u, s_nsc);
  K2R_STAMP(5)

  // ---- symbol passes over the live range, warp w owns [v0, v1) ----
  if (nsc) {
    for (uint32_t base = v0; base < v1; base += 32) {
      const uint32_t s = base + lane;
      const uint32_t k = s < v1 ? a.cls16[s] : 0xFFFFu;
      uint32_t sc = 0xFFu;
      if (k != 0xFFFFu) {
        const uint32_t ci = LW[k];
        if (ci & 0x100u) sc = ci >> 9;
      }
      const unsigned peers = __match_any_sync(0xffffffffu, sc);
      if (sc != 0xFFu && lane == __ffs(peers) - 1) cntA[warp * 64 + sc] += __popc(peers);
    }
    __syncthreads();
    if (tid < (int)nsc) {
      uint32_t run = 0;
      for (int w = 0; w < NW; w++) {
        const uint32_t t = cntA[w * 64 + tid];
        cntA[w * 64 + tid] = run;
        run += t;
      }
    }
    __syncthreads();
  }
  // pass B: code lengths, per-warp length counts, RLE run starts
  {
    uint32_t prevlen = 0, starts = 0, firstlen = 0;
    bool first = true;
    for (uint32_t base = v0; base < v1; base += 32) {
      const uint32_t s = base + lane;
      const bool in = s < v1;
      const uint32_t k = in ? a.cls16[s] : 0xFFFFu;
      uint32_t len = 0, sc = 0xFFu;
      if (k != 0xFFFFu) {
        const uint32_t ci = LW[k];
        len = ci & 0xFFu;
        if (ci & 0x100u) sc = ci >> 9;
      }
      const unsigned ps = __match_any_sync(0xffffffffu, sc);
      if (sc != 0xFFu) {
        const uint32_t r = cntA[warp * 64 + sc] + __popc(ps & lt);
        // depth = dl + #{cut levels x in [da, db) with t = LB[x] - s0 > r}
        uint32_t extra = 0;
        for (uint32_t x = sc_da[sc]; x < sc_db[sc]; x++) extra += (s_LB[x] - sc_s0[sc]) > r;
        len = sc_dl[sc] + extra;
      }
      __syncwarp();
      if (sc != 0xFFu && lane == __ffs(ps) - 1) cntA[warp * 64 + sc] += __popc(ps);
      len = min(len, 63u);
      if (k != 0xFFFFu) {
        a.len8[s] = (uint8_t)len;
        if (a.out_lengths) a.out_lengths[s] = (uint16_t)len;
      }
      const unsigned pl = __match_any_sync(0xffffffffu, in ? len : 0xFFu);
      if (in && len && lane == __ffs(pl) - 1) cntL[warp * 64 + len] += __popc(pl);
      // run starts inside this warp's range (its first symbol is judged later)
      uint32_t up = __shfl_up_sync(0xffffffffu, len, 1);
      if (lane == 0) up = prevlen;
      const bool st = in && !(first && lane == 0) && len != up;
      starts += __popc(__ballot_sync(0xffffffffu, st));
      if (first) firstlen = __shfl_sync(0xffffffffu, len, 0);
      const uint32_t nin = min(32u, v1 - base);
      prevlen = __shfl_sync(0xffffffffu, len, nin - 1);
      first = false;
      __syncwarp();
    }
    if (lane == 0) {
      w_has[warp] = v0 < v1;
      w_first[warp] = firstlen;
      w_last[warp] = prevlen;
      w_starts[warp] = starts;
    }
  }
  __syncthreads();
  if (tid < 64) {
    uint32_t run = s_base[tid];
    for (int w = 0; w < NW; w++) {
      const uint32_t t = cntL[w * 64 + tid];
      cntL[w * 64 + tid] = run;
      run += t;
    }
  }
  __syncthreads();
  // pass C: canonical ranks -> canon[], ctab[]
  for (uint32_t base = v0; base < v1; base += 32) {
    const uint32_t s = base + lane;
    const bool live = s < v1 && a.cls16[s] != 0xFFFFu;
    const uint32_t len = live ? a.len8[s] : 0xFFu;
    const unsigned pl = __match_any_sync(0xffffffffu, len);
    if (live) {
      const uint32_t ci = cntL[warp * 64 + len] + __popc(pl & lt);
      a.canon[ci] = s;
      if (a.ctab && len <= 56) a.ctab[s] = ((s_first[len] + (ci - s_base[len])) << 8) | len;
    }
    __syncwarp();
    if (live && lane == __ffs(pl) - 1) cntL[warp * 64 + len] += __popc(pl);
    __syncwarp();
  }
  if (tid < 64) a.len_counts[tid] = tid ? s_lencnt[tid] : 0u;
  K2R_STAMP(6)
  if (tid == 0) {
    // RLE records over the whole alphabet: zero run before lo, runs inside
    // [lo, hi], zero run after hi; a run longer than 65535 splits
    uint64_t recs = 1 + (lo > 0) + (hi + 1 < A);
    int prev = -1;
    for (int w = 0; w < NW; w++) {
      if (!w_has[w]) continue;
      recs += w_starts[w];
      if (prev >= 0 && w_first[w] != w_last[prev]) recs++;
      prev = w;
    }
    if (recs == 1 && A > 65535) recs = (A + 65534) / 65535;
    actc_plan_t *pl = a.plan;
    pl->n = a.n_symbols;
    pl->sym_bytes = a.sym_bytes;
    pl->live_symbols = L;
    pl->max_len = maxlen;
    pl->payload_bits = tb;
    pl->rle_runs = recs;
    pl->entropy_bits = L > 1 ? -te : 0.0;
    if (pl->entropy_bits == 0.0) pl->entropy_bits = 0.0;
    pl->status = (s_err & 1u) ? ACTC_EPARAM : ((s_err & 2u) ? ACTC_ECUDA : ACTC_OK);
    if (maxlen > 56) pl->status = ACTC_EPARAM;
    if (a.n_outliers) pl->n_outliers = *a.n_outliers;
    if (a.nonfinite && *a.nonfinite) pl->status = ACTC_EDATA;
    pl->sym_lo = lo;
    pl->sym_hi = hi;
    *a.fallback = 0u;
    if (a.dbg) {
      a.dbg[7] = clock64();
      a.dbg[8] = s_nph;
      a.dbg[9] = L;
      a.dbg[10] = R;
      a.dbg[11] = ni;
      a.dbg[12] = nsc;
    }
  }
#undef K2R_STAMP
}

}  // namespace actc
