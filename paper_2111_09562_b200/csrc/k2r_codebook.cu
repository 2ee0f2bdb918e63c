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
// pairs with the lightest remaining item ("carry").  Phases of <= 32 runs
// run on one warp without block barriers.  The activation alphabets of the
// bench have 0.5-5 K classes for 12-64 K live symbols.
//
// Depths need no tree walk: depth is non-increasing in creation order
// (internals) and in sorted order (leaves), so with B_0 = root and
// B_d = min{ j : pos(j) >= 2 B_{d-1} } (pos = merge position), the nodes of
// depth <= d are exactly those popped at positions >= 2 B_{d-1}.  One
// search per level over the run arrays gives the level boundaries; a
// frequency class then has one depth, or (if a boundary cuts it) its first
// t symbols in symbol order are one level deeper.
//
// Symbol passes: thread t owns a contiguous symbol segment; per-thread
// length counters + column prefix sums give the canonical rank by (length,
// symbol) without warp voting.
//
// Limits of this fast path (else the host-launched k2_codebook runs: the
// kernel leaves *fallback = 1): alphabet <= 65536, sum of freqs < 2^32,
// <= kRCap classes, <= kICap internal runs, <= kBigCap symbols with freq >=
// 2^18, <= 32 distinct code lengths, <= 8 cut classes.
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
constexpr uint32_t kHot = 384;            // classes counted in per-warp counters
constexpr int kNL = K2R_NL;               // max distinct code lengths (symbol passes)
constexpr int kTS = K2R_TS;               // per-thread length-counter stride (odd word count)
constexpr int kNS = 8;                    // max cut classes
constexpr int kSS = kNS + 2;              // per-thread cut-class counter stride

struct Side {
  uint32_t run, pos, leaf;
};

// first k in [0, nr) with pred(k) (pred monotone), warp-cooperative 32-ary search
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

// phase scan element: item count c and the number of runs emitted when the
// segment starts at an even (e0) or odd (e1) merge position
struct PhS {
  uint32_t c, e0, e1;
};
__device__ __forceinline__ PhS ph_combine(PhS a, PhS b) {
  const bool odd = a.c & 1u;
  return PhS{a.c + b.c, a.e0 + (odd ? b.e1 : b.e0), a.e1 + (odd ? b.e0 : b.e1)};
}
__device__ __forceinline__ PhS ph_shfl_up(PhS v, int o) {
  return PhS{__shfl_up_sync(0xffffffffu, v.c, o), __shfl_up_sync(0xffffffffu, v.e0, o),
             __shfl_up_sync(0xffffffffu, v.e1, o)};
}
// block exclusive scan of PhS; *tot = block total
__device__ PhS ph_block_excl(PhS v, PhS *wb, PhS *tot) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  PhS inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const PhS t = ph_shfl_up(inc, o);
    if (lane >= o) inc = ph_combine(t, inc);
  }
  if (lane == 31) wb[w] = inc;
  __syncthreads();
  if (w == 0) {
    const PhS x = wb[lane];
    PhS xi = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const PhS t = ph_shfl_up(xi, o);
      if (lane >= o) xi = ph_combine(t, xi);
    }
    PhS xe = ph_shfl_up(xi, 1);
    if (lane == 0) xe = PhS{0, 0, 0};
    wb[lane] = xe;
    if (lane == 31) wb[32] = xi;
  }
  __syncthreads();
  PhS le = ph_shfl_up(inc, 1);
  if (lane == 0) le = PhS{0, 0, 0};
  const PhS r = ph_combine(wb[w], le);
  *tot = wb[32];
  __syncthreads();
  return r;
}

// exclusive prefix down the rows (threads) of one column of a per-thread u16
// table, plus a column base; one warp per column, 32 rows per round
__device__ void column_prefix(uint16_t *tab, uint32_t stride, uint32_t ncol, const uint32_t *colbase) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t col = warp; col < ncol; col += NW) {
    uint32_t run = colbase ? colbase[col] : 0u;
    for (int r0 = 0; r0 < NT; r0 += 32) {
      uint16_t *p = tab + (r0 + lane) * stride + col;
      const uint32_t v = *p;
      const uint32_t inc = warp_incl_sum(v);
      *p = (uint16_t)(run + inc - v);
      run += __shfl_sync(0xffffffffu, inc, 31);
    }
  }
}

}  // namespace

__global__ void __launch_bounds__(NT, 1) k2r_codebook(CodebookArgs a) {
  extern __shared__ __align__(16) uint32_t sm[];
  // run arrays: leaf (class) runs and internal runs: weight, count, position
  uint32_t *LW = sm, *LC = LW + (kRCap + 1), *LM = LC + (kRCap + 1);
  uint32_t *IW = LM + (kRCap + 1), *IC = IW + (kICap + 1), *IM = IC + (kICap + 1);
  // class-building scratch aliases the internal-run region (dead until the phases)
  uint32_t *bm = IW, *bpre = bm + kBMW, *BL = bpre + kBMW, *SB = BL + kBigCap, *wcnt = SB + kBigCap;
  // symbol-pass tables alias LC.. after the per-class stage
  uint16_t *cntT = reinterpret_cast<uint16_t *>(LC);  // [NT][kTS] length counters
  uint16_t *cntS = cntT + NT * kTS;                      // [NT][kSS] cut-class counters
  uint8_t *t_first = reinterpret_cast<uint8_t *>(cntS + NT * kSS), *t_last = t_first + NT;

  __shared__ uint32_t s_wb[NW + 1];
  __shared__ unsigned long long s_wbl[NW + 1];
  __shared__ double s_wbd[NW + 1];
  __shared__ PhS s_wbp[NW + 1];
  __shared__ uint32_t s_lastw_t[NT];
  __shared__ uint32_t s_dummy[NW];
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
  __shared__ uint32_t s_starts, s_minlen, s_maxlen;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const uint32_t A = (uint32_t)a.A;
#define K2R_STAMP(i) \
  if (a.dbg && tid == 0) a.dbg[i] = clock64();
  K2R_STAMP(0)
  // the plan's K1 counters: loaded early, used at the very end
  unsigned long long n_out = 0;
  unsigned nonfin = 0;
  if (tid == 0) {
    if (a.n_outliers) n_out = *a.n_outliers;
    if (a.nonfinite) nonfin = *a.nonfinite;
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
    s_starts = 0;
  }
  if (tid < 64) s_lencnt[tid] = 0;
  for (uint32_t i = tid; i < kBMW; i += NT) bm[i] = 0;
  for (uint32_t i = tid; i < NW * kHot; i += NT) wcnt[i] = 0;
  __syncthreads();

  // ---- S1: live range, frequency bitmap, heavy frequencies (warp-strided) ----
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
            const uint32_t bit = 1u << (f & 31);
            if (!(bm[f >> 5] & bit)) atomicOr(&bm[f >> 5], bit);
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
    if (tid == 0 && a.dbg) {
      a.dbg[20] = 1;
      a.dbg[21] = nbig;
      a.dbg[22] = L;
    }
    if (tid == 0) {
      *a.fallback = 1u;
      a.plan->status = ACTC_EAGAIN;  // k2_codebook (if queued) rewrites the plan
    }
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
    if (tid == 0 && a.dbg) {
      a.dbg[20] = 2;
      a.dbg[21] = R;
      a.dbg[22] = L;
    }
    if (tid == 0) {
      *a.fallback = 1u;
      a.plan->status = ACTC_EAGAIN;  // k2_codebook (if queued) rewrites the plan
    }
    return;
  }
  for (uint32_t i = tid; i < R; i += NT) LC[i] = 0;
  __syncthreads();
  K2R_STAMP(1)

  // symbol-pass geometry: thread t owns [p0 + t*SEG, p0 + (t+1)*SEG), SEG % 16 == 0
  const uint32_t p0 = lo & ~15u;
  const uint32_t SEG = ((((hi + 1 - p0) + NT - 1) / NT) + 15) & ~15u;

  // ---- S2: class id per live symbol, class sizes and weights (warp-strided) ----
  {
    const uint32_t span = hi + 1 - p0;
    const uint32_t WS2 = (((span + NW - 1) / NW) + 31) & ~31u;
    const uint32_t v0 = min(hi + 1, p0 + warp * WS2), v1 = min(hi + 1, v0 + WS2);
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
        // one unconditional constant add per lane: ptxas turns it into
        // ATOMS.POPC.INC, which aggregates a warp's equal addresses in the
        // atomic unit (a __match_any_sync + leader update cost ~1.4 K cycles
        // per symbol and thread on wide alphabets); dead lanes count into a
        // per-warp dummy.  Warp-private counters for the lightest (hottest)
        // classes keep the warps off each other's addresses.
        uint32_t *ctr = !f ? &s_dummy[warp] : (k < kHot ? &wcnt[warp * kHot + k] : &LC[k]);
        atomicAdd(ctr, 1u);
        if (f) LW[k] = f;
        if (s < v1) a.cls16[s] = f ? (uint16_t)k : (uint16_t)0xFFFF;
      }
    }
  }
  __syncthreads();
  if (tid < (int)min(kHot, R)) {
    uint32_t c = LC[tid];
    for (int w = 0; w < NW; w++) c += wcnt[w * kHot + tid];
    LC[tid] = c;
  }
  K2R_STAMP(2)

  // ---- phases over runs ----
  const uint32_t target = 2 * (L - 1);
  // range of the upcoming phase (warp 0): runs lighter than twice the lightest item
  auto next_range = [&]() {
    const uint32_t li = s_li, ii = s_ii, ni = s_ni;
    const unsigned long long wl = li < R ? LW[li] : ~0ull, wi = ii < ni ? IW[ii] : ~0ull;
    const unsigned long long lim = 2ull * min(wl, wi);
    const uint32_t le = li + warp_first(R - li, [&](uint32_t k) { return (unsigned long long)LW[li + k] >= lim; });
    const uint32_t ie = ii + warp_first(ni - ii, [&](uint32_t k) { return (unsigned long long)IW[ii + k] >= lim; });
    if (lane == 0) {
      s_le = le;
      s_ie = ie;
      if (++s_nph > 96) s_fail = 1;
    }
    __syncwarp();
  };
  // odd leftover (weight s_lastw) pairs with the lightest remaining item
  // (leaf on ties); one thread, then the state advances
  auto finish_phase = [&](uint32_t P, uint32_t C, uint32_t E) {
    const uint32_t li = s_li, lh = s_lh, ii = s_ii, ih = s_ih, ni = s_ni, le = s_le, ie = s_ie;
    uint32_t Pn = P + C, nli = le, nlh = le == li ? lh : 0u, nii = ie, nih = ie == ii ? ih : 0u, nni = ni + E;
    if (C & 1u) {
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
  };
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
  if (warp == 0 && target > 0) next_range();
  __syncthreads();
  while (true) {
    if (s_P >= target || s_fail) break;
    const uint32_t T0 = (s_le - s_li) + (s_ie - s_ii);
    if (T0 <= 32) {
      // ---- one warp runs consecutive small phases (lane = merged run) ----
      if (warp == 0) {
        while (true) {
          const uint32_t P = s_P, li = s_li, lh = s_lh, ii = s_ii, ih = s_ih, ni = s_ni, le = s_le, ie = s_ie;
          const uint32_t nL = le - li, nI = ie - ii, T = nL + nI;
          uint32_t w = 0, c = 0, run = 0;
          bool tl = false;
          if ((uint32_t)lane < T) {
            const uint32_t j = lane;
            uint32_t l2 = j > nI ? j - nI : 0, h2 = min(j, nL);
            while (l2 < h2) {
              const uint32_t m = (l2 + h2) >> 1;
              if (LW[li + m] <= IW[ii + j - 1 - m]) l2 = m + 1; else h2 = m;
            }
            const uint32_t ax = l2, bx = j - l2;
            tl = ax < nL && (bx >= nI || LW[li + ax] <= IW[ii + bx]);
            if (tl) {
              run = li + ax;
              w = LW[run];
              c = LC[run] - (ax == 0 ? lh : 0u);
            } else {
              run = ii + bx;
              w = IW[run];
              c = IC[run] - (bx == 0 ? ih : 0u);
            }
          }
          const uint32_t cin = warp_incl_sum(c);
          const uint32_t C = __shfl_sync(0xffffffffu, cin, 31);
          const uint32_t p = P + cin - c;
          const uint32_t bnd = ((uint32_t)lane < T) ? (p & 1u) : 0u;
          const uint32_t rem = c - bnd;
          const uint32_t nbk = ((uint32_t)lane < T && rem >= 2u) ? 1u : 0u;
          const uint32_t e = bnd + nbk;
          const uint32_t ein = warp_incl_sum(e);
          const uint32_t E = __shfl_sync(0xffffffffu, ein, 31);
          if (ni + E + 1 > kICap) {
            if (lane == 0) s_fail = 1;
            __syncwarp();
            break;
          }
          const uint32_t prevw = __shfl_up_sync(0xffffffffu, w, 1);
          const uint32_t lastw = __shfl_sync(0xffffffffu, w, (T - 1) & 31);
          if ((uint32_t)lane < T) {
            if (tl) LM[run] = p | ((run == li && lh) ? kHT : 0u);
            else IM[run] = p | ((run == ii && ih) ? kHT : 0u);
            uint32_t o = ni + ein - e;
            if (bnd) {
              IW[o] = prevw + w;
              IC[o] = 1;
              o++;
            }
            if (nbk) {
              IW[o] = 2u * w;
              IC[o] = rem >> 1;
            }
          }
          __syncwarp();
          if (lane == 0) {
            s_lastw = lastw;
            finish_phase(P, C, E);
          }
          __syncwarp();
          if (s_P >= target || s_fail) break;
          next_range();
          if ((s_le - s_li) + (s_ie - s_ii) > 32) break;
        }
      }
      __syncthreads();
      continue;
    }
    // ---- block phase: thread t owns merged runs [j0, j1) ----
    const uint32_t P = s_P, li = s_li, lh = s_lh, ii = s_ii, ih = s_ih, ni = s_ni, le = s_le, ie = s_ie;
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
    PhS loc{0, 0, 0};
    uint32_t lastw = 0;
    {
      uint32_t ax = a0, bx = j0 - a0, q0 = 0, q1 = 1;
      for (uint32_t j = j0; j < j1; j++) {
        K2R_NEXT
        if (tl) ax++; else bx++;
        const uint32_t b0 = q0 & 1u, b1 = q1 & 1u;
        loc.e0 += b0 + ((c - b0) >= 2u);
        loc.e1 += b1 + ((c - b1) >= 2u);
        q0 += c;
        q1 += c;
        loc.c += c;
        lastw = w;
      }
    }
    s_lastw_t[tid] = lastw;
    if (j0 < j1 && j1 == T) s_lastw = lastw;
    PhS tot;
    const PhS ex = ph_block_excl(loc, s_wbp, &tot);
    const uint32_t C = tot.c, E = tot.e0;
    if (ni + E + 1 > kICap) {
      if (tid == 0) s_fail = 1;
      __syncthreads();
      break;
    }
    {
      uint32_t ax = a0, bx = j0 - a0, p = P + ex.c, o = ni + ex.e0;
      uint32_t prevw = (tid > 0 && j0 < j1) ? s_lastw_t[tid - 1] : 0u;
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
    if (warp == 0) {
      if (lane == 0) finish_phase(P, C, E);
      __syncwarp();
      if (s_P < target && !s_fail) next_range();
    }
    __syncthreads();
  }
  if (s_fail) {
    if (tid == 0 && a.dbg) {
      a.dbg[20] = 3;
      a.dbg[21] = ((unsigned long long)s_ni << 32) | s_nside;
      a.dbg[22] = L;
      a.dbg[23] = s_nph;
      a.dbg[24] = R;
    }
    if (tid == 0) {
      *a.fallback = 1u;
      a.plan->status = ACTC_EAGAIN;  // k2_codebook (if queued) rewrites the plan
    }
    return;
  }
  K2R_STAMP(3)

  // ---- depth levels ----
  const uint32_t ni = s_ni, nside = s_nside;
  prefix_inplace(LC, R, s_wb);  // LC -> first sorted-leaf index of each class (LC[R] = L)
  if (L >= 2) prefix_inplace(IC, ni, s_wb);  // IC -> first internal index of each run
  // position of a head-taken run's first item (side table)
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

  // ---- per class: depth, cut points, bits, entropy, length counts ----
  unsigned long long bits = 0;
  double ent = 0.0;
  const double total = (double)a.n_symbols;
  for (uint32_t k0 = 0; k0 < R; k0 += NT) {
    const uint32_t k = k0 + tid;
    uint32_t dl = 0xFFu, cnt = 0;
    if (k < R) {
      const uint32_t s0 = LC[k], s1 = LC[k + 1], f = LW[k];
      cnt = s1 - s0;
      // depth(i) = 1 + #{levels with LB > i}; LB non-increasing over levels
      auto depth_of = [&](uint32_t i) -> uint32_t {
        uint32_t l2 = 0, h2 = nlv;
        while (l2 < h2) {
          const uint32_t m = (l2 + h2) >> 1;
          if (s_LB[m] > i) l2 = m + 1; else h2 = m;
        }
        return 1u + l2;
      };
      dl = depth_of(s1 - 1);
      const uint32_t df = depth_of(s0);
      uint32_t ci = dl;
      unsigned long long sumt = 0;
      if (df != dl) {
        // level indices x in [dl-1, df-1) have s0 < LB[x] <= s1-1: they cut the
        // class at rank t = LB[x] - s0 (t decreasing in x); ranks [t, prev)
        // are j levels deeper than the class's last symbol
        const uint32_t da = dl - 1, db = df - 1;
        const uint32_t sc = atomicAdd(&s_nsc, 1u);
        if (sc < 64) {
          sc_s0[sc] = s0;
          sc_da[sc] = da;
          sc_db[sc] = db;
          sc_dl[sc] = dl;
        }
        ci = dl | 0x100u | (min(sc, 63u) << 9);
        uint32_t prev = cnt, j = 0;
        for (uint32_t x = da; x < db; x++) {
          const uint32_t t = s_LB[x] - s0;
          sumt += t;
          atomicAdd(&s_lencnt[min(63u, dl + j)], prev - t);
          prev = t;
          j++;
        }
        atomicAdd(&s_lencnt[min(63u, dl + j)], prev);
        dl = 0xFFu;  // counted above
      }
      bits += (unsigned long long)f * ((unsigned long long)cnt * (ci & 0xFFu) + sumt);
      const double p = (double)f / total;
      ent += (double)cnt * (p * log2(p));
      LW[k] = ci;
    }
    // uncut classes: one atomic per distinct length per warp
    const unsigned pk = __match_any_sync(0xffffffffu, dl);
    const uint32_t sumc = __reduce_add_sync(pk, cnt);
    if (dl != 0xFFu && lane == __ffs(pk) - 1) atomicAdd(&s_lencnt[min(63u, dl)], sumc);
  }
  unsigned long long tb;
  block_excl_sum<unsigned long long>(bits, s_wbl, &tb);
  double te;
  block_excl_sum<double>(ent, s_wbd, &te);
  if (tid == 0) {
    unsigned long long code = 0;
    uint32_t idx = 0, mx = 0, mn = 64;
    for (int l = 0; l < 64; l++) {
      code <<= 1;
      s_first[l] = code;
      s_base[l] = idx;
      code += s_lencnt[l];
      idx += s_lencnt[l];
      if (s_lencnt[l]) {
        mx = l;
        mn = min(mn, (uint32_t)l);
      }
    }
    s_minlen = mn;
    s_maxlen = mx;
    if (mx + 1 - mn > (uint32_t)kNL || s_nsc > (uint32_t)kNS) s_fail = 1;
  }
  __syncthreads();
  if (s_fail) {
    if (tid == 0 && a.dbg) {
      a.dbg[20] = 4;
      a.dbg[21] = ((unsigned long long)s_minlen << 32) | s_maxlen;
      a.dbg[22] = L;
      a.dbg[23] = s_nsc;
    }
    if (tid == 0) {
      *a.fallback = 1u;
      a.plan->status = ACTC_EAGAIN;  // k2_codebook (if queued) rewrites the plan
    }
    return;
  }
  const uint32_t minlen = s_minlen, maxlen = s_maxlen, nsc = s_nsc;
  {
    // per-thread counters (LC.. is dead now)
    uint32_t *z = reinterpret_cast<uint32_t *>(cntT);
    const uint32_t words = (NT * kTS + NT * kSS) / 2;
    for (uint32_t i = tid; i < words; i += NT) z[i] = 0;
  }
  __syncthreads();
  K2R_STAMP(5)

  // ---- symbol passes: thread t owns [q0, q0 + SEG) ----
  const uint32_t q0 = p0 + tid * SEG;
  const uint32_t q1 = min(hi + 1, q0 + SEG);  // live-range part of my segment
  uint16_t *myT = cntT + tid * kTS;
  uint16_t *myS = cntS + tid * kSS;
  if (nsc) {
    // pass A: cut-class membership counts
    for (uint32_t c0 = q0; c0 < q1; c0 += 8) {
      const uint4 v = *reinterpret_cast<const uint4 *>(a.cls16 + c0);
      const uint32_t wv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int u = 0; u < 8; u++) {
        const uint32_t s = c0 + u;
        const uint32_t k = (wv[u >> 1] >> (16 * (u & 1))) & 0xFFFFu;
        if (s >= lo && s < q1 && k != 0xFFFFu) {
          const uint32_t ci = LW[k];
          if (ci & 0x100u) myS[ci >> 9]++;
        }
      }
    }
    __syncthreads();
    K2R_STAMP(13)
    column_prefix(cntS, kSS, nsc, nullptr);
    __syncthreads();
  }
  K2R_STAMP(14)
  // pass B: lengths (len8 written 16 at a time), per-thread length counts, run starts
  {
    uint32_t prevlen = 0, starts = 0;
    for (uint32_t c0 = q0; c0 < q1; c0 += 16) {
      const uint4 va = *reinterpret_cast<const uint4 *>(a.cls16 + c0);
      const uint4 vb = *reinterpret_cast<const uint4 *>(a.cls16 + c0 + 8);
      const uint32_t wv[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
      uint32_t out[4] = {0, 0, 0, 0};
#pragma unroll
      for (int u = 0; u < 16; u++) {
        const uint32_t s = c0 + u;
        const uint32_t k = (wv[u >> 1] >> (16 * (u & 1))) & 0xFFFFu;
        uint32_t len = 0;
        if (s >= lo && s < q1 && k != 0xFFFFu) {
          const uint32_t ci = LW[k];
          len = ci & 0xFFu;
          if (ci & 0x100u) {
            const uint32_t sc = ci >> 9;
            const uint32_t r = myS[sc];
            myS[sc] = (uint16_t)(r + 1);
            uint32_t extra = 0;
            for (uint32_t x = sc_da[sc]; x < sc_db[sc]; x++) extra += (s_LB[x] - sc_s0[sc]) > r;
            len += extra;
          }
          myT[len - minlen]++;
        }
        out[u >> 2] |= len << (8 * (u & 3));
        if (s < q1) {
          if (s == q0) t_first[tid] = (uint8_t)len;
          else if (s > lo && len != prevlen) starts++;
          prevlen = len;
        }
      }
      *reinterpret_cast<uint4 *>(a.len8 + c0) = make_uint4(out[0], out[1], out[2], out[3]);
      if (a.out_lengths) {
        for (int u = 0; u < 16; u++) {
          const uint32_t s = c0 + u;
          if (s >= lo && s < q1) a.out_lengths[s] = (uint16_t)((out[u >> 2] >> (8 * (u & 3))) & 0xFFu);
        }
      }
    }
    if (q0 < q1) t_last[tid] = (uint8_t)prevlen;
    __syncthreads();
    // a run starts at my first symbol when it differs from the previous thread's last
    if (q0 < q1 && q0 > lo && tid > 0 && t_first[tid] != t_last[tid - 1]) starts++;
    starts = warp_sum(starts);
    if (lane == 0 && starts) atomicAdd(&s_starts, starts);
  }
  K2R_STAMP(15)
  column_prefix(cntT, kTS, maxlen + 1 - minlen, s_base + minlen);
  K2R_STAMP(16)
  __syncthreads();
  // pass C (canonical ranks -> canon[], ctab[]) is k2s_emit's: one SM's
  // store pipe is too narrow for ~2 scattered stores per symbol.  Hand over
  // this thread's starting rank per length (column prefix + base).
  {
    // the [thread][length] table is contiguous in shared memory: copy it coalesced
    __syncthreads();
    const uint32_t *src = reinterpret_cast<const uint32_t *>(cntT);
    uint32_t *dst = reinterpret_cast<uint32_t *>(a.rank_tab);
    for (uint32_t i = tid; i < (uint32_t)(NT * kTS / 2); i += NT) dst[i] = src[i];
  }
  if (tid < 64) a.len_counts[tid] = s_lencnt[tid];
  __syncthreads();
  K2R_STAMP(6)
  if (tid == 0) {
    // RLE records over the whole alphabet: zero run before lo, runs inside
    // [lo, hi] (the one starting at lo + later starts), zero run after hi; a
    // run longer than 65535 splits
    uint64_t recs = (lo > 0) + 1 + s_starts + (hi + 1 < A);
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
    pl->status = (s_err & 1u) ? ACTC_EPARAM : ACTC_OK;
    if (maxlen > 56) pl->status = ACTC_EPARAM;
    if (a.n_outliers) pl->n_outliers = n_out;
    if (a.nonfinite && nonfin) pl->status = ACTC_EDATA;
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

// K2s: canonical codes for the symbols of the k2r threads' segments
// (huffman.py:78-94 rule: code = first[len] + rank among the symbols of that
// length in symbol order); thread t of the grid replays k2r thread t's
// segment with the starting ranks k2r left in rank_tab.  32 CTAs of one warp:
// the scattered stores spread over 32 SMs.
__global__ void __launch_bounds__(32) k2s_emit(CodebookArgs a) {
  if (*a.fallback) return;  // k2_codebook built the tables
  __shared__ uint16_t s_row[32 * kTS];
  __shared__ unsigned long long s_first[64];
  __shared__ uint32_t s_base[64];
  const EmitArgs e{a.fallback, a.rank_tab, a.len_counts, a.len8, a.plan, a.canon, a.ctab};
  k2s_emit_warp(e, blockIdx.x, s_row, s_first, s_base);
}

}  // namespace actc
