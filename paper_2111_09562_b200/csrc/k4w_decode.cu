// K4 (fast path): warp-cooperative canonical-Huffman decode fused with the
// inverse Lorenzo reconstruction, outlier splice and re-zero filter.
//
// Replaces huffman_decode/_decode_bits (huffman.py:120-142, 210-236), the
// marker check (codec.py:356-359), lorenzo_decode (codec.py:275-293) and
// recon / splice / re-zero (codec.py:360-369) for streams that carry the
// device-side decode index (bit offset + starting lattice value of every
// ACTC_CHUNK-th symbol, both recorded at compress time).
//
// Work unit: one warp owns 32 consecutive chunks (8192 symbols), lane l
// decodes chunk l.  Per round each lane decodes 64 symbols of its chunk into
// a per-warp shared buffer (u16 pairs, rows padded to 33 words: conflict-free
// lane stores and row reads); then the warp walks the 32 rows: a warp scan of
// the deltas plus the chunk's running lattice value gives 64 consecutive
// lattice values, reconstructed in fp64 and stored coalesced.  No block
// barriers, no look-back: chunk start values come from the index.
//
// Decode step (one path for every lane): a 12-bit LUT gives (symbol, length)
// for codes <= 12 bits and a starting length l0 for longer prefixes; three
// comparisons against the left-aligned canonical limits finish the length
// (for a short code they are all false: the limits are non-decreasing), and
// the symbol of a long code comes from canon[off[l] + (W >> (32-l))] (shared
// cache of the first codes in canonical order).  Only invalid streams and
// codes longer than l0+3 take the warp-voted bit-serial fallback.  The next
// payload word is loaded one refill ahead and byte-swapped when consumed.
#include "kernels.cuh"

namespace actc {

namespace {

constexpr int ROUND = 64;             // symbols per lane per round
constexpr int ROW16 = ROUND / 2 + 1;  // words per row, u16 symbols
constexpr int ROW32 = ROUND + 1;      // words per row, u32 symbols
constexpr int NW4 = K4W_THREADS / 32;

__device__ __forceinline__ uint64_t read_bits64(const uint32_t *__restrict__ pw, uint64_t pos) {
  uint64_t wi = pos >> 5;
  unsigned sh = pos & 31;
  uint64_t hi = ((uint64_t)bswap32(pw[wi]) << 32) | bswap32(pw[wi + 1]);
  if (!sh) return hi;
  uint32_t lo = bswap32(pw[wi + 2]);
  return (hi << sh) | ((uint64_t)lo >> (32 - sh));
}

// 32-bit shared-window addressing: the tables and row buffers are addressed
// through addresses computed once, so the compiler does not rematerialise the
// shared window base (S2R SR_CgaCtaId + LEA) on every access.
__device__ __forceinline__ uint32_t saddr(const void *p) {
  // the opaque mov keeps the address in a register (otherwise the compiler
  // recomputes it from SR_CgaCtaId at every use inside the decode loop)
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mov.u32 %0, %1;" : "=r"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ uint32_t lds_u32(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_u16(uint32_t a) {
  unsigned short v;
  asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t lds_row(uint32_t a) {  // row buffer: ordered w.r.t. the stores
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a) : "memory");
  return v;
}
__device__ __forceinline__ void sts_row(uint32_t a, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(a), "r"(v) : "memory");
}

}  // namespace

template <int MODE, int SW, bool CIR>
__global__ void __launch_bounds__(K4W_THREADS, 3) k4w_decode(DecodeArgs a) {
  __shared__ uint32_t lut[kLutSize];
  __shared__ uint16_t ccache[K4W_CANON_CACHE];  // canon[0 .. ncache): the most frequent codes
  __shared__ uint32_t s_limm1[64];              // ((first+count) << (32-l)) - 1, saturated
  __shared__ int32_t s_off[64];                 // base[l] - first[l]
  __shared__ unsigned long long s_first[64];    // for the reference-rule fallback
  __shared__ uint32_t s_count[64], s_base[64];
  __shared__ uint32_t s_maxlen, s_zci;
  extern __shared__ __align__(16) uint32_t wbuf_all[];  // NW4 * 32 rows
  constexpr int ROW = SW == 16 ? ROW16 : ROW32;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  {
    constexpr int PER = kLutSize / 4 / K4W_THREADS;  // 16-byte loads per thread, all in flight
    uint4 l4[PER];
#pragma unroll
    for (int u = 0; u < PER; u++) l4[u] = __ldg(reinterpret_cast<const uint4 *>(a.lut) + tid + u * K4W_THREADS);
#pragma unroll
    for (int u = 0; u < PER; u++) reinterpret_cast<uint4 *>(lut)[tid + u * K4W_THREADS] = l4[u];
  }
  if (tid == 0) {
    unsigned long long code = 0;
    uint32_t idx = 0, mx = 0;
    for (int l = 0; l < 64; l++) {
      code <<= 1;
      const uint32_t c = a.len_counts[l];
      s_first[l] = code;
      s_count[l] = c;
      s_base[l] = idx;
      if (l >= 1 && l <= 32) {
        const unsigned long long lim = (code + c) << (32 - l);
        s_limm1[l] = lim == 0 ? 0u : (uint32_t)min(lim - 1, 0xFFFFFFFFull);
        s_off[l] = (int32_t)idx - (int32_t)(uint32_t)code;
      } else {
        s_limm1[l] = 0xFFFFFFFFu;
        s_off[l] = 0;
      }
      code += c;
      idx += c;
      if (c && l > 0) mx = l;
    }
    s_maxlen = mx;
    s_zci = 0xFFFFFFFFu;
  }
  const uint32_t ncache = SW == 16 ? min((uint32_t)K4W_CANON_CACHE, a.live) : 0u;
  // canonical-symbol cache: 8 x 16-byte loads in flight per thread
  for (uint32_t i0 = 4 * tid; i0 < ncache; i0 += 4 * 8 * K4W_THREADS) {
    uint4 c4[8];
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const uint32_t i = i0 + 4 * u * K4W_THREADS;
      c4[u] = i + 3 < ncache ? __ldg(reinterpret_cast<const uint4 *>(a.canon + i)) : make_uint4(0, 0, 0, 0);
      if (i < ncache && i + 3 >= ncache) {  // ragged tail
        c4[u].x = a.canon[i];
        if (i + 1 < ncache) c4[u].y = a.canon[i + 1];
        if (i + 2 < ncache) c4[u].z = a.canon[i + 2];
      }
    }
#pragma unroll
    for (int u = 0; u < 8; u++) {
      const uint32_t i = i0 + 4 * u * K4W_THREADS;
      if (i < ncache) ccache[i] = (uint16_t)c4[u].x;
      if (i + 1 < ncache) ccache[i + 1] = (uint16_t)c4[u].y;
      if (i + 2 < ncache) ccache[i + 2] = (uint16_t)c4[u].z;
      if (i + 3 < ncache) ccache[i + 3] = (uint16_t)c4[u].w;
    }
  }
  __syncthreads();
  // canonical index of the outlier marker (symbol 0): the smallest symbol, so
  // the first of its length in canonical order (only live with outliers)
  if (a.k && tid < 64 && s_count[tid] && a.canon[s_base[tid]] == 0u) s_zci = s_base[tid];
  __syncthreads();
  const uint32_t zci = s_zci;

  const bool fast_long = a.lut[kLutSize] != 0;
  const bool fin_scale = isfinite(a.two_eb);
  const int maxlen = (int)s_maxlen;
  const uint64_t nchunks = (a.n + ACTC_CHUNK - 1) / ACTC_CHUNK;
  const uint64_t nwt = (nchunks + 31) / 32;
  const long long radius = a.radius;
  const uint32_t rbase = saddr(wbuf_all) + 4u * (warp * 32 * ROW);  // this warp's rows
  const uint32_t mbase = rbase + 4u * (lane * ROW);                    // my row
  const uint32_t lut_s = saddr(lut), lim_s = saddr(s_limm1), off_s = saddr(s_off), cc_s = saddr(ccache);
  const uint32_t *__restrict__ pw = a.payload;
  // canonical index -> symbol (the most frequent codes come first in canonical order)
  // CIR: rows hold canonical indices (translated in the reconstruct, off the
  // decode chain); otherwise the decode chain resolves symbols itself
  auto sym_of = [&](uint32_t ci) -> uint32_t {
    if (!CIR) return ci;
    return ci < ncache ? lds_u16(cc_s + 2u * ci) : __ldg(&a.canon[ci]);
  };
  const uint32_t zmark = CIR ? zci : 0u;
  const uint32_t ncm1 = ncache ? ncache - 1 : 0u;
  unsigned long long nonzero = 0, markers = 0;
  bool bad = false;

  for (uint64_t wt = (uint64_t)blockIdx.x * NW4 + warp; wt < nwt; wt += (uint64_t)gridDim.x * NW4) {
    const uint64_t c = wt * 32 + lane;
    const bool valid = c < nchunks;
    const uint64_t e0 = c * ACTC_CHUNK;
    const uint32_t cnt = valid ? (uint32_t)min((uint64_t)ACTC_CHUNK, a.n - e0) : 0u;
    // a full warp tile: 32 complete chunks, no bounds checks in the row loop
    const bool full_tile = (wt + 1) * 32 * ACTC_CHUNK <= a.n;
    uint64_t endp = 0;
    const uint32_t *__restrict__ src = pw;  // next word to load into nextw
    unsigned long long buf = 0;
    int nb = 0;
    uint32_t nextw = 0;
    long long P = 0;    // running lattice value of my chunk
    uint32_t ordn = 0;  // ordinal of my chunk's next outlier
    bool ord_known = false;
    if (valid) {
      const uint64_t pos = a.chunk_off[c];
      endp = (c + 1 < nchunks) ? a.chunk_off[c + 1] : a.payload_bits;
      src = pw + (pos >> 5);
      const char *lp = reinterpret_cast<const char *>(src);
      for (uint64_t off = 128; off < ((endp - pos) >> 3) + 16; off += 128)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(lp + off));
      buf = ((unsigned long long)bswap32(__ldg(src)) << 32) | bswap32(__ldg(src + 1));
      buf <<= (pos & 31);
      nb = 64 - (int)(pos & 31);
      nextw = __ldg(src + 2);  // kept raw (big-endian); swapped when consumed
      src += 3;
      if (MODE != 2) P = a.chunk_lat[c];
    }
    for (int r = 0; r * ROUND < ACTC_CHUNK; r++) {
      // ---------------- decode up to ROUND symbols of my chunk ----------------
      const uint32_t i0 = r * ROUND;
      const uint32_t iend = max(i0, min(cnt, i0 + ROUND));  // empty once the chunk is exhausted
      uint32_t zr = 0;
#define ACTC_DEC(SYM)                                                                             \
  {                                                                                               \
    if (nb < 32) {                                                                                \
      buf |= (unsigned long long)bswap32(nextw) << (32 - nb);                                     \
      nb += 32;                                                                                   \
      nextw = __ldg(src); /* raw: swapped at the next refill, so the load latency is hidden */   \
      ++src;                                                                                      \
    }                                                                                             \
    const uint32_t W = (uint32_t)(buf >> 32);                                                     \
    const uint32_t e = lds_u32(lut_s + ((W >> (32 - kLutBits)) << 2));                            \
    const uint32_t l6 = e & 63u, hv = e >> 6;                                                     \
    const bool lng = l6 == 63u;                                                                   \
    /* a long code behind an exact-length prefix resolves without a branch: every lane */         \
    /* forms the canonical index (with a dummy length 1 for short codes) and reads the */         \
    /* symbol cache, so the warp never splits on the common long codes */                         \
    const uint32_t lc = lng ? hv : 1u;                                                            \
    const uint32_t ci = lds_u32(off_s + 4u * lc) + (W >> (32 - lc));                              \
    int len = lng ? (int)hv : (int)l6;                                                            \
    uint32_t sv;                                                                                  \
    if (CIR) {                                                                                    \
      sv = lng ? ci : hv;                                                                         \
    } else {                                                                                      \
      const uint32_t sl = lds_u16(cc_s + 2u * min(ci, ncm1));                                     \
      sv = lng ? sl : hv;                                                                         \
    }                                                                                             \
    if (__any_sync(__activemask(), l6 == 0u || (!CIR && lng && ci >= ncache))) {                  \
      if (!CIR && lng && ci >= ncache) sv = __ldg(&a.canon[ci]);                                  \
      if (l6 == 0u) {                                                                             \
        /* long code behind a mixed prefix: the LUT gives the shortest length l0; */              \
        /* three comparisons with the left-aligned canonical limits finish it */                  \
        const uint32_t l0 = hv;                                                                   \
        const uint32_t lb = lim_s + 4u * l0;                                                      \
        const uint32_t l = l0 + (W > lds_u32(lb)) + (W > lds_u32(lb + 4u)) + (W > lds_u32(lb + 8u)); \
        const bool ok = fast_long && l0 >= 1 && !(W > lds_u32(lb + 12u)) && (int)l <= maxlen;    \
        if (ok) {                                                                                 \
          const uint32_t cj = lds_u32(off_s + 4u * l) + (W >> (32 - l));                         \
          sv = CIR ? cj : (cj < ncache ? lds_u16(cc_s + 2u * cj) : __ldg(&a.canon[cj]));          \
          len = (int)l;                                                                           \
        } else {                                                                                  \
          /* rare: longer than l0+3, over-subscribed table, codes > 32 bits, or invalid */        \
          const uint64_t pos = ((uint64_t)(src - pw) << 5) - 32 - (uint64_t)nb;                   \
          const uint64_t win = read_bits64(pw, pos);                                              \
          len = 0;                                                                                \
          for (int ll = kLutBits + 1; ll <= maxlen; ll++) {                                       \
            const unsigned long long cd = win >> (64 - ll), of = cd - s_first[ll];                \
            if (of < s_count[ll]) {                                                               \
              sv = CIR ? s_base[ll] + (uint32_t)of : a.canon[s_base[ll] + of];                    \
              len = ll;                                                                           \
              break;                                                                              \
            }                                                                                     \
          }                                                                                       \
          if (!len) {                                                                             \
            bad = true;                                                                           \
            len = 1;                                                                              \
            sv = CIR ? 0u : a.radius;                                                             \
          }                                                                                       \
          const uint64_t np = pos + len;                                                          \
          src = pw + (np >> 5);                                                                   \
          buf = ((unsigned long long)bswap32(src[0]) << 32) | bswap32(src[1]);                    \
          buf <<= (np & 31);                                                                      \
          nb = 64 - (int)(np & 31);                                                               \
          nextw = src[2];                                                                         \
          src += 3;                                                                               \
          len = 0;                                                                                \
        }                                                                                         \
      }                                                                                           \
    }                                                                                             \
    buf <<= len;                                                                                  \
    nb -= len;                                                                                    \
    SYM = sv;                                                                                     \
  }
#define ACTC_ZERO(SYM, IDX)                                                                       \
  if (MODE != 2 && SYM == zmark) {                                                                \
    if (!ord_known) {                                                                             \
      uint64_t lo = 0, hi = a.k;                                                                  \
      while (lo < hi) {                                                                           \
        uint64_t mid = (lo + hi) >> 1;                                                            \
        if (a.out_idx[mid] < e0) lo = mid + 1; else hi = mid;                                     \
      }                                                                                           \
      ordn = (uint32_t)lo;                                                                        \
      ord_known = true;                                                                           \
    }                                                                                             \
    if (ordn >= a.k || a.out_idx[ordn] != e0 + (IDX)) bad = true;                                 \
    ordn++;                                                                                       \
    zr++;                                                                                         \
  }
      uint32_t i = i0;
      for (; i + 1 < iend; i += 2) {
        uint32_t sa, sb;
        ACTC_DEC(sa)
        ACTC_DEC(sb)
        ACTC_ZERO(sa, i)
        ACTC_ZERO(sb, i + 1)
        if (SW == 32) {
          sts_row(mbase + 4u * (i - i0), sa);
          sts_row(mbase + 4u * (i - i0 + 1), sb);
        } else {
          sts_row(mbase + 4u * ((i - i0) >> 1), sa | (sb << 16));
        }
      }
      if (i < iend) {
        uint32_t sa;
        ACTC_DEC(sa)
        ACTC_ZERO(sa, i)
        if (SW == 32)
          sts_row(mbase + 4u * (i - i0), sa);
        else
          sts_row(mbase + 4u * ((i - i0) >> 1), sa);
      }
#undef ACTC_DEC
#undef ACTC_ZERO
      markers += zr;
      const uint32_t ordr = ordn - zr;  // ordinal of my first outlier in this round (if zr > 0)
      __syncwarp();
      const unsigned zmask = __ballot_sync(0xffffffffu, zr != 0);

      // ---------------- reconstruct row by row (coalesced) ----------------
      // 32-bit lattice arithmetic when every chunk's running value is small
      // (a round moves it by at most ROUND * radius <= 2^22)
      const bool small_lat = __all_sync(0xffffffffu, P > -(1ll << 29) && P < (1ll << 29));
      if (MODE != 2 && SW == 16 && full_tile && zmask == 0 && small_lat && fin_scale) {
        // fast path: 32 complete chunks, no outliers in this round; lane owns
        // 4 consecutive elements of each row (ROUND = 128).  The re-zero
        // filter is a no-op here: a lattice value L != 0 reconstructs to
        // |fl(L*2eb)| >= 2eb > eb, L == 0 to +0 (or NaN when 2eb = inf) --
        // so it is skipped, and "nonzero" is L != 0 (or 2eb = inf).
        int P32 = (int)P;
        const int R32 = (int)radius;
        for (int cc = 0; cc < 32; cc++) {
          // lane owns elements 2*lane, 2*lane+1 of row cc (ROUND = 64)
          const uint32_t wa = lds_row(rbase + 4u * (cc * ROW + lane));
          const int d0 = (int)sym_of(wa & 0xFFFFu) - R32;
          const int d1 = (int)sym_of(wa >> 16) - R32;
          const int p1 = d0 + d1;
          const int inc = warp_incl_sum(p1);
          const int tot = __shfl_sync(0xffffffffu, inc, 31);
          const int Pc = __shfl_sync(0xffffffffu, P32, cc);
          const int B = Pc + (inc - p1);
          if (lane == cc) P32 = Pc + tot;
          const int L0 = B + d0, L1 = B + p1;
          const double r0 = __dmul_rn((double)L0, a.two_eb);
          const double r1 = __dmul_rn((double)L1, a.two_eb);
          nonzero += (L0 != 0) + (L1 != 0);
          const uint64_t eg = (wt * 32 + cc) * ACTC_CHUNK + i0 + 2 * lane;
          if (MODE == 0) {
            __stcs(reinterpret_cast<float2 *>(reinterpret_cast<float *>(a.out) + eg), make_float2((float)r0, (float)r1));
          } else {
            __stcs(reinterpret_cast<double2 *>(reinterpret_cast<double *>(a.out) + eg), make_double2(r0, r1));
          }
        }
        P = P32;
      } else {
        for (int cc = 0; cc < 32; cc++) {
          const uint64_t ch = wt * 32 + cc;
          if (ch >= nchunks) break;
          const uint32_t ccnt = (uint32_t)min((uint64_t)ACTC_CHUNK, a.n - ch * ACTC_CHUNK);
          if (i0 >= ccnt) continue;
          // running outlier ordinal of chunk cc within this round
          uint32_t ordc = __shfl_sync(0xffffffffu, ordr, cc);
          for (int h = 0; h < ROUND / 64; h++) {
          const uint32_t k0 = i0 + 64 * h + 2 * lane;  // element index inside the chunk
          if (i0 + 64 * h >= ccnt) break;
          const bool v0 = k0 < ccnt, v1 = k0 + 1 < ccnt;
          uint32_t s0, s1;
          if (SW == 16) {
            const uint32_t w = lds_row(rbase + 4u * (cc * ROW + 32 * h + lane));
            s0 = w & 0xFFFFu;
            s1 = w >> 16;
          } else {
            s0 = lds_row(rbase + 4u * (cc * ROW + 64 * h + 2 * lane));
            s1 = lds_row(rbase + 4u * (cc * ROW + 64 * h + 2 * lane + 1));
          }
          const uint64_t eg = ch * ACTC_CHUNK + k0;  // global element index
          // row entries are canonical indices: outlier markers by index,
          // everything else translated to its symbol
          const bool m0 = v0 && s0 == zmark, m1 = v1 && s1 == zmark;
          s0 = v0 ? sym_of(s0) : 0u;
          s1 = v1 ? sym_of(s1) : 0u;
          if (MODE == 2) {
            uint32_t *out = reinterpret_cast<uint32_t *>(a.out) + eg;
            if (v1)
              *reinterpret_cast<uint2 *>(out) = make_uint2(s0, s1);
            else if (v0)
              *out = s0;
            continue;
          }
          const long long Pc = __shfl_sync(0xffffffffu, P, cc);
          long long L0, L1, Pn;
          bool z0 = false, z1 = false;
          uint32_t o0 = 0, o1 = 0;
          if (SW == 16 && !((zmask >> cc) & 1u)) {
            const int d0 = v0 ? (int)s0 - (int)radius : 0;
            const int d1 = v1 ? (int)s1 - (int)radius : 0;
            const int inc = warp_incl_sum(d0 + d1);
            L0 = Pc + (inc - d1);
            L1 = L0 + d1;
            Pn = Pc + __shfl_sync(0xffffffffu, inc, 31);
          } else {
            z0 = m0;
            z1 = m1;
            const int nzl = (int)z0 + (int)z1;
            const int zi = warp_incl_sum(nzl);
            o0 = ordc + (uint32_t)(zi - nzl);
            o1 = o0 + (uint32_t)z0;
            ordc += (uint32_t)__shfl_sync(0xffffffffu, zi, 31);
            bool dummy;
            const Seg e0s = z0 ? Seg{quant_exact((double)a.out_val[o0], a.two_eb, a.eb, dummy), 1}
                               : Seg{v0 ? (long long)s0 - radius : 0, 0};
            const Seg e1s = z1 ? Seg{quant_exact((double)a.out_val[o1], a.two_eb, a.eb, dummy), 1}
                               : Seg{v1 ? (long long)s1 - radius : 0, 0};
            const Seg inc = warp_incl_seg(seg_combine(e0s, e1s));
            const long long pv = __shfl_up_sync(0xffffffffu, inc.v, 1);
            const int pr = __shfl_up_sync(0xffffffffu, inc.r, 1);
            const Seg ex = lane ? Seg{pv, pr} : Seg{0, 0};
            const Seg a0 = seg_combine(ex, e0s);
            const Seg a1 = seg_combine(a0, e1s);
            L0 = a0.r ? a0.v : Pc + a0.v;
            L1 = a1.r ? a1.v : Pc + a1.v;
            const long long tv = __shfl_sync(0xffffffffu, inc.v, 31);
            const int tr = __shfl_sync(0xffffffffu, inc.r, 31);
            Pn = tr ? tv : Pc + tv;
          }
          if (lane == cc) P = Pn;
          double r0 = z0 ? (double)a.out_val[o0] : __dmul_rn((double)L0, a.two_eb);
          double r1 = z1 ? (double)a.out_val[o1] : __dmul_rn((double)L1, a.two_eb);
          if (a.preserve) {
            if (fabs(r0) <= a.eb) r0 = 0.0;
            if (fabs(r1) <= a.eb) r1 = 0.0;
          }
          nonzero += (v0 && r0 != 0.0) + (v1 && r1 != 0.0);
          if (MODE == 0) {
            float *out = reinterpret_cast<float *>(a.out) + eg;
            if (v1)
              __stcs(reinterpret_cast<float2 *>(out), make_float2((float)r0, (float)r1));
            else if (v0)
              *out = (float)r0;
          } else {
            double *out = reinterpret_cast<double *>(a.out) + eg;
            if (v1)
              __stcs(reinterpret_cast<double2 *>(out), make_double2(r0, r1));
            else if (v0)
              *out = r0;
          }
          }
        }
      }
      __syncwarp();
    }
    if (valid) {
      const uint64_t pos_end = ((uint64_t)(src - pw) << 5) - 32 - (uint64_t)nb;
      if (pos_end != endp || pos_end > a.payload_bits) bad = true;
    }
  }
  if (bad) report_format_error(a);
  const unsigned long long ws = warp_sum(nonzero), wm = warp_sum(markers);
  if (lane == 0) {
    if (ws) atomicAdd(a.nonzero, ws);
    if (wm) atomicAdd(a.markers, wm);
  }
}

template __global__ void k4w_decode<0, 16, false>(DecodeArgs);
template __global__ void k4w_decode<1, 16, false>(DecodeArgs);
template __global__ void k4w_decode<0, 32, false>(DecodeArgs);
template __global__ void k4w_decode<1, 32, false>(DecodeArgs);
template __global__ void k4w_decode<2, 32, false>(DecodeArgs);
template __global__ void k4w_decode<0, 16, true>(DecodeArgs);
template __global__ void k4w_decode<1, 16, true>(DecodeArgs);

}  // namespace actc
