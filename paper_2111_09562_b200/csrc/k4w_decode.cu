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
// a 4 KB per-warp shared buffer (u16 pairs, rows padded to 33 words so lane
// stores and row reads are bank-conflict free); then the warp walks the 32
// rows: a warp inclusive scan of the deltas plus the chunk's running lattice
// value gives 64 consecutive lattice values, reconstructed in fp64 and
// stored coalesced (256 B / 512 B per warp store).  No block barriers, no
// look-back: chunk start values come from the index, so warps run free.
#include "kernels.cuh"

namespace actc {

namespace {

constexpr int ROUND = 64;                  // symbols per lane per round
constexpr int ROW16 = ROUND / 2 + 1;       // words per row, u16 symbols
constexpr int ROW32 = ROUND + 1;           // words per row, u32 symbols
constexpr int NW4 = K4W_THREADS / 32;

struct Tables {
  unsigned long long first[64];
  unsigned long long lim[64];
  uint32_t count[64];
  uint32_t base[64];
  uint32_t maxlen;
  uint32_t n_short;  // number of codes with length <= kLutBits (canon index of the first long code)
};

__device__ __forceinline__ uint64_t read_bits64(const uint32_t *__restrict__ pw, uint64_t pos) {
  uint64_t wi = pos >> 5;
  unsigned sh = pos & 31;
  uint64_t hi = ((uint64_t)bswap32(pw[wi]) << 32) | bswap32(pw[wi + 1]);
  if (!sh) return hi;
  uint32_t lo = bswap32(pw[wi + 2]);
  return (hi << sh) | ((uint64_t)lo >> (32 - sh));
}

// reference first-match rule from memory (over-subscribed tables, codes > 32 bits)
__device__ __forceinline__ int slow_decode(const uint32_t *__restrict__ pw, uint64_t pos, const Tables &t,
                                           const uint32_t *__restrict__ canon, uint32_t &sym) {
  uint64_t win = read_bits64(pw, pos);
  for (int l = kLutBits + 1; l <= (int)t.maxlen; l++) {
    unsigned long long code = win >> (64 - l);
    unsigned long long off = code - t.first[l];
    if (off < t.count[l]) {
      sym = canon[t.base[l] + off];
      return l;
    }
  }
  return 0;
}

}  // namespace

template <int MODE, int SW>
__global__ void __launch_bounds__(K4W_THREADS, 3) k4w_decode(DecodeArgs a) {
  __shared__ uint32_t lut[kLutSize];
  __shared__ uint16_t ccache[K4W_CANON_CACHE];  // canon[n_short ...], the most frequent long codes
  __shared__ Tables t;
  extern __shared__ __align__(16) uint32_t wbuf_all[];  // NW4 * 32 rows
  constexpr int ROW = SW == 16 ? ROW16 : ROW32;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kLutSize / 4; i += K4W_THREADS)
    reinterpret_cast<uint4 *>(lut)[i] = reinterpret_cast<const uint4 *>(a.lut)[i];
  if (tid == 0) {
    unsigned long long code = 0;
    uint32_t idx = 0, mx = 0, ns = 0;
    for (int l = 0; l < 64; l++) {
      code <<= 1;
      uint32_t c = a.len_counts[l];
      t.first[l] = code;
      t.count[l] = c;
      t.base[l] = idx;
      t.lim[l] = l <= 32 ? (code + c) << (32 - l) : 0;
      code += c;
      idx += c;
      if (c && l > 0) mx = l;
      if (l <= kLutBits) ns = idx;
    }
    t.maxlen = mx;
    t.n_short = ns;
  }
  __syncthreads();
  const uint32_t n_short = t.n_short;
  const uint32_t ncache = SW == 16 ? (uint32_t)min((long long)K4W_CANON_CACHE, (long long)a.live - (long long)n_short) : 0u;
  for (uint32_t i = tid; i < ncache; i += K4W_THREADS) ccache[i] = (uint16_t)a.canon[n_short + i];
  __syncthreads();

  const bool fast_long = a.lut[kLutSize] != 0;
  const uint64_t nchunks = (a.n + ACTC_CHUNK - 1) / ACTC_CHUNK;
  const uint64_t nwt = (nchunks + 31) / 32;
  const long long radius = a.radius;
  uint32_t *rows = wbuf_all + warp * 32 * ROW;
  uint32_t *myrow = rows + lane * ROW;
  unsigned long long nonzero = 0, markers = 0;
  bool bad = false;

  for (uint64_t wt = (uint64_t)blockIdx.x * NW4 + warp; wt < nwt; wt += (uint64_t)gridDim.x * NW4) {
    const uint64_t c = wt * 32 + lane;
    const bool valid = c < nchunks;
    const uint64_t e0 = c * ACTC_CHUNK;
    const uint32_t cnt = valid ? (uint32_t)min((uint64_t)ACTC_CHUNK, a.n - e0) : 0u;
    uint64_t pos = 0, endp = 0;
    const uint32_t *pw = a.payload;
    uint64_t wi = 0;
    unsigned long long buf = 0;
    int nb = 0;
    uint32_t nextw = 0;
    long long P = 0;       // running lattice value of my chunk
    uint32_t ordn = 0;     // ordinal of my chunk's next outlier
    bool ord_known = false;
    if (valid) {
      pos = a.chunk_off[c];
      endp = (c + 1 < nchunks) ? a.chunk_off[c + 1] : a.payload_bits;
      wi = pos >> 5;
      // pull the chunk's bitstream lines towards L1 while the first words load
      const char *lp = reinterpret_cast<const char *>(pw + wi);
      for (uint64_t off = 128; off < ((endp - pos) >> 3) + 16; off += 128)
        asm volatile("prefetch.global.L1 [%0];" ::"l"(lp + off));
      buf = ((unsigned long long)bswap32(pw[wi]) << 32) | bswap32(pw[wi + 1]);
      buf <<= (pos & 31);
      nb = 64 - (int)(pos & 31);
      wi += 2;
      nextw = bswap32(pw[wi++]);
      if (MODE != 2) P = a.chunk_lat[c];
    }
    for (int r = 0; r * ROUND < ACTC_CHUNK; r++) {
      // ---------------- decode up to ROUND symbols of my chunk ----------------
      const uint32_t i0 = r * ROUND;
      const uint32_t iend = max(i0, min(cnt, i0 + ROUND));  // empty once the chunk is exhausted
      uint32_t zr = 0;
      // One symbol, straight-line: 12-bit LUT hit, else the LUT gives the
      // first candidate length l0 and up to 4 predicated limit steps finish it
      // (uniform instruction stream across the warp); anything rarer takes the
      // divergent fallback.
#define ACTC_DEC(SYM)                                                                                  \
  {                                                                                                    \
    if (nb < 32) {                                                                                     \
      buf |= (unsigned long long)nextw << (32 - nb);                                                   \
      nb += 32;                                                                                        \
      nextw = bswap32(pw[wi++]);                                                                       \
    }                                                                                                  \
    const uint32_t W = (uint32_t)(buf >> 32);                                                          \
    const uint32_t e = lut[W >> (32 - kLutBits)];                                                      \
    int len = e & 63;                                                                                  \
    uint32_t sv = e >> 6;                                                                              \
    if (len == 0) {                                                                                    \
      int l = (int)sv;                                                                                 \
      if (fast_long && l) {                                                                            \
        l += (unsigned long long)W >= t.lim[l];                                                        \
        l += (unsigned long long)W >= t.lim[l];                                                        \
        l += (unsigned long long)W >= t.lim[l];                                                        \
        while (l <= (int)t.maxlen && (unsigned long long)W >= t.lim[l]) l++;                            \
        if (l <= (int)t.maxlen) {                                                                      \
          const uint32_t ci = t.base[l] + ((W >> (32 - l)) - (uint32_t)t.first[l]);                    \
          sv = (ci - n_short < ncache) ? (uint32_t)ccache[ci - n_short] : __ldg(&a.canon[ci]);          \
          len = l;                                                                                     \
        }                                                                                              \
      }                                                                                                \
      if (len == 0) {                                                                                  \
        const uint64_t pos = (wi << 5) - 32 - (uint64_t)nb;                                            \
        len = slow_decode(pw, pos, t, a.canon, sv);                                                    \
        if (!len) {                                                                                    \
          bad = true;                                                                                  \
          len = 1;                                                                                     \
          sv = a.radius;                                                                               \
        }                                                                                              \
        const uint64_t np = pos + len;                                                                 \
        wi = np >> 5;                                                                                  \
        buf = ((unsigned long long)bswap32(pw[wi]) << 32) | bswap32(pw[wi + 1]);                       \
        buf <<= (np & 31);                                                                             \
        nb = 64 - (int)(np & 31);                                                                      \
        wi += 2;                                                                                       \
        nextw = bswap32(pw[wi++]);                                                                     \
        len = 0;                                                                                       \
      }                                                                                                \
    }                                                                                                  \
    buf <<= len;                                                                                       \
    nb -= len;                                                                                         \
    SYM = sv;                                                                                          \
  }
#define ACTC_ZERO(SYM, IDX)                                                                            \
  if (MODE != 2 && SYM == 0) {                                                                         \
    if (!ord_known) {                                                                                  \
      uint64_t lo = 0, hi = a.k;                                                                       \
      while (lo < hi) {                                                                                \
        uint64_t mid = (lo + hi) >> 1;                                                                 \
        if (a.out_idx[mid] < e0) lo = mid + 1; else hi = mid;                                          \
      }                                                                                                \
      ordn = (uint32_t)lo;                                                                             \
      ord_known = true;                                                                                \
    }                                                                                                  \
    if (ordn >= a.k || a.out_idx[ordn] != e0 + (IDX)) bad = true;                                      \
    ordn++;                                                                                            \
    zr++;                                                                                              \
  }
      uint32_t i = i0;
      for (; i + 1 < iend; i += 2) {
        uint32_t sa, sb;
        ACTC_DEC(sa)
        ACTC_DEC(sb)
        ACTC_ZERO(sa, i)
        ACTC_ZERO(sb, i + 1)
        if (SW == 32) {
          myrow[i - i0] = sa;
          myrow[i - i0 + 1] = sb;
        } else {
          myrow[(i - i0) >> 1] = sa | (sb << 16);
        }
      }
      if (i < iend) {
        uint32_t sa;
        ACTC_DEC(sa)
        ACTC_ZERO(sa, i)
        if (SW == 32)
          myrow[i - i0] = sa;
        else
          myrow[(i - i0) >> 1] = sa;
      }
#undef ACTC_DEC
#undef ACTC_ZERO
      markers += zr;
      // ordinal of my first outlier in this round (valid whenever zr > 0)
      const uint32_t ordr = ordn - zr;
      __syncwarp();
      const unsigned zmask = __ballot_sync(0xffffffffu, zr != 0);

      // ---------------- reconstruct row by row (coalesced) ----------------
      for (int cc = 0; cc < 32; cc++) {
        const uint64_t ch = wt * 32 + cc;
        if (ch >= nchunks) break;
        const uint32_t ccnt = (uint32_t)min((uint64_t)ACTC_CHUNK, a.n - ch * ACTC_CHUNK);
        if (i0 >= ccnt) continue;
        const uint32_t k0 = i0 + 2 * lane;  // element index inside the chunk
        const bool v0 = k0 < ccnt, v1 = k0 + 1 < ccnt;
        uint32_t s0, s1;
        const uint32_t *row = rows + cc * ROW;
        if (SW == 16) {
          const uint32_t w = row[lane];
          s0 = w & 0xFFFFu;
          s1 = w >> 16;
        } else {
          s0 = row[2 * lane];
          s1 = row[2 * lane + 1];
        }
        const uint64_t eg = ch * ACTC_CHUNK + k0;  // global element index
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
          z0 = v0 && s0 == 0;
          z1 = v1 && s1 == 0;
          const int nzl = (int)z0 + (int)z1;
          const int zi = warp_incl_sum(nzl);
          o0 = __shfl_sync(0xffffffffu, ordr, cc) + (uint32_t)(zi - nzl);
          o1 = o0 + (uint32_t)z0;
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
      __syncwarp();
    }
    if (valid) {
      const uint64_t pos_end = (wi << 5) - 32 - (uint64_t)nb;
      if (pos_end != endp || pos_end > a.payload_bits) bad = true;
    }
  }
  if (bad) atomicOr(a.status, (unsigned)ACTC_EFORMAT);
  const unsigned long long ws = warp_sum(nonzero), wm = warp_sum(markers);
  if (lane == 0) {
    if (ws) atomicAdd(a.nonzero, ws);
    if (wm) atomicAdd(a.markers, wm);
  }
}

template __global__ void k4w_decode<0, 16>(DecodeArgs);
template __global__ void k4w_decode<1, 16>(DecodeArgs);
template __global__ void k4w_decode<0, 32>(DecodeArgs);
template __global__ void k4w_decode<1, 32>(DecodeArgs);
template __global__ void k4w_decode<2, 32>(DecodeArgs);

}  // namespace actc
