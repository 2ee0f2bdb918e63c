// K4x: lane-per-chunk canonical-Huffman decode fused with the *sequential*
// inverse Lorenzo reconstruction (indexed streams).
//
// Replaces huffman_decode/_decode_bits (huffman.py:120-142, 210-236), the
// marker check (codec.py:356-359), lorenzo_decode (codec.py:275-293) and
// recon / splice / re-zero (codec.py:360-369).
//
// Lane l of the grid owns chunk c (ACTC_CHUNK symbols, bit offset and
// starting lattice value from the device index): it decodes its symbols,
// keeps the running lattice value P in a register (the inverse Lorenzo of a
// chunk is a sequential sum), reconstructs fp64(P)*2eb and stores 4 values
// at a time.  No shared-memory row buffers and no warp scans: the only
// shared state is the decode tables, so many warps fit per SM.
//
// Decode step (identical for every lane): an 12-bit prefix table gives the
// code length l0 of short codes, or the shortest length of the long codes
// behind the prefix; three comparisons of the left-aligned 32-bit window W
// with the canonical limits finish the length (they are all false for a
// short code), and the canonical index is off[l] + (W >> (32 - l)).  The
// table holds 0 for prefixes whose codes span more than four lengths and for
// invalid prefixes: those lanes take the reference's bit-serial rule
// (warp-voted, rare).  Canonical index -> symbol comes from a shared cache of
// the first kXCache canonical entries (the most frequent codes) or from L2;
// the lookups of a group of 4 symbols are issued before the next group is
// decoded, so their latency overlaps the decode chain.
#include "kernels.cuh"

namespace actc {

namespace {

static_assert(kXBits == 12, "k4x prefix width");
constexpr int kXCache = 16384;

__device__ __forceinline__ uint64_t x_read_bits64(const uint32_t *__restrict__ pw, uint64_t pos) {
  const uint64_t wi = pos >> 5;
  const unsigned sh = pos & 31;
  const uint64_t hi = ((uint64_t)bswap32(pw[wi]) << 32) | bswap32(pw[wi + 1]);
  if (!sh) return hi;
  const uint32_t lo = bswap32(pw[wi + 2]);
  return (hi << sh) | ((uint64_t)lo >> (32 - sh));
}

// 32-bit shared-window addressing computed once (generic pointers to
// __shared__ arrays make the compiler rebuild the window base from
// SR_CgaCtaId at every access)
__device__ __forceinline__ uint32_t x_saddr(const void *p) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mov.u32 %0, %1;" : "=r"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ uint32_t x_lds_u8(uint32_t a) {
  unsigned short v;
  asm("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t x_lds_u16(uint32_t a) {
  unsigned short v;
  asm("ld.shared.u16 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ uint32_t x_lds_u32(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}

}  // namespace

// u8 length table: lut8[p] = l0 when every code whose left-aligned 32-bit
// value starts with the 12-bit prefix p has length in [l0, l0+3] (maxlen <=
// 32); 0 otherwise (long spread, invalid prefix, or codes > 32 bits).
__global__ void k_build_lut8(const uint32_t *__restrict__ len_counts, uint8_t *__restrict__ lut8) {
  lut8_body(len_counts, lut8, blockIdx.x);
}

template <int MODE>
__global__ void __launch_bounds__(K4X_THREADS) k4x_decode(DecodeArgs a) {
  __shared__ uint8_t s_lut[1 << kXBits];
  __shared__ uint16_t s_cc[kXCache];
  __shared__ uint32_t s_limm1[40];  // W > s_limm1[l]: the code is longer than l
  __shared__ int32_t s_off[36];     // base[l] - first[l]
  __shared__ unsigned long long s_first[64];
  __shared__ uint32_t s_count[64], s_base[64];
  __shared__ uint32_t s_maxlen, s_zci;
  const int tid = threadIdx.x, lane = tid & 31;
  {
    const uint4 *src = reinterpret_cast<const uint4 *>(a.lut);  // the u8 table sits in the LUT buffer
    reinterpret_cast<uint4 *>(s_lut)[tid] = __ldg(src + tid);   // 256 x 16 B = 4 KB
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
      if (l < 40) {
        if (l >= 1 && l <= 32) {
          const unsigned long long lim = (code + c) << (32 - l);
          s_limm1[l] = lim == 0 ? 0u : (uint32_t)min(lim - 1, 0xFFFFFFFFull);
        } else {
          s_limm1[l] = 0xFFFFFFFFu;
        }
      }
      if (l < 36) s_off[l] = (l >= 1 && l <= 32) ? (int32_t)idx - (int32_t)(uint32_t)code : 0;
      code += c;
      idx += c;
      if (c && l > 0) mx = l;
    }
    s_maxlen = mx;
    s_zci = 0xFFFFFFFFu;
  }
  const bool cache16 = 2ull * a.radius <= 65536;
  const uint32_t ncache = cache16 ? min((uint32_t)kXCache, a.live) : 0u;
  for (uint32_t i0 = 4 * tid; i0 < ncache; i0 += 4 * K4X_THREADS) {
    if (i0 + 3 < ncache) {
      const uint4 v = __ldg(reinterpret_cast<const uint4 *>(a.canon + i0));
      reinterpret_cast<uint2 *>(s_cc)[i0 >> 2] = make_uint2(v.x | (v.y << 16), v.z | (v.w << 16));
    } else {
      for (uint32_t i = i0; i < ncache; i++) s_cc[i] = (uint16_t)a.canon[i];
    }
  }
  __syncthreads();
  // canonical index of the outlier marker (symbol 0, only live with outliers)
  if (a.k && tid < 64 && s_count[tid] && a.canon[s_base[tid]] == 0u) s_zci = s_base[tid];
  __syncthreads();
  const uint32_t zci = s_zci;
  const int maxlen = (int)s_maxlen;
  const bool general = !isfinite(a.two_eb);  // 2eb = inf: keep the reference's per-element rules
  const uint64_t nchunks = (a.n + ACTC_CHUNK - 1) / ACTC_CHUNK;
  const long long radius = a.radius;
  const uint32_t *__restrict__ pw = a.payload;
  unsigned long long nonzero = 0, markers = 0;
  bool bad = false;
  const uint32_t lut_s = x_saddr(s_lut), lim_s = x_saddr(s_limm1), off_s = x_saddr(s_off), cc_s = x_saddr(s_cc);
  auto sym_of = [&](uint32_t ci) -> uint32_t { return ci < ncache ? x_lds_u16(cc_s + 2u * ci) : __ldg(&a.canon[ci]); };

  for (uint64_t c = (uint64_t)blockIdx.x * K4X_THREADS + tid; c < nchunks; c += (uint64_t)gridDim.x * K4X_THREADS) {
    const uint64_t e0 = c * ACTC_CHUNK;
    const uint32_t cnt = (uint32_t)min((uint64_t)ACTC_CHUNK, a.n - e0);
    const uint64_t pos0 = a.chunk_off[c];
    const uint64_t endp = (c + 1 < nchunks) ? a.chunk_off[c + 1] : a.payload_bits;
    {
      // this chunk's payload lines: one DRAM round trip for all of them
      const char *pb = reinterpret_cast<const char *>(pw);
      for (uint64_t b = (pos0 >> 3) & ~127ull; b <= (endp >> 3); b += 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(pb + b));
    }
    const uint32_t *__restrict__ src = pw + (pos0 >> 5);
    unsigned long long buf = ((unsigned long long)bswap32(__ldg(src)) << 32) | bswap32(__ldg(src + 1));
    buf <<= (pos0 & 31);
    int nb = 64 - (int)(pos0 & 31);
    uint32_t nextw = __ldg(src + 2);  // raw (big-endian); swapped when consumed
    src += 3;
    long long P = MODE != 2 ? a.chunk_lat[c] : 0;
    uint32_t ord = 0;
    bool ord_known = false;

#define K4X_DEC(CI)                                                                        \
  {                                                                                        \
    if (nb < 32) {                                                                         \
      buf |= (unsigned long long)bswap32(nextw) << (32 - nb);                              \
      nb += 32;                                                                            \
      nextw = __ldg(src);                                                                  \
      ++src;                                                                               \
    }                                                                                      \
    const uint32_t W = (uint32_t)(buf >> 32);                                              \
    const uint32_t l0 = x_lds_u8(lut_s + (W >> (32 - kXBits)));                            \
    const uint32_t lb = lim_s + 4u * l0;                                                   \
    const uint32_t l = l0 + (W > x_lds_u32(lb)) + (W > x_lds_u32(lb + 4u)) + (W > x_lds_u32(lb + 8u)); \
    int len = (int)l;                                                                      \
    CI = x_lds_u32(off_s + 4u * l) + (W >> ((32 - l) & 31));                               \
    {                                                                                      \
      if (l0 == 0) {                                                                       \
        /* rare: codes spanning > 4 lengths behind the prefix, > 32 bits, or invalid */    \
        const uint64_t pos = ((uint64_t)(src - pw) << 5) - 32 - (uint64_t)nb;              \
        const uint64_t win = x_read_bits64(pw, pos);                                       \
        len = 0;                                                                           \
        for (int ll = 1; ll <= maxlen; ll++) {                                             \
          const unsigned long long cd = win >> (64 - ll), of = cd - s_first[ll];           \
          if (of < s_count[ll]) {                                                          \
            CI = s_base[ll] + (uint32_t)of;                                                \
            len = ll;                                                                      \
            break;                                                                         \
          }                                                                                \
        }                                                                                  \
        if (!len) {                                                                        \
          bad = true;                                                                      \
          len = 1;                                                                         \
          CI = 0;                                                                          \
        }                                                                                  \
        const uint64_t np = pos + len;                                                     \
        src = pw + (np >> 5);                                                              \
        buf = ((unsigned long long)bswap32(src[0]) << 32) | bswap32(src[1]);               \
        buf <<= (np & 31);                                                                 \
        nb = 64 - (int)(np & 31);                                                          \
        nextw = src[2];                                                                    \
        src += 3;                                                                          \
        len = 0;                                                                           \
      }                                                                                    \
    }                                                                                      \
    buf <<= len;                                                                           \
    nb -= len;                                                                             \
  }

    // reconstruct one element from its symbol (or outlier marker)
    auto recon = [&](uint32_t ci, uint32_t sv, uint32_t idx) -> double {
      double r;
      if (ci == zci) {
        if (!ord_known) {
          uint64_t lo = 0, hi = a.k;
          while (lo < hi) {
            const uint64_t mid = (lo + hi) >> 1;
            if (a.out_idx[mid] < e0) lo = mid + 1; else hi = mid;
          }
          ord = (uint32_t)lo;
          ord_known = true;
        }
        float ov = 0.0f;
        if (ord >= a.k || a.out_idx[ord] != e0 + idx) bad = true;
        else ov = a.out_val[ord];
        ord++;
        markers++;
        bool dummy;
        P = quant_exact((double)ov, a.two_eb, a.eb, dummy);
        r = (double)ov;
        if (a.preserve && fabs(r) <= a.eb) r = 0.0;
      } else {
        P += (long long)sv - radius;
        r = __dmul_rn((double)P, a.two_eb);
        if (general && a.preserve && fabs(r) <= a.eb) r = 0.0;
      }
      nonzero += (r != 0.0);
      return r;
    };

    uint32_t i = 0;
    if (cnt == ACTC_CHUNK) {
      // full chunk: groups of 4, symbol lookups one group ahead
      uint32_t ci[4], sv[4];
      K4X_DEC(ci[0]) K4X_DEC(ci[1]) K4X_DEC(ci[2]) K4X_DEC(ci[3])
#pragma unroll
      for (int u = 0; u < 4; u++) sv[u] = sym_of(ci[u]);
      for (i = 0; i < ACTC_CHUNK; i += 4) {
        uint32_t cn[4] = {0, 0, 0, 0};
        if (i + 4 < ACTC_CHUNK) {
          K4X_DEC(cn[0]) K4X_DEC(cn[1]) K4X_DEC(cn[2]) K4X_DEC(cn[3])
        }
        if (MODE == 2) {
          *reinterpret_cast<uint4 *>(reinterpret_cast<uint32_t *>(a.out) + e0 + i) = make_uint4(sv[0], sv[1], sv[2], sv[3]);
        } else {
          const double r0 = recon(ci[0], sv[0], i), r1 = recon(ci[1], sv[1], i + 1);
          const double r2 = recon(ci[2], sv[2], i + 2), r3 = recon(ci[3], sv[3], i + 3);
          if (MODE == 0) {
            __stcs(reinterpret_cast<float4 *>(reinterpret_cast<float *>(a.out) + e0 + i),
                   make_float4((float)r0, (float)r1, (float)r2, (float)r3));
          } else {
            double2 *o = reinterpret_cast<double2 *>(reinterpret_cast<double *>(a.out) + e0 + i);
            __stcs(o, make_double2(r0, r1));
            __stcs(o + 1, make_double2(r2, r3));
          }
        }
#pragma unroll
        for (int u = 0; u < 4; u++) {
          ci[u] = cn[u];
          sv[u] = sym_of(cn[u]);
        }
      }
    } else {
      for (i = 0; i < cnt; i++) {
        uint32_t ci;
        K4X_DEC(ci)
        const uint32_t sv = sym_of(ci);
        if (MODE == 2) {
          reinterpret_cast<uint32_t *>(a.out)[e0 + i] = sv;
        } else {
          const double r = recon(ci, sv, i);
          if (MODE == 0) reinterpret_cast<float *>(a.out)[e0 + i] = (float)r;
          else reinterpret_cast<double *>(a.out)[e0 + i] = r;
        }
      }
    }
#undef K4X_DEC
    const uint64_t pos_end = ((uint64_t)(src - pw) << 5) - 32 - (uint64_t)nb;
    if (pos_end != endp || pos_end > a.payload_bits) bad = true;
  }
  if (bad) report_format_error(a);
  const unsigned long long ws = warp_sum(nonzero), wm = warp_sum(markers);
  if (lane == 0) {
    if (ws) atomicAdd(a.nonzero, ws);
    if (wm) atomicAdd(a.markers, wm);
  }
}

template __global__ void k4x_decode<0>(DecodeArgs);
template __global__ void k4x_decode<1>(DecodeArgs);
template __global__ void k4x_decode<2>(DecodeArgs);

}  // namespace actc
