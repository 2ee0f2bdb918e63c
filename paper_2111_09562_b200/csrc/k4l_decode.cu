// K4L: lane-serial canonical-Huffman decode fused with the inverse Lorenzo
// reconstruction, outlier splice and re-zero filter, for streams that carry
// the device-side decode index (bit offset + lattice value before every
// ACTC_CHUNK-th symbol, recorded at compress time).
//
// Replaces huffman_decode/_decode_bits (huffman.py:120-142, 210-236), the
// marker check (codec.py:356-359), lorenzo_decode (codec.py:275-293) and
// recon / splice / re-zero (codec.py:360-369).
//
// Work unit: a warp owns 32 consecutive chunks (4096 symbols); lane l decodes
// chunk l sequentially.  The decode is bound by the L1 data pipe (shared and
// global wavefronts), then by instruction issue, so both are budgeted per
// symbol:
//
//   window W     two payload words from the lane's ring    2 LDS (conflict-free)
//   entry e      T1[W >> 20] (4 B)                         1 LDS (random banks)
//   advance      pos += e                                  IADD (len in e's low bits)
//   delta        the int16 canonical delta at
//                ((e >> 16) + (W >> (32 - len))) mod 2^16     LDS.S16
//   value        P += delta; fp32(fp64(P) * 2eb)           IADD, I2F, DMUL, F2F
//   store        16 B per 4 values into a swizzled box     STS.128
//
// T1 entry (kernels.cuh, k4l_table_rows): bits 0-4 the code length (0: slow
// path), bits 16-31 (base[len] - first[len]) mod 2^16 (or, slow path, the
// shortest length a code under the prefix can have).  `pos` holds the
// chunk's bit position in its low 15 bits (a chunk spans < 2^13 bits), so
// `pos += e` advances it by len and lets the rest of e spill into bits >= 15.
// Wide alphabets keep the deltas of their leading canonical indices in
// shared memory (the shared memory the warps leave) and read the tail from
// the global canonical table.
//
// Payload staging: each lane streams its own chunk through a 32-word ring in
// shared memory, layout [slot][lane] (a warp's ring reads are conflict-free),
// with a mirror of slot 0 behind slot 31 so the window's second word is always
// at +128 B.  Words are fetched 32 B per lane per load (LDG.256, one sector),
// byte-swapped once, issued a round ahead and never past the chunk's end.
//
// Output: lanes store their values into a per-warp 32-row x 64-B box
// (hardware 64-B swizzle, conflict-free STS.128), and one lane hands every
// box (two rounds) to the tensor memory accelerator (cp.async.bulk.tensor
// store): the transposition to the tensor's layout costs no load wavefronts
// and no uncoalesced global stores.
#include <cuda.h>

#include <type_traits>

#include "kernels.cuh"

namespace actc {

namespace {

constexpr int kRingSlots = 32;                              // payload words per lane in the ring
constexpr int kRingBytesPerWarp = (kRingSlots + 1) * 128;   // + the mirror of slot 0
constexpr int kBoxBytes = 32 * 64;                          // one TMA box: 32 chunk rows x 64 B
constexpr int kOutBytesPerWarp = kBoxBytes;                 // one box per warp (its store is read out long before the box is refilled)
constexpr uint32_t kSeedGroups = 3;  // 32-B groups staged at a chunk's start
constexpr uint32_t kNeed = 15;       // words past a round's first word it may touch
constexpr uint32_t kTopUp = 17;      // ... staged by the rare synchronous top-up
constexpr uint32_t kAhead = 24;      // refill while staged words <= round word + kAhead
constexpr uint32_t kPosMask = 0x7FFFu;

static_assert(kSeedGroups == 3 && 8 * kSeedGroups >= 7 + kTopUp, "seed covers the first round");
static_assert(kAhead + 8 <= kRingSlots, "refill never overwrites a word still needed");

__device__ __forceinline__ uint32_t shr_clamp(uint32_t x, uint32_t n) {  // x >> n, 0 for n >= 32
  uint32_t r;
  asm("shr.b32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(n));
  return r;
}

__device__ __forceinline__ uint64_t k4l_bits64(const uint32_t *__restrict__ pw, uint64_t pos, uint64_t nwords) {
  const uint64_t wi = pos >> 5;
  if (wi + 3 > nwords) return 0;  // past the buffer (a corrupt stream): no code matches
  const unsigned sh = pos & 31;
  const uint64_t hi = ((uint64_t)bswap32(__ldg(pw + wi)) << 32) | bswap32(__ldg(pw + wi + 1));
  if (!sh) return hi;
  const uint32_t lo = bswap32(__ldg(pw + wi + 2));
  return (hi << sh) | ((uint64_t)lo >> (32 - sh));
}

template <int MODE>
struct OutT;
template <>
struct OutT<0> {
  typedef float T;
};
template <>
struct OutT<1> {
  typedef double T;
};
template <>
struct OutT<2> {
  typedef uint32_t T;
};

// shared-window address kept in a register (otherwise the compiler rebuilds
// it from SR_CgaCtaId at every access inside the decode loop)
__device__ __forceinline__ uint32_t k4l_saddr(const void *p) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mov.u32 %0, %1;" : "=r"(r) : "r"(a));
  return r;
}
// ring reads (volatile: ordered after the lane's own ring stores)
__device__ __forceinline__ uint32_t k4l_lds(uint32_t addr) {
  uint32_t v;
  asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
// read-only tables (written before the __syncthreads ahead of the tile loop)
__device__ __forceinline__ uint32_t k4l_lds_t(uint32_t addr) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ int k4l_lds_s16(uint32_t addr) {
  int v;
  asm("ld.shared.s16 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}
__device__ __forceinline__ int k4l_lds_s16_if(uint32_t addr, int v, bool on) {
  asm("{\n\t.reg .pred p;\n\tsetp.ne.u32 p, %2, 0;\n\t@p ld.shared.s16 %0, [%1];\n\t}"
      : "+r"(v)
      : "r"(addr), "r"((uint32_t)on));
  return v;
}
__device__ __forceinline__ void k4l_sts(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
struct U8 {
  uint32_t w[8];
};
// one 32-B sector, predicated (r keeps its value when !on)
__device__ __forceinline__ void k4l_ldg256_if(U8 &r, const unsigned char *p, bool on) {
  asm volatile(
      "{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %9, 0;\n\t"
      "@q ld.global.nc.L1::no_allocate.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n\t}"
      : "+r"(r.w[0]), "+r"(r.w[1]), "+r"(r.w[2]), "+r"(r.w[3]), "+r"(r.w[4]), "+r"(r.w[5]), "+r"(r.w[6]),
        "+r"(r.w[7])
      : "l"(p), "r"((uint32_t)on));
}

}  // namespace

__global__ void k4l_build_table(const uint32_t *__restrict__ len_counts, const uint32_t *__restrict__ canon,
                                uint32_t radius, uint32_t *__restrict__ table) {
  k4l_table_rows(len_counts, canon, radius, table, blockIdx.x);
}

struct K4LShared {
  unsigned long long first[64];
  uint32_t count[64], base[64];
  uint32_t maxlen;
};

// per-lane decode state of one chunk
template <bool NARROW>
struct K4LLane {
  typedef typename std::conditional<NARROW, int, long long>::type Lat;
  uint32_t pos;   // bit position relative to the ring origin (low 15 bits)
  uint32_t G;     // 32-B groups staged or in flight
  uint32_t pend;  // a group was issued at the last round start (landing now)
  U8 p;
  Lat P;
  uint32_t ordn;
  bool ord_known;
};

// the lane's payload ring (layout [slot][lane], slot 32 mirrors slot 0)
struct K4LRing {
  uint32_t base;             // shared address of this lane's slot 0
  const unsigned char *src;  // the ring origin: the 32-B sector holding the chunk's first bit
  uint32_t endg;             // groups up to the chunk's end (loads stop there)
  __device__ __forceinline__ void load_if(U8 &v, uint32_t g, bool on) const { k4l_ldg256_if(v, src + 32ull * g, on); }
  // group g's words into slots 8g .. 8g+7 (mod 32), big-endian -> value order
  __device__ __forceinline__ void store(uint32_t g, const U8 &v) const {
    const uint32_t s0 = (8u * g) & (kRingSlots - 1);
    const uint32_t ad = base + s0 * 128u;
    const uint32_t w0 = bswap32(v.w[0]);
    k4l_sts(ad, w0);
#pragma unroll
    for (int k = 1; k < 8; k++) k4l_sts(ad + 128u * k, bswap32(v.w[k]));
    if (s0 == 0) k4l_sts(base + kRingSlots * 128u, w0);
  }
  // the 32-bit window at bit position pos (relative)
  __device__ __forceinline__ uint32_t window(uint32_t pos) const {
    const uint32_t ad = base + ((pos & 0x3E0u) << 2);
    const uint32_t w0 = k4l_lds(ad), w1 = k4l_lds(ad + 128u);
    return __funnelshift_l(w1, w0, pos);  // shift = pos & 31
  }
};

// Refill at a round's start: store the group that landed, top up
// synchronously if a run of long codes got ahead of the staging (rare), and
// issue the next load (at most one group; it lands by the next round).
// Groups past the chunk's end are counted as staged without a load (the
// window's look-ahead bits past the last code never decide a code).
template <bool NARROW>
__device__ __forceinline__ void k4l_refill(const K4LRing &rg, K4LLane<NARROW> &L) {
  if (L.pend) rg.store(L.G - 1, L.p);
  const uint32_t aw = (L.pos & kPosMask) >> 5;
  if (8u * L.G < aw + kNeed) {
    while (8u * L.G < aw + kTopUp) {
      if (L.G < rg.endg) {
        U8 t = {};
        rg.load_if(t, L.G, true);
        rg.store(L.G, t);
      }
      L.G++;
    }
  }
  const bool want = 8u * L.G <= aw + kAhead;
  L.pend = want && L.G < rg.endg;
  rg.load_if(L.p, L.G, L.pend);
  L.G += want;
}

// Phase A's rare path (lane-divergent): the reference's bit rule for a
// prefix the table does not resolve (scan from the prefix's shortest length
// l0; huffman.py:129-141).  Returns {canonical index, length | bad << 31};
// the caller advances the position.
__device__ __forceinline__ uint2 k4l_resolve(const K4LShared &sh, const uint32_t *__restrict__ payload, uint64_t nwords,
                                          uint32_t live, uint64_t abs_pos, uint32_t W, uint32_t l0) {
  const int maxlen = (int)sh.maxlen;
  int l = max(1, (int)l0);
  uint32_t ci = 0, len = 0, bad = 0;
  for (; l <= min(maxlen, 32); l++) {
    const uint32_t code = shr_clamp(W, 32u - (uint32_t)l);
    if ((unsigned long long)code >= sh.first[l] && code - (uint32_t)sh.first[l] < sh.count[l]) {
      ci = sh.base[l] + (code - (uint32_t)sh.first[l]);
      len = (uint32_t)l;
      break;
    }
  }
  if (!len && maxlen > 32) {
    // codes longer than 32 bits: a 64-bit window from the payload
    const uint64_t win = k4l_bits64(payload, abs_pos, nwords);
    for (l = max(l, 33); l <= maxlen; l++) {
      const unsigned long long cd = win >> (64 - l), of = cd - sh.first[l];
      if (of < sh.count[l]) {
        ci = sh.base[l] + (uint32_t)of;
        len = (uint32_t)l;
        break;
      }
    }
  }
  if (!len) {
    bad = 1u;  // invalid code (-2), or a stream cut short
    len = 1;
  }
  return make_uint2(min(ci, live - 1), len | (bad << 31));
}

// Phase B's rare path: an outlier marker.  The chain rebases on
// prequantize(value) and the value is spliced, then re-zeroed
// (codec.py:286-292, 356-368); the marker must sit at the next stored index.
template <bool NARROW>
__device__ __forceinline__ double k4l_marker(const DecodeArgs &a, K4LLane<NARROW> &L, uint64_t e_idx, uint64_t e0,
                                             bool &bad, unsigned long long &markers) {
  if (!L.ord_known) {
    uint64_t lo = 0, hi = a.k;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (a.out_idx[mid] < e0) lo = mid + 1; else hi = mid;
    }
    L.ordn = (uint32_t)lo;
    L.ord_known = true;
  }
  float ov = 0.0f;
  if (L.ordn >= a.k || a.out_idx[L.ordn] != e_idx) bad = true;
  else ov = a.out_val[L.ordn];
  L.ordn++;
  markers++;
  bool dummy;
  L.P = (typename K4LLane<NARROW>::Lat)quant_exact((double)ov, a.two_eb, a.eb, dummy);
  double rv = (double)ov;
  if (a.preserve && fabs(rv) <= a.eb) rv = 0.0;
  return rv;
}

struct K4LCtx {
  uint32_t t1_s, cd_s;  // shared addresses: prefix table, canonical deltas
  uint32_t obox;        // this warp's output box
  uint64_t nwords;      // payload words incl. the buffers' 32-byte pad
  const CUtensorMap *tm;
};

// decode one lane's chunk (ACTC_CHUNK symbols, or cnt when !FULL) of a
// 32-chunk tile; FULL tiles leave through the TMA boxes, the partial tile
// through plain stores
template <int MODE, bool GCANON, bool FULL, bool NARROW, bool NZ>
__device__ __forceinline__ void k4l_tile(const DecodeArgs &a, const K4LShared &sh, const K4LRing &rg,
                                         const K4LCtx &cx, uint64_t tile, uint32_t cnt, uint64_t e0, uint64_t abs0,
                                         K4LLane<NARROW> &L, unsigned long long &nonzero,
                                         unsigned long long &markers, bool &bad) {
  typedef typename OutT<MODE>::T T;
  constexpr int VPU = 16 / (int)sizeof(T);  // values per 16-B unit
  constexpr int R = 2 * VPU;                // symbols per lane per round (32 B)
  const int lane = threadIdx.x & 31;
  const int radius = (int)a.radius;
  const double two_eb = a.two_eb;
  // this lane's row of the boxes, and the 64-B swizzle of its 16-B units
  const uint32_t myrow = cx.obox + lane * 64u;
  const uint32_t swz = (uint32_t)((lane >> 1) & 3);
  uint32_t nzc = 0;
  for (int r = 0; r < ACTC_CHUNK / R; r++) {
    k4l_refill<NARROW>(rg, L);
    // phase A: the window chain -- R codes resolved to their deltas (the
    // delta lookups hang off the chain: nothing waits on them until phase B)
    int dl[R];
#pragma unroll
    for (int j = 0; j < R; j++) {
      const uint32_t W = rg.window(L.pos);
      uint32_t e = k4l_lds_t(cx.t1_s + ((W >> 20) << 2));
      const bool in = FULL || (uint32_t)(r * R + j) < cnt;
      if (!in) e = 0x8000u;  // past the chunk: no advance in the position's low 15 bits, never the slow path
      uint32_t ci;
      if ((e & 31u) == 0u && in) {
        const uint2 rs = k4l_resolve(sh, a.payload, cx.nwords, a.live, abs0 + (L.pos & kPosMask), W, e >> 16);
        bad |= (rs.y >> 31) != 0u;
        L.pos += rs.y & 0x7FFFFFFFu;
        ci = rs.x;
      } else {
        L.pos += e;
        ci = ((e >> 16) + __funnelshift_l(W, 0u, e)) & 0xFFFFu;  // W >> (32 - len)
      }
      if (GCANON) {
        // the leading (most frequent) canonical indices from shared memory,
        // the tail of a wide alphabet from the global table
        const bool sm = ci < a.cd_lim;
        int g = k4l_lds_s16_if(cx.cd_s + 2u * ci, 0, sm);
        if (!sm) g = (int)__ldg(a.canon + ci) - radius;
        dl[j] = g;
      } else {
        dl[j] = k4l_lds_s16(cx.cd_s + 2u * ci);
      }
      if (!in) dl[j] = 0;
    }
    // phase B: the lattice running sum and the reconstruction.  Outlier
    // markers only occur in streams with outliers (not NARROW); a round
    // holding one is redone with the splice rule.
    T vals[R];
    const typename K4LLane<NARROW>::Lat P0 = L.P;
    const uint32_t nz0 = nzc;
#pragma unroll
    for (int j = 0; j < R; j++) {
      L.P += dl[j];
      if (MODE == 2) {
        vals[j] = (T)(uint32_t)(dl[j] + radius);
      } else {
        vals[j] = (T)__dmul_rn((double)L.P, two_eb);
        if (NZ && (FULL || (uint32_t)(r * R + j) < cnt)) nzc += L.P != 0;
      }
    }
    if (!NARROW && MODE != 2) {
      bool mk = false;
#pragma unroll
      for (int j = 0; j < R; j++) mk |= dl[j] == -radius && (FULL || (uint32_t)(r * R + j) < cnt);
      if (__any_sync(0xffffffffu, mk)) {
        L.P = P0;
        nzc = nz0;
#pragma unroll
        for (int j = 0; j < R; j++) {
          const uint32_t i = (uint32_t)(r * R + j);
          const bool in = FULL || i < cnt;
          uint32_t nzi;
          if (in && dl[j] == -radius) {
            const double rv = k4l_marker<NARROW>(a, L, e0 + i, e0, bad, markers);
            vals[j] = (T)rv;
            nzi = rv != 0.0;
          } else {
            L.P += dl[j];
            vals[j] = (T)__dmul_rn((double)L.P, two_eb);
            nzi = L.P != 0;
          }
          if (NZ && in) nzc += nzi;
        }
      }
    }
    if (FULL) {
      // units 2(r&1), 2(r&1)+1 of this lane's row of the box
      const uint32_t box = 0;
      if ((r & 1) == 0) {
        // the TMA store of the previous box (two rounds ago) must have read it
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncwarp();
      }
#pragma unroll
      for (int u = 0; u < 2; u++) {
        uint4 pk;
        memcpy(&pk, vals + u * VPU, 16);
        const uint32_t unit = ((uint32_t)(2 * (r & 1) + u)) ^ swz;
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(myrow + box + 16u * unit), "r"(pk.x),
                     "r"(pk.y), "r"(pk.z), "r"(pk.w)
                     : "memory");
      }
      if (r & 1) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          const int x = (r >> 1) * (64 / (int)sizeof(T));
          const int y = (int)(tile * 32);
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"((uint64_t)cx.tm),
              "r"(x), "r"(y), "r"(cx.obox + box)
              : "memory");
          asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        }
      }
    } else {
      T *dst = reinterpret_cast<T *>(a.out) + e0 + (uint64_t)r * R;
#pragma unroll
      for (int j = 0; j < R; j++)
        if ((uint32_t)(r * R + j) < cnt) dst[j] = vals[j];
    }
  }
  if (NZ) nonzero += nzc;
}

template <int MODE, bool GCANON, bool NZ>
__global__ void __launch_bounds__(K4L_THREADS, 1) k4l_decode(DecodeArgs a, const __grid_constant__ CUtensorMap tm) {
  const int NW = blockDim.x >> 5;  // warps per CTA (fewer for small streams or big delta tables)
  extern __shared__ __align__(1024) unsigned char k4l_sm[];
  // boxes first, on a 1024-B boundary (the 64-B swizzle atom spans 512 B)
  unsigned char *obox = k4l_sm + ((1024u - (k4l_saddr(k4l_sm) & 1023u)) & 1023u);
  unsigned char *t1 = obox + NW * kOutBytesPerWarp;
  unsigned char *ring = t1 + kLutSize * 4;
  int16_t *cdelta = reinterpret_cast<int16_t *>(ring + NW * kRingBytesPerWarp);
  __shared__ K4LShared sh;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (int i = tid; i < kLutSize / 4; i += blockDim.x)
    reinterpret_cast<uint4 *>(t1)[i] = __ldg(reinterpret_cast<const uint4 *>(a.lut) + i);
  const int radius = (int)a.radius;
  {
    // canonical deltas (symbol - radius; the outlier marker is -radius) of
    // every code, or (wide alphabets) of the leading cd_lim codes
    // (four 16-B loads in flight per thread)
    const uint32_t live = GCANON ? a.cd_lim : a.live;
    const uint32_t step = 4 * blockDim.x;
    for (uint32_t i0 = 4 * tid; i0 < live; i0 += 4 * step) {
      uint4 c[4];
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const uint32_t i = i0 + u * step;
        c[u] = i + 4 <= live ? __ldg(reinterpret_cast<const uint4 *>(a.canon + i)) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 4; u++) {
        const uint32_t i = i0 + u * step;
        if (i + 4 <= live) {
          const uint32_t lo = ((uint32_t)(c[u].x - radius) & 0xFFFFu) | ((uint32_t)(c[u].y - radius) << 16);
          const uint32_t hi = ((uint32_t)(c[u].z - radius) & 0xFFFFu) | ((uint32_t)(c[u].w - radius) << 16);
          *reinterpret_cast<uint2 *>(cdelta + i) = make_uint2(lo, hi);
        } else {
          for (uint32_t k = i; k < live; k++) cdelta[k] = (int16_t)((int)a.canon[k] - radius);
        }
      }
    }
  }
  stage_len_counts(sh.count, a.len_counts);
  __syncthreads();
  if (tid == 0) {
    unsigned long long code = 0;
    uint32_t idx = 0, mx = 0;
    for (int l = 0; l < 64; l++) {
      code <<= 1;
      const uint32_t c = sh.count[l];
      sh.first[l] = code;
      sh.base[l] = idx;
      code += c;
      idx += c;
      if (c && l > 0) mx = l;
    }
    sh.maxlen = mx;
  }
  __syncthreads();

  const uint64_t n = a.n;
  const uint64_t nchunks = (n + ACTC_CHUNK - 1) / ACTC_CHUNK;
  const uint64_t ntiles = (nchunks + 31) / 32;
  K4LCtx cx;
  cx.t1_s = k4l_saddr(t1);
  cx.cd_s = k4l_saddr(cdelta);
  cx.obox = k4l_saddr(obox + warp * kOutBytesPerWarp);
  cx.nwords = (a.payload_bits + 31) / 32 + 8;
  cx.tm = &tm;
  const uint32_t rbase = k4l_saddr(ring + warp * kRingBytesPerWarp) + lane * 4u;
  const uint64_t pay = (uint64_t)a.payload;  // byte address of the payload
  unsigned long long nonzero = 0, markers = 0;
  bool bad = false;
  // 32-bit lattice arithmetic: no outliers (no rebase) and 16-bit deltas, so
  // a chunk moves its running value by < 2^22 from a start below 2^30
  const bool narrow_ok = MODE == 2 || (a.k == 0 && radius <= 32768);

  // tile of pass k: k * (grid * NW) + warp * grid + block -- the tiles of a
  // last, partial pass spread over every SM (one SM holding all of them
  // would run alone at the end)
  for (uint64_t tile = (uint64_t)warp * gridDim.x + blockIdx.x; tile < ntiles; tile += (uint64_t)gridDim.x * NW) {
    const uint64_t c = tile * 32 + lane;
    const bool valid = c < nchunks;
    const uint64_t e0 = c * ACTC_CHUNK;
    const uint32_t cnt = valid ? (uint32_t)min((uint64_t)ACTC_CHUNK, n - e0) : 0u;
    const bool full = (tile + 1) * 32 * ACTC_CHUNK <= n;  // warp-uniform
    uint64_t pos0 = 0, endp = 0;
    long long P0 = 0;
    if (valid) {
      pos0 = a.chunk_off[c];
      endp = (c + 1 < nchunks) ? a.chunk_off[c + 1] : a.payload_bits;
      if (MODE != 2) P0 = a.chunk_lat[c];
      if (pos0 > endp || endp > a.payload_bits) {  // a corrupt index: nothing is read past the buffer
        bad = true;
        pos0 = endp = 0;
      }
    }
    const bool narrow = narrow_ok && __all_sync(0xffffffffu, P0 > -(1ll << 30) && P0 < (1ll << 30));
    // the ring origin: the 32-B sector holding the chunk's first bit
    const uint64_t byte0 = pay + (pos0 >> 3);
    const uint64_t org = byte0 & ~31ull;
    const uint32_t rel0 = (uint32_t)(((byte0 - org) << 3) + (pos0 & 7));  // pos0 relative to the origin
    K4LRing rg;
    rg.base = rbase;
    rg.src = reinterpret_cast<const unsigned char *>(org);
    rg.endg = (uint32_t)((rel0 + (endp - pos0) + 255) >> 8);
    const uint64_t abs0 = pos0 - rel0;  // payload bit position of the origin (mod 2^64)
    uint64_t pos_end;
#define K4L_RUN(FULLV, NARROWV)                                                                              \
  {                                                                                                        \
    K4LLane<NARROWV> L;                                                                                    \
    L.pos = rel0;                                                                                          \
    {                                                                                                      \
      U8 s0 = {}, s1 = {}, s2 = {}; /* groups past the chunk's end are not loaded (don't-care words) */   \
      rg.load_if(s0, 0, 0 < rg.endg);                                                                      \
      rg.load_if(s1, 1, 1 < rg.endg);                                                                      \
      rg.load_if(s2, 2, 2 < rg.endg);                                                                      \
      rg.store(0, s0);                                                                                     \
      rg.store(1, s1);                                                                                     \
      rg.store(2, s2);                                                                                     \
    }                                                                                                      \
    L.G = kSeedGroups;                                                                                     \
    L.pend = 0;                                                                                            \
    L.p = U8{};                                                                                            \
    L.P = (typename K4LLane<NARROWV>::Lat)P0;                                                              \
    L.ordn = 0;                                                                                            \
    L.ord_known = false;                                                                                   \
    k4l_tile<MODE, GCANON, FULLV, NARROWV, NZ>(a, sh, rg, cx, tile, cnt, e0, abs0, L, nonzero, markers, bad); \
    pos_end = abs0 + (L.pos & kPosMask);                                                                   \
  }
    if (full && narrow) K4L_RUN(true, true)
    else if (full) K4L_RUN(true, false)
    else K4L_RUN(false, false)
#undef K4L_RUN
    if (valid && pos_end != endp) bad = true;
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  if (bad) report_format_error(a);
  const unsigned long long ws = NZ ? warp_sum(nonzero) : 0ull, wm = warp_sum(markers);
  if (lane == 0) {
    if (ws) atomicAdd(a.nonzero, ws);
    if (wm) atomicAdd(a.markers, wm);
    if (wm && a.mcount) atomicAdd(a.mcount, wm);
  }
  // the last CTA checks that every stored outlier met its marker
  // (codec.py:356-359: the marker positions must equal the stored indices)
  if (a.mcount && MODE != 2) {
    __shared__ unsigned s_last;
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      s_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (s_last && tid == 0) {
      __threadfence();
      const unsigned long long tot = atomicAdd(a.mcount, 0ull);
      if (tot != a.k) report_format_error(a);
      *a.mcount = 0;  // self-resetting for the next launch on this context
      *a.ticket = 0;
    }
  }
}

// dynamic shared memory of a launch with `warps` warps and the deltas of
// `cd_entries` canonical indices
size_t k4l_smem_bytes(uint32_t cd_entries, int warps) {
  return 1024 + (size_t)warps * (kOutBytesPerWarp + kRingBytesPerWarp) + (size_t)kLutSize * 4 +
         (((size_t)cd_entries * 2 + 15) & ~(size_t)15);
}
// warps per CTA: as many as `dyn_max` bytes of dynamic shared memory hold
// (up to K4L_THREADS / 32)
int k4l_max_warps(uint32_t cd_entries, size_t dyn_max) {
  const size_t fixed = k4l_smem_bytes(cd_entries, 0);
  if (dyn_max <= fixed) return 0;
  const size_t per = kOutBytesPerWarp + kRingBytesPerWarp;
  return (int)std::min<size_t>((size_t)(K4L_THREADS / 32), (dyn_max - fixed) / per);
}

template __global__ void k4l_decode<0, false, false>(DecodeArgs, const __grid_constant__ CUtensorMap);
template __global__ void k4l_decode<0, false, true>(DecodeArgs, const __grid_constant__ CUtensorMap);
template __global__ void k4l_decode<1, false, false>(DecodeArgs, const __grid_constant__ CUtensorMap);
template __global__ void k4l_decode<1, false, true>(DecodeArgs, const __grid_constant__ CUtensorMap);
template __global__ void k4l_decode<0, true, false>(DecodeArgs, const __grid_constant__ CUtensorMap);
template __global__ void k4l_decode<0, true, true>(DecodeArgs, const __grid_constant__ CUtensorMap);
template __global__ void k4l_decode<1, true, false>(DecodeArgs, const __grid_constant__ CUtensorMap);
template __global__ void k4l_decode<1, true, true>(DecodeArgs, const __grid_constant__ CUtensorMap);
template __global__ void k4l_decode<2, true, false>(DecodeArgs, const __grid_constant__ CUtensorMap);

}  // namespace actc
