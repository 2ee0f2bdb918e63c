// K3: canonical-Huffman encode + MSB-first bit packing + outlier
// extraction + decode chunk index, as reduce-then-scan:
//
//   k3_count   each CTA owns a contiguous range of tiles; sums code lengths
//              and outlier markers of its range (symbols read once)
//   k_excl_scan_u64   tiny scan of the per-CTA totals -> each CTA's first
//              bit / first outlier rank
//   k3_pack    each CTA re-walks its range with its exact start bit:
//              (code, len) from a shared-memory copy of the code table
//              (live symbol range), block scan, codes packed into a shared
//              word buffer (plain stores for words a thread owns, atomicOr
//              for the two it shares), big-endian word stores (byte order ==
//              np.packbits, huffman.py:206).  The partial word between two
//              tiles of one CTA is carried in shared memory; the first/last
//              word of each CTA go to side slots merged by
//   k3_fixup   one CTA, one thread per CTA boundary.
// No CTA ever waits on another, so there is no look-back latency on the
// critical path.  Replaces huffman.py:188-207 and codec.py:321-322.
#include "kernels.cuh"

namespace actc {

namespace {

template <bool WIDE>
struct Ent;
template <>
struct Ent<false> {
  using T = uint32_t;
};
template <>
struct Ent<true> {
  using T = unsigned long long;
};

struct Packer {
  uint32_t *words;
  uint32_t w;
  uint32_t first_w;
  unsigned long long buf;
  int nb;
  __device__ __forceinline__ void emit(uint32_t v) {
    if (w == first_w)
      atomicOr(&words[w], v);
    else
      words[w] = v;  // fully owned by this thread
    w++;
  }
  __device__ __forceinline__ void put(uint32_t code, int len) {  // len <= 32, nb <= 31
    buf |= (unsigned long long)code << (64 - nb - len);
    nb += len;
    if (nb >= 32) {
      emit((uint32_t)(buf >> 32));
      buf <<= 32;
      nb -= 32;
    }
  }
  __device__ __forceinline__ void finish() {
    if (nb > 0) atomicOr(&words[w], (uint32_t)(buf >> 32));
  }
};

template <typename SymT>
__device__ __forceinline__ void load_syms(const SymT *__restrict__ sym, uint64_t base, uint64_t n,
                                          uint32_t (&s)[K3_EPT]) {
  if (base + K3_EPT <= n) {
    if (sizeof(SymT) == 2) {
      const uint4 *p = reinterpret_cast<const uint4 *>(sym + base);
#pragma unroll
      for (int j = 0; j < K3_EPT / 8; j++) {
        uint4 v = __ldg(p + j);
        uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; k++) {
          s[8 * j + 2 * k] = w4[k] & 0xFFFFu;
          s[8 * j + 2 * k + 1] = w4[k] >> 16;
        }
      }
    } else {
      const uint4 *p = reinterpret_cast<const uint4 *>(sym + base);
#pragma unroll
      for (int j = 0; j < K3_EPT / 4; j++) {
        uint4 v = __ldg(p + j);
        s[4 * j] = v.x; s[4 * j + 1] = v.y; s[4 * j + 2] = v.z; s[4 * j + 3] = v.w;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < K3_EPT; j++) s[j] = (base + j < n) ? (uint32_t)sym[base + j] : 0u;
  }
}

template <bool WIDE>
__device__ __forceinline__ void load_table(typename Ent<WIDE>::T *sh, const unsigned long long *__restrict__ ctab,
                                           uint32_t win_lo, uint32_t win_n) {
  for (uint32_t i = threadIdx.x; i < win_n; i += blockDim.x) {
    unsigned long long e = ctab[win_lo + i];
    if (WIDE)
      sh[i] = (typename Ent<WIDE>::T)e;
    else
      sh[i] = (typename Ent<WIDE>::T)(((e >> 8) << 6) | (e & 63));  // (code << 6) | len
  }
}

template <bool WIDE>
__device__ __forceinline__ void lookup(const typename Ent<WIDE>::T *sh, const unsigned long long *__restrict__ ctab,
                                       uint32_t win_lo, uint32_t win_n, uint32_t s, unsigned long long &code,
                                       uint32_t &len) {
  const uint32_t wi = s - win_lo;
  if (WIDE) {
    unsigned long long e = wi < win_n ? (unsigned long long)sh[wi] : __ldg(&ctab[s]);
    len = (uint32_t)(e & 0xFF);
    code = e >> 8;
  } else {
    uint32_t e;
    if (wi < win_n) {
      e = (uint32_t)sh[wi];
    } else {
      unsigned long long g = __ldg(&ctab[s]);
      e = (uint32_t)(((g >> 8) << 6) | (g & 63));
    }
    len = e & 63;
    code = e >> 6;
  }
}

}  // namespace

template <typename SymT, bool WIDE>
__global__ void __launch_bounds__(K3_THREADS) k3_count(const SymT *__restrict__ sym, uint64_t n,
                                                       const unsigned long long *__restrict__ ctab,
                                                       uint32_t win_lo, uint32_t win_n, uint64_t tiles_per_cta,
                                                       unsigned long long *__restrict__ cta_bits,
                                                       unsigned long long *__restrict__ cta_nz) {
  // code lengths only: one byte per symbol of the window (whole 64K alphabet fits)
  extern __shared__ __align__(16) unsigned char len8[];
  __shared__ unsigned long long wb[K3_THREADS / 32], wz[K3_THREADS / 32];
  for (uint32_t i = threadIdx.x; i < win_n; i += K3_THREADS) len8[i] = (unsigned char)(ctab[win_lo + i] & 0xFF);
  __syncthreads();
  const uint64_t ntiles = (n + K3_TILE - 1) / K3_TILE;
  const uint64_t t0 = blockIdx.x * tiles_per_cta, t1 = min(ntiles, t0 + tiles_per_cta);
  uint32_t bits = 0, nz = 0;  // per tile <= 16 * 63 bits, flushed to 64-bit per tile
  unsigned long long bits64 = 0, nz64 = 0;
  for (uint64_t tile = t0; tile < t1; tile++) {
    const uint64_t base = tile * K3_TILE + (uint64_t)threadIdx.x * K3_EPT;
    uint32_t s[K3_EPT];
    load_syms(sym, base, n, s);
    bits = 0;
    nz = 0;
    if (base + K3_EPT <= n) {
#pragma unroll
      for (int j = 0; j < K3_EPT; j++) {
        const uint32_t wi = s[j] - win_lo;
        bits += wi < win_n ? (uint32_t)len8[wi] : (uint32_t)(__ldg(&ctab[s[j]]) & 0xFF);
        nz += s[j] == 0;
      }
    } else {
#pragma unroll
      for (int j = 0; j < K3_EPT; j++) {
        if (base + j < n) {
          const uint32_t wi = s[j] - win_lo;
          bits += wi < win_n ? (uint32_t)len8[wi] : (uint32_t)(__ldg(&ctab[s[j]]) & 0xFF);
          nz += s[j] == 0;
        }
      }
    }
    bits64 += bits;
    nz64 += nz;
  }
  const unsigned long long vb = warp_sum(bits64), vz = warp_sum(nz64);
  if ((threadIdx.x & 31) == 0) {
    wb[threadIdx.x >> 5] = vb;
    wz[threadIdx.x >> 5] = vz;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long tb = 0, tz = 0;
    for (int w = 0; w < K3_THREADS / 32; w++) {
      tb += wb[w];
      tz += wz[w];
    }
    cta_bits[blockIdx.x] = tb;
    cta_nz[blockIdx.x] = tz;
  }
}

constexpr int PK_EPT = 2 * K3_EPT;  // symbols per thread per pack tile
constexpr int PK_TILE = K3_THREADS * PK_EPT;

template <typename SymT>
__device__ __forceinline__ void load_syms32(const SymT *__restrict__ sym, uint64_t base, uint64_t n,
                                            uint32_t (&s)[PK_EPT]) {
  if (base + PK_EPT <= n) {
    const uint4 *p = reinterpret_cast<const uint4 *>(sym + base);
    if (sizeof(SymT) == 2) {
#pragma unroll
      for (int j = 0; j < PK_EPT / 8; j++) {
        uint4 v = __ldg(p + j);
        uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; k++) {
          s[8 * j + 2 * k] = w4[k] & 0xFFFFu;
          s[8 * j + 2 * k + 1] = w4[k] >> 16;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < PK_EPT / 4; j++) {
        uint4 v = __ldg(p + j);
        s[4 * j] = v.x; s[4 * j + 1] = v.y; s[4 * j + 2] = v.z; s[4 * j + 3] = v.w;
      }
    }
  } else {
#pragma unroll
    for (int j = 0; j < PK_EPT; j++) s[j] = (base + j < n) ? (uint32_t)sym[base + j] : 0xFFFFFFFFu;
  }
}

template <typename SymT, bool WIDE>
__global__ void __launch_bounds__(K3_THREADS) k3_pack(
    const SymT *__restrict__ sym, uint64_t n, const unsigned long long *__restrict__ ctab, uint32_t win_lo,
    uint32_t win_n, uint32_t word_cap, uint64_t tiles_per_cta, const float *__restrict__ x,
    const unsigned long long *__restrict__ cta_bit0, const unsigned long long *__restrict__ cta_nz0,
    uint32_t *__restrict__ payload, unsigned long long *__restrict__ out_idx, float *__restrict__ out_val,
    unsigned long long *__restrict__ chunk_off, uint32_t *__restrict__ head, uint32_t *__restrict__ tail,
    int extract_outliers) {
  // tiles_per_cta counts K3_TILE units (the count pass's granularity); the
  // pack pass walks the same symbol range in PK_TILE steps
  extern __shared__ __align__(16) unsigned char smem[];
  using E = typename Ent<WIDE>::T;
  E *sh = reinterpret_cast<E *>(smem);
  uint32_t *words = reinterpret_cast<uint32_t *>(smem + (((size_t)win_n * sizeof(E) + 15) & ~size_t(15)));
  __shared__ unsigned long long wbuf[K3_THREADS / 32 + 1];
  __shared__ uint32_t s_carry;
  const int tid = threadIdx.x;
  load_table<WIDE>(sh, ctab, win_lo, win_n);
  if (tid == 0) s_carry = 0;
  __syncthreads();
  const uint64_t r0 = min(n, blockIdx.x * tiles_per_cta * (uint64_t)K3_TILE);
  const uint64_t r1 = min(n, (blockIdx.x + 1) * tiles_per_cta * (uint64_t)K3_TILE);
  unsigned long long bit = cta_bit0[blockIdx.x];  // start bit of the current tile
  unsigned long long nzb = cta_nz0[blockIdx.x];
  const unsigned long long cta_start = bit;
  for (uint64_t tb = r0; tb < r1; tb += PK_TILE) {
    const uint64_t base = tb + (uint64_t)tid * PK_EPT;
    const uint64_t lim = min(r1, tb + (uint64_t)PK_TILE);
    uint32_t s[PK_EPT];
    load_syms32(sym, base, lim, s);
    // pass 1: lengths (the table lookup is repeated in pass 2 to save registers)
    uint32_t nbits = 0, nz = 0;
#pragma unroll
    for (int j = 0; j < PK_EPT; j++) {
      if (s[j] != 0xFFFFFFFFu) {
        unsigned long long code;
        uint32_t len;
        lookup<WIDE>(sh, ctab, win_lo, win_n, s[j], code, len);
        nbits += len;
        nz += s[j] == 0;
      }
    }
    unsigned long long tot;
    const unsigned long long excl =
        block_excl_sum<unsigned long long>(((unsigned long long)nbits << 32) | nz, wbuf, &tot);
    const unsigned long long tile_bits = tot >> 32;
    const uint32_t start_off = (uint32_t)(bit & 31);
    const uint32_t nwords = (uint32_t)((start_off + tile_bits + 31) >> 5);
    for (uint32_t i = tid; i < nwords && i < word_cap; i += K3_THREADS) words[i] = 0;
    __syncthreads();
    const unsigned long long my_bit0 = bit + (excl >> 32);
    // decode chunk index: bit offsets of the ACTC_CHUNK-th symbols this thread starts
    if ((base % ACTC_CHUNK) == 0 && base < lim) chunk_off[base / ACTC_CHUNK] = my_bit0;
    if (extract_outliers && nz) {
      unsigned long long o = nzb + (excl & 0xFFFFFFFFull);
#pragma unroll
      for (int j = 0; j < PK_EPT; j++) {
        if (s[j] == 0) {
          out_idx[o] = base + j;
          out_val[o] = x[base + j];
          o++;
        }
      }
    }
    if (nbits) {
      const uint32_t rel = start_off + (uint32_t)(excl >> 32);
      if (!WIDE) {
        // codes <= 26 bits complete at most one word each: predicated emits;
        // only the first (shared with the previous thread) and the final
        // partial word (shared with the next) are atomic
        uint32_t w = rel >> 5;
        const uint32_t w0 = w;
        int nb = rel & 31;
        unsigned long long acc = 0;
#pragma unroll
        for (int j = 0; j < PK_EPT; j++) {
          unsigned long long cj;
          uint32_t lj;
          const bool pad = s[j] == 0xFFFFFFFFu;  // past the range end
          lookup<WIDE>(sh, ctab, win_lo, win_n, pad ? win_lo : s[j], cj, lj);
          if (pad) lj = 0;
          acc |= lj ? cj << (64 - nb - (int)lj) : 0ull;
          nb += (int)lj;
          const bool ready = nb >= 32;
          const uint32_t hiw = (uint32_t)(acc >> 32);
          if (ready && w == w0) atomicOr(&words[w], hiw);
          if (ready && w != w0) words[w] = hiw;
          acc = ready ? (acc << 32) : acc;
          nb = ready ? nb - 32 : nb;
          w += ready;
        }
        if (nb > 0) atomicOr(&words[w], (uint32_t)(acc >> 32));
      } else {
        Packer pk;
        pk.words = words;
        pk.w = rel >> 5;
        pk.first_w = pk.w;
        pk.nb = rel & 31;
        pk.buf = 0;
#pragma unroll
        for (int j = 0; j < PK_EPT; j++) {
          if (s[j] == 0xFFFFFFFFu) continue;
          unsigned long long cj;
          uint32_t lj;
          lookup<WIDE>(sh, ctab, win_lo, win_n, s[j], cj, lj);
          if (lj > 32) {
            pk.put((uint32_t)(cj >> 32), (int)lj - 32);
            pk.put((uint32_t)cj, 32);
          } else {
            pk.put((uint32_t)cj, (int)lj);
          }
        }
        pk.finish();
      }
    }
    __syncthreads();
    // word 0 continues the previous tile's partial word; the CTA's very first
    // word and its final partial word go to the side slots
    const bool first_tile = tb == r0, last_tile = tb + PK_TILE >= r1;
    const uint32_t end_off = (uint32_t)((start_off + tile_bits) & 31);
    if (tid == 0 && !first_tile) words[0] |= s_carry;
    __syncthreads();
    const uint64_t gw0 = bit >> 5;
    const bool head_word = first_tile && ((cta_start & 31) != 0 || nwords == 1);
    const uint32_t wlo = head_word ? 1 : 0;
    const uint32_t whi = end_off ? nwords - 1 : nwords;  // last partial word is carried
    for (uint32_t i = wlo + tid; i < whi; i += K3_THREADS) payload[gw0 + i] = bswap32(words[i]);
    __syncthreads();
    if (tid == 0) {
      if (head_word) head[blockIdx.x] = words[0];
      uint32_t carry = end_off ? words[nwords - 1] : 0u;
      if (head_word && nwords == 1) carry = 0;  // already in head
      s_carry = carry;
      if (last_tile) tail[blockIdx.x] = carry;
    }
    bit += tile_bits;
    nzb += tot & 0xFFFFFFFFull;
    __syncthreads();
  }
}

// Merge the CTA boundary words: head[b] goes into the word holding CTA b's
// first bit, tail[b] into the word holding its last bit (both partial).
__global__ void k3_fixup(uint32_t *__restrict__ payload, const unsigned long long *__restrict__ cta_bit0,
                         const unsigned long long *__restrict__ cta_bits, const uint32_t *__restrict__ head,
                         const uint32_t *__restrict__ tail, uint32_t ncta) {
  // pass 1: zero every word a side slot lands in; pass 2: OR the slots in
  for (int pass = 0; pass < 2; pass++) {
    for (uint32_t b = threadIdx.x; b < ncta; b += blockDim.x) {
      const unsigned long long s = cta_bit0[b], nb = cta_bits[b];
      if (!nb) continue;
      const unsigned long long e = s + nb;
      const uint64_t wf = s >> 5, wl = (e - 1) >> 5;
      const bool has_head = (s & 31) != 0 || wf == wl;
      const bool has_tail = (e & 31) != 0 && !(wf == wl && has_head);
      if (pass == 0) {
        if (has_head) payload[wf] = 0;
        if (has_tail) payload[wl] = 0;
      } else {
        if (has_head) atomicOr(&payload[wf], bswap32(head[b]));
        if (has_tail) atomicOr(&payload[wl], bswap32(tail[b]));
      }
    }
    __syncthreads();
  }
}

#define K3_INST(T, W)                                                                                          \
  template __global__ void k3_count<T, W>(const T *, uint64_t, const unsigned long long *, uint32_t, uint32_t, \
                                          uint64_t, unsigned long long *, unsigned long long *);                 \
  template __global__ void k3_pack<T, W>(const T *, uint64_t, const unsigned long long *, uint32_t, uint32_t,  \
                                         uint32_t, uint64_t, const float *, const unsigned long long *,         \
                                         const unsigned long long *, uint32_t *, unsigned long long *, float *, \
                                         unsigned long long *, uint32_t *, uint32_t *, int);
K3_INST(uint16_t, false)
K3_INST(uint16_t, true)
K3_INST(uint32_t, false)
K3_INST(uint32_t, true)

}  // namespace actc
