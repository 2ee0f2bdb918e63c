// K3: canonical-Huffman encode + MSB-first bit packing + outlier
// extraction + decode chunk index.
//
// Replaces huffman_encode's bit expansion and np.packbits
// (huffman.py:188-207) and the outlier gather of compress
// (codec.py:321-322).  One pass over the symbol stream:
//   * per thread: 16 symbols -> (code, len) from a shared-memory copy of the
//     code table covering the live symbol range (u32 entries when every code
//     fits 26 bits; global fallback outside the window);
//   * block exclusive scan of (bits, outliers) packed in one u64;
//   * decoupled look-back across tiles for the global bit offset (u64) and
//     outlier rank;
//   * codes packed into a shared word buffer (plain stores for words a
//     thread owns, atomicOr only for the two it shares with neighbours),
//     written back as big-endian 32-bit words (byte order == np.packbits).
// The word a tile shares with its successor is not stored by the tile: its
// bits are published in the look-back record ("tail") and merged by the
// successor, so no output pre-zeroing and no global atomics are needed and
// the dependency is strictly backwards.
#include "kernels.cuh"

namespace actc {

namespace {

struct Packer {
  uint32_t *words;
  uint32_t w;        // current word index
  uint32_t first_w;  // first word this thread touches (shared with predecessor)
  unsigned long long buf;
  int nb;
  __device__ __forceinline__ void emit(uint32_t v) {
    if (w == first_w)
      atomicOr(&words[w], v);
    else
      words[w] = v;  // fully owned
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
    if (nb > 0) atomicOr(&words[w], (uint32_t)(buf >> 32));  // shared with successor
  }
};

}  // namespace

template <typename SymT, bool WIDE>
__global__ void __launch_bounds__(K3_THREADS) k3_encode(
    const SymT *__restrict__ sym, uint64_t n, const unsigned long long *__restrict__ ctab,
    uint32_t win_lo, uint32_t win_n, uint32_t word_cap, const float *__restrict__ x,
    uint32_t *__restrict__ payload, unsigned long long *__restrict__ out_idx,
    float *__restrict__ out_val, unsigned long long *__restrict__ chunk_off, EncStatus st,
    unsigned *__restrict__ ticket, uint64_t ntiles, int extract_outliers) {
  extern __shared__ __align__(16) unsigned char smem[];
  using Ent = typename std::conditional<WIDE, unsigned long long, uint32_t>::type;
  Ent *sh_ctab = reinterpret_cast<Ent *>(smem);
  uint32_t *sh_words = reinterpret_cast<uint32_t *>(smem + (((size_t)win_n * sizeof(Ent) + 15) & ~size_t(15)));
  __shared__ unsigned long long wbuf[K3_THREADS / 32 + 1];
  __shared__ unsigned long long s_excl_bits, s_excl_nz;
  __shared__ unsigned s_tile;

  const int tid = threadIdx.x, lane = tid & 31;
  for (uint32_t i = tid; i < win_n; i += K3_THREADS) {
    unsigned long long e = ctab[win_lo + i];
    if (WIDE)
      sh_ctab[i] = (Ent)e;
    else
      sh_ctab[i] = (Ent)(((e >> 8) << 6) | (e & 63));  // (code << 6) | len, code <= 26 bits
  }
  __syncthreads();

  while (true) {
    if (tid == 0) s_tile = atomicAdd(ticket, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    if (tile >= ntiles) break;
    const uint64_t base = tile * K3_TILE + (uint64_t)tid * K3_EPT;

    uint32_t s[K3_EPT];
    if (base + K3_EPT <= n) {
      if (sizeof(SymT) == 2) {
        const uint4 *p = reinterpret_cast<const uint4 *>(sym + base);
#pragma unroll
        for (int j = 0; j < K3_EPT / 8; j++) {
          uint4 v = __ldcs(p + j);
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
          uint4 v = __ldcs(p + j);
          s[4 * j] = v.x; s[4 * j + 1] = v.y; s[4 * j + 2] = v.z; s[4 * j + 3] = v.w;
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < K3_EPT; j++) s[j] = (base + j < n) ? (uint32_t)sym[base + j] : 0u;
    }
    // (code, len) per symbol; code kept in the low bits of e
    unsigned long long code[K3_EPT];
    uint32_t len[K3_EPT];
    uint32_t nbits = 0, nz = 0;
#pragma unroll
    for (int j = 0; j < K3_EPT; j++) {
      if (base + j < n) {
        uint32_t wi = s[j] - win_lo;
        if (WIDE) {
          unsigned long long e = wi < win_n ? sh_ctab[wi] : __ldg(&ctab[s[j]]);
          len[j] = (uint32_t)(e & 0xFF);
          code[j] = e >> 8;
        } else {
          uint32_t e;
          if (wi < win_n) {
            e = (uint32_t)sh_ctab[wi];
          } else {
            unsigned long long g = __ldg(&ctab[s[j]]);
            e = (uint32_t)(((g >> 8) << 6) | (g & 63));
          }
          len[j] = e & 63;
          code[j] = e >> 6;
        }
        nbits += len[j];
        nz += s[j] == 0;
      } else {
        len[j] = 0;
        code[j] = 0;
      }
    }
    unsigned long long tot;
    const unsigned long long mine = ((unsigned long long)nbits << 32) | nz;
    const unsigned long long excl = block_excl_sum<unsigned long long>(mine, wbuf, &tot);
    const unsigned long long tile_bits = tot >> 32, tile_nz = tot & 0xFFFFFFFFull;

    // ---- decoupled look-back (warp 0) ----
    if (tid < 32) {
      unsigned long long eb = 0, en = 0;
      if (tile == 0) {
        if (lane == 0) {
          st.inc_bits[0] = tile_bits;
          st.inc_nz[0] = tile_nz;
          st_release(&st.flag[0], kFlagAgg | kFlagInc);
        }
      } else {
        if (lane == 0) {
          st.agg_bits[tile] = tile_bits;
          st.agg_nz[tile] = tile_nz;
          st_release(&st.flag[tile], kFlagAgg);
        }
        long long pred = (long long)tile - 1;
        while (true) {
          long long idx = pred - lane;
          unsigned f = kFlagInc;
          if (idx >= 0) {
            do {
              f = ld_acquire(&st.flag[idx]);
            } while (f == 0);
          }
          unsigned incm = __ballot_sync(0xffffffffu, (f & kFlagInc) != 0);
          int stop = incm ? __ffs(incm) - 1 : 32;
          unsigned long long vb = 0, vn = 0;
          if (idx >= 0 && lane <= stop) {
            if (lane == stop) {
              vb = ld_relaxed_u64(&st.inc_bits[idx]);
              vn = ld_relaxed_u64(&st.inc_nz[idx]);
            } else {
              vb = ld_relaxed_u64(&st.agg_bits[idx]);
              vn = ld_relaxed_u64(&st.agg_nz[idx]);
            }
          }
          eb += warp_sum(vb);
          en += warp_sum(vn);
          if (incm) break;
          pred -= 32;
        }
        if (lane == 0) {
          st.inc_bits[tile] = eb + tile_bits;
          st.inc_nz[tile] = en + tile_nz;
          st_release(&st.flag[tile], kFlagAgg | kFlagInc);
        }
      }
      if (lane == 0) {
        s_excl_bits = eb;
        s_excl_nz = en;
      }
    }
    // zero the word buffer while warp 0 looks back
    const uint32_t zwords = min(word_cap, (uint32_t)((tile_bits + 63) >> 5));
    for (uint32_t i = tid; i < zwords; i += K3_THREADS) sh_words[i] = 0;
    __syncthreads();
    const unsigned long long tile_bit0 = s_excl_bits;
    const unsigned long long my_bit0 = tile_bit0 + (excl >> 32);

    // decode chunk index: bit offset of every ACTC_CHUNK-th symbol
    if ((base % ACTC_CHUNK) == 0 && base < n) chunk_off[base / ACTC_CHUNK] = my_bit0;
    // outliers in stream order (codec.py:321-322)
    if (extract_outliers && nz) {
      unsigned long long o = s_excl_nz + (excl & 0xFFFFFFFFull);
#pragma unroll
      for (int j = 0; j < K3_EPT; j++) {
        if (base + j < n && s[j] == 0) {
          out_idx[o] = base + j;
          out_val[o] = x[base + j];
          o++;
        }
      }
    }

    // ---- pack into the shared word buffer ----
    const uint32_t start_off = (uint32_t)(tile_bit0 & 31);
    const uint32_t nwords = (uint32_t)((start_off + tile_bits + 31) >> 5);
    if (nbits) {
      uint32_t rel = start_off + (uint32_t)(excl >> 32);
      Packer pk;
      pk.words = sh_words;
      pk.w = rel >> 5;
      pk.first_w = pk.w;
      pk.nb = rel & 31;
      pk.buf = 0;
#pragma unroll
      for (int j = 0; j < K3_EPT; j++) {
        if (!len[j]) continue;
        if (WIDE && len[j] > 32) {
          pk.put((uint32_t)(code[j] >> 32), (int)len[j] - 32);
          pk.put((uint32_t)code[j], 32);
        } else {
          pk.put((uint32_t)code[j], (int)len[j]);
        }
      }
      pk.finish();
    }
    __syncthreads();

    // ---- boundary words ----
    const bool last = tile + 1 == ntiles;
    const uint32_t end_off = (uint32_t)((start_off + tile_bits) & 31);
    const bool keep_tail = !last && end_off != 0;  // successor merges our last word
    if (tid == 0) {
      // publish our own bits of the shared last word first (never waits),
      // then merge the predecessor's tail into our first word
      if (!last) {
        st.tail[tile] = keep_tail ? sh_words[nwords - 1] : 0u;
        __threadfence();
        atomicOr(&st.flag[tile], kFlagTail);
      }
      if (start_off != 0) {
        unsigned f;
        do {
          f = ld_acquire(&st.flag[tile - 1]);
        } while (!(f & kFlagTail));
        sh_words[0] |= ld_relaxed_u32(&st.tail[tile - 1]);
      }
    }
    __syncthreads();
    const uint32_t nstore = keep_tail ? nwords - 1 : nwords;
    const uint64_t gw0 = tile_bit0 >> 5;
    for (uint32_t i = tid; i < nstore; i += K3_THREADS) payload[gw0 + i] = bswap32(sh_words[i]);
    __syncthreads();
  }
}

#define K3_INST(T, W)                                                                                        \
  template __global__ void k3_encode<T, W>(const T *, uint64_t, const unsigned long long *, uint32_t, uint32_t, \
                                           uint32_t, const float *, uint32_t *, unsigned long long *, float *,  \
                                           unsigned long long *, EncStatus, unsigned *, uint64_t, int);
K3_INST(uint16_t, false)
K3_INST(uint16_t, true)
K3_INST(uint32_t, false)
K3_INST(uint32_t, true)

}  // namespace actc
