// K4: chunked canonical-Huffman decode fused with the inverse Lorenzo
// (segmented int64 prefix sum), reconstruction, outlier splice and the
// re-zero filter.
//
// Replaces huffman_decode/_decode_bits (huffman.py:120-142, 210-236), the
// marker check (codec.py:356-359), lorenzo_decode (codec.py:275-293) and
// recon / splice / re-zero (codec.py:360-369).
//
// Tile = K4_THREADS chunks of ACTC_CHUNK symbols.
//  Phase A  each thread decodes one chunk sequentially from its recorded bit
//           offset with a 12-bit shared-memory LUT (canonical slow path for
//           longer codes), writes the symbols to shared memory and keeps the
//           chunk's segmented lattice aggregate (an outlier rebases the chain
//           on prequantize(outlier value)).
//  Phase B  block segmented scan over chunk aggregates + decoupled look-back
//           across tiles -> absolute lattice value before every chunk.
//  Phase C  one warp per chunk, 64 elements per round: warp scan of the
//           deltas, lattice*2eb in fp64, splice/re-zero, coalesced stores.
#include "kernels.cuh"

namespace actc {

namespace {

// shared-memory words per staged chunk: u16 symbol pairs (+1 pad word so the
// per-thread rows land in distinct banks) or one u32 per symbol (+1 pad)
template <int SW>
__host__ __device__ constexpr int words_per_chunk() { return SW == 16 ? ACTC_CHUNK / 2 + 1 : ACTC_CHUNK + 1; }

__device__ __forceinline__ uint64_t read_bits64(const uint32_t *__restrict__ pw, uint64_t pos) {
  uint64_t wi = pos >> 5;
  unsigned sh = pos & 31;
  uint64_t hi = ((uint64_t)bswap32(pw[wi]) << 32) | bswap32(pw[wi + 1]);
  if (!sh) return hi;
  uint32_t lo = bswap32(pw[wi + 2]);
  return (hi << sh) | ((uint64_t)lo >> (32 - sh));
}

// Canonical decode of one code starting at absolute bit `pos` for lengths
// beyond the LUT (huffman.py:127-141 rule: the first length whose code
// offset is in range).  Returns length or 0 if invalid.
__device__ __forceinline__ int slow_decode(const uint32_t *__restrict__ pw, uint64_t pos,
                                           const CodeTables &t, const uint32_t *__restrict__ canon,
                                           uint32_t &sym) {
  uint64_t win = read_bits64(pw, pos);
  for (int l = kLutBits + 1; l <= (int)t.maxlen; l++) {
    unsigned long long code = win >> (64 - l);
    unsigned long long off = code - t.first[l];
    if (off < t.count[l]) {
      sym = canon ? canon[t.base[l] + off] : 0u;
      return l;
    }
  }
  return 0;
}

}  // namespace

__global__ void k_build_lut(const uint32_t *__restrict__ canon, const uint32_t *__restrict__ len_counts,
                            uint32_t *__restrict__ lut, int mode) {
  lut32_body(canon, len_counts, lut, mode, blockIdx.x);
}

template <int MODE, int SW>
__global__ void __launch_bounds__(K4_THREADS) k4_decode(DecodeArgs a) {
  constexpr int kWPC = words_per_chunk<SW>();
  __shared__ uint32_t lut[kLutSize];
  __shared__ CodeTables t;
  extern __shared__ __align__(16) uint32_t symbuf[];  // K4_THREADS * kWPC
  __shared__ long long s_prefix[K4_THREADS];
  __shared__ uint32_t s_ord0[K4_THREADS];
  __shared__ uint8_t s_haszero[K4_THREADS];
  __shared__ long long w_v[K4_THREADS / 32];
  __shared__ int w_r[K4_THREADS / 32];
  __shared__ long long s_tile_prefix;
  __shared__ unsigned s_tile;
  __shared__ unsigned long long s_nz[K4_THREADS / 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NW = K4_THREADS / 32;
  for (int i = tid; i < kLutSize / 4; i += K4_THREADS)
    reinterpret_cast<uint4 *>(lut)[i] = reinterpret_cast<const uint4 *>(a.lut)[i];
  build_tables(t, a.len_counts);
  __syncthreads();

  const uint64_t nchunks = (a.n + ACTC_CHUNK - 1) / ACTC_CHUNK;
  const long long radius = a.radius;
  const bool fast_long = a.lut[kLutSize] != 0;
  unsigned long long nonzero = 0;

  while (true) {
    if (tid == 0) s_tile = atomicAdd(a.ticket, 1u);
    __syncthreads();
    const uint64_t tile = s_tile;
    if (tile >= a.ntiles) break;

    // ---------------- Phase A: decode one chunk per thread ----------------
    const uint64_t c = tile * K4_THREADS + tid;
    Seg agg{0, 0};
    uint32_t zc = 0, ord0 = 0;
    uint32_t *my = symbuf + tid * kWPC;
    if (c < nchunks) {
      const uint64_t e0 = c * ACTC_CHUNK;
      const uint32_t cnt = (uint32_t)min((uint64_t)ACTC_CHUNK, a.n - e0);
      if (MODE != 2 && a.k) {
        uint64_t lo = 0, hi = a.k;
        while (lo < hi) {
          uint64_t mid = (lo + hi) >> 1;
          if (a.out_idx[mid] < e0) lo = mid + 1; else hi = mid;
        }
        ord0 = (uint32_t)lo;
      }
      uint64_t pos = a.chunk_off[c];
      const uint64_t endp = (c + 1 < nchunks) ? a.chunk_off[c + 1] : a.payload_bits;
      const uint32_t *pw = a.payload;
      uint64_t wi = pos >> 5;
      unsigned long long buf = ((unsigned long long)bswap32(pw[wi]) << 32) | bswap32(pw[wi + 1]);
      buf <<= (pos & 31);
      int nb = 64 - (int)(pos & 31);
      wi += 2;
      uint32_t nextw = bswap32(pw[wi++]);  // one-word lookahead hides the load latency
      long long acc = 0;
      int reset = 0;
      bool bad = false;
      uint32_t pair = 0;
      for (uint32_t i = 0; i < cnt; i++) {
        if (nb < 32) {
          buf |= (unsigned long long)nextw << (32 - nb);
          nb += 32;
          nextw = bswap32(pw[wi++]);
        }
        const uint32_t W = (uint32_t)(buf >> 32);
        uint32_t e = lut[W >> (32 - kLutBits)];
        int len = e & 63;
        uint32_t s = e >> 6;
        if (!len) {
          if (fast_long && s) {
            // canonical decode from the register window: first length whose
            // left-aligned limit exceeds the window
            int l = (int)s;
            while (l <= (int)t.maxlen && (unsigned long long)W >= t.lim[l]) l++;
            if (l <= (int)t.maxlen) {
              len = l;
              s = __ldg(&a.canon[t.base[l] + ((W >> (32 - l)) - (uint32_t)t.first[l])]);
            }
          }
          if (!len) {
            // reference first-match rule from memory (over-subscribed tables, codes > 32 bits)
            len = slow_decode(pw, pos, t, a.canon, s);
            if (!len) {
              bad = true;
              break;
            }
            pos += len;
            wi = pos >> 5;
            buf = ((unsigned long long)bswap32(pw[wi]) << 32) | bswap32(pw[wi + 1]);
            buf <<= (pos & 31);
            nb = 64 - (int)(pos & 31);
            wi += 2;
            nextw = bswap32(pw[wi++]);
            len = 0;
          }
        }
        buf <<= len;
        nb -= len;
        pos += len;
        if (MODE != 2) {
          if (s == 0) {
            uint32_t ord = ord0 + zc;
            zc++;
            if (ord >= a.k || a.out_idx[ord] != e0 + i) {
              bad = true;
            } else {
              bool v;
              acc = quant_exact((double)a.out_val[ord], a.two_eb, a.eb, v);
              reset = 1;
            }
          } else {
            acc += (long long)s - radius;
          }
        }
        if (SW == 32) {
          my[i] = s;
        } else if (i & 1) {
          my[i >> 1] = pair | (s << 16);
        } else {
          pair = s;
        }
      }
      if (SW == 16 && (cnt & 1) && !bad) my[cnt >> 1] = pair;
      if (pos != endp || pos > a.payload_bits) bad = true;
      if (bad) report_format_error(a);
      agg = Seg{acc, reset};
    }
    if (MODE != 2) {
      s_ord0[tid] = ord0;
      s_haszero[tid] = zc != 0;
      if (zc) atomicAdd(a.markers, (unsigned long long)zc);
    }

    // ---------------- Phase B: segmented scan + look-back ----------------
    if (MODE != 2) {
      Seg inc = warp_incl_seg(agg);
      if (lane == 31) {
        w_v[warp] = inc.v;
        w_r[warp] = inc.r;
      }
      __syncthreads();
      if (tid == 0) {
        Seg run{0, 0};
        for (int w = 0; w < NW; w++) {
          Seg ww{w_v[w], w_r[w]};
          w_v[w] = run.v;
          w_r[w] = run.r;
          run = seg_combine(run, ww);
        }
        // tile aggregate -> look-back (single thread; tiles are large)
        long long excl_v = 0;
        if (tile == 0) {
          a.st.inc_v[0] = run.r ? run.v : run.v;  // absolute from lattice 0
          st_release(&a.st.flag[0], kFlagAgg | kFlagInc);
          excl_v = 0;
        } else {
          a.st.agg_v[tile] = run.v;
          a.st.agg_r[tile] = run.r;
          st_release(&a.st.flag[tile], kFlagAgg);
          Seg acc{0, 0};
          long long idx = (long long)tile - 1;
          while (true) {
            unsigned f;
            do {
              f = ld_acquire(&a.st.flag[idx]);
            } while (f == 0);
            if (f & kFlagInc) {
              long long iv = (long long)ld_relaxed_u64((const unsigned long long *)&a.st.inc_v[idx]);
              acc = seg_combine(Seg{iv, 1}, acc);
              break;
            }
            long long av = (long long)ld_relaxed_u64((const unsigned long long *)&a.st.agg_v[idx]);
            int ar = (int)ld_relaxed_u32((const unsigned *)&a.st.agg_r[idx]);
            acc = seg_combine(Seg{av, ar}, acc);
            if (ar) break;  // a reset makes everything earlier irrelevant
            idx--;
          }
          excl_v = acc.v;  // acc.r == 1 always (absolute)
          Seg incl = seg_combine(Seg{excl_v, 1}, run);
          a.st.inc_v[tile] = incl.v;
          st_release(&a.st.flag[tile], kFlagAgg | kFlagInc);
        }
        s_tile_prefix = excl_v;
      }
      __syncthreads();
      // exclusive prefix of this chunk inside the tile
      Seg ex;
      {
        long long pv = __shfl_up_sync(0xffffffffu, inc.v, 1);
        int pr = __shfl_up_sync(0xffffffffu, inc.r, 1);
        Seg wp{w_v[warp], w_r[warp]};
        ex = lane ? seg_combine(wp, Seg{pv, pr}) : wp;
      }
      s_prefix[tid] = ex.r ? ex.v : s_tile_prefix + ex.v;
    }
    __syncthreads();

    // ---------------- Phase C: coalesced reconstruction ----------------
    for (int cl = warp; cl < K4_THREADS; cl += NW) {
      const uint64_t cc = tile * K4_THREADS + cl;
      if (cc >= nchunks) break;
      const uint64_t e0 = cc * ACTC_CHUNK;
      const uint32_t cnt = (uint32_t)min((uint64_t)ACTC_CHUNK, a.n - e0);
      const uint32_t *buf = symbuf + cl * kWPC;
      if (MODE == 2) {
        uint32_t *out = reinterpret_cast<uint32_t *>(a.out) + e0;
        for (uint32_t i = lane; i < cnt; i += 32) out[i] = buf[i];
        continue;
      }
      long long P = s_prefix[cl];
      uint32_t ordb = s_ord0[cl];
      const bool slow = SW == 32 || s_haszero[cl];
#pragma unroll
      for (int r = 0; r < ACTC_CHUNK / 64; r++) {
        const uint32_t i0 = 64 * r + 2 * lane;
        uint32_t s0, s1;
        if (SW == 16) {
          const uint32_t w = buf[32 * r + lane];
          s0 = w & 0xFFFFu;
          s1 = w >> 16;
        } else {
          s0 = buf[i0];
          s1 = buf[i0 + 1];
        }
        const bool v0 = i0 < cnt, v1 = i0 + 1 < cnt;
        long long L0, L1;
        bool z0 = false, z1 = false;
        uint32_t o0 = 0, o1 = 0;
        if (!slow) {
          int d0 = v0 ? (int)s0 - (int)radius : 0;
          int d1 = v1 ? (int)s1 - (int)radius : 0;
          int inc = warp_incl_sum(d0 + d1);
          int tot = __shfl_sync(0xffffffffu, inc, 31);
          L0 = P + (inc - d1);
          L1 = L0 + d1;
          P += tot;
        } else {
          z0 = v0 && s0 == 0;
          z1 = v1 && s1 == 0;
          int nzl = (int)z0 + (int)z1;
          int zi = warp_incl_sum(nzl);
          int ztot = __shfl_sync(0xffffffffu, zi, 31);
          o0 = ordb + (uint32_t)(zi - nzl);
          o1 = o0 + (uint32_t)z0;
          bool dummy;
          Seg e0s = z0 ? Seg{quant_exact((double)a.out_val[o0], a.two_eb, a.eb, dummy), 1}
                       : Seg{v0 ? (long long)s0 - radius : 0, 0};
          Seg e1s = z1 ? Seg{quant_exact((double)a.out_val[o1], a.two_eb, a.eb, dummy), 1}
                       : Seg{v1 ? (long long)s1 - radius : 0, 0};
          Seg ls = seg_combine(e0s, e1s);
          Seg inc = warp_incl_seg(ls);
          long long pv = __shfl_up_sync(0xffffffffu, inc.v, 1);
          int pr = __shfl_up_sync(0xffffffffu, inc.r, 1);
          Seg ex = lane ? Seg{pv, pr} : Seg{0, 0};
          Seg a0 = seg_combine(ex, e0s);
          Seg a1 = seg_combine(a0, e1s);
          L0 = a0.r ? a0.v : P + a0.v;
          L1 = a1.r ? a1.v : P + a1.v;
          long long tv = __shfl_sync(0xffffffffu, inc.v, 31);
          int tr = __shfl_sync(0xffffffffu, inc.r, 31);
          P = tr ? tv : P + tv;
          ordb += (uint32_t)ztot;
        }
        double r0 = z0 ? (double)a.out_val[o0] : __dmul_rn((double)L0, a.two_eb);
        double r1 = z1 ? (double)a.out_val[o1] : __dmul_rn((double)L1, a.two_eb);
        if (a.preserve) {
          if (fabs(r0) <= a.eb) r0 = 0.0;
          if (fabs(r1) <= a.eb) r1 = 0.0;
        }
        nonzero += (v0 && r0 != 0.0) + (v1 && r1 != 0.0);
        if (MODE == 0) {
          float *out = reinterpret_cast<float *>(a.out) + e0 + i0;
          if (v1)
            __stcs(reinterpret_cast<float2 *>(out), make_float2((float)r0, (float)r1));
          else if (v0)
            *out = (float)r0;
        } else {
          double *out = reinterpret_cast<double *>(a.out) + e0 + i0;
          if (v1)
            __stcs(reinterpret_cast<double2 *>(out), make_double2(r0, r1));
          else if (v0)
            *out = r0;
        }
      }
    }
    __syncthreads();
  }
  if (MODE != 2) {
    unsigned long long ws = warp_sum(nonzero);
    if (lane == 0) s_nz[warp] = ws;
    __syncthreads();
    if (tid == 0) {
      unsigned long long tsum = 0;
      for (int w = 0; w < NW; w++) tsum += s_nz[w];
      if (tsum) atomicAdd(a.nonzero, tsum);
    }
  }
}

template __global__ void k4_decode<0, 16>(DecodeArgs);
template __global__ void k4_decode<1, 16>(DecodeArgs);
template __global__ void k4_decode<0, 32>(DecodeArgs);
template __global__ void k4_decode<1, 32>(DecodeArgs);
template __global__ void k4_decode<2, 32>(DecodeArgs);

// lorenzo_decode debug entry (codec.py:275-293), sequential on one thread.
__global__ void k_lorenzo_decode_seq(const uint32_t *__restrict__ sym, uint64_t n,
                                     const long long *__restrict__ olat, uint64_t k,
                                     uint32_t radius, long long *__restrict__ out,
                                     unsigned *__restrict__ status) {
  if (threadIdx.x || blockIdx.x) return;
  uint64_t markers = 0;
  for (uint64_t i = 0; i < n; i++) markers += sym[i] == 0;
  if (markers != k) {
    *status = ACTC_EFORMAT;
    return;
  }
  long long acc = 0;
  uint64_t j = 0;
  for (uint64_t i = 0; i < n; i++) {
    if (sym[i] == 0)
      acc = olat[j++];
    else
      acc += (long long)sym[i] - (long long)radius;
    out[i] = acc;
  }
}

// ------------------------------------------------------------------------
// Chunk-index rebuild for streams without one (from_bytes).  Segments of
// seg_bits bits are decoded speculatively from a start position; the start
// of segment s+1 is the first code boundary at or after its nominal start
// reached from segment s.  Iterate until no start changes (Huffman codes
// self-synchronise quickly; worst case one segment per iteration).
// ------------------------------------------------------------------------
__global__ void k_sync_pass(const uint32_t *__restrict__ payload, uint64_t payload_bits,
                            const uint32_t *__restrict__ lut, const uint32_t *__restrict__ len_counts,
                            uint64_t seg_bits, uint64_t nseg, unsigned long long *__restrict__ start,
                            unsigned long long *__restrict__ end_pos,
                            unsigned long long *__restrict__ count, unsigned *__restrict__ changed,
                            unsigned *__restrict__ status, int first) {
  __shared__ CodeTables t;
  __shared__ uint32_t sl[kLutSize];
  for (int i = threadIdx.x; i < kLutSize; i += blockDim.x) sl[i] = lut[i];
  build_tables(t, len_counts);
  __syncthreads();
  uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  uint64_t st = first ? (s ? s * seg_bits : 0) : start[s];
  if (!first && s > 0) {
    unsigned long long prev_end = end_pos[s - 1];
    if (prev_end != st) {
      st = prev_end;
      start[s] = st;
      atomicOr(changed, 1u);
    } else {
      return;  // unchanged start: keep previous result
    }
  } else if (first) {
    start[s] = st;
  }
  const uint64_t lim = min((s + 1) * seg_bits, payload_bits);
  uint64_t pos = st;
  unsigned long long cnt = 0;
  while (pos < lim) {
    uint64_t win = read_bits64(payload, pos);
    uint32_t e = sl[win >> (64 - kLutBits)];
    int len = e & 63;
    uint32_t sym;
    if (!len) len = slow_decode(payload, pos, t, nullptr, sym);
    if (!len) {
      // not a valid code from here: only possible from a wrong start
      len = 1;
      if (s == 0) atomicOr(status, (unsigned)ACTC_EFORMAT);
    }
    pos += len;
    cnt++;
  }
  end_pos[s] = pos;
  count[s] = cnt;
}

__global__ void k_index_emit(const uint32_t *__restrict__ payload, uint64_t payload_bits,
                             const uint32_t *__restrict__ lut, const uint32_t *__restrict__ len_counts,
                             uint64_t seg_bits, uint64_t nseg,
                             const unsigned long long *__restrict__ start,
                             const unsigned long long *__restrict__ sym_base, uint64_t n,
                             unsigned long long *__restrict__ chunk_off) {
  __shared__ CodeTables t;
  __shared__ uint32_t sl[kLutSize];
  for (int i = threadIdx.x; i < kLutSize; i += blockDim.x) sl[i] = lut[i];
  build_tables(t, len_counts);
  __syncthreads();
  uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (s >= nseg) return;
  const uint64_t lim = min((s + 1) * seg_bits, payload_bits);
  uint64_t pos = start[s];
  uint64_t idx = sym_base[s];
  while (pos < lim && idx < n) {
    if ((idx % ACTC_CHUNK) == 0) chunk_off[idx / ACTC_CHUNK] = pos;
    uint64_t win = read_bits64(payload, pos);
    uint32_t e = sl[win >> (64 - kLutBits)];
    int len = e & 63;
    uint32_t sym;
    if (!len) len = slow_decode(payload, pos, t, nullptr, sym);
    if (!len) len = 1;
    pos += len;
    idx++;
  }
}

}  // namespace actc
