// K3: canonical-Huffman encode + MSB-first bit packing + outlier
// extraction + decode chunk index.
//
// Replaces huffman.py:188-207 (code lookup, np.packbits) and codec.py:321-322
// (outlier indices / values).  Two barrier-free passes over 1024-symbol
// segments (see the section comment below).
#include "kernels.cuh"

namespace actc {

namespace {

constexpr uint32_t kSent = 0xFFFFFFFFu;  // symbol past the end of the stream

// a lane's K3L_EPT symbols, 16-bit ones kept two per register; cnt < K3L_EPT
// only in the stream's last segment (symbols past the end read as 0 and are
// masked by cnt)
template <typename SymT>
struct SymBuf {
  static constexpr int W = sizeof(SymT) == 2 ? K3L_EPT / 2 : K3L_EPT;
  uint32_t w[W];
  uint32_t cnt;
  __device__ __forceinline__ uint32_t get(int j) const {
    if (sizeof(SymT) == 2) return (j & 1) ? (w[j >> 1] >> 16) : (w[j >> 1] & 0xFFFFu);
    return w[j];
  }
  __device__ __forceinline__ void load(const SymT *__restrict__ sym, uint64_t base, uint64_t n) {
    if (base + K3L_EPT <= n) {
      cnt = K3L_EPT;
      const uint4 *p = reinterpret_cast<const uint4 *>(sym + base);
#pragma unroll
      for (int j = 0; j < W / 4; j++) {
        const uint4 v = __ldcs(p + j);  // streaming: the symbol buffer is read once more
        w[4 * j] = v.x; w[4 * j + 1] = v.y; w[4 * j + 2] = v.z; w[4 * j + 3] = v.w;
      }
    } else {
      cnt = base < n ? (uint32_t)(n - base) : 0u;
#pragma unroll
      for (int j = 0; j < W; j++) w[j] = 0;
#pragma unroll
      for (int j = 0; j < K3L_EPT; j++) {
        const uint32_t v = (uint32_t)j < cnt ? (uint32_t)sym[base + j] : 0u;
        if (sizeof(SymT) == 2) w[j >> 1] |= v << (16 * (j & 1));
        else w[j] = v;
      }
    }
  }
};

}  // namespace

// ===========================================================================
// Two-pass, barrier-free variant (the production path for codes <= 26 bits):
//   k3_seg_count  CTA b owns segments [b*spc, (b+1)*spc); warp per 1024-symbol
//                 segment sums code lengths (byte table of the live range in
//                 shared memory) and outlier markers; the CTA then turns its
//                 segment counts into exclusive in-CTA prefixes and writes its
//                 totals
//                 (the last count CTA turns the CTA totals into exclusive prefixes)
//   k3_seg_pack   warp per segment at bit cta_prefix + in-CTA prefix: one
//                 (code, len) lookup per symbol into registers, pack, store
// Symbols are read twice (2 x 2 B), but no warp ever waits for another.
// ===========================================================================

constexpr uint32_t K3S_L8MAX = 65536;  // byte length table in shared memory (u16 symbol range)

// pack-pass table entry of a (code << 8 | len) code-table word of a code of
// <= 26 bits: the code left-aligned in 32 bits, its length in the low 6 bits
// (which a left-aligned code of <= 26 bits leaves zero)
__device__ __forceinline__ uint32_t k3_entry(unsigned long long g) {
  const uint32_t len = (uint32_t)(g & 63);
  return len ? ((uint32_t)(g >> 8) << (32 - len)) | len : 0u;
}

__device__ __forceinline__ void k3_load_window(uint32_t *tab, const unsigned long long *__restrict__ ctab,
                                               uint32_t win_lo, uint32_t win_n, int nthreads) {
  for (uint32_t i0 = threadIdx.x; i0 < win_n; i0 += 16 * nthreads) {
    unsigned long long e[16];
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const uint32_t i = i0 + u * nthreads;
      e[u] = i < win_n ? __ldg(&ctab[win_lo + i]) : 0ull;
    }
#pragma unroll
    for (int u = 0; u < 16; u++) {
      const uint32_t i = i0 + u * nthreads;
      if (i < win_n) tab[i] = k3_entry(e[u]);
    }
  }
}

__device__ __forceinline__ uint32_t k3c_saddr(const void *p) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mov.u32 %0, %1;" : "=r"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ uint32_t k3c_ldsb(uint32_t a) {
  unsigned short v;
  asm("ld.shared.u8 %0, [%1];" : "=h"(v) : "r"(a));
  return v;
}

template <typename SymT>
__global__ void __launch_bounds__(K3L_THREADS) k3_seg_count(const SymT *__restrict__ sym, SegArgs a) {
  extern __shared__ __align__(16) uint8_t k3c_l8[];
  __shared__ unsigned long long wsum_b[K3L_THREADS / 32 + 1], wsum_z[K3L_THREADS / 32 + 1];
  if (!seg_resolve(a)) return;
  if (a.dplan) {
    // device-planned: zero the payload (the pack ORs boundary words)
    const uint64_t nw = (a.dplan->payload_bits + 31) / 32 + 2;
    const uint64_t stride = (uint64_t)gridDim.x * K3L_THREADS;
    if (!(reinterpret_cast<uintptr_t>(a.payload) & 15)) {
      // 16-byte stores (the buffer carries a 32-byte pad past its last word)
      uint4 *p4 = reinterpret_cast<uint4 *>(a.payload);
      for (uint64_t i = (uint64_t)blockIdx.x * K3L_THREADS + threadIdx.x; i < (nw + 3) / 4; i += stride)
        p4[i] = make_uint4(0u, 0u, 0u, 0u);
    } else {
      for (uint64_t i = (uint64_t)blockIdx.x * K3L_THREADS + threadIdx.x; i < nw; i += stride) a.payload[i] = 0u;
    }
    if (a.canon_src) {
      // the table is in ctx scratch: copy it to the caller's buffers
      const uint32_t live = a.dplan->live_symbols;
      for (uint32_t i = blockIdx.x * K3L_THREADS + threadIdx.x; i < live; i += gridDim.x * K3L_THREADS)
        a.canon_out[i] = a.canon_src[i];
      if (blockIdx.x == 0 && threadIdx.x < 64) a.lencnt_out[threadIdx.x] = a.lencnt_src[threadIdx.x];
    }
  }
  if (a.emit.rank_tab && threadIdx.x < 32 && !*a.emit.fallback) {
    // the codebook's canonical-code emission (k2s_emit's work), warp 0 of
    // the first CTAs: this pass reads only len8; the pack reads ctab
    __shared__ uint16_t e_row[32 * K2R_TS];
    __shared__ unsigned long long e_first[64];
    __shared__ uint32_t e_base[64];
    for (uint32_t wb = blockIdx.x; wb < K2_THREADS / 32; wb += gridDim.x) k2s_emit_warp(a.emit, wb, e_row, e_first, e_base);
  }
  const bool smem_tab = a.span <= K3S_L8MAX;
  uint32_t shift = 0;
  if (smem_tab) {
    // len8[lo, lo+span) -> shared, 16-byte loads from an aligned start (the
    // global table is padded by 64 bytes), 16 in flight per thread
    const uint32_t a0 = a.lo & ~15u;
    shift = a.lo - a0;
    const uint32_t nv = (shift + a.span + 15) >> 4;
    const uint4 *src = reinterpret_cast<const uint4 *>(a.len8 + a0);
    for (uint32_t i0 = threadIdx.x; i0 < nv; i0 += 16 * K3L_THREADS) {
      uint4 v[16];
#pragma unroll
      for (int u = 0; u < 16; u++) {
        const uint32_t i = i0 + u * K3L_THREADS;
        v[u] = i < nv ? __ldg(src + i) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int u = 0; u < 16; u++) {
        const uint32_t i = i0 + u * K3L_THREADS;
        if (i < nv) reinterpret_cast<uint4 *>(k3c_l8)[i] = v[u];
      }
    }
  }
  __syncthreads();
  const uint8_t *l8 = k3c_l8 + shift;  // l8[s - lo]
  const uint32_t l8_rel = k3c_saddr(k3c_l8) + shift - a.lo;  // l8[s - lo] at l8_rel + s (mod 2^32)
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t nseg = (a.n + K3L_SEG - 1) / K3L_SEG;
  const uint64_t s0 = (uint64_t)blockIdx.x * a.spc, s1 = min(nseg, s0 + a.spc);
  unsigned long long tb = 0, tz = 0;
  // the next segment's symbols are loaded while this one is counted
  SymBuf<SymT> nxt;
  if (s0 + warp < s1) nxt.load(sym, (s0 + warp) * K3L_SEG + (uint64_t)lane * K3L_EPT, a.n);
  for (uint64_t seg = s0 + warp; seg < s1; seg += K3L_THREADS / 32) {
    const SymBuf<SymT> sb = nxt;
    if (seg + K3L_THREADS / 32 < s1) nxt.load(sym, (seg + K3L_THREADS / 32) * K3L_SEG + (uint64_t)lane * K3L_EPT, a.n);
    uint32_t bits = 0, nz = 0, mx = 0;
    if (smem_tab && __all_sync(0xffffffffu, sb.cnt == (uint32_t)K3L_EPT)) {
      // full segment, byte table in shared memory: one LDS.U8 per symbol
#pragma unroll
      for (int j = 0; j < K3L_EPT; j++) {
        const uint32_t l = k3c_ldsb(l8_rel + sb.get(j));
        bits += l;
        mx = max(mx, l);
      }
      if (a.k) {
#pragma unroll
        for (int j = 0; j < K3L_EPT; j++) nz += sb.get(j) == 0;
      }
    } else {
#pragma unroll
      for (int j = 0; j < K3L_EPT; j++) {
        if ((uint32_t)j < sb.cnt) {
          const uint32_t sj = sb.get(j);
          const uint32_t l = smem_tab ? (uint32_t)l8[sj - a.lo] : (uint32_t)(__ldg(&a.ctab[sj]) & 63);
          bits += l;
          mx = max(mx, l);
          nz += sj == 0;
        }
      }
    }
    bits = warp_sum(bits);
    if (a.k || !__all_sync(0xffffffffu, nz == 0)) nz = warp_sum(nz);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) {
      a.seg_long[seg] = mx > (uint32_t)K3_SHORT_MAXLEN;  // the pack takes its u64 path
      a.seg_bits[seg] = bits;
      a.seg_nz[seg] = nz;
      tb += bits;
      tz += nz;
    }
  }
  __syncthreads();  // this CTA's segment counts are visible to the whole CTA
  // in-CTA exclusive prefixes (u32: spc * 1024 * 26 bits < 2^32 for spc < 2^17)
  unsigned long long runb = 0, runz = 0;
  for (uint64_t c0 = s0; c0 < s1; c0 += K3L_THREADS) {
    const uint64_t i = c0 + threadIdx.x;
    const uint32_t vb = i < s1 ? a.seg_bits[i] : 0u, vz = i < s1 ? a.seg_nz[i] : 0u;
    unsigned long long allb, allz;
    const unsigned long long eb = block_excl_sum<unsigned long long>(vb, wsum_b, &allb);
    const unsigned long long ez = block_excl_sum<unsigned long long>(vz, wsum_z, &allz);
    if (i < s1) {
      a.seg_bits[i] = (uint32_t)(runb + eb);
      a.seg_nz[i] = (uint32_t)(runz + ez);
    }
    runb += allb;
    runz += allz;
  }
  // the last CTA to finish turns the per-CTA totals into exclusive prefixes
  // (in place) -- no separate scan launch waiting for a free SM
  __shared__ unsigned k3c_last;
  if (threadIdx.x == 0) {
    a.cta_bits[blockIdx.x] = runb;
    a.cta_nz[blockIdx.x] = runz;
    __threadfence();
    k3c_last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!k3c_last) return;
  __threadfence();
  runb = runz = 0;
  for (uint32_t c0 = 0; c0 < a.ncta; c0 += K3L_THREADS) {
    const uint32_t i = c0 + threadIdx.x;
    const unsigned long long vb = i < a.ncta ? __ldcg(&a.cta_bits[i]) : 0ull;
    const unsigned long long vz = i < a.ncta ? __ldcg(&a.cta_nz[i]) : 0ull;
    unsigned long long allb, allz;
    const unsigned long long eb = block_excl_sum<unsigned long long>(vb, wsum_b, &allb);
    const unsigned long long ez = block_excl_sum<unsigned long long>(vz, wsum_z, &allz);
    if (i < a.ncta) {
      a.cta_bits[i] = runb + eb;
      a.cta_nz[i] = runz + ez;
    }
    runb += allb;
    runz += allz;
  }
  if (threadIdx.x == 0) *a.ticket = 0u;  // ready for the next launch
}

__device__ __forceinline__ uint32_t k3_saddr(const void *p) {
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mov.u32 %0, %1;" : "=r"(r) : "r"(a));
  return r;
}
__device__ __forceinline__ uint32_t k3_lds(uint32_t a) {
  uint32_t v;
  asm("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void k3_sts(uint32_t addr, uint32_t v) {
  asm volatile("st.shared.u32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}
// OR v into the warp buffer
__device__ __forceinline__ void k3_red_or(uint32_t addr, uint32_t v) {
  asm volatile("red.shared.or.b32 [%0], %1;" ::"r"(addr), "r"(v) : "memory");
}

__device__ __forceinline__ void k3_plan_out(const SegArgs &a) {
  constexpr int W = (int)(sizeof(actc_plan_t) / 4);
  if (threadIdx.x < W)
    reinterpret_cast<volatile uint32_t *>(a.plan_host)[threadIdx.x] = reinterpret_cast<const uint32_t *>(a.dplan)[threadIdx.x];
  __threadfence_system();
}

template <typename SymT>
__global__ void __launch_bounds__(K3L_THREADS, 2) k3_seg_pack(const SymT *__restrict__ sym, SegArgs a) {
  extern __shared__ __align__(16) uint32_t k3p_sm[];
  if (!seg_resolve(a)) {
    if (a.plan_host && blockIdx.x == 0) k3_plan_out(a);  // the host redoes this stream: it needs the plan
    return;
  }
  if (a.table && a.dplan) {
    // the stream's decode table (kLutSize entries, 16 rows of 256), built
    // here by the first CTAs instead of a launch of its own
    for (uint32_t b = blockIdx.x; b < (uint32_t)(kLutSize / K3L_THREADS); b += gridDim.x) {
      table_rows_plan(a.canon_out, a.lencnt_out, a.radius, a.table, b);
      __syncthreads();
    }
  }
  uint32_t *tab = k3p_sm;
  k3_load_window(tab, a.ctab, a.win_lo, a.win_n, K3L_THREADS);
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t *wb = k3p_sm + ((a.win_n + 3) & ~3u) + warp * K3L_WORDS;
  const uint64_t nseg = (a.n + K3L_SEG - 1) / K3L_SEG;
  const uint64_t nwarps = (uint64_t)gridDim.x * (K3L_THREADS / 32);
  const uint32_t wlast = a.win_n - 1;
  const uint32_t tab_s = k3_saddr(tab);
  const uint32_t wb_s = k3_saddr(wb);
  // the next segment's symbols are loaded while this one is encoded (16-bit
  // symbols: two per register leave room for the second set)
  constexpr bool kPrefetch = sizeof(SymT) == 2;
  uint64_t seg = (uint64_t)blockIdx.x * (K3L_THREADS / 32) + warp;
  SymBuf<SymT> nxt;
  if (kPrefetch && seg < nseg) nxt.load(sym, seg * K3L_SEG + (uint64_t)lane * K3L_EPT, a.n);
  for (; seg < nseg; seg += nwarps) {
    const uint64_t base = seg * K3L_SEG + (uint64_t)lane * K3L_EPT;
    SymBuf<SymT> sb;
    if (kPrefetch) {
      sb = nxt;
      if (seg + nwarps < nseg) nxt.load(sym, (seg + nwarps) * K3L_SEG + (uint64_t)lane * K3L_EPT, a.n);
    } else {
      sb.load(sym, base, a.n);
    }
    const uint64_t r = seg / a.spc;
    const unsigned long long pb = a.cta_bits[r] + a.seg_bits[seg], pz = a.cta_nz[r] + a.seg_nz[seg];
    if (a.seg_long[seg]) {
      // rare: a code longer than 26 bits in this segment.  u64 (code, len)
      // entries from the global table, every word OR-ed straight into the
      // (zeroed) payload, codes fed in <= 32-bit chunks.
      uint32_t bits = 0, zm = 0;
#pragma unroll
      for (int j = 0; j < K3L_EPT; j++) {
        if ((uint32_t)j < sb.cnt) {
          bits += (uint32_t)(__ldg(&a.ctab[sb.get(j)]) & 0xFF);
          zm |= (uint32_t)(sb.get(j) == 0) << j;
        }
      }
      const uint32_t nzl = __popc(zm);
      const uint32_t ib = warp_incl_sum(bits), iz = warp_incl_sum(nzl);
      const uint32_t lane_ex = ib - bits;
      if (((lane * K3L_EPT) % ACTC_CHUNK) == 0 && base < a.n) a.chunk_off[base / ACTC_CHUNK] = pb + lane_ex;
      if (a.extract && nzl) {
        unsigned long long o = pz + (iz - nzl);
        for (uint32_t m = zm; m; m &= m - 1) {
          const uint64_t e_idx = base + (uint32_t)(__ffs(m) - 1);
          a.out_idx[o] = e_idx;
          a.out_val[o] = a.x[e_idx];
          o++;
        }
      }
      unsigned long long P = pb + lane_ex;
#pragma unroll
      for (int j = 0; j < K3L_EPT; j++) {
        if ((uint32_t)j >= sb.cnt) continue;
        const unsigned long long g = __ldg(&a.ctab[sb.get(j)]);
        const unsigned long long code = g >> 8;
        int len = (int)(g & 0xFF);
        while (len > 0) {
          const int c = len > 32 ? 32 : len;
          const uint32_t chunk = (uint32_t)((code >> (len - c)) & ((1ull << c) - 1));
          const uint32_t off = (uint32_t)(P & 31);
          const unsigned long long v = (unsigned long long)chunk << (64 - off - c);
          uint32_t *w = a.payload + (P >> 5);
          atomicOr(w, bswap32((uint32_t)(v >> 32)));
          if (off + c > 32) atomicOr(w + 1, bswap32((uint32_t)v));
          P += c;
          len -= c;
        }
      }
      continue;
    }
    // one (left-aligned code | len) lookup per symbol, clamped into the
    // shared window; the few symbols outside it (the tails of the
    // distribution) are fixed up from the global table, sentinels past the
    // end get length 0
    uint32_t e[K3L_EPT];
    uint32_t zmask = 0, oow = 0;
    if (__all_sync(0xffffffffu, sb.cnt == (uint32_t)K3L_EPT)) {
#pragma unroll
      for (int j = 0; j < K3L_EPT; j++) {
        const uint32_t wi = sb.get(j) - a.win_lo;
        e[j] = k3_lds(tab_s + 4u * min(wi, wlast));
        oow |= (uint32_t)(wi > wlast) << j;
      }
      if (a.k) {
#pragma unroll
        for (int j = 0; j < K3L_EPT; j++) zmask |= (uint32_t)(sb.get(j) == 0) << j;
      }
    } else {
#pragma unroll
      for (int j = 0; j < K3L_EPT; j++) {
        const uint32_t wi = sb.get(j) - a.win_lo;
        const bool sent = (uint32_t)j >= sb.cnt;
        e[j] = sent ? 0u : tab[min(wi, wlast)];
        oow |= (uint32_t)(wi > wlast && !sent) << j;
        zmask |= (uint32_t)(sb.get(j) == 0 && !sent) << j;
      }
    }
    if (oow) {
#pragma unroll
      for (int j = 0; j < K3L_EPT; j++) {
        if ((oow >> j) & 1u) e[j] = k3_entry(__ldg(&a.ctab[sb.get(j)]));
      }
    }
    uint32_t bits = 0;
#pragma unroll
    for (int j = 0; j < K3L_EPT; j++) bits += e[j] & 63;
    const uint32_t nz = __popc(zmask);
    const uint32_t ib = warp_incl_sum(bits), iz = warp_incl_sum(nz);
    const uint32_t seg_bits = __shfl_sync(0xffffffffu, ib, 31);
    const uint32_t lane_ex = ib - bits;
    const uint32_t off0 = (uint32_t)(pb & 31);
    const uint32_t nw = (off0 + seg_bits + 31) >> 5;
    // only the segment's last word can be left without a plain store (no
    // code completes it): it alone is zeroed for the shared ORs
    if (lane == 0) wb[nw - 1] = 0;
    __syncwarp();
    if (((lane * K3L_EPT) % ACTC_CHUNK) == 0 && base < a.n) a.chunk_off[base / ACTC_CHUNK] = pb + lane_ex;  // every ACTC_CHUNK-th symbol
    if (a.extract && nz) {
      unsigned long long o = pz + (iz - nz);
      for (uint32_t m = zmask; m; m &= m - 1) {
        const uint64_t e_idx = base + (uint32_t)(__ffs(m) - 1);
        a.out_idx[o] = e_idx;
        a.out_val[o] = a.x[e_idx];
        o++;
      }
    }
    {
      // Codes accumulate in a register word at the lane's bit position; a
      // word the lane completes is written by a plain shared store (exactly
      // one lane completes each word), and after a warp barrier the lane's
      // last, partial word is OR-ed in (it may share the word with the next
      // lanes, or be the segment's zeroed last word).  A left-aligned code of
      // <= 26 bits completes at most one word.  A length-0 entry (past the
      // end) has code 0.
      uint32_t pos = off0 + lane_ex;
      uint32_t wad = wb_s + ((pos >> 3) & ~3u);
      uint32_t fill = pos & 31u, hi = 0u;
#pragma unroll
      for (int j = 0; j < K3L_EPT; j++) {
        const uint32_t cl = e[j] & ~63u;
        hi |= __funnelshift_r(cl, 0u, fill);          // cl >> fill
        const uint32_t ov = __funnelshift_r(0u, cl, fill);  // the bits past the word (0 unless it completes)
        const uint32_t t = fill + (e[j] & 63u);
        if (t >= 32u) {
          k3_sts(wad, hi);
          wad += 4u;
          hi = ov;
        }
        fill = t & 31u;
      }
      __syncwarp();
      if (fill) k3_red_or(wad, hi);
    }
    __syncwarp();
    // copy-out: interior words by plain stores, the two words the segment
    // shares with its neighbours by global ORs (the payload was zeroed)
    uint32_t *dst = a.payload + (pb >> 5);
    const uint32_t end_off = (off0 + seg_bits) & 31;
    const uint32_t i_lo = off0 ? 1u : 0u, i_hi = end_off ? nw - 1 : nw;
    for (uint32_t i = i_lo + lane; i < i_hi; i += 32) dst[i] = bswap32(wb[i]);
    if (lane == 0 && off0) atomicOr(dst, bswap32(wb[0]));
    if (lane == 31 && end_off && (nw > 1 || !off0)) atomicOr(dst + nw - 1, bswap32(wb[nw - 1]));
    __syncwarp();
  }
  if (a.plan_host) {
    // the last CTA to finish hands the plan to the mapped host mailbox
    __shared__ unsigned k3p_last;
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence();
      k3p_last = atomicAdd(a.pack_ticket, 1u) == gridDim.x - 1;
    }
    __syncthreads();
    if (k3p_last) {
      k3_plan_out(a);
      if (threadIdx.x == 0) *a.pack_ticket = 0u;
    }
  }
}


}  // namespace actc

namespace actc {
template __global__ void k3_seg_count<uint16_t>(const uint16_t *, SegArgs);
template __global__ void k3_seg_count<uint32_t>(const uint32_t *, SegArgs);
template __global__ void k3_seg_pack<uint16_t>(const uint16_t *, SegArgs);
template __global__ void k3_seg_pack<uint32_t>(const uint32_t *, SegArgs);
}  // namespace actc
