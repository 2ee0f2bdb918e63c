// K1: fused prequantize + bound check + 1-D Lorenzo + outlier flag +
// quant-code histogram (shared-memory window + global tail).
//
// Replaces, per element of the flattened fp32 stream:
//   prequantize          codec.py:238-251
//   bound check          codec.py:311-312
//   lorenzo_encode       codec.py:254-272 (delta vs own predecessor lattice)
//   bincount             huffman.py:183
// Memory traffic: 4 B read + sizeof(Sym) written per element; the lattice
// never leaves registers.  Each thread owns 16 consecutive elements
// (4 x 128-bit loads); the predecessor lattice value of the first element
// comes from the neighbouring lane by shuffle, lane 0 recomputes it from
// x[i-1] (deterministic, identical result).
#include "kernels.cuh"

namespace actc {

__device__ __forceinline__ uint32_t k1_saddr(const void *p) {
  // opaque: keeps the shared base in a register (no SR_CgaCtaId rematerialisation)
  uint32_t a = (uint32_t)__cvta_generic_to_shared(p), r;
  asm volatile("mov.u32 %0, %1;" : "=r"(r) : "r"(a));
  return r;
}
// one histogram count for symbol sj: an unconditional shared add (ptxas
// emits ATOMS.POPC.INC, which counts the lanes of a warp that hit one bin in
// one operation -- the dominant zero-delta bin costs no serialisation).
// Elements that must not count here (outside the window, or not valid) add
// into a per-lane scratch bin past the window; returns "outside the window"
__device__ __forceinline__ bool k1_hist_add(uint32_t hbase, uint32_t win_lo, uint32_t win_n, uint32_t sj,
                                            bool valid) {
  const uint32_t w = sj - win_lo;
  const bool in = w < win_n;
  const uint32_t bin = (in && valid) ? w : win_n + (threadIdx.x & 31);
  asm volatile("red.shared.add.u32 [%0], 1;" ::"r"(hbase + 4u * bin) : "memory");
  return !in;
}

// the tile's elements outside the histogram window (rare): global adds.
// Outliers (symbol 0) are excluded when bin 0 is outside the window: the
// kernel adds their count once at the end
__device__ __forceinline__ void k1_hist_misses(unsigned long long *__restrict__ ghist, uint32_t win_lo,
                                               uint32_t win_n, const uint32_t (&s)[K1_EPT], uint64_t base,
                                               uint64_t n) {
#pragma unroll
  for (int j = 0; j < K1_EPT; j++) {
    const uint32_t sj = s[j];
    if (sj - win_lo >= win_n && sj != 0 && base + j < n) atomicAdd(&ghist[sj], 1ull);
  }
}

template <typename SymT>
__device__ __forceinline__ void k1_store(SymT *__restrict__ sym, uint64_t base, const uint32_t (&s)[K1_EPT]) {
  if (sizeof(SymT) == 2) {
    uint4 *d = reinterpret_cast<uint4 *>(sym + base);
#pragma unroll
    for (int j = 0; j < K1_EPT / 8; j++)
      d[j] = make_uint4(s[8 * j] | (s[8 * j + 1] << 16), s[8 * j + 2] | (s[8 * j + 3] << 16),
                        s[8 * j + 4] | (s[8 * j + 5] << 16), s[8 * j + 6] | (s[8 * j + 7] << 16));
  } else {
    uint4 *d = reinterpret_cast<uint4 *>(sym + base);
#pragma unroll
    for (int j = 0; j < K1_EPT / 4; j++) d[j] = make_uint4(s[4 * j], s[4 * j + 1], s[4 * j + 2], s[4 * j + 3]);
  }
}

template <typename SymT>
__global__ void __launch_bounds__(K1_THREADS, 3) k1_quant_lorenzo_hist(
    const float *__restrict__ x, uint64_t n, QParams P, uint32_t radius, SymT *__restrict__ sym,
    unsigned long long *__restrict__ ghist, unsigned long long *__restrict__ n_outliers,
    uint32_t win_lo, uint32_t win_n, unsigned *__restrict__ nonfinite,
    long long *__restrict__ chunk_lat) {
  extern __shared__ unsigned sh_hist[];
  for (uint32_t i = threadIdx.x; i < win_n; i += blockDim.x) sh_hist[i] = 0;
  __syncthreads();
  const uint32_t hbase = k1_saddr(sh_hist);
  const int lane = threadIdx.x & 31;
  const uint64_t ntiles = (n + K1_TILE - 1) / K1_TILE;
  const uint64_t nfull = n / K1_TILE;  // tiles with no element past n
  const int R = (int)min(radius, 0x40000000u);
  unsigned outl = 0;
  bool fin_all = true;
  for (uint64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const uint64_t base = tile * K1_TILE + (uint64_t)threadIdx.x * K1_EPT;
    const bool full_tile = tile < nfull;  // warp-uniform
    float xv[K1_EPT];
    if (full_tile) {
      const float4 *p = reinterpret_cast<const float4 *>(x + base);
#pragma unroll
      for (int j = 0; j < K1_EPT / 4; j++) {
        float4 v = __ldcs(p + j);  // streaming: read once
        xv[4 * j] = v.x; xv[4 * j + 1] = v.y; xv[4 * j + 2] = v.z; xv[4 * j + 3] = v.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < K1_EPT; j++) xv[j] = (base + j < n) ? x[base + j] : 0.0f;
    }
    // fp32-pair quantizer for all 16 elements, the fp64 multiply tier for
    // the few it declines, exact fp64 only where both decline
    int q32[K1_EPT];
    unsigned slow = 0;
    if (P.dfast) {
#pragma unroll
      for (int j = 0; j < K1_EPT; j++) slow |= (unsigned)!quant_df(xv[j], P.ih, P.il, q32[j]) << j;
      if (slow) {
#pragma unroll
        for (int j = 0; j < K1_EPT; j++)
          if ((slow >> j) & 1u) slow &= ~((unsigned)quant_fast32(xv[j], P.inv, q32[j]) << j);
      }
    } else if (P.fast) {
#pragma unroll
      for (int j = 0; j < K1_EPT; j++) slow |= (unsigned)!quant_fast32(xv[j], P.inv, q32[j]) << j;
    } else {
      slow = (1u << K1_EPT) - 1;
#pragma unroll
      for (int j = 0; j < K1_EPT; j++) q32[j] = 0;
    }
    // non-finite inputs always fail the fast path (|v| < 2^29 is false for
    // inf and NaN), so only the lanes that took the slow path are checked
    if (slow) {
#pragma unroll
      for (int j = 0; j < K1_EPT; j++) fin_all &= !((slow >> j) & 1u) || isfinite(xv[j]);
    }
    long long prev64;
    {
      long long lastq = q32[K1_EPT - 1];
      if (slow >> (K1_EPT - 1)) {
        bool v;
        lastq = quant_exact((double)xv[K1_EPT - 1], P.two_eb, P.eb, v);
      }
      prev64 = __shfl_up_sync(0xffffffffu, lastq, 1);
      if (lane == 0) {
        bool dummy;
        prev64 = (base > 0 && base - 1 < n) ? quant_elem(x[base - 1], P, dummy) : 0;
      }
    }
    uint32_t s[K1_EPT];
    const bool fast32 = __all_sync(0xffffffffu, slow == 0 && prev64 >= -(1ll << 29) && prev64 <= (1ll << 29));
    if (fast32 && full_tile) {
      // every lattice value fits int32 (|q| < 2^19): 32-bit Lorenzo + histogram
      if (chunk_lat) {
        if (base == 0) chunk_lat[0] = 0;
        if (((base + K1_EPT) % ACTC_CHUNK) == 0 && base + K1_EPT < n) chunk_lat[(base + K1_EPT) / ACTC_CHUNK] = q32[K1_EPT - 1];
      }
      int prev = (int)prev64;
      bool miss = false;
#pragma unroll
      for (int j = 0; j < K1_EPT; j++) {
        const int d = q32[j] - prev;
        prev = q32[j];
        const bool o = (uint32_t)(d + R - 1) >= (uint32_t)(2 * R - 1);  // |d| >= radius
        const uint32_t sj = o ? 0u : (uint32_t)(d + R);
        s[j] = sj;
        outl += o;
        miss |= k1_hist_add(hbase, win_lo, win_n, sj, true) && !o;
      }
      k1_store<SymT>(sym, base, s);
      if (miss) k1_hist_misses(ghist, win_lo, win_n, s, base, n);
    } else {
      // general path: exact fp64 where the fast path declined, int64 deltas
      long long q[K1_EPT];
      unsigned viol = 0;
#pragma unroll
      for (int j = 0; j < K1_EPT; j++) {
        q[j] = q32[j];
        if ((slow >> j) & 1u) {
          bool vj;
          q[j] = quant_exact((double)xv[j], P.two_eb, P.eb, vj);
          viol |= (unsigned)vj << j;
        }
      }
      if (chunk_lat) {
        if (base == 0) chunk_lat[0] = 0;
        if (((base + K1_EPT) % ACTC_CHUNK) == 0 && base + K1_EPT < n) chunk_lat[(base + K1_EPT) / ACTC_CHUNK] = q[K1_EPT - 1];
      }
      long long prev = prev64;
      bool miss = false;
#pragma unroll
      for (int j = 0; j < K1_EPT; j++) {
        long long d = q[j] - prev;
        prev = q[j];
        unsigned long long ad = d < 0 ? (unsigned long long)(-d) : (unsigned long long)d;
        bool o = ad >= radius || ((viol >> j) & 1u);
        uint32_t sj = o ? 0u : (uint32_t)(d + (long long)radius);
        s[j] = sj;
        const bool valid = base + j < n;
        outl += valid && o;
        miss |= k1_hist_add(hbase, win_lo, win_n, sj, valid) && valid && !o;
      }
      if (miss) k1_hist_misses(ghist, win_lo, win_n, s, base, n);
      if (full_tile) {
        k1_store<SymT>(sym, base, s);
      } else {
#pragma unroll
        for (int j = 0; j < K1_EPT; j++)
          if (base + j < n) sym[base + j] = (SymT)s[j];
      }
    }
  }
  if (!__all_sync(0xffffffffu, fin_all) && !fin_all) atomicOr(nonfinite, 1u);  // tensor.py:56-57
  unsigned wsum = warp_sum(outl);
  if (lane == 0 && wsum) atomicAdd(n_outliers, (unsigned long long)wsum);
  // outliers are symbol 0 (bincount counts them too): counted in the window
  // when bin 0 is in it, else added here
  if (lane == 0 && wsum && win_lo != 0) atomicAdd(&ghist[0], (unsigned long long)wsum);
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < win_n; i += blockDim.x) {
    unsigned c = sh_hist[i];
    if (c) atomicAdd(&ghist[win_lo + i], (unsigned long long)c);
  }
}

template __global__ void k1_quant_lorenzo_hist<uint16_t>(const float *, uint64_t, QParams, uint32_t,
                                                         uint16_t *, unsigned long long *,
                                                         unsigned long long *, uint32_t, uint32_t,
                                                         unsigned *, long long *);
template __global__ void k1_quant_lorenzo_hist<uint32_t>(const float *, uint64_t, QParams, uint32_t,
                                                         uint32_t *, unsigned long long *,
                                                         unsigned long long *, uint32_t, uint32_t,
                                                         unsigned *, long long *);

// Histogram of an arbitrary u32 symbol stream (huffman_encode's bincount,
// huffman.py:181-183) with the out-of-range check.
__global__ void k_hist_u32(const uint32_t *__restrict__ s, uint64_t n, uint64_t alphabet,
                           unsigned long long *__restrict__ ghist, unsigned *__restrict__ bad,
                           uint32_t win_n) {
  extern __shared__ unsigned sh_hist[];
  for (uint32_t i = threadIdx.x; i < win_n; i += blockDim.x) sh_hist[i] = 0;
  __syncthreads();
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint32_t v = s[i];
    if (v >= alphabet) {
      atomicOr(bad, 1u);
      continue;
    }
    if (v < win_n)
      atomicAdd(&sh_hist[v], 1u);
    else
      atomicAdd(&ghist[v], 1ull);
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < win_n; i += blockDim.x)
    if (sh_hist[i]) atomicAdd(&ghist[i], (unsigned long long)sh_hist[i]);
}

// prequantize only (codec.py:238-251), fp32 or fp64 input, exact path.
__global__ void k_prequantize(const void *__restrict__ x, int dtype, uint64_t n, double eb,
                              long long *__restrict__ q) {
  const double two_eb = 2.0 * eb;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    double v = dtype == ACTC_DTYPE_F32 ? (double)((const float *)x)[i] : ((const double *)x)[i];
    bool viol;
    q[i] = quant_exact(v, two_eb, eb, viol);
  }
}

// Exhaustive check of K1's fast quantizer tiers: every finite fp32 bit
// pattern in [lo, lo + count) through quant_df, else quant_fast32 (when one
// claims the element; the order K1 uses) vs the exact restatement
// quant_exact (q and "no bound violation").  out[0] += mismatches, out[1]
// += elements a fast tier took.
__global__ void k_quant_check(uint64_t lo, uint64_t count, QParams P, unsigned long long *__restrict__ out) {
  unsigned long long bad = 0, fast = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < count;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const float xf = __uint_as_float((uint32_t)(lo + i));
    if (!isfinite(xf)) continue;
    int q32;
    if (!((P.dfast && quant_df(xf, P.ih, P.il, q32)) || (P.fast && quant_fast32(xf, P.inv, q32)))) continue;
    fast++;
    bool viol;
    const long long qe = quant_exact((double)xf, P.two_eb, P.eb, viol);
    bad += (qe != (long long)q32) || viol;
  }
  bad = warp_sum(bad);
  fast = warp_sum(fast);
  if ((threadIdx.x & 31) == 0) {
    if (bad) atomicAdd(&out[0], bad);
    if (fast) atomicAdd(&out[1], fast);
  }
}

// lorenzo_encode over an int64 lattice (codec.py:254-272).
__global__ void k_lorenzo_encode(const long long *__restrict__ lat, uint64_t n, uint32_t radius,
                                 const uint8_t *__restrict__ force, uint32_t *__restrict__ sym,
                                 unsigned long long *__restrict__ n_out) {
  unsigned cnt = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    long long prev = i ? lat[i - 1] : 0;
    long long d = (long long)((unsigned long long)lat[i] - (unsigned long long)prev);
    unsigned long long ad = d < 0 ? (unsigned long long)(-d) : (unsigned long long)d;
    bool o = ad >= radius || (force && force[i]);
    sym[i] = o ? 0u : (uint32_t)(d + (long long)radius);
    cnt += o;
  }
  cnt = warp_sum(cnt);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(n_out, (unsigned long long)cnt);
}

}  // namespace actc
