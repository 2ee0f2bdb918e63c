// actc_internal.cuh -- shared device helpers for the sm_100a codec kernels.
//
// Numerics: every fp64 operation that must match numpy bit for bit is an
// explicit round-to-nearest intrinsic (__ddiv_rn, __dadd_rn, __dmul_rn,
// __dsub_rn) and the library is compiled with -fmad=false, so nothing is
// contracted into an FMA.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/actc.h"

namespace actc {

constexpr double kLatticeLimit = 2305843009213693952.0;  // 2^61, codec.py:37
constexpr int kLutBits = 12;                             // decoder LUT prefix width
constexpr int kLutSize = 1 << kLutBits;
constexpr int kSymKeyBits = 26;  // live-symbol index / symbol field in 64-bit sort keys
constexpr uint32_t kMaxAlphabet = 1u << kSymKeyBits;

// ---------------------------------------------------------------------
// prequantize (codec.py:248-251) + bound check (codec.py:311-312)
// ---------------------------------------------------------------------
struct QParams {
  double eb;
  double two_eb;   // 2.0 * eb (exact scaling; may be +inf like numpy)
  double inv;      // fl64(1 / two_eb) -- fast-path multiplier
  int fast;        // inv is finite and normal
  float ih, il;    // inv as an unevaluated fp32 pair: ih = fl32(inv), il = fl32(inv - ih)
  int dfast;       // the fp32-pair tier applies (ih finite and normal)
};

// Exact restatement: v = x / (2eb); q = sign(v)*floor(fl(|v| + 0.5));
// clip +-2^61; recon = q*(2eb); viol = |x - recon| > eb.
__device__ __forceinline__ long long quant_exact(double x, double two_eb, double eb, bool &viol) {
  double v = __ddiv_rn(x, two_eb);
  double f = floor(__dadd_rn(fabs(v), 0.5));
  double q = v > 0.0 ? f : (v < 0.0 ? -f : 0.0);
  q = fmax(fmin(q, kLatticeLimit), -kLatticeLimit);
  double recon = __dmul_rn(q, two_eb);
  viol = fabs(__dsub_rn(x, recon)) > eb;
  return (long long)q;
}

// Fast path in fp64 with a multiply instead of the division.
// v' = x * fl64(1/(2eb)) is within |v|*2^-51 of the true quotient; when the
// distance of |v'| to the rounding boundary exceeds (|v'|+1)*2^-44 the exact
// path (x / 2eb, floor(fl(|v|+0.5))) provably yields the same q, and
// |x - q*2eb| <= eb*(1 - m) so the bound check cannot fire.  With |v'| <
// 2^29 that margin is below 2^-14, which is used as a constant (three fp64
// operations fewer per element; ~1e-4 of elements take the exact path
// instead).  Returns false when the caller must take quant_exact.
__device__ __forceinline__ bool quant_fast32(float xf, double inv, int &q) {
  const double v = __dmul_rn((double)xf, inv);
  const double a = fabs(v);
  const double f = floor(__dadd_rn(a, 0.5));
  const double r = __dsub_rn(a, f);
  const bool safe = (a < 0x1p29) && (fabs(r) < 0.49993896484375);  // 0.5 - 2^-14
  const int qi = (int)f;
  q = xf > 0.0f ? qi : -qi;
  return safe;
}
// First tier, all fp32 at full rate (no fp64, no conversion-pipe op):
// v ~ x*(ih + il) as p + e (p = fl32(x*ih), e = the product's exact error by
// FMA plus x*il), rounded to the nearest integer r by the 1.5*2^23 magic
// add (|p| < 2^22), d = (p - r) + e.  |(ih + il) - 1/two_eb| <= inv*2^-47.9,
// and with |p| < 2^22 the rounding errors of e and d stay below 2^-23, so
// |v - r| < 0.5 - 2^-21 whenever |d| < 0.5 - 2^-20: then q = r is numpy's
// sign(v)*floor(|v| + 0.5) (fl64(|v| + 0.5) cannot reach the next integer)
// and |x - q*2eb| <= eb*(1 - 2^-20) rules out a bound violation.  Returns
// false (caller takes quant_fast32 / quant_exact) otherwise, and for
// non-finite x.  Verified for every fp32 pattern by k_quant_check.
__device__ __forceinline__ bool quant_df(float xf, float ih, float il, int &q) {
  const float p = __fmul_rn(xf, ih);
  float e = __fmaf_rn(xf, ih, -p);
  e = __fmaf_rn(xf, il, e);
  const float m = __fadd_rn(p, 12582912.0f);  // 1.5 * 2^23: rounds p to an integer
  const float r = __fsub_rn(m, 12582912.0f);
  const float d = __fadd_rn(__fsub_rn(p, r), e);
  q = __float_as_int(m) - 0x4B400000;
  return fabsf(p) < 0x1p22f && fabsf(d) < 0.49999904632568359375f;  // 0.5 - 2^-20
}

__device__ __forceinline__ bool quant_fast(float xf, double inv, long long &q) {
  int q32;
  const bool safe = quant_fast32(xf, inv, q32);
  q = q32;
  return safe;
}

__device__ __forceinline__ long long quant_elem(float xf, const QParams &P, bool &viol) {
  long long q;
  viol = false;
  int qd;
  if (P.dfast && quant_df(xf, P.ih, P.il, qd)) return qd;
  if (P.fast && quant_fast(xf, P.inv, q)) return q;
  return quant_exact((double)xf, P.two_eb, P.eb, viol);
}

// ---------------------------------------------------------------------
// bit / memory helpers
// ---------------------------------------------------------------------
__device__ __forceinline__ uint32_t bswap32(uint32_t w) { return __byte_perm(w, 0, 0x0123); }

__device__ __forceinline__ unsigned ld_acquire(const unsigned *p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned *p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_relaxed_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_u64(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_relaxed_u32(const unsigned *p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// lookback flag bits
constexpr unsigned kFlagAgg = 1u;
constexpr unsigned kFlagInc = 2u;
constexpr unsigned kFlagTail = 4u;

// ---------------------------------------------------------------------
// warp / block scans
// ---------------------------------------------------------------------
template <typename T>
__device__ __forceinline__ T warp_incl_sum(T v) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    T t = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += t;
  }
  return v;
}

template <typename T>
__device__ __forceinline__ T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Block-wide exclusive sum; `warp_buf` needs blockDim/32 + 1 entries of T.
// Returns the exclusive prefix; *total receives the block total.
template <typename T>
__device__ __forceinline__ T block_excl_sum(T v, T *warp_buf, T *total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  T inc = warp_incl_sum(v);
  if (lane == 31) warp_buf[wid] = inc;
  __syncthreads();
  if (wid == 0) {
    T w = lane < nw ? warp_buf[lane] : T(0);
    T wi = warp_incl_sum(w);
    if (lane < nw) warp_buf[lane] = wi - w;
    if (lane == nw - 1) warp_buf[nw] = wi;
  }
  __syncthreads();
  T res = warp_buf[wid] + inc - v;
  *total = warp_buf[nw];
  __syncthreads();
  return res;
}

// Segmented scan element for the inverse Lorenzo chain (codec.py:286-292):
// reset=1 means "value is an absolute lattice value" (an outlier rebased
// the chain inside the segment); otherwise value is a relative sum.
struct Seg {
  long long v;
  int r;
};
__device__ __forceinline__ Seg seg_combine(Seg a, Seg b) {
  Seg o;
  o.r = a.r | b.r;
  o.v = b.r ? b.v : a.v + b.v;
  return o;
}

__device__ __forceinline__ Seg warp_incl_seg(Seg s) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    long long tv = __shfl_up_sync(0xffffffffu, s.v, o);
    int tr = __shfl_up_sync(0xffffffffu, s.r, o);
    if (lane >= o) {
      Seg t{tv, tr};
      s = seg_combine(t, s);
    }
  }
  return s;
}

}  // namespace actc
