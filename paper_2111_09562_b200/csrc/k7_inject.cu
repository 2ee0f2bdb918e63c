// K7: uniform error injection on the device, bit-identical to the
// reference's inject_uniform_error (errorprop.py:127-139):
//   rng   = np.random.default_rng(seed)            (PCG64, SeedSequence-seeded)
//   noise = rng.uniform(-eb, eb, size=n)           low + (high-low) * next_double
//   noise[data == 0] = 0        if preserve_zeros
//   out   = f64(x) + noise
// The host hands over the PCG64 state numpy derives from the seed (128-bit
// state and increment).  PCG64 is an LCG on 2^128 with the XSL-RR output
// (numpy pcg64.h: step, then output of the new state); element i uses draw
// i+1, so each thread jumps its own copy of the generator to its first
// element in O(log n) (the LCG advance: (A, C) composed by squaring) and
// then steps through K consecutive elements.
#include "kernels.cuh"

namespace actc {

namespace {

typedef unsigned __int128 u128;

constexpr int kInjThreads = 256;
constexpr int kInjPer = 64;  // consecutive elements per thread

__device__ __forceinline__ u128 pcg_mult() {
  return ((u128)2549297995355413924ull << 64) | (u128)4865540595714422341ull;
}

// state after `delta` steps of s <- s * M + inc
__device__ __forceinline__ u128 pcg_advance(u128 s, u128 inc, unsigned long long delta) {
  u128 cur_mult = pcg_mult(), cur_plus = inc, acc_mult = 1, acc_plus = 0;
  while (delta) {
    if (delta & 1ull) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * s + acc_plus;
}

__device__ __forceinline__ unsigned long long pcg_out(u128 s) {
  const unsigned long long x = (unsigned long long)(s >> 64) ^ (unsigned long long)s;
  const unsigned r = (unsigned)(s >> 122);
  return (x >> r) | (x << ((64u - r) & 63u));
}

template <typename T>
__global__ void __launch_bounds__(kInjThreads) k7_inject(const T *__restrict__ x, uint64_t n, double low,
                                                       double range, int preserve, unsigned long long st_hi,
                                                       unsigned long long st_lo, unsigned long long inc_hi,
                                                       unsigned long long inc_lo, double *__restrict__ out) {
  const uint64_t t = (uint64_t)blockIdx.x * kInjThreads + threadIdx.x;
  const uint64_t e0 = t * kInjPer;
  if (e0 >= n) return;
  const u128 inc = ((u128)inc_hi << 64) | inc_lo;
  u128 s = pcg_advance(((u128)st_hi << 64) | st_lo, inc, e0);
  const u128 M = pcg_mult();
  const uint64_t e1 = min(n, e0 + kInjPer);
  for (uint64_t e = e0; e < e1; e++) {
    s = s * M + inc;
    const double u = (double)(pcg_out(s) >> 11) * (1.0 / 9007199254740992.0);
    double noise = __dadd_rn(low, __dmul_rn(range, u));
    const double d = (double)x[e];
    if (preserve && d == 0.0) noise = 0.0;
    out[e] = __dadd_rn(d, noise);
  }
}

}  // namespace

int inject_launch(const void *x, int dtype, uint64_t n, double eb, int preserve, const uint64_t state[4],
                  double *out, cudaStream_t s) {
  if (!n) return 0;
  const uint64_t threads = (n + kInjPer - 1) / kInjPer;
  const uint64_t grid = (threads + kInjThreads - 1) / kInjThreads;
  const double low = -eb, range = eb - (-eb);  // numpy: low + (high - low) * u
  if (dtype == ACTC_DTYPE_F64)
    k7_inject<double><<<(unsigned)grid, kInjThreads, 0, s>>>((const double *)x, n, low, range, preserve, state[0],
                                                              state[1], state[2], state[3], out);
  else
    k7_inject<float><<<(unsigned)grid, kInjThreads, 0, s>>>((const float *)x, n, low, range, preserve, state[0],
                                                             state[1], state[2], state[3], out);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace actc
