// K5: per-layer statistics that feed the adaptive error-bound controller.
//
//   R      count_nonzero / size          tensor.py:180-181, training.py:351-352
//   L_bar  mean over samples of max|g|   training.py:358-361
//   M_avg  mean(|v|) of the velocity     nn.py:249-253, controller.py:169
//
// Bit-exactness of the means: numpy reduces with pairwise summation (blocks
// of <= 128 elements summed with 8 strided accumulators, split point
// n2 = n/2 - (n/2) % 8) in the input dtype; the fp32 mean is
// f32(f64(sum)/n).  We replay that exact tree: the top `depth` levels are
// enumerated by thread index, each thread sums its subtree sequentially in
// the same order, and one thread folds the partials back up the tree.
#include "kernels.cuh"

namespace actc {

namespace {

template <typename T>
__device__ __forceinline__ T absv(T v) { return v < T(0) ? -v : (v == T(0) ? T(0) : v); }

// numpy pairwise sum of |a[0..n)| (loops_utils.h.src pairwise_sum), iterative
template <typename T>
__device__ T pairwise_abs(const T *__restrict__ a, uint64_t n) {
  // explicit stack of (offset, length, state) emulating the recursion
  struct Fr { uint64_t off, len; T left; int st; };
  Fr stk[48];
  int sp = 0;
  stk[0] = {0, n, T(0), 0};
  T ret = T(0);
  while (sp >= 0) {
    Fr &f = stk[sp];
    if (f.st == 0) {
      if (f.len < 8) {
        T r = T(0);
        for (uint64_t i = 0; i < f.len; i++) r = r + absv(a[f.off + i]);
        ret = r;
        sp--;
        continue;
      }
      if (f.len <= 128) {
        T r[8];
#pragma unroll
        for (int j = 0; j < 8; j++) r[j] = absv(a[f.off + j]);
        uint64_t i;
        const uint64_t lim = f.len - (f.len % 8);
        for (i = 8; i < lim; i += 8) {
#pragma unroll
          for (int j = 0; j < 8; j++) r[j] = r[j] + absv(a[f.off + i + j]);
        }
        T res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
        for (; i < f.len; i++) res = res + absv(a[f.off + i]);
        ret = res;
        sp--;
        continue;
      }
      uint64_t n2 = f.len / 2;
      n2 -= n2 % 8;
      f.st = 1;
      stk[sp + 1] = {f.off, n2, T(0), 0};
      sp++;
      continue;
    }
    if (f.st == 1) {
      f.left = ret;
      f.st = 2;
      uint64_t n2 = f.len / 2;
      n2 -= n2 % 8;
      stk[sp + 1] = {f.off + n2, f.len - n2, T(0), 0};
      sp++;
      continue;
    }
    ret = f.left + ret;
    sp--;
  }
  return ret;
}

// descend `depth` levels following the bits of t (MSB first); returns false
// if the path ends at a leaf above `depth` and t is not the leaf's canonical
// (lowest) index.
__device__ __forceinline__ bool node_of(uint64_t n, int depth, uint64_t t, uint64_t &off,
                                        uint64_t &len) {
  off = 0;
  len = n;
  for (int d = 0; d < depth; d++) {
    if (len <= 128) {
      uint64_t rest = t & ((1ull << (depth - d)) - 1);
      return rest == 0;
    }
    uint64_t n2 = len / 2;
    n2 -= n2 % 8;
    if ((t >> (depth - 1 - d)) & 1) {
      off += n2;
      len -= n2;
    } else {
      len = n2;
    }
  }
  return true;
}

template <typename T>
__device__ T fold(const double *__restrict__ partial, uint64_t len, int d, int depth, uint64_t p) {
  // iterative post-order fold of the top levels
  struct Fr { uint64_t len, p; int d; T left; int st; };
  Fr stk[40];
  int sp = 0;
  stk[0] = {len, p, d, T(0), 0};
  T ret = T(0);
  while (sp >= 0) {
    Fr &f = stk[sp];
    if (f.st == 0) {
      if (f.d == depth || f.len <= 128) {
        ret = (T)partial[f.p << (depth - f.d)];
        sp--;
        continue;
      }
      uint64_t n2 = f.len / 2;
      n2 -= n2 % 8;
      f.st = 1;
      stk[sp + 1] = {n2, f.p * 2, f.d + 1, T(0), 0};
      sp++;
      continue;
    }
    if (f.st == 1) {
      f.left = ret;
      f.st = 2;
      uint64_t n2 = f.len / 2;
      n2 -= n2 % 8;
      stk[sp + 1] = {f.len - n2, f.p * 2 + 1, f.d + 1, T(0), 0};
      sp++;
      continue;
    }
    ret = f.left + ret;
    sp--;
  }
  return ret;
}

}  // namespace

__global__ void k_count_nonzero(const void *__restrict__ x, int dtype, uint64_t n,
                                unsigned long long *__restrict__ out) {
  unsigned long long c = 0;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (dtype == ACTC_DTYPE_F32)
      c += ((const float *)x)[i] != 0.0f;
    else
      c += ((const double *)x)[i] != 0.0;
  }
  c = warp_sum(c);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void k_pairwise_partials(const void *__restrict__ x, int dtype, uint64_t n, int depth,
                                    double *__restrict__ partial) {
  uint64_t t = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (t >= (1ull << depth)) return;
  uint64_t off, len;
  if (!node_of(n, depth, t, off, len)) return;
  if (dtype == ACTC_DTYPE_F32)
    partial[t] = (double)pairwise_abs<float>((const float *)x + off, len);
  else
    partial[t] = pairwise_abs<double>((const double *)x + off, len);
}

__global__ void k_pairwise_finish(const double *__restrict__ partial, int dtype, uint64_t n,
                                  int depth, double *__restrict__ out) {
  if (threadIdx.x || blockIdx.x) return;
  if (dtype == ACTC_DTYPE_F32) {
    float s = fold<float>(partial, n, 0, depth, 0);
    *out = (double)(float)((double)s / (double)n);  // numpy _mean for float32
  } else {
    double s = fold<double>(partial, n, 0, depth, 0);
    *out = s / (double)n;
  }
}

// per-sample max |g| via integer atomicMax on the IEEE bits (values >= 0)
__global__ void k_sample_max(const void *__restrict__ g, int dtype, uint64_t N, uint64_t per,
                             unsigned long long *__restrict__ bits) {
  const uint64_t total = N * per;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < total;
       i += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t s = i / per;
    if (dtype == ACTC_DTYPE_F32) {
      float v = fabsf(((const float *)g)[i]);
      unsigned u = __float_as_uint(v);
      if (u) atomicMax(&bits[s], (unsigned long long)u);
    } else {
      double v = fabs(((const double *)g)[i]);
      unsigned long long u = (unsigned long long)__double_as_longlong(v);
      if (u) atomicMax(&bits[s], u);
    }
  }
}

// mean of the N per-sample maxima with numpy's pairwise order
__global__ void k_lbar_finish(const unsigned long long *__restrict__ bits, int dtype, uint64_t N,
                              void *__restrict__ per_sample_max, double *__restrict__ out) {
  if (threadIdx.x || blockIdx.x) return;
  // maxima are non-negative, so |m| == m and pairwise_abs is the plain sum
  if (dtype == ACTC_DTYPE_F32) {
    float *m = (float *)per_sample_max;
    for (uint64_t s = 0; s < N; s++) m[s] = __uint_as_float((unsigned)bits[s]);
    float sum = pairwise_abs<float>(m, N);
    *out = (double)(float)((double)sum / (double)N);
  } else {
    double *m = (double *)per_sample_max;
    for (uint64_t s = 0; s < N; s++) m[s] = __longlong_as_double((long long)bits[s]);
    double sum = pairwise_abs<double>(m, N);
    *out = sum / (double)N;
  }
}

__global__ void k_excl_scan_u64(const unsigned long long *__restrict__ in, uint64_t m,
                                unsigned long long *__restrict__ out,
                                unsigned long long *__restrict__ total) {
  __shared__ unsigned long long wb[33];
  unsigned long long run = 0;
  for (uint64_t c = 0; c < m; c += blockDim.x) {
    uint64_t i = c + threadIdx.x;
    unsigned long long v = i < m ? in[i] : 0;
    unsigned long long tot;
    unsigned long long ex = block_excl_sum<unsigned long long>(v, wb, &tot);
    if (i < m) out[i] = run + ex;
    run += tot;
  }
  if (threadIdx.x == 0) *total = run;
}

}  // namespace actc
