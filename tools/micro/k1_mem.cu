// Memory-pattern bound of K1: read fp32, write u16, same tiling as K1
// (256 threads x 16 elements, grid-stride over 4096-element tiles).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int EPT, bool CS>
__global__ void __launch_bounds__(256) rw(const float *__restrict__ x, uint16_t *__restrict__ y, uint64_t n) {
  const uint64_t tile = 256 * EPT;
  const uint64_t nt = n / tile;
  for (uint64_t t = blockIdx.x; t < nt; t += gridDim.x) {
    const uint64_t base = t * tile + threadIdx.x * EPT;
    float v[EPT];
    const float4 *p = reinterpret_cast<const float4 *>(x + base);
#pragma unroll
    for (int j = 0; j < EPT / 4; j++) {
      float4 a = CS ? __ldcs(p + j) : p[j];
      v[4 * j] = a.x; v[4 * j + 1] = a.y; v[4 * j + 2] = a.z; v[4 * j + 3] = a.w;
    }
    uint32_t s[EPT / 2];
#pragma unroll
    for (int j = 0; j < EPT / 2; j++) s[j] = (__float_as_uint(v[2 * j]) >> 16) | (__float_as_uint(v[2 * j + 1]) & 0xFFFF0000u);
    uint4 *d = reinterpret_cast<uint4 *>(y + base);
#pragma unroll
    for (int j = 0; j < EPT / 8; j++) d[j] = make_uint4(s[4 * j], s[4 * j + 1], s[4 * j + 2], s[4 * j + 3]);
  }
}

// coalesced mapping: each thread one float4 per row, rows strided by the CTA
__global__ void __launch_bounds__(256) rw_coal(const float4 *__restrict__ x, uint2 *__restrict__ y, uint64_t n4) {
  for (uint64_t i = blockIdx.x * 256ull + threadIdx.x; i < n4; i += (uint64_t)gridDim.x * 256) {
    float4 a = __ldcs(x + i);
    y[i] = make_uint2((__float_as_uint(a.x) >> 16) | (__float_as_uint(a.y) & 0xFFFF0000u),
                      (__float_as_uint(a.z) >> 16) | (__float_as_uint(a.w) & 0xFFFF0000u));
  }
}

template <typename F>
float timeit(F f) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  f();
  cudaDeviceSynchronize();
  float best = 1e9;
  for (int r = 0; r < 10; r++) {
    cudaEventRecord(a);
    f();
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms < best ? ms : best;
  }
  return best * 1e3f;
}

int main() {
  const uint64_t n = 49561600ull;  // conv1 of the bench (49.6 M elements)
  float *x;
  uint16_t *y;
  cudaMalloc(&x, n * 4);
  cudaMalloc(&y, n * 2);
  cudaMemset(x, 0, n * 4);
  const double bytes = n * 6.0;
  for (int g : {148 * 2, 148 * 3, 148 * 4, 148 * 8}) {
    float t1 = timeit([&] { rw<16, true><<<g, 256>>>(x, y, n); });
    float t2 = timeit([&] { rw<16, false><<<g, 256>>>(x, y, n); });
    float t3 = timeit([&] { rw<8, true><<<g, 256>>>(x, y, n); });
    float t4 = timeit([&] { rw_coal<<<g, 256>>>((const float4 *)x, (uint2 *)y, n / 4); });
    printf("grid %d: ept16 cs %.1f us (%.0f GB/s)  ept16 %.1f  ept8 cs %.1f  coalesced %.1f us (%.0f GB/s)\n", g, t1,
           bytes / t1 / 1e3, t2, t3, t4, bytes / t4 / 1e3);
  }
  return 0;
}
