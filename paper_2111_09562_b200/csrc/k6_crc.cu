// K6: CRC-32 (zlib polynomial, reflected) of a device buffer, bit-identical
// to zlib.crc32(data, value) -- the checksum CMTZ appends (codec.py:118) and
// verifies (codec.py:126).
//
// The raw CRC (register starts at 0, no final xor) is linear over GF(2):
//   raw(A || B) = Z_|B|(raw(A)) ^ raw(B)
// where Z_n is the 32x32 bit matrix "feed n zero bytes through the register".
// So every thread checksums its own 256-byte piece (slicing-by-8 tables in
// shared memory), a warp folds its 32 piece values with Z_256, Z_512, ...
// (a log-depth tree, one matrix per level), the CTA folds its 8 warps, and
// the last CTA to finish folds the per-CTA values.  The stream is padded with
// zeros at the END to a whole number of 64 KiB blocks, so every piece and
// block has the same size; the padding is undone with the inverse matrices
// (x is invertible modulo the CRC polynomial).  Finally the caller's running
// value enters as Z_L(~value) and the result is complemented, as in zlib.
//
// Z_{2^k} and Z_{2^k}^{-1} for k < 48 live in constant memory (uniform
// indices: broadcast reads); built on the host once per device.
#include <mutex>

#include "kernels.cuh"

namespace actc {

namespace {

constexpr uint32_t kPoly = 0xEDB88320u;  // reflected 0x04C11DB7
constexpr int kPiece = 256;              // bytes per thread
constexpr int kCrcThreads = 256;
constexpr uint64_t kBlock = (uint64_t)kPiece * kCrcThreads;  // 64 KiB per CTA
constexpr int kLogPiece = 8, kLogWarp = 13, kLogBlock = 16;
constexpr int kMats = 48;

__constant__ uint32_t c_z[kMats][32];     // c_z[k][i]  = Z_{2^k} applied to bit i
__constant__ uint32_t c_zinv[kMats][32];  // c_zinv[k][i] = Z_{2^k}^{-1} applied to bit i
__device__ uint32_t g_tab[8][256];        // slicing-by-8

__device__ __forceinline__ uint32_t zmul(const uint32_t (&m)[32], uint32_t c) {
  uint32_t r = 0;
#pragma unroll
  for (int i = 0; i < 32; i++) r ^= (0u - ((c >> i) & 1u)) & m[i];
  return r;
}

// raw CRC of 8 bytes (w0 = bytes 0..3, w1 = bytes 4..7, little-endian)
__device__ __forceinline__ uint32_t crc8(const uint32_t *t, uint32_t c, uint32_t w0, uint32_t w1) {
  c ^= w0;
  return t[7 * 256 + (c & 0xFF)] ^ t[6 * 256 + ((c >> 8) & 0xFF)] ^ t[5 * 256 + ((c >> 16) & 0xFF)] ^
         t[4 * 256 + (c >> 24)] ^ t[3 * 256 + (w1 & 0xFF)] ^ t[2 * 256 + ((w1 >> 8) & 0xFF)] ^
         t[1 * 256 + ((w1 >> 16) & 0xFF)] ^ t[w1 >> 24];
}

// warp fold: lane l holds the raw CRC of segment l (2^lg bytes each);
// lane 0 returns the raw CRC of the 32 segments in order
__device__ __forceinline__ uint32_t warp_fold(uint32_t v, int lg) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int j = 0; j < 5; j++) {
    const uint32_t u = __shfl_down_sync(0xffffffffu, v, 1 << j);
    const uint32_t sh = zmul(c_z[lg + j], v);
    if ((lane & ((2 << j) - 1)) == 0) v = sh ^ u;
  }
  return v;
}

__global__ void __launch_bounds__(kCrcThreads) k6_crc32(const uint8_t *__restrict__ data, uint64_t len,
                                                      uint32_t crc_in, uint32_t *__restrict__ part,
                                                      unsigned *__restrict__ ticket, uint32_t *__restrict__ out) {
  __shared__ uint32_t tab[8 * 256];
  __shared__ uint32_t wv[kCrcThreads / 32];
  __shared__ unsigned s_last;
  for (int i = threadIdx.x; i < 8 * 256; i += kCrcThreads) tab[i] = (&g_tab[0][0])[i];
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint64_t p0 = (uint64_t)blockIdx.x * kBlock + (uint64_t)threadIdx.x * kPiece;
  uint32_t c = 0;
  if (p0 + kPiece <= len) {
    const uint4 *src = reinterpret_cast<const uint4 *>(data + p0);
#pragma unroll 4
    for (int u = 0; u < kPiece / 16; u++) {
      const uint4 v = __ldg(src + u);
      c = crc8(tab, c, v.x, v.y);
      c = crc8(tab, c, v.z, v.w);
    }
  } else if (p0 < len) {
    // the piece holding the end: bytes past `len` count as zero padding
    const uint4 *src = reinterpret_cast<const uint4 *>(data + p0);
    for (int u = 0; u < kPiece / 16; u++) {
      const uint64_t o = p0 + 16ull * u;
      uint4 v = make_uint4(0, 0, 0, 0);
      if (o < len) {
        v = __ldg(src + u);
        const uint64_t keep = len - o;  // valid bytes in this 16-byte word (may be >= 16)
        uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int q = 0; q < 4; q++) {
          const int64_t kb = (int64_t)keep - 4 * q;
          if (kb <= 0) w[q] = 0;
          else if (kb < 4) w[q] &= (1u << (8 * kb)) - 1u;
        }
        v = make_uint4(w[0], w[1], w[2], w[3]);
      }
      c = crc8(tab, c, v.x, v.y);
      c = crc8(tab, c, v.z, v.w);
    }
  } else {
    // all padding: the raw CRC of zeros fed into a zero register is zero
  }
  c = warp_fold(c, kLogPiece);
  if (lane == 0) wv[warp] = c;
  __syncthreads();
  if (warp == 0) {
    uint32_t v = lane < kCrcThreads / 32 ? wv[lane] : 0u;
    // 8 warps: fold as 32 lanes whose first 24 are leading zeros -- leading
    // zero segments do not change a raw CRC, so shift the 8 values to the top
    v = __shfl_up_sync(0xffffffffu, v, 32 - kCrcThreads / 32);
    if (lane < 32 - kCrcThreads / 32) v = 0u;
    v = warp_fold(v, kLogWarp);
    if (lane == 0) {
      part[blockIdx.x] = v;
      __threadfence();
      s_last = atomicAdd(ticket, 1u) == gridDim.x - 1;
    }
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // last CTA: fold the nb block values.  Thread t takes m consecutive blocks
  // (m a power of two) of a sequence front-padded with zero blocks to 256*m
  const uint32_t nb = gridDim.x;
  uint32_t m = 1;
  int lgm = 0;
  while ((uint64_t)m * kCrcThreads < nb) {
    m <<= 1;
    lgm++;
  }
  const int64_t pad = (int64_t)m * kCrcThreads - nb;
  uint32_t acc = 0;
  for (uint32_t i = 0; i < m; i++) {
    const int64_t b = (int64_t)threadIdx.x * m + i - pad;
    acc = zmul(c_z[kLogBlock], acc);
    if (b >= 0) acc ^= __ldcg(&part[b]);
  }
  acc = warp_fold(acc, kLogBlock + lgm);
  if (lane == 0) wv[warp] = acc;
  __syncthreads();
  if (warp == 0) {
    uint32_t v = lane < kCrcThreads / 32 ? wv[lane] : 0u;
    v = __shfl_up_sync(0xffffffffu, v, 32 - kCrcThreads / 32);
    if (lane < 32 - kCrcThreads / 32) v = 0u;
    v = warp_fold(v, kLogBlock + lgm + 5);
    if (lane == 0) {
      // undo the trailing zero padding, then bring in the running value
      const uint64_t z = (uint64_t)nb * kBlock - len;
      for (int k = 0; k < kMats; k++)
        if ((z >> k) & 1ull) v = zmul(c_zinv[k], v);
      uint32_t r = ~crc_in;
      for (int k = 0; k < kMats; k++)
        if ((len >> k) & 1ull) r = zmul(c_z[k], r);
      *out = ~(v ^ r);
      *ticket = 0u;  // ready for the next launch
    }
  }
}

// ---- host: tables and matrices (once per device) ----
void gf2_square(uint32_t *sq, const uint32_t *m) {
  for (int i = 0; i < 32; i++) {
    uint32_t r = 0, c = m[i];
    for (int j = 0; j < 32; j++)
      if ((c >> j) & 1u) r ^= m[j];
    sq[i] = r;
  }
}

int crc_init_device(int dev) {
  static std::mutex mu;
  static uint64_t done = 0;
  std::lock_guard<std::mutex> g(mu);
  if (dev < 64 && ((done >> dev) & 1ull)) return 0;
  static uint32_t tab[8][256], z[kMats][32], zi[kMats][32];
  static bool built = false;
  if (!built) {
    for (uint32_t n = 0; n < 256; n++) {
      uint32_t c = n;
      for (int k = 0; k < 8; k++) c = (c >> 1) ^ ((c & 1u) ? kPoly : 0u);
      tab[0][n] = c;
    }
    for (int k = 1; k < 8; k++)
      for (int n = 0; n < 256; n++) tab[k][n] = (tab[k - 1][n] >> 8) ^ tab[0][tab[k - 1][n] & 0xFF];
    // one zero byte = eight zero bits: forward c -> (c >> 1) ^ (c & 1 ? P : 0);
    // inverse: bit 31 of the image says whether P was folded in
    for (int i = 0; i < 32; i++) {
      uint32_t c = 1u << i, d = 1u << i;
      for (int b = 0; b < 8; b++) {
        c = (c >> 1) ^ ((c & 1u) ? kPoly : 0u);
        d = (d & 0x80000000u) ? (((d ^ kPoly) << 1) | 1u) : (d << 1);
      }
      z[0][i] = c;
      zi[0][i] = d;
    }
    for (int k = 1; k < kMats; k++) {
      gf2_square(z[k], z[k - 1]);
      gf2_square(zi[k], zi[k - 1]);
    }
    built = true;
  }
  if (cudaMemcpyToSymbol(c_z, z, sizeof(z)) != cudaSuccess) return -1;
  if (cudaMemcpyToSymbol(c_zinv, zi, sizeof(zi)) != cudaSuccess) return -1;
  if (cudaMemcpyToSymbol(g_tab, tab, sizeof(tab)) != cudaSuccess) return -1;
  if (dev < 64) done |= 1ull << dev;
  return 0;
}

}  // namespace

// number of per-CTA scratch words crc32_launch needs for `len` bytes
uint64_t crc32_blocks(uint64_t len) { return len ? (len + kBlock - 1) / kBlock : 1; }

// data must be 16-byte aligned; part holds crc32_blocks(len) words; ticket
// is zero (and left zero); *out_dev receives zlib.crc32(data, crc_in)
int crc32_launch(const uint8_t *data, uint64_t len, uint32_t crc_in, uint32_t *part, unsigned *ticket,
                 uint32_t *out_dev, cudaStream_t s) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || crc_init_device(dev)) return -1;
  const uint64_t nb = crc32_blocks(len);
  if (nb > 0x7FFFFFFFull) return -1;
  k6_crc32<<<(unsigned)nb, kCrcThreads, 0, s>>>(data, len, crc_in, part, ticket, out_dev);
  return cudaPeekAtLastError() == cudaSuccess ? 0 : -1;
}

}  // namespace actc
