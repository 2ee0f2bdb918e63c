// actc_api.cu -- the C ABI (include/actc.h): context, scratch management and
// launch orchestration of K1..K5.  No torch types cross this boundary.
#include <float.h>
#include <stddef.h>
#include <stdarg.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <atomic>
#include <mutex>
#include <vector>

#include "kernels.cuh"

using namespace actc;

namespace {

thread_local char g_err[512];

int set_err(int code, const char *fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
  return code;
}

#define CK(call)                                                                 \
  do {                                                                           \
    cudaError_t e_ = (call);                                                     \
    if (e_ != cudaSuccess)                                                       \
      return set_err(ACTC_ECUDA, "%s failed: %s", #call, cudaGetErrorString(e_)); \
  } while (0)

#define CKL()                                                                   \
  do {                                                                          \
    cudaError_t e_ = cudaGetLastError();                                        \
    if (e_ != cudaSuccess)                                                      \
      return set_err(ACTC_ECUDA, "launch failed: %s", cudaGetErrorString(e_)); \
  } while (0)

struct Buf {
  void *p = nullptr;
  size_t cap = 0;
};

int grow(Buf &b, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (b.cap >= bytes) return ACTC_OK;
  if (b.p) cudaFree(b.p);
  b.p = nullptr;
  b.cap = 0;
  size_t want = bytes + bytes / 8 + 256;  // headroom to avoid re-growing by a few bytes
  cudaError_t e = cudaMalloc(&b.p, want);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_err(ACTC_ENOMEM, "cudaMalloc(%zu) failed: %s", want, cudaGetErrorString(e));
  }
  b.cap = want;
  return ACTC_OK;
}

// ---- launch instrumentation (actc_timing_enable / actc_kernel_stats) ----
struct KRec {
  int kind;
  cudaEvent_t a, b;
  cudaStream_t s;
};
std::atomic<unsigned long long> g_launches[ACTC_KIND_NKINDS];
std::atomic<bool> g_timing{false};
std::mutex g_tmu;
std::vector<KRec> g_recs;
std::vector<cudaEvent_t> g_pool;

cudaEvent_t pool_event() {
  cudaEvent_t e = nullptr;
  if (!g_pool.empty()) {
    e = g_pool.back();
    g_pool.pop_back();
  } else if (cudaEventCreate(&e) != cudaSuccess) {
    cudaGetLastError();
    e = nullptr;
  }
  return e;
}

// Scope guard around one kernel launch: counts it and, when timing is on,
// brackets it with events on its own stream.
struct KTimer {
  int kind;
  cudaStream_t s;
  cudaEvent_t a = nullptr, b = nullptr;
  KTimer(int k, cudaStream_t st) : kind(k), s(st) {
    g_launches[k].fetch_add(1, std::memory_order_relaxed);
    if (g_timing.load(std::memory_order_relaxed)) {
      std::lock_guard<std::mutex> g(g_tmu);
      a = pool_event();
      b = pool_event();
      if (a && b) cudaEventRecord(a, s);
    }
  }
  ~KTimer() {
    if (a && b) {
      cudaEventRecord(b, s);
      std::lock_guard<std::mutex> g(g_tmu);
      g_recs.push_back({kind, a, b, s});
    } else {
      std::lock_guard<std::mutex> g(g_tmu);
      if (a) g_pool.push_back(a);
      if (b) g_pool.push_back(b);
    }
  }
};
#define KT(kind) KTimer kt_guard_(kind, s)

// memoised cudaOccupancyMaxActiveBlocksPerMultiprocessor (the query costs
// microseconds of host time and sits on every encode/decode launch)
int occupancy(const void *f, int threads, size_t smem) {
  struct Key {
    const void *f;
    int t;
    size_t s;
    int v;
  };
  static std::mutex mu;
  static std::vector<Key> memo;
  {
    std::lock_guard<std::mutex> g(mu);
    for (const Key &k : memo)
      if (k.f == f && k.t == threads && k.s == smem) return k.v;
  }
  int v = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, f, threads, smem);
  std::lock_guard<std::mutex> g(mu);
  if (memo.size() < 256) memo.push_back({f, threads, smem, v});
  return v;
}

inline uint64_t cdiv(uint64_t a, uint64_t b) { return (a + b - 1) / b; }
inline uint64_t pow2_ge(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

struct DecResult {
  unsigned long long nonzero;
  unsigned long long markers;
  unsigned status;  // this call (reset when the caller asks for the result)
  unsigned sticky;  // every decode on the context since the last actc_ctx_take_status
};
static_assert(offsetof(DecResult, sticky) == offsetof(DecResult, status) + 4, "report_format_error layout");

}  // namespace

struct actc_ctx {
  int device = 0;
  int num_sms = 148;
  Buf sym, hist, cb, ctab, len8, canon, lencnt, status, misc, lut, idx, part, crc, crc_copy;
  actc_plan_t *plan_dev = nullptr;  // inside misc (kMiscPlanOff)
  bool plan_zeroed = false;          // launch_k1 zeroed it: the next codebook launch skips its memset
  DecResult *dres_dev = nullptr;
  // state carried from plan to encode
  uint64_t n = 0, A = 0;
  uint32_t radius = 0, sym_bytes = 2, win_lo = 0, win_n = 0;
  int mode = 0;  // 1 = codec, 2 = huffman debug
  int k1_blocks = 0, k3_blocks = 0, k4_blocks[5] = {0, 0, 0, 0, 0};
  // when set (actc_compress_async), the codebook writes the canonical table
  // straight into the caller's buffers instead of the ctx scratch
  uint32_t *canon_out = nullptr, *lencnt_out = nullptr;
  // when set (actc_compress_async), the codebook leaves the canonical-code
  // emission to the segment count pass that follows it
  bool defer_emit = false;
  bool no_fallback = false;  // actc_compress_async ACTC_ASYNC_NO_FALLBACK
  EmitArgs emit{};
  // caller-provided symbol scratch for the next K1 (actc_ctx_set_scratch;
  // consumed by that launch), and the buffer the current stream's symbols live in
  void *sym_ext = nullptr;
  size_t sym_ext_bytes = 0;
  void *sym_cur = nullptr;
  // decode-table output for the next async compression (actc_ctx_set_table_out)
  void *table_out = nullptr;
  int smem_optin = 0;  // dynamic shared memory a CTA may opt in to
  int k4l_dyn_max = 0; // ... for the K4L decoders (opt-in limit minus their static shared memory)
};

namespace {

// codebook scratch carve-up for alphabet A
struct CbLayout {
  size_t live_sym, live_freq, keys, keys2, vals, vals2, nf, lpar, npar, llen, ndepth, cls16, rank_tab, total;
};
CbLayout cb_layout(uint64_t A) {
  CbLayout l;
  uint64_t P = pow2_ge(A);
  size_t o = 0;
  auto take = [&](size_t bytes) {
    size_t r = o;
    o += (bytes + 255) & ~size_t(255);
    return r;
  };
  (void)P;
  l.live_sym = take(4 * A);
  l.live_freq = take(8 * A);
  l.keys = take(8 * A);
  l.keys2 = take(8 * A);
  l.vals = take(4 * A);
  l.vals2 = take(4 * A);
  l.nf = take(8 * A);
  l.lpar = take(4 * A);
  l.npar = take(4 * A);
  l.llen = take(A);
  l.ndepth = take(4 * A);
  l.cls16 = take(2 * A + 64);
  l.rank_tab = take(1024 * 34 * 2);
  l.total = o;
  return l;
}

// misc counters layout (u64 slots)
enum { M_NOUT = 0, M_TICKET = 1, M_BAD = 2, M_SCAN_TOT = 3, M_CHANGED = 4, M_STATUS = 5, M_SCAN_TOT2 = 6, M_K2GATE = 7, M_SEGTICKET = 8, M_PACKTICKET = 9, M_K4LTICKET = 10, M_K4LMCOUNT = 11, M_SLOTS = 12 };
constexpr size_t kMiscPlanOff = (8 * M_SLOTS + 63) & ~(size_t)63;  // device plan inside the misc buffer

constexpr size_t kK2Smem = 4096 * (8 + 8 + 8 + 4 + 4 + 4 + 4 + 4 + 1) + 64;

// Plan hand-off to pinned host memory.  A cudaMemcpyAsync D2H would queue
// behind every earlier device-to-host copy on the copy engine (e.g. a
// caller's 200 MB D2H of a reconstructed tensor on another stream); a kernel
// storing into the mapped pinned buffer (UVA) lands as soon as the stream
// reaches it.  Falls back to the copy for host memory the device cannot map.
__global__ void k_plan_out(const actc_plan_t *__restrict__ src, actc_plan_t *dst) {
  constexpr int W = (int)(sizeof(actc_plan_t) / 4);
  static_assert(sizeof(actc_plan_t) % 4 == 0, "plan size");
  if (threadIdx.x < W) reinterpret_cast<volatile uint32_t *>(dst)[threadIdx.x] = reinterpret_cast<const uint32_t *>(src)[threadIdx.x];
  __threadfence_system();
}

// device alias of a pinned host buffer (UVA-mapped), or null
void *mapped_alias(const void *host) {
  // a few recent answers per thread: a batch cycles through one plan
  // mailbox per context (cudaPointerGetAttributes costs a few us a call)
  constexpr int kN = 16;
  static thread_local const void *hosts[kN] = {};
  static thread_local void *devs[kN] = {};
  static thread_local int next = 0;
  for (int i = 0; i < kN; i++)
    if (hosts[i] == host && host) return devs[i];
  cudaPointerAttributes at{};
  void *dev = nullptr;
  if (cudaPointerGetAttributes(&at, host) == cudaSuccess && at.type == cudaMemoryTypeHost)
    dev = at.devicePointer;
  cudaGetLastError();
  hosts[next] = host;
  devs[next] = dev;
  next = (next + 1) % kN;
  return dev;
}

int plan_to_host(actc_ctx *c, actc_plan_t *plan_host, cudaStream_t s) {
  void *last_dev = mapped_alias(plan_host);
  if (last_dev) {
    KT(ACTC_KIND_CODEBOOK);  // the plan hand-off is the codebook's output
    k_plan_out<<<1, 32, 0, s>>>(c->plan_dev, (actc_plan_t *)last_dev);
    CKL();
  } else {
    CK(cudaMemcpyAsync(plan_host, c->plan_dev, sizeof(actc_plan_t), cudaMemcpyDeviceToHost, s));
  }
  return ACTC_OK;
}

int run_codebook(actc_ctx *c, const unsigned long long *hist, uint64_t A, const uint16_t *in_lengths,
                 uint16_t *out_lengths, const unsigned long long *n_out, uint64_t n_symbols,
                 uint32_t sym_bytes, cudaStream_t s, const unsigned *nonfinite = nullptr) {
  CbLayout l = cb_layout(A);
  int rc;
  if ((rc = grow(c->cb, l.total))) return rc;
  if ((rc = grow(c->ctab, 8 * A))) return rc;
  if ((rc = grow(c->len8, A + 64))) return rc;
  if ((rc = grow(c->canon, 4 * A))) return rc;
  if ((rc = grow(c->lencnt, 4 * 64))) return rc;
  char *b = (char *)c->cb.p;
  CodebookArgs a;
  a.hist = hist;
  a.A = A;
  a.in_lengths = in_lengths;
  a.ctab = (unsigned long long *)c->ctab.p;
  a.len8 = (uint8_t *)c->len8.p;
  a.canon = c->canon_out ? c->canon_out : (uint32_t *)c->canon.p;
  a.len_counts = c->lencnt_out ? c->lencnt_out : (uint32_t *)c->lencnt.p;
  a.out_lengths = out_lengths;
  a.plan = c->plan_dev;
  a.n_outliers = n_out;
  a.nonfinite = nonfinite;
  a.live_sym = (uint32_t *)(b + l.live_sym);
  a.live_freq = (unsigned long long *)(b + l.live_freq);
  a.keys = (unsigned long long *)(b + l.keys);
  a.keys2 = (unsigned long long *)(b + l.keys2);
  a.vals = (uint32_t *)(b + l.vals);
  a.vals2 = (uint32_t *)(b + l.vals2);
  a.nf = (unsigned long long *)(b + l.nf);
  a.lpar = (uint32_t *)(b + l.lpar);
  a.npar = (uint32_t *)(b + l.npar);
  a.llen = (uint8_t *)(b + l.llen);
  a.ndepth = (uint8_t *)(b + l.ndepth);
  a.n_symbols = n_symbols;
  a.sym_bytes = sym_bytes;
  a.dbg = nullptr;
  a.cls16 = (uint16_t *)(b + l.cls16);
  a.rank_tab = (uint16_t *)(b + l.rank_tab);
  a.fallback = (unsigned *)((unsigned long long *)c->misc.p + M_K2GATE);
  a.gate = nullptr;
  if (getenv("ACTC_K2_TIMING")) {
    int rc2 = grow(c->idx, 4096);
    if (rc2) return rc2;
    a.dbg = (unsigned long long *)c->idx.p;
  }
  if (!c->plan_zeroed) CK(cudaMemsetAsync(c->plan_dev, 0, sizeof(actc_plan_t), s));
  c->plan_zeroed = false;
  // frequency-class codebook first; it hands over to k2_codebook (gated)
  // when its capacities are exceeded
  // the single-CTA codebooks sit on the critical path of their tensor's
  // chain: highest execution priority, so a freed SM goes to them before the
  // pending CTAs of other tensors' bandwidth kernels (the gated fallback
  // too: it needs a whole SM's shared memory, and at default priority it
  // waited ~5 us per chain for one to drain)
  static int hi = [] {
    int lo = 0, h = 0;
    cudaDeviceGetStreamPriorityRange(&lo, &h);
    return h;
  }();
  if (!in_lengths && A <= 65536 && n_symbols < (1ull << 32)) {
    KT(ACTC_KIND_CODEBOOK);
    {
      cudaLaunchConfig_t cfg{};
      cfg.gridDim = dim3(1);
      cfg.blockDim = dim3(K2_THREADS);
      cfg.dynamicSmemBytes = kK2rSmem;
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributePriority;
      at[0].val.priority = hi;
      cfg.attrs = at;
      cfg.numAttrs = 1;
      CK(cudaLaunchKernelEx(&cfg, k2r_codebook, a));
    }
    a.gate = a.fallback;
  }
  if (!(a.gate && c->no_fallback)) {
    KT(ACTC_KIND_CODEBOOK);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(1);
    cfg.blockDim = dim3(K2_THREADS);
    cfg.dynamicSmemBytes = kK2Smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributePriority;
    at[0].val.priority = hi;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, k2_codebook, a));
  }
  c->emit = EmitArgs{};
  if (a.gate && c->defer_emit) {
    c->emit = EmitArgs{a.fallback, a.rank_tab, a.len_counts, a.len8, a.plan, a.canon, a.ctab};
  } else if (a.gate) {
    KT(ACTC_KIND_CODEBOOK);
    k2s_emit<<<K2_THREADS / 32, 32, 0, s>>>(a);
  }
  CKL();
  return ACTC_OK;
}


}  // namespace

extern "C" {

const char *actc_last_error(void) { return g_err; }
int actc_version(void) { return 1; }

/* debug: copy the K2 stage timestamps of the last codebook build (ACTC_K2_TIMING=1) */
int actc_debug_k2_timing(actc_ctx *c, uint64_t *out32) {
  if (!c->idx.p) return ACTC_EPARAM;
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out32, c->idx.p, 32 * 8, cudaMemcpyDeviceToHost));
  return ACTC_OK;
}

// 1 if the last codebook on this ctx came from the frequency-class kernel (synchronizes)
int actc_debug_k2r_used(actc_ctx *c) {
  unsigned v = 0xFFFFFFFFu;
  cudaDeviceSynchronize();
  cudaMemcpy(&v, (unsigned long long *)c->misc.p + M_K2GATE, 4, cudaMemcpyDeviceToHost);
  return v == 0u ? 1 : 0;
}

// debug: per-launch timeline of the timed launches since the last call
// (kind, start ms, end ms, stream slot) relative to the earliest start;
// consumes the records like actc_kernel_stats.  Returns the record count.
int actc_debug_timeline(double *out, int cap) {
  std::vector<KRec> recs;
  {
    std::lock_guard<std::mutex> g(g_tmu);
    recs.swap(g_recs);
  }
  int n = 0;
  if (!recs.empty()) {
    for (const KRec &r : recs) cudaEventSynchronize(r.b);
    cudaEvent_t ref = recs[0].a;
    float best = 0.f;
    for (const KRec &r : recs) {
      float t = 0.f;
      if (cudaEventElapsedTime(&t, ref, r.a) == cudaSuccess && t < best) {
        best = t;
      }
    }
    std::vector<cudaStream_t> slots;
    for (const KRec &r : recs) {
      if (n >= cap) break;
      float t0 = 0.f, t1 = 0.f;
      cudaEventElapsedTime(&t0, ref, r.a);
      cudaEventElapsedTime(&t1, ref, r.b);
      int slot = -1;
      for (size_t q = 0; q < slots.size(); q++)
        if (slots[q] == r.s) slot = (int)q;
      if (slot < 0) {
        slot = (int)slots.size();
        slots.push_back(r.s);
      }
      out[4 * n] = r.kind;
      out[4 * n + 1] = t0 - best;
      out[4 * n + 2] = t1 - best;
      out[4 * n + 3] = slot;
      n++;
    }
  }
  cudaGetLastError();
  {
    std::lock_guard<std::mutex> g(g_tmu);
    for (const KRec &r : recs) {
      g_pool.push_back(r.a);
      g_pool.push_back(r.b);
    }
  }
  return n;
}

int actc_timing_enable(int on) {
  g_timing.store(on != 0);
  return ACTC_OK;
}

int actc_kernel_stats(uint64_t *launches, double *ms, int nkinds) {
  double acc[ACTC_KIND_NKINDS] = {0};
  std::vector<KRec> recs;
  {
    std::lock_guard<std::mutex> g(g_tmu);
    recs.swap(g_recs);
  }
  int rc = ACTC_OK;
  for (const KRec &r : recs) {
    float t = 0.f;
    if (cudaEventSynchronize(r.b) == cudaSuccess && cudaEventElapsedTime(&t, r.a, r.b) == cudaSuccess)
      acc[r.kind] += t;
    else
      rc = set_err(ACTC_ECUDA, "kernel timing event failed: %s", cudaGetErrorString(cudaGetLastError()));
  }
  {
    std::lock_guard<std::mutex> g(g_tmu);
    for (const KRec &r : recs) {
      g_pool.push_back(r.a);
      g_pool.push_back(r.b);
    }
  }
  for (int k = 0; k < ACTC_KIND_NKINDS; k++) {
    unsigned long long l = g_launches[k].exchange(0);
    if (k < nkinds) {
      if (launches) launches[k] = l;
      if (ms) ms[k] = acc[k];
    }
  }
  return rc;
}

int actc_ctx_create(int device, actc_ctx **out) {
  *out = nullptr;
  CK(cudaSetDevice(device));
  actc_ctx *c = new actc_ctx();
  c->device = device;
  cudaDeviceGetAttribute(&c->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaMalloc(&c->dres_dev, sizeof(DecResult)) != cudaSuccess) {
    delete c;
    return set_err(ACTC_ENOMEM, "ctx alloc failed");
  }
  cudaMemset(c->dres_dev, 0, sizeof(DecResult));
  int rc;
  // the device plan lives right after the misc words: launch_k1 zeroes both
  // with one memset (no separate zeroing step between K1 and the codebook)
  if ((rc = grow(c->misc, kMiscPlanOff + sizeof(actc_plan_t))) ||
      (rc = grow(c->lut, std::max<size_t>(4 * kLutWords, kK4lTableBytes)))) {
    delete c;
    return rc;
  }
  CK(cudaMemset(c->misc.p, 0, c->misc.cap));  // self-resetting tickets start at 0
  c->plan_dev = (actc_plan_t *)((char *)c->misc.p + kMiscPlanOff);
  CK(cudaFuncSetAttribute(k2_codebook, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kK2Smem));
  CK(cudaFuncSetAttribute(k2r_codebook, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kK2rSmem));
  int nb = 0;
  int optin = 0;
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  c->smem_optin = optin;
  const void *big[] = {(const void *)k4l_decode<0, false, false>, (const void *)k4l_decode<0, false, true>,
                       (const void *)k4l_decode<1, false, false>, (const void *)k4l_decode<1, false, true>,
                       (const void *)k4l_decode<0, true, false>,  (const void *)k4l_decode<0, true, true>,
                       (const void *)k4l_decode<1, true, false>,  (const void *)k4l_decode<1, true, true>,
                       (const void *)k4l_decode<2, true, false>,  (const void *)k3_seg_pack<uint16_t>,
                       (const void *)k3_seg_pack<uint32_t>,     (const void *)k3_seg_count<uint16_t>,
                       (const void *)k3_seg_count<uint32_t>,    (const void *)k1_quant_lorenzo_hist<uint16_t>,
                       (const void *)k1_quant_lorenzo_hist<uint32_t>, (const void *)k_hist_u32};
  c->k4l_dyn_max = optin;
  for (int i = 0; i < (int)(sizeof(big) / sizeof(big[0])); i++) {
    const void *f = big[i];
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, f));
    CK(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, optin - (int)fa.sharedSizeBytes));
    if (i < 9) c->k4l_dyn_max = std::min(c->k4l_dyn_max, optin - (int)fa.sharedSizeBytes);  // the K4L variants
  }
  // occupancy-derived persistent grid sizes
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k1_quant_lorenzo_hist<uint16_t>, K1_THREADS, (size_t)(K1_WIN + 32) * 4);
  c->k1_blocks = std::max(1, nb) * c->num_sms;
  size_t s16 = (size_t)K4_THREADS * (ACTC_CHUNK / 2 + 1) * 4, s32 = (size_t)K4_THREADS * (ACTC_CHUNK + 1) * 4;
  CK(cudaFuncSetAttribute(k4_decode<0, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s16));
  CK(cudaFuncSetAttribute(k4_decode<1, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s16));
  CK(cudaFuncSetAttribute(k4_decode<0, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s32));
  CK(cudaFuncSetAttribute(k4_decode<1, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s32));
  CK(cudaFuncSetAttribute(k4_decode<2, 32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)s32));
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k4_decode<0, 16>, K4_THREADS, s16);
  c->k4_blocks[0] = std::max(1, nb) * c->num_sms;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, k4_decode<0, 32>, K4_THREADS, s32);
  c->k4_blocks[1] = std::max(1, nb) * c->num_sms;
  cudaGetLastError();
  *out = c;
  return ACTC_OK;
}

int actc_ctx_set_table_out(actc_ctx *c, void *table_dev, uint64_t bytes) {
  if (table_dev && bytes < ACTC_TABLE_BYTES) return set_err(ACTC_EPARAM, "decode table buffer too small");
  if (((uintptr_t)table_dev & 15u) != 0) return set_err(ACTC_EPARAM, "decode table buffer must be 16-byte aligned");
  c->table_out = table_dev;
  return ACTC_OK;
}

int actc_ctx_set_scratch(actc_ctx *c, void *sym_dev, uint64_t bytes) {
  c->sym_ext = sym_dev;
  c->sym_ext_bytes = sym_dev ? bytes : 0;
  return ACTC_OK;
}

int actc_ctx_take_status(actc_ctx *c, uint32_t *status_host, actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  CK(cudaMemcpyAsync(status_host, &c->dres_dev->sticky, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaMemsetAsync(&c->dres_dev->sticky, 0, 4, s));
  return ACTC_OK;
}

uint64_t actc_ctx_device_bytes(const actc_ctx *c) {
  if (!c) return 0;
  const Buf *bufs[] = {&c->sym, &c->hist, &c->cb, &c->ctab, &c->len8, &c->canon, &c->lencnt,
                       &c->status, &c->misc, &c->lut, &c->idx, &c->part, &c->crc, &c->crc_copy};
  uint64_t t = sizeof(actc_plan_t) + sizeof(DecResult);
  for (const Buf *b : bufs) t += b->p ? b->cap : 0;
  return t;
}

void actc_ctx_destroy(actc_ctx *c) {
  if (!c) return;
  Buf *bufs[] = {&c->sym, &c->hist, &c->cb, &c->ctab, &c->len8, &c->canon, &c->lencnt,
                 &c->status, &c->misc, &c->lut, &c->idx, &c->part, &c->crc, &c->crc_copy};
  for (Buf *b : bufs)
    if (b->p) cudaFree(b->p);
  cudaFree(c->dres_dev);
  delete c;
}

// K1's quantizer parameters for error bound eb (actc_internal.cuh QParams)
static QParams make_qparams(double eb) {
  QParams P;
  P.eb = eb;
  P.two_eb = 2.0 * eb;
  const double inv = 1.0 / P.two_eb;
  P.inv = inv;
  P.fast = (isfinite(inv) && inv >= DBL_MIN) ? 1 : 0;
  P.ih = (float)inv;
  P.il = (float)(inv - (double)P.ih);
  P.dfast = (P.fast && isfinite(P.ih) && P.ih >= FLT_MIN) ? 1 : 0;
  return P;
}

static int launch_k1(actc_ctx *c, const float *x, uint64_t n, double eb, uint32_t radius, int64_t *chunk_lat,
                     cudaStream_t s) {
  if (!(eb > 0 && isfinite(eb))) return set_err(ACTC_EPARAM, "eb must be a positive finite real, got %g", eb);
  if (radius < 2) return set_err(ACTC_EPARAM, "radius must be >= 2, got %u", radius);
  if (n == 0) return set_err(ACTC_EPARAM, "empty tensor");
  if (n >= (1ull << 38)) return set_err(ACTC_EPARAM, "tensor too large");
  const uint64_t A = 2ull * radius;
  if (A > kMaxAlphabet) return set_err(ACTC_EPARAM, "radius %u too large for the device codebook (max %u)", radius, kMaxAlphabet / 2);
  const uint32_t sb = A <= 65536 ? 2 : 4;
  int rc;
  const size_t sym_need = (size_t)sb * n + 64;
  if (c->sym_ext && c->sym_ext_bytes >= sym_need) {
    c->sym_cur = c->sym_ext;
  } else {
    if ((rc = grow(c->sym, sym_need))) return rc;
    c->sym_cur = c->sym.p;
  }
  c->sym_ext = nullptr;  // one launch only
  c->sym_ext_bytes = 0;
  if ((rc = grow(c->hist, 8 * A))) return rc;
  CK(cudaMemsetAsync(c->hist.p, 0, 8 * A, s));
  CK(cudaMemsetAsync(c->misc.p, 0, kMiscPlanOff + sizeof(actc_plan_t), s));  // counters + device plan
  c->plan_zeroed = true;
  unsigned long long *misc = (unsigned long long *)c->misc.p;

  const QParams P = make_qparams(eb);
  uint32_t win_n = (uint32_t)std::min<uint64_t>(A, K1_WIN);
  uint32_t win_lo = A <= K1_WIN ? 0 : radius - K1_WIN / 2;
  uint64_t ntiles = cdiv(n, K1_TILE);
  int grid = (int)std::min<uint64_t>(ntiles, (uint64_t)c->k1_blocks);
  {
    KT(ACTC_KIND_QUANT);
    if (sb == 2)
      k1_quant_lorenzo_hist<uint16_t><<<grid, K1_THREADS, (win_n + 32) * 4, s>>>(
          x, n, P, radius, (uint16_t *)c->sym_cur, (unsigned long long *)c->hist.p, misc + M_NOUT, win_lo, win_n,
          (unsigned *)(misc + M_BAD), (long long *)chunk_lat);
    else
      k1_quant_lorenzo_hist<uint32_t><<<grid, K1_THREADS, (win_n + 32) * 4, s>>>(
          x, n, P, radius, (uint32_t *)c->sym_cur, (unsigned long long *)c->hist.p, misc + M_NOUT, win_lo, win_n,
          (unsigned *)(misc + M_BAD), (long long *)chunk_lat);
  }
  CKL();
  c->n = n;
  c->A = A;
  c->radius = radius;
  c->sym_bytes = sb;
  return ACTC_OK;
}

// codebook for the histogram the last launch_k1 on this ctx produced
static int launch_cb(actc_ctx *c, cudaStream_t s) {
  unsigned long long *misc = (unsigned long long *)c->misc.p;
  int rc = run_codebook(c, (const unsigned long long *)c->hist.p, c->A, nullptr, nullptr, misc + M_NOUT, c->n,
                        c->sym_bytes, s, (const unsigned *)(misc + M_BAD));
  if (rc) return rc;
  c->mode = 1;
  return ACTC_OK;
}

static int launch_plan(actc_ctx *c, const float *x, uint64_t n, double eb, uint32_t radius, int64_t *chunk_lat,
                       cudaStream_t s) {
  int rc = launch_k1(c, x, n, eb, radius, chunk_lat, s);
  if (rc) return rc;
  return launch_cb(c, s);
}

int actc_compress_plan(actc_ctx *c, const float *x, uint64_t n, double eb, uint32_t radius,
                       uint32_t flags, int64_t *chunk_lat, actc_plan_t *plan_host, actc_stream stream) {
  (void)flags;
  cudaStream_t s = (cudaStream_t)stream;
  int rc = launch_plan(c, x, n, eb, radius, chunk_lat, s);
  if (rc) return rc;
  if ((rc = plan_to_host(c, plan_host, s))) return rc;
  return ACTC_OK;
}

static int launch_encode(actc_ctx *c, const void *sym, uint32_t sb, uint64_t n, const float *x,
                         const actc_plan_t *plan, uint8_t *payload, uint64_t *out_idx, float *out_val,
                         uint64_t *chunk_off, int extract, cudaStream_t s) {
  int rc;
  // the segment encoder's (code << 8 | len) table holds codes of up to 56
  // bits; a longer Huffman code needs > Fib(58) ~ 5.9e11 symbols, more than
  // a tensor in 180 GB of HBM can hold -- rejected loudly, never truncated
  if (plan->max_len > 56) return set_err(ACTC_EPARAM, "Huffman code length %u exceeds the device encoder's 56 bits",
                                         plan->max_len);
  uint32_t lo = plan->sym_lo, hi = plan->sym_hi;
  uint32_t span = hi >= lo ? hi - lo + 1 : 1;
  // code-table window of the pack pass: the live range, capped and centred
  // on the radius (symbol of a zero delta)
  uint32_t lwin_lo = lo, lwin_n = std::min<uint32_t>(span, K3L_WIN);
  if (span > K3L_WIN) {
    uint32_t centre = c->radius ? c->radius : (lo + hi) / 2;
    uint32_t wl = centre > K3L_WIN / 2 ? centre - K3L_WIN / 2 : 0;
    if (wl < lo) wl = lo;
    if (wl + K3L_WIN > hi + 1) wl = hi + 1 - K3L_WIN;
    lwin_lo = wl;
  }
  // two passes over 1024-symbol segments, no inter-warp waiting
  const uint64_t nseg = cdiv(n, K3L_SEG);
  SegArgs g{};
  g.n = n;
  g.ctab = (const unsigned long long *)c->ctab.p;
  g.len8 = (const uint8_t *)c->len8.p;
  g.lo = lo;
  g.span = span;
  g.win_lo = lwin_lo;
  g.win_n = lwin_n;
  const bool l8 = span <= 65536;
  const size_t csm = l8 ? (size_t)((((lo & 15u) + span + 15) & ~15u)) : 16;
  const size_t psm = (size_t)((lwin_n + 3) & ~3u) * 4 + (size_t)(K3L_THREADS / 32) * K3L_WORDS * 4;
  const void *fc = sb == 2 ? (const void *)k3_seg_count<uint16_t> : (const void *)k3_seg_count<uint32_t>;
  const void *fp = sb == 2 ? (const void *)k3_seg_pack<uint16_t> : (const void *)k3_seg_pack<uint32_t>;
  const int occ_c = occupancy(fc, K3L_THREADS, csm), occ_p = occupancy(fp, K3L_THREADS, psm);
  const uint64_t want_c = (uint64_t)std::max(1, occ_c) * c->num_sms;
  g.spc = std::max<uint64_t>(K3L_THREADS / 32, cdiv(nseg, want_c));
  g.ncta = (uint32_t)cdiv(nseg, g.spc);
  if ((rc = grow(c->status, nseg * 9 + (size_t)g.ncta * 16 + 1024))) return rc;
  g.cta_bits = (unsigned long long *)c->status.p;
  g.cta_nz = g.cta_bits + g.ncta;
  g.seg_bits = (uint32_t *)(g.cta_nz + g.ncta);
  g.seg_nz = g.seg_bits + nseg;
  g.seg_long = (uint8_t *)(g.seg_nz + nseg);
  g.ticket = (unsigned *)((unsigned long long *)c->misc.p + M_SEGTICKET);
  g.x = x;
  g.payload = (uint32_t *)payload;
  g.out_idx = (unsigned long long *)out_idx;
  g.out_val = out_val;
  g.chunk_off = (unsigned long long *)chunk_off;
  g.extract = extract;
  g.k = plan->n_outliers;
  CK(cudaMemsetAsync(payload, 0, 4 * cdiv(plan->payload_bits, 32) + 8, s));
  const int gp = (int)std::max<uint64_t>(
      1, std::min<uint64_t>(cdiv(nseg, K3L_THREADS / 32), (uint64_t)std::max(1, occ_p) * c->num_sms));
  {
    KT(ACTC_KIND_COUNT);
    if (sb == 2)
      k3_seg_count<uint16_t><<<g.ncta, K3L_THREADS, csm, s>>>((const uint16_t *)sym, g);
    else
      k3_seg_count<uint32_t><<<g.ncta, K3L_THREADS, csm, s>>>((const uint32_t *)sym, g);
  }
  {
    KT(ACTC_KIND_PACK);
    if (sb == 2)
      k3_seg_pack<uint16_t><<<gp, K3L_THREADS, psm, s>>>((const uint16_t *)sym, g);
    else
      k3_seg_pack<uint32_t><<<gp, K3L_THREADS, psm, s>>>((const uint32_t *)sym, g);
  }
  CKL();
  return ACTC_OK;
}

int actc_compress_encode(actc_ctx *c, const float *x, const actc_plan_t *plan, uint8_t *payload,
                         uint64_t *out_idx, float *out_val, uint32_t *canon, uint32_t *len_counts,
                         uint64_t *chunk_off, actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (c->mode != 1 || plan->n != c->n) return set_err(ACTC_EPARAM, "actc_compress_encode without a matching plan");
  if (plan->status != ACTC_OK) return set_err(plan->status, "Huffman code length exceeds 63 bits");
  int rc = launch_encode(c, c->sym_cur, c->sym_bytes, c->n, x, plan, payload, out_idx, out_val, chunk_off, 1, s);
  if (rc) return rc;
  if (plan->live_symbols)
    CK(cudaMemcpyAsync(canon, c->canon.p, 4ull * plan->live_symbols, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(len_counts, c->lencnt.p, 4 * 64, cudaMemcpyDeviceToDevice, s));
  return ACTC_OK;
}

int actc_compress_async(actc_ctx *c, const float *x, uint64_t n, double eb, uint32_t radius, uint32_t flags,
                        int64_t *chunk_lat, uint8_t *payload, uint64_t payload_cap_bytes, uint64_t *out_idx,
                        float *out_val, uint64_t k_cap, uint32_t *canon, uint32_t *len_counts, uint64_t *chunk_off,
                        actc_plan_t *plan_host, actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  int rc;
  // ACTC_ASYNC_K1_ONLY / ACTC_ASYNC_REST split the launch in two so a batch
  // can put every tensor's K1 on the GPU before the rest of any chain
  if (!(flags & ACTC_ASYNC_REST)) {
    if ((rc = launch_k1(c, x, n, eb, radius, chunk_lat, s))) return rc;
    if (flags & ACTC_ASYNC_K1_ONLY) return ACTC_OK;
  } else if (c->n != n) {
    return set_err(ACTC_EPARAM, "actc_compress_async(REST) without a matching K1 launch");
  }
  c->canon_out = canon;
  c->lencnt_out = len_counts;
  c->defer_emit = true;
  c->no_fallback = (flags & ACTC_ASYNC_NO_FALLBACK) != 0;
  rc = launch_cb(c, s);
  c->canon_out = c->lencnt_out = nullptr;
  c->defer_emit = false;
  c->no_fallback = false;
  if (rc) return rc;
  // K3 segment encoder planned on the device: live range / windows from the
  // device plan, shared-memory sizes and grids at their caps
  const uint32_t sb = c->sym_bytes;
  const void *sym = c->sym_cur;
  const uint64_t nseg = cdiv(n, K3L_SEG);
  SegArgs g{};
  g.n = n;
  g.ctab = (const unsigned long long *)c->ctab.p;
  g.len8 = (const uint8_t *)c->len8.p;
  g.dplan = c->plan_dev;
  g.radius = radius;
  g.cap_bits = payload_cap_bytes >= 32 ? 8 * (payload_cap_bytes - 32) : 0;
  g.k_cap = k_cap;
  g.canon_src = nullptr;  // the codebook wrote the caller's table directly
  g.lencnt_src = nullptr;
  g.canon_out = canon;
  g.lencnt_out = len_counts;
  const size_t csm = 65536 + 16;
  const size_t psm = (size_t)K3L_WIN * 4 + (size_t)(K3L_THREADS / 32) * K3L_WORDS * 4;
  const void *fc = sb == 2 ? (const void *)k3_seg_count<uint16_t> : (const void *)k3_seg_count<uint32_t>;
  const void *fp = sb == 2 ? (const void *)k3_seg_pack<uint16_t> : (const void *)k3_seg_pack<uint32_t>;
  const int occ_c = occupancy(fc, K3L_THREADS, csm), occ_p = occupancy(fp, K3L_THREADS, psm);
  const uint64_t want_c = (uint64_t)std::max(1, occ_c) * c->num_sms;
  g.spc = std::max<uint64_t>(K3L_THREADS / 32, cdiv(nseg, want_c));
  g.ncta = (uint32_t)cdiv(nseg, g.spc);
  if ((rc = grow(c->status, nseg * 9 + (size_t)g.ncta * 16 + 1024))) return rc;
  g.cta_bits = (unsigned long long *)c->status.p;
  g.cta_nz = g.cta_bits + g.ncta;
  g.seg_bits = (uint32_t *)(g.cta_nz + g.ncta);
  g.seg_nz = g.seg_bits + nseg;
  g.seg_long = (uint8_t *)(g.seg_nz + nseg);
  g.ticket = (unsigned *)((unsigned long long *)c->misc.p + M_SEGTICKET);
  g.emit = c->emit;  // the count pass emits the canonical codes
  c->emit = EmitArgs{};
  // the pack's last CTA hands the plan to the mapped mailbox (one launch
  // less per tensor than the plan_to_host kernel)
  g.plan_host = (actc_plan_t *)mapped_alias(plan_host);
  g.pack_ticket = (unsigned *)((unsigned long long *)c->misc.p + M_PACKTICKET);
  g.table = c->table_out;  // the first pack CTAs build the decode table
  g.sw16 = 2ull * radius <= 65536 ? 1 : 0;
  c->table_out = nullptr;
  g.x = x;
  g.payload = (uint32_t *)payload;
  g.out_idx = (unsigned long long *)out_idx;
  g.out_val = out_val;
  g.chunk_off = (unsigned long long *)chunk_off;
  g.extract = 1;
  const int gp = (int)std::max<uint64_t>(
      1, std::min<uint64_t>(cdiv(nseg, K3L_THREADS / 32), (uint64_t)std::max(1, occ_p) * c->num_sms));
  {
    KT(ACTC_KIND_COUNT);
    if (sb == 2)
      k3_seg_count<uint16_t><<<g.ncta, K3L_THREADS, csm, s>>>((const uint16_t *)sym, g);
    else
      k3_seg_count<uint32_t><<<g.ncta, K3L_THREADS, csm, s>>>((const uint32_t *)sym, g);
  }
  {
    KT(ACTC_KIND_PACK);
    if (sb == 2)
      k3_seg_pack<uint16_t><<<gp, K3L_THREADS, psm, s>>>((const uint16_t *)sym, g);
    else
      k3_seg_pack<uint32_t><<<gp, K3L_THREADS, psm, s>>>((const uint32_t *)sym, g);
  }
  CKL();
  if (!g.plan_host && (rc = plan_to_host(c, plan_host, s))) return rc;
  c->mode = 0;  // the ctx holds no pending plan for actc_compress_encode
  return ACTC_OK;
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no libcuda link)
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_tiled() {
  static const EncodeTiledFn fn = []() -> EncodeTiledFn {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess)
      return nullptr;
    return (EncodeTiledFn)p;
  }();
  return fn;
}

// the decoder's output as a 2-D tensor of chunk rows (k4l_decode's TMA
// stores): rows x ACTC_CHUNK values, box 32 rows x 64 B, 64-B swizzle
static int make_chunk_rows_map(CUtensorMap *tm, void *out, uint64_t rows, int mode) {
  memset(tm, 0, sizeof(*tm));
  if (rows == 0) return ACTC_OK;  // no full tile: the map is never used
  if ((uintptr_t)out & 15u) return set_err(ACTC_EPARAM, "decode output must be 16-byte aligned");
  const EncodeTiledFn enc = encode_tiled();
  if (!enc) return set_err(ACTC_ECUDA, "cuTensorMapEncodeTiled unavailable");
  const uint32_t elem = mode == 1 ? 8u : 4u;
  const CUtensorMapDataType dt = mode == 1   ? CU_TENSOR_MAP_DATA_TYPE_FLOAT64
                                 : mode == 0 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                             : CU_TENSOR_MAP_DATA_TYPE_UINT32;
  const cuuint64_t dims[2] = {(cuuint64_t)ACTC_CHUNK, (cuuint64_t)rows};
  const cuuint64_t strides[1] = {(cuuint64_t)ACTC_CHUNK * elem};
  const cuuint32_t box[2] = {64u / elem, 32u};
  const cuuint32_t es[2] = {1u, 1u};
  const CUresult r = enc(tm, dt, 2, out, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) return set_err(ACTC_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
  return ACTC_OK;
}

// phase: 0 = table + decoder, 1 = table only, 2 = decoder only (table built by a phase-1 call)
static int launch_decode(actc_ctx *c, const actc_stream_t *st_in, void *out, int mode,
                         actc_decode_result_t *res_host, cudaStream_t s, int phase = 0,
                         bool no_nonzero = false) {
  const actc_stream_t &S = *st_in;
  if (S.n == 0) return set_err(ACTC_EPARAM, "empty stream");
  if (!S.chunk_offsets_dev) return set_err(ACTC_EPARAM, "stream has no chunk index (call actc_build_chunk_index)");
  if (S.live_symbols == 0) return set_err(ACTC_EFORMAT, "empty code table with nonzero symbol count");
  const uint64_t nchunks = cdiv(S.n, ACTC_CHUNK);
  const uint64_t ntiles = cdiv(nchunks, K4_THREADS);
  int rc;
  size_t need = ntiles * (4 + 4 + 8 + 8) + 1024;
  if ((rc = grow(c->status, need))) return rc;
  char *b = (char *)c->status.p;
  DecStatus st;
  st.flag = (unsigned *)b;
  size_t o = ((ntiles * 4 + 255) / 256) * 256;
  st.agg_r = (int *)(b + o); o += ((ntiles * 4 + 255) / 256) * 256;
  st.agg_v = (long long *)(b + o); o += ntiles * 8;
  st.inc_v = (long long *)(b + o);
  // indexed streams (compress-time chunk lattice, or the raw-symbol debug
  // mode) decode with K4L; streams from bytes (bit offsets rebuilt, no
  // lattice) and the absurd-eb case (2*eb = inf: every value is +-inf/NaN)
  // with the look-back scan decoder K4
  const bool lane_dec = (S.chunk_lat_dev || mode == 2) && (mode == 2 || isfinite(2.0 * S.eb));
  unsigned *ticket = (unsigned *)((unsigned long long *)c->misc.p + M_TICKET);
  if (!lane_dec && phase != 1) {  // look-back state of the scan decoder
    CK(cudaMemsetAsync(st.flag, 0, ntiles * 4, s));
    CK(cudaMemsetAsync(ticket, 0, 8, s));
  }
  // the result mailbox is only read back when the caller asks for it
  if ((res_host || !lane_dec) && phase != 1) CK(cudaMemsetAsync(c->dres_dev, 0, offsetof(DecResult, sticky), s));
  const bool sw16 = 2ull * S.radius <= 65536 && mode != 2;
  // a table built at compress time (the pack kernel's first CTAs) is the K4L table
  const bool prebuilt = S.table_dev && lane_dec && mode != 2;
  if (prebuilt && phase == 1) return ACTC_OK;
  // batches skip the table-only call for streams that carry a table
  if (!prebuilt && (phase != 2 || S.table_dev)) {
    KT(ACTC_KIND_LUT);
    if (lane_dec)
      k4l_build_table<<<kLutSize / 256, 256, 0, s>>>(S.len_counts_dev, S.canon_syms_dev, mode == 2 ? 0u : S.radius,
                                                     (uint32_t *)c->lut.p);
    else
      k_build_lut<<<kLutSize / 256, 256, 0, s>>>(S.canon_syms_dev, S.len_counts_dev, (uint32_t *)c->lut.p, 0);
  }
  CKL();
  if (phase == 1) return ACTC_OK;
  DecodeArgs a;
  a.n = S.n;
  a.eb = S.eb;
  a.two_eb = 2.0 * S.eb;
  a.radius = mode == 2 ? 0u : S.radius;  // raw symbols: delta = symbol
  a.preserve = (S.flags & ACTC_FLAG_PRESERVE_ZEROS) ? 1 : 0;
  a.k = S.n_outliers;
  a.out_idx = (const unsigned long long *)S.outlier_idx_dev;
  a.out_val = S.outlier_val_dev;
  a.canon = S.canon_syms_dev;
  a.len_counts = S.len_counts_dev;
  a.lut = prebuilt ? (const uint32_t *)S.table_dev : (const uint32_t *)c->lut.p;
  a.payload = (const uint32_t *)S.payload_dev;
  a.payload_bits = S.payload_bits;
  a.chunk_off = (const unsigned long long *)S.chunk_offsets_dev;
  a.out = out;
  a.st = st;
  a.ticket = ticket;
  a.ntiles = ntiles;
  a.nonzero = &c->dres_dev->nonzero;
  a.markers = &c->dres_dev->markers;
  a.status = &c->dres_dev->status;
  a.chunk_lat = (const long long *)S.chunk_lat_dev;
  a.live = S.live_symbols;
  a.mcount = nullptr;
  a.cd_lim = 0;
  KT(ACTC_KIND_DECODE);
  if (lane_dec) {
    // K4L: one CTA per SM (persistent over 32-chunk warp tiles).  Warps
    // first: every warp runs the same number of 32-chunk tiles -- the fewest
    // passes the shared memory allows without a delta table, then the fewest
    // warps per SM that still finish in that many passes (a partial last pass
    // on some SMs would leave the others idle).  The canonical deltas (16-bit
    // symbols) then take the shared memory left: all of them, or the leading
    // (most frequent) canonical indices with the tail from the global table.
    const uint64_t ntl = cdiv(nchunks, 32);
    const int wmax = k4l_max_warps(0u, (size_t)c->k4l_dyn_max);
    if (wmax < 1) return set_err(ACTC_EPARAM, "decode tables exceed shared memory");
    const uint64_t passes = cdiv(ntl, (uint64_t)c->num_sms * (uint64_t)wmax);
    const int warps = (int)std::max<uint64_t>(1, std::min<uint64_t>((uint64_t)wmax, cdiv(ntl, (uint64_t)c->num_sms * passes)));
    const int grid = (int)std::max<uint64_t>(1, std::min<uint64_t>(cdiv(ntl, warps), (uint64_t)c->num_sms));
    const size_t used = k4l_smem_bytes(0, warps);
    const size_t room = (size_t)c->k4l_dyn_max > used ? (size_t)c->k4l_dyn_max - used : 0;
    a.cd_lim = sw16 ? (uint32_t)std::min<size_t>(S.live_symbols, (room / 2) & ~(size_t)7) : 0u;
    const bool gcanon = a.cd_lim < S.live_symbols;
    if (mode != 2 && S.n_outliers) {
      a.ticket = (unsigned *)((unsigned long long *)c->misc.p + M_K4LTICKET);
      a.mcount = (unsigned long long *)c->misc.p + M_K4LMCOUNT;
    }
    // the nonzero count (R) only when the caller reads the result back
    const bool nz = res_host && !no_nonzero;
    const void *f;
    if (mode == 2) f = (const void *)k4l_decode<2, true, false>;
    else if (mode == 1)
      f = gcanon ? (nz ? (const void *)k4l_decode<1, true, true> : (const void *)k4l_decode<1, true, false>)
                 : (nz ? (const void *)k4l_decode<1, false, true> : (const void *)k4l_decode<1, false, false>);
    else
      f = gcanon ? (nz ? (const void *)k4l_decode<0, true, true> : (const void *)k4l_decode<0, true, false>)
                 : (nz ? (const void *)k4l_decode<0, false, true> : (const void *)k4l_decode<0, false, false>);
    const size_t smem = k4l_smem_bytes(a.cd_lim, warps);
    // full tiles leave through TMA stores: the output as [n / ACTC_CHUNK][ACTC_CHUNK]
    CUtensorMap tm;
    int rc2;
    if ((rc2 = make_chunk_rows_map(&tm, out, S.n / ACTC_CHUNK, mode))) return rc2;
    void *args[] = {&a, &tm};
    CK(cudaLaunchKernel(f, dim3(grid), dim3(32 * warps), args, smem, s));
  } else {
    const size_t smem = (size_t)K4_THREADS * (sw16 ? ACTC_CHUNK / 2 + 1 : ACTC_CHUNK + 1) * 4;
    const int grid = (int)std::min<uint64_t>(ntiles, (uint64_t)(sw16 ? c->k4_blocks[0] : c->k4_blocks[1]));
    if (mode == 0)
      sw16 ? k4_decode<0, 16><<<grid, K4_THREADS, smem, s>>>(a) : k4_decode<0, 32><<<grid, K4_THREADS, smem, s>>>(a);
    else
      sw16 ? k4_decode<1, 16><<<grid, K4_THREADS, smem, s>>>(a) : k4_decode<1, 32><<<grid, K4_THREADS, smem, s>>>(a);
  }
  CKL();
  if (res_host) CK(cudaMemcpyAsync(res_host, c->dres_dev, sizeof(DecResult), cudaMemcpyDeviceToHost, s));
  return ACTC_OK;
}

int actc_decompress(actc_ctx *c, const actc_stream_t *stream, void *out, int out_dtype,
                    actc_decode_result_t *result_host, actc_stream s) {
  const int phase = (out_dtype & ACTC_DEC_LUT_ONLY) ? 1 : (out_dtype & ACTC_DEC_REST) ? 2 : 0;
  const bool no_nonzero = (out_dtype & ACTC_DEC_NO_NONZERO) != 0;
  out_dtype &= ~(ACTC_DEC_LUT_ONLY | ACTC_DEC_REST | ACTC_DEC_NO_NONZERO);
  if (out_dtype != ACTC_DTYPE_F32 && out_dtype != ACTC_DTYPE_F64) return set_err(ACTC_EPARAM, "bad out dtype");
  if (!(stream->eb > 0 && isfinite(stream->eb)) || stream->radius < 2)
    return set_err(ACTC_EFORMAT, "invalid codec params in stream");
  if (2ull * stream->radius > kMaxAlphabet) return set_err(ACTC_EPARAM, "radius too large for the device decoder");
  return launch_decode(c, stream, out, out_dtype == ACTC_DTYPE_F32 ? 0 : 1, result_host, (cudaStream_t)s, phase,
                       no_nonzero);
}

int actc_memcpy_batch(void *const *dst, const void *const *src, const uint64_t *bytes, int count, actc_stream stream) {
  if (count < 0 || count > 16) return set_err(ACTC_EPARAM, "memcpy_batch: count %d not in [0, 16]", count);
  cudaStream_t s = (cudaStream_t)stream;
  for (int i = 0; i < count; i++)
    if (bytes[i]) CK(cudaMemcpyAsync(dst[i], src[i], bytes[i], cudaMemcpyDeviceToDevice, s));
  return ACTC_OK;
}

int actc_crc32(actc_ctx *c, const void *data_dev, uint64_t len, uint32_t crc_in, uint32_t *crc_out_host,
               actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (len && !data_dev) return set_err(ACTC_EPARAM, "null buffer");
  const uint64_t nb = crc32_blocks(len);
  int rc;
  // [ticket][result][pad][per-CTA values]
  if ((rc = grow(c->crc, 16 + 4 * nb))) return rc;
  uint32_t *w = (uint32_t *)c->crc.p;
  const uint8_t *src = (const uint8_t *)data_dev;
  if (len && ((uintptr_t)src & 15u)) {  // the kernel loads 16-byte words
    if ((rc = grow(c->crc_copy, len + 16))) return rc;
    CK(cudaMemcpyAsync(c->crc_copy.p, src, len, cudaMemcpyDeviceToDevice, s));
    src = (const uint8_t *)c->crc_copy.p;
  }
  CK(cudaMemsetAsync(w, 0, 4, s));
  {
    KT(ACTC_KIND_CRC);
    if (crc32_launch(src, len, crc_in, w + 4, (unsigned *)w, w + 1, s))
      return set_err(ACTC_ECUDA, "crc32 launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  }
  CK(cudaMemcpyAsync(crc_out_host, w + 1, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  return ACTC_OK;
}

int actc_inject_uniform(actc_ctx *c, const void *x_dev, int dtype, uint64_t n, double eb, int preserve_zeros,
                        const uint64_t *pcg_state, double *out_dev, actc_stream stream) {
  (void)c;
  cudaStream_t s = (cudaStream_t)stream;
  if (!(eb > 0.0) || !isfinite(eb)) return set_err(ACTC_EPARAM, "eb must be > 0 and finite");
  if (dtype != ACTC_DTYPE_F32 && dtype != ACTC_DTYPE_F64) return set_err(ACTC_EPARAM, "bad dtype");
  if (n && (!x_dev || !out_dev || !pcg_state)) return set_err(ACTC_EPARAM, "null buffer");
  KT(ACTC_KIND_INJECT);
  if (inject_launch(x_dev, dtype, n, eb, preserve_zeros, pcg_state, out_dev, s))
    return set_err(ACTC_ECUDA, "inject launch failed: %s", cudaGetErrorString(cudaGetLastError()));
  return ACTC_OK;
}

int actc_codebook_from_lengths(actc_ctx *c, const uint16_t *lengths, uint64_t A, uint32_t *canon,
                               uint32_t *len_counts, uint32_t *live_host, actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (A > kMaxAlphabet || A == 0) return set_err(ACTC_EPARAM, "alphabet too large");
  int rc = run_codebook(c, nullptr, A, lengths, nullptr, nullptr, 0, 0, s);
  if (rc) return rc;
  actc_plan_t plan;
  CK(cudaMemcpyAsync(&plan, c->plan_dev, sizeof(plan), cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (plan.status == ACTC_EPARAM) return set_err(ACTC_EFORMAT, "code length exceeds 63 bits");
  if (plan.live_symbols) CK(cudaMemcpyAsync(canon, c->canon.p, 4ull * plan.live_symbols, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(len_counts, c->lencnt.p, 4 * 64, cudaMemcpyDeviceToDevice, s));
  *live_host = plan.live_symbols;
  return ACTC_OK;
}

int actc_build_chunk_index(actc_ctx *c, const actc_stream_t *S, uint64_t *chunk_off, uint32_t *status_host,
                           actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  *status_host = ACTC_OK;
  if (S->n == 0) return ACTC_OK;
  const uint64_t seg_bits = 4096;
  const uint64_t nseg = std::max<uint64_t>(1, cdiv(S->payload_bits, seg_bits));
  int rc;
  if ((rc = grow(c->idx, nseg * 8 * 4 + 1024))) return rc;
  unsigned long long *start = (unsigned long long *)c->idx.p;
  unsigned long long *endp = start + nseg, *cnt = endp + nseg, *base = cnt + nseg;
  unsigned long long *misc = (unsigned long long *)c->misc.p;
  unsigned *changed = (unsigned *)(misc + M_CHANGED);
  unsigned *status = (unsigned *)(misc + M_STATUS);
  CK(cudaMemsetAsync(misc + M_STATUS, 0, 8, s));
  {
    KT(ACTC_KIND_LUT);
    k_build_lut<<<kLutSize / 256, 256, 0, s>>>(S->canon_syms_dev, S->len_counts_dev, (uint32_t *)c->lut.p, 0);
  }
  CKL();
  const int tpb = 128;
  const int grid = (int)cdiv(nseg, tpb);
  const uint32_t *pw = (const uint32_t *)S->payload_dev;
  {
    KT(ACTC_KIND_INDEX);
    k_sync_pass<<<grid, tpb, 0, s>>>(pw, S->payload_bits, (const uint32_t *)c->lut.p, S->len_counts_dev, seg_bits,
                                     nseg, start, endp, cnt, changed, status, 1);
  }
  CKL();
  unsigned h_changed = 1;
  for (uint64_t it = 0; it <= nseg + 1 && h_changed; it++) {
    CK(cudaMemsetAsync(changed, 0, 4, s));
    {
      KT(ACTC_KIND_INDEX);
      k_sync_pass<<<grid, tpb, 0, s>>>(pw, S->payload_bits, (const uint32_t *)c->lut.p, S->len_counts_dev, seg_bits,
                                       nseg, start, endp, cnt, changed, status, 0);
    }
    CKL();
    CK(cudaMemcpyAsync(&h_changed, changed, 4, cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  }
  {
    KT(ACTC_KIND_INDEX);
    k_excl_scan_u64<<<1, 1024, 0, s>>>(cnt, nseg, base, misc + M_SCAN_TOT);
  }
  CKL();
  unsigned long long total = 0, last_end = 0;
  unsigned st = 0;
  CK(cudaMemcpyAsync(&total, misc + M_SCAN_TOT, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&last_end, endp + nseg - 1, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaMemcpyAsync(&st, status, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (st || total < S->n || (total == S->n && last_end != S->payload_bits) || h_changed) {
    *status_host = ACTC_EFORMAT;
    return ACTC_OK;
  }
  {
    KT(ACTC_KIND_INDEX);
    k_index_emit<<<grid, tpb, 0, s>>>(pw, S->payload_bits, (const uint32_t *)c->lut.p, S->len_counts_dev, seg_bits,
                                      nseg, start, base, S->n, (unsigned long long *)chunk_off);
  }
  CKL();
  return ACTC_OK;
}

int actc_prequantize(const void *x, int dtype, uint64_t n, double eb, int64_t *q, actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!(eb > 0 && isfinite(eb))) return set_err(ACTC_EPARAM, "eb must be a positive finite real, got %g", eb);
  if (!n) return ACTC_OK;
  int grid = (int)std::min<uint64_t>(cdiv(n, 256), 148 * 16);
  KT(ACTC_KIND_DEBUG);
  k_prequantize<<<grid, 256, 0, s>>>(x, dtype, n, eb, (long long *)q);
  CKL();
  return ACTC_OK;
}

int actc_debug_quant_check(double eb, uint64_t lo, uint64_t count, uint64_t *out_host, actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (!(eb > 0 && isfinite(eb))) return set_err(ACTC_EPARAM, "eb must be a positive finite real, got %g", eb);
  const QParams P = make_qparams(eb);  // exactly as launch_k1 builds it
  unsigned long long *d = nullptr;
  CK(cudaMallocAsync((void **)&d, 16, s));
  CK(cudaMemsetAsync(d, 0, 16, s));
  if (count) {
    KT(ACTC_KIND_DEBUG);
    k_quant_check<<<148 * 16, 256, 0, s>>>(lo, count, P, d);
    CKL();
  }
  CK(cudaMemcpyAsync(out_host, d, 16, cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(d, s));
  return ACTC_OK;
}

int actc_lorenzo_encode(const int64_t *lat, uint64_t n, uint32_t radius, const uint8_t *force, uint32_t *sym,
                        uint64_t *n_out_host, actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (radius < 2) return set_err(ACTC_EPARAM, "radius must be >= 2, got %u", radius);
  // stream-ordered scratch word on the stream's device (no per-thread
  // cache: a thread may drive several devices and streams)
  unsigned long long *d_cnt = nullptr;
  CK(cudaMallocAsync((void **)&d_cnt, 8, s));
  CK(cudaMemsetAsync(d_cnt, 0, 8, s));
  if (n) {
    int grid = (int)std::min<uint64_t>(cdiv(n, 256), 148 * 16);
    KT(ACTC_KIND_DEBUG);
    k_lorenzo_encode<<<grid, 256, 0, s>>>((const long long *)lat, n, radius, force, sym, d_cnt);
    CKL();
  }
  CK(cudaMemcpyAsync(n_out_host, d_cnt, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(d_cnt, s));
  return ACTC_OK;
}

int actc_lorenzo_decode(const uint32_t *sym, uint64_t n, const int64_t *olat, uint64_t k, uint32_t radius,
                        int64_t *out, uint32_t *status_host, actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  unsigned *d_st = nullptr;  // stream-ordered scratch word
  CK(cudaMallocAsync((void **)&d_st, 4, s));
  CK(cudaMemsetAsync(d_st, 0, 4, s));
  {
    KT(ACTC_KIND_DEBUG);
    k_lorenzo_decode_seq<<<1, 1, 0, s>>>(sym, n, (const long long *)olat, k, radius, (long long *)out, d_st);
  }
  CKL();
  CK(cudaMemcpyAsync(status_host, d_st, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(d_st, s));
  return ACTC_OK;
}

int actc_huffman_plan(actc_ctx *c, const uint32_t *sym, uint64_t n, uint64_t A, uint16_t *lengths,
                      actc_plan_t *plan_host, actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (A < 1) return set_err(ACTC_EPARAM, "alphabet_size must be >= 1");
  if (A > kMaxAlphabet) return set_err(ACTC_EPARAM, "alphabet too large for the device codebook");
  int rc;
  if ((rc = grow(c->hist, 8 * A))) return rc;
  CK(cudaMemsetAsync(c->hist.p, 0, 8 * A, s));
  CK(cudaMemsetAsync(c->misc.p, 0, 8 * M_SLOTS, s));
  unsigned long long *misc = (unsigned long long *)c->misc.p;
  uint32_t win_n = (uint32_t)std::min<uint64_t>(A, K1_WIN);
  if (n) {
    int grid = (int)std::min<uint64_t>(cdiv(n, 256), (uint64_t)c->num_sms * 4);
    KT(ACTC_KIND_DEBUG);
    k_hist_u32<<<grid, 256, win_n * 4, s>>>(sym, n, A, (unsigned long long *)c->hist.p, (unsigned *)(misc + M_BAD), win_n);
    CKL();
  }
  unsigned bad = 0;
  CK(cudaMemcpyAsync(&bad, misc + M_BAD, 4, cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  if (bad) return set_err(ACTC_EPARAM, "symbol out of alphabet range");
  if ((rc = run_codebook(c, (const unsigned long long *)c->hist.p, A, nullptr, lengths, nullptr, n, 4, s))) return rc;
  if ((rc = plan_to_host(c, plan_host, s))) return rc;
  c->n = n;
  c->A = A;
  c->radius = 0;
  c->sym_bytes = 4;
  c->mode = 2;
  return ACTC_OK;
}

int actc_huffman_encode(actc_ctx *c, const uint32_t *sym, const actc_plan_t *plan, uint8_t *payload,
                        uint32_t *canon, uint32_t *len_counts, uint64_t *chunk_off, actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (c->mode != 2 || plan->n != c->n) return set_err(ACTC_EPARAM, "actc_huffman_encode without a matching plan");
  if (plan->status != ACTC_OK) return set_err(plan->status, "Huffman code length exceeds 63 bits");
  if (c->n) {
    int rc = launch_encode(c, sym, 4, c->n, nullptr, plan, payload, nullptr, nullptr, chunk_off, 0, s);
    if (rc) return rc;
  }
  if (plan->live_symbols)
    CK(cudaMemcpyAsync(canon, c->canon.p, 4ull * plan->live_symbols, cudaMemcpyDeviceToDevice, s));
  CK(cudaMemcpyAsync(len_counts, c->lencnt.p, 4 * 64, cudaMemcpyDeviceToDevice, s));
  return ACTC_OK;
}

int actc_huffman_decode(actc_ctx *c, const actc_stream_t *stream, uint32_t *symbols,
                        actc_decode_result_t *result_host, actc_stream s) {
  return launch_decode(c, stream, symbols, 2, result_host, (cudaStream_t)s);
}

int actc_code_lengths(actc_ctx *c, const uint64_t *freqs, uint64_t A, uint16_t *lengths, actc_plan_t *plan_host,
                      actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (A < 1 || A > kMaxAlphabet) return set_err(ACTC_EPARAM, "bad alphabet size");
  int rc = run_codebook(c, (const unsigned long long *)freqs, A, nullptr, lengths, nullptr, 1, 4, s);
  if (rc) return rc;
  if ((rc = plan_to_host(c, plan_host, s))) return rc;
  return ACTC_OK;
}

int actc_count_nonzero(const void *x, int dtype, uint64_t n, uint64_t *out_host, actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  unsigned long long *d = nullptr;  // stream-ordered scratch word
  CK(cudaMallocAsync((void **)&d, 8, s));
  CK(cudaMemsetAsync(d, 0, 8, s));
  if (n) {
    int grid = (int)std::min<uint64_t>(cdiv(n, 256), 148 * 8);
    KT(ACTC_KIND_STATS);
    k_count_nonzero<<<grid, 256, 0, s>>>(x, dtype, n, d);
    CKL();
  }
  CK(cudaMemcpyAsync(out_host, d, 8, cudaMemcpyDeviceToHost, s));
  CK(cudaFreeAsync(d, s));
  return ACTC_OK;
}

int actc_mean_abs(actc_ctx *c, const void *x, int dtype, uint64_t n, double *out_host, actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) return set_err(ACTC_EPARAM, "empty tensor");
  int depth = 0;
  while (depth < 16 && (n >> depth) > 4096) depth++;
  int rc;
  if ((rc = grow(c->part, 8ull * ((1ull << depth) + 1)))) return rc;
  double *part = (double *)c->part.p;
  uint64_t nt = 1ull << depth;
  {
    KT(ACTC_KIND_STATS);
    k_pairwise_partials<<<(int)cdiv(nt, 128), 128, 0, s>>>(x, dtype, n, depth, part);
  }
  CKL();
  {
    KT(ACTC_KIND_STATS);
    k_pairwise_finish<<<1, 1, 0, s>>>(part, dtype, n, depth, part + nt);
  }
  CKL();
  CK(cudaMemcpyAsync(out_host, part + nt, 8, cudaMemcpyDeviceToHost, s));
  return ACTC_OK;
}

int actc_lbar(actc_ctx *c, const void *g, int dtype, uint64_t N, uint64_t per, void *per_sample_max,
              double *out_host, actc_stream stream) {
  cudaStream_t s = (cudaStream_t)stream;
  if (N == 0) return set_err(ACTC_EPARAM, "empty batch");
  int rc;
  if ((rc = grow(c->part, 8 * N + 8 * N + 64))) return rc;
  unsigned long long *bits = (unsigned long long *)c->part.p;
  double *res = (double *)(bits + N);
  void *psm = per_sample_max ? per_sample_max : (void *)(res + 1);
  CK(cudaMemsetAsync(bits, 0, 8 * N, s));
  uint64_t total = N * per;
  if (total) {
    int grid = (int)std::min<uint64_t>(cdiv(total, 256), 148 * 8);
    KT(ACTC_KIND_STATS);
    k_sample_max<<<grid, 256, 0, s>>>(g, dtype, N, per, bits);
    CKL();
  }
  {
    KT(ACTC_KIND_STATS);
    k_lbar_finish<<<1, 1, 0, s>>>(bits, dtype, N, psm, res);
  }
  CKL();
  CK(cudaMemcpyAsync(out_host, res, 8, cudaMemcpyDeviceToHost, s));
  return ACTC_OK;
}

}  // extern "C"
