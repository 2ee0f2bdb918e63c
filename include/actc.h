/*
 * actc.h -- C ABI of the B200-native COMET activation codec (libactc.so).
 *
 * The reference (/root/reference/pkg, Python) exposes this path as Python
 * functions; this header is the native boundary its FFI would bind
 * (see INTEGRATION.md for the ctypes binding).  Each entry point cites the
 * reference interface it replaces.
 *
 * Conventions
 *  - Every pointer named *_dev is CUDA device memory; every call is
 *    stream-ordered on the given cudaStream_t and does not block the host
 *    unless stated.  Buffers are caller-owned (the host wrapper allocates
 *    them from the PyTorch caching allocator); the context owns only
 *    scratch.
 *  - Return value: ACTC_OK or an error class mirroring the reference's
 *    exception taxonomy (errors.py:4-33).  actc_last_error() gives text.
 *  - Device-detected errors (decode faults, marker mismatch, code length
 *    > 63) are reported in the `status` field of the host-visible structs
 *    below after the caller synchronizes the stream.
 */
#ifndef ACTC_H
#define ACTC_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ACTC_OK 0
#define ACTC_EPARAM 1  /* -> ParameterError (errors.py:12) */
#define ACTC_EDATA 2   /* -> DataError      (errors.py:16) */
#define ACTC_EFORMAT 3 /* -> FormatError    (errors.py:20) */
#define ACTC_ENOMEM 4
#define ACTC_ECUDA 5
#define ACTC_EAGAIN 6  /* plan status only: the async codebook needs its fallback, redo (actc_compress_async) */

#define ACTC_FLAG_PRESERVE_ZEROS 1u /* CMTZ flags bit0 (codec.py:96) */

#define ACTC_DTYPE_F32 0
#define ACTC_DTYPE_F64 1

/* Symbols per decode chunk: the encoder records the bit offset of every
 * ACTC_CHUNK-th symbol in a device-side index (not part of CMTZ). */
#define ACTC_CHUNK 128
#define ACTC_MAX_CODE_LENGTH 63 /* huffman.py:34 */

typedef void *actc_stream; /* a cudaStream_t */
typedef struct actc_ctx actc_ctx;

/* Result of compress phase 1 (quantize + Lorenzo + histogram + codebook);
 * valid on the host after the stream is synchronized. */
typedef struct {
  uint64_t n;             /* element count (= symbol_count, codec.py:323) */
  uint64_t n_outliers;    /* len(outlier_indices) (codec.py:321) */
  uint64_t payload_bits;  /* sum_s hist[s]*len[s] (huffman.py:189) */
  uint32_t live_symbols;  /* number of symbols with a code */
  uint32_t max_len;       /* longest code length */
  uint64_t rle_runs;      /* CMTZ RLE records incl. 65535-splits (codec.py:201-226) */
  double entropy_bits;    /* stream_entropy_bits(hist) (huffman.py:239-246) */
  uint32_t status;        /* ACTC_OK or ACTC_EPARAM (code length > 63) */
  uint32_t sym_bytes;     /* 2 (u16 symbols, radius <= 2^15) or 4 */
  uint32_t sym_lo;        /* smallest / largest live symbol */
  uint32_t sym_hi;
} actc_plan_t;

/* A compressed stream as the decoder sees it (all arrays on the device).
 * Field meaning follows CompressedActivation (codec.py:74-86); the code
 * table is kept in canonical form (symbols ordered by (length, symbol),
 * huffman.py:78-94) instead of the per-symbol length table. */
typedef struct {
  uint64_t n;
  double eb;
  uint32_t radius;
  uint32_t flags;
  uint64_t n_outliers;
  const uint64_t *outlier_idx_dev; /* ascending, codec.py:321 */
  const float *outlier_val_dev;    /* exact originals, codec.py:322 */
  uint32_t live_symbols;
  const uint32_t *canon_syms_dev;  /* [live_symbols] */
  const uint32_t *len_counts_dev;  /* [64]: number of codes of each length */
  const uint8_t *payload_dev;      /* MSB-first bitstream; 4-byte aligned, >=32 B tail pad */
  uint64_t payload_bits;
  const uint64_t *chunk_offsets_dev; /* [ceil(n/ACTC_CHUNK)] or NULL (rebuilt) */
  const int64_t *chunk_lat_dev;      /* [ceil(n/ACTC_CHUNK)] lattice before each chunk, or NULL */
  const void *table_dev;             /* decode table built at compress time (actc_ctx_set_table_out), or NULL */
} actc_stream_t;

/* Result of a decompression; valid after the stream is synchronized. */
typedef struct {
  uint64_t nonzero;  /* count_nonzero(reconstruction) -> R (training.py:351-352) */
  uint64_t markers;  /* number of outlier markers decoded */
  uint32_t status;   /* ACTC_OK or ACTC_EFORMAT */
  uint32_t reserved;
} actc_decode_result_t;

const char *actc_last_error(void);
int actc_version(void);

/* One context per stream: owns grow-on-demand device scratch. */
int actc_ctx_create(int device, actc_ctx **out);
void actc_ctx_destroy(actc_ctx *ctx);
/* device bytes the context's scratch currently holds (cudaMalloc'ed by the
 * library, outside the caller's allocator) */
uint64_t actc_ctx_device_bytes(const actc_ctx *ctx);
/* Decode faults of every decoder launched on this context since the last
 * call (ACTC_OK or ACTC_EFORMAT), including launches made without a result
 * mailbox (batched decompression): the sticky word is copied to
 * status_host (pinned; valid after the stream is synchronized) and reset.
 * Replaces the FormatError huffman_decode / decompress raise at once
 * (huffman.py:228-235, codec.py:356-359) for callers that defer the check
 * to their next synchronisation point. */
int actc_ctx_take_status(actc_ctx *ctx, uint32_t *status_host, actc_stream s);
/* symbol scratch for the NEXT compress launch on this context (K1 writes
 * the n symbols, u16 when 2*radius <= 65536 else u32, plus 64 bytes; the
 * encoder reads them): lets a caller hand in stream-ordered memory from its
 * own allocator instead of the context's persistent buffer.  Consumed by
 * that launch; must stay valid until the compression completes. */
int actc_ctx_set_scratch(actc_ctx *ctx, void *sym_dev, uint64_t bytes);
/* buffer (ACTC_TABLE_BYTES) for the decode table of the NEXT compression on
 * this context: the codebook's tail builds the table actc_decompress will
 * pick for the stream (prefix LUT, or the u8 length table for wide
 * alphabets), so decompression launches only the decoder (pass it back as
 * actc_stream_t.table_dev).  Consumed by that launch. */
#define ACTC_TABLE_BYTES 16400
int actc_ctx_set_table_out(actc_ctx *ctx, void *table_dev, uint64_t bytes);

/* compress(), phase 1 -- replaces codec.py:296-316 up to the codebook:
 * prequantize (:238-251), bound check (:311-312), lorenzo_encode
 * (:254-272), bincount (huffman.py:183), build_code_lengths
 * (huffman.py:37-75), canonical_codes (huffman.py:78-94).
 * chunk_lat_dev (may be NULL) receives the decode index's lattice value
 * before every ACTC_CHUNK-th element ([ceil(n/ACTC_CHUNK)] int64).
 * plan_host must be pinned host memory; it is written asynchronously. */
int actc_compress_plan(actc_ctx *ctx, const float *x_dev, uint64_t n, double eb,
                       uint32_t radius, uint32_t flags, int64_t *chunk_lat_dev,
                       actc_plan_t *plan_host, actc_stream s);

/* compress(), phase 2 -- huffman_encode bit packing (huffman.py:188-207)
 * plus outlier extraction (codec.py:321-322) and the decode chunk index.
 * `plan` is the synchronized phase-1 result; buffers are sized from it:
 *   payload_dev      >= 4*ceil(payload_bits/32) + 32 bytes, 4-byte aligned
 *   outlier_idx_dev  [n_outliers], outlier_val_dev [n_outliers]
 *   canon_syms_dev   [live_symbols], len_counts_dev [64]
 *   chunk_offsets_dev [ceil(n/ACTC_CHUNK)]
 * Must follow actc_compress_plan on the same ctx and stream. */
int actc_compress_encode(actc_ctx *ctx, const float *x_dev, const actc_plan_t *plan,
                         uint8_t *payload_dev, uint64_t *outlier_idx_dev,
                         float *outlier_val_dev, uint32_t *canon_syms_dev,
                         uint32_t *len_counts_dev, uint64_t *chunk_offsets_dev,
                         actc_stream s);

/* compress(), both phases without a host round trip (for batches): K1,
 * the codebook and the K3 segment encoder are launched back to back, the
 * encoder taking its live symbol range from the device plan.  Output
 * buffers are sized by caps instead of the plan:
 *   payload_dev >= payload_cap_bytes (a Huffman payload is at most
 *     n*ceil(log2 L) bits for L live symbols; the caller passes that bound + 32)
 *   outlier_idx_dev / outlier_val_dev [k_cap]
 *   canon_syms_dev [min(alphabet, n)], len_counts_dev [64], chunk_offsets_dev
 * The plan lands in plan_host (pinned) when the stream reaches it.  If the
 * stream needs the wide (> 26-bit) encoder, exceeds a cap, or the plan
 * status is not ACTC_OK, nothing is encoded and the caller redoes the
 * tensor with actc_compress_plan/actc_compress_encode.  Same inputs and
 * ownership rules as actc_compress_plan.
 * ACTC_ASYNC_NO_FALLBACK: do not queue the symbol-level fallback codebook
 * behind the frequency-class one (its launch needs a whole SM and waits for
 * one to drain); if the fast codebook's capacities are exceeded the plan
 * status is ACTC_EAGAIN and the caller redoes the tensor. */
#define ACTC_ASYNC_K1_ONLY 0x100u /* flags: launch only K1 (quantize/Lorenzo/histogram) */
#define ACTC_ASYNC_REST 0x200u    /* flags: launch the codebook + encoder after a K1_ONLY call */
#define ACTC_ASYNC_NO_FALLBACK 0x400u
int actc_compress_async(actc_ctx *ctx, const float *x_dev, uint64_t n, double eb, uint32_t radius,
                        uint32_t flags, int64_t *chunk_lat_dev, uint8_t *payload_dev,
                        uint64_t payload_cap_bytes, uint64_t *outlier_idx_dev, float *outlier_val_dev,
                        uint64_t k_cap, uint32_t *canon_syms_dev, uint32_t *len_counts_dev,
                        uint64_t *chunk_offsets_dev, actc_plan_t *plan_host, actc_stream s);

/* decompress() -- replaces codec.py:343-369: huffman_decode
 * (huffman.py:210-236), marker check (codec.py:356-359), lorenzo_decode
 * (codec.py:275-293), recon/splice/re-zero (codec.py:364-368).
 * out_dtype ACTC_DTYPE_F64 is bit-identical to the reference's fp64
 * output; ACTC_DTYPE_F32 stores fp32(that value).  result_host is pinned
 * host memory written asynchronously.  out_dtype may carry
 * ACTC_DEC_LUT_ONLY (build only the decode table into ctx) or ACTC_DEC_REST
 * (launch only the decoder, after a LUT_ONLY call with the same ctx, stream
 * and actc_stream_t): a batch puts every table build on the GPU before any
 * decoder fills it.  The nonzero count of the result (R) is only formed when
 * result_host is given and ACTC_DEC_NO_NONZERO is not set. */
#define ACTC_DEC_LUT_ONLY 0x100
#define ACTC_DEC_REST 0x200
#define ACTC_DEC_NO_NONZERO 0x400
int actc_decompress(actc_ctx *ctx, const actc_stream_t *stream, void *out_dev,
                    int out_dtype, actc_decode_result_t *result_host, actc_stream s);

/* zlib.crc32(data, crc_in) of a device buffer -- the CMTZ checksum
 * (codec.py:118 writes it over every preceding byte, codec.py:126 checks it).
 * A running value continues a checksum begun elsewhere (the host-built
 * header), exactly as zlib.crc32's second argument.  Synchronizes. */
int actc_crc32(actc_ctx *ctx, const void *data_dev, uint64_t len, uint32_t crc_in,
               uint32_t *crc_out_host, actc_stream s);

/* Utility (no reference counterpart): count <= 16 device-to-device copies
 * queued on one stream in one call -- the exact-size container compaction
 * after an asynchronous compression (codec.py compress_end, compact=True).
 * Asynchronous. */
int actc_memcpy_batch(void *const *dst_dev, const void *const *src_dev, const uint64_t *bytes, int count,
                      actc_stream s);

/* Build the canonical code table from a per-symbol length table (the
 * form CMTZ stores, codec.py:164) -- used after from_bytes
 * (codec.py:121-179).  canon_syms_dev needs [count of nonzero lengths]. */
int actc_codebook_from_lengths(actc_ctx *ctx, const uint16_t *lengths_dev, uint64_t alphabet,
                               uint32_t *canon_syms_dev, uint32_t *len_counts_dev,
                               uint32_t *live_host, actc_stream s);

/* Rebuild the chunk index of a stream that lacks one (blobs parsed by
 * from_bytes): self-synchronising parallel decode.  Synchronizes. */
int actc_build_chunk_index(actc_ctx *ctx, const actc_stream_t *stream,
                           uint64_t *chunk_offsets_dev, uint32_t *status_host, actc_stream s);

/* ---- debug / conformance entry points (reference internals) ---- */

/* prequantize (codec.py:238-251); x_dtype ACTC_DTYPE_F32 or _F64 */
int actc_prequantize(const void *x_dev, int x_dtype, uint64_t n, double eb, int64_t *q_dev,
                     actc_stream s);
/* exhaustive check of the fp32 fast quantizer used by compress: every
 * finite fp32 bit pattern u in [lo, lo+count) (count <= 2^32 - lo) that the
 * fast path claims is compared with the exact restatement of prequantize +
 * bound check (codec.py:248-251, 311-312).  out_host (pinned, 2 x u64,
 * written async): {mismatches, elements the fast path took}. */
int actc_debug_quant_check(double eb, uint64_t lo, uint64_t count, uint64_t *out_host, actc_stream s);
/* lorenzo_encode (codec.py:254-272); symbols_dev u32, force_dev may be NULL;
 * n_outliers_host pinned, written async */
int actc_lorenzo_encode(const int64_t *lattice_dev, uint64_t n, uint32_t radius,
                        const uint8_t *force_dev, uint32_t *symbols_dev,
                        uint64_t *n_outliers_host, actc_stream s);
/* lorenzo_decode (codec.py:275-293); status_host gets ACTC_EFORMAT on a
 * marker/value count mismatch */
int actc_lorenzo_decode(const uint32_t *symbols_dev, uint64_t n, const int64_t *outlier_lattice_dev,
                        uint64_t k, uint32_t radius, int64_t *out_dev, uint32_t *status_host,
                        actc_stream s);
/* huffman_encode (huffman.py:171-207) over an arbitrary u32 symbol stream:
 * phase 1 builds histogram + codebook; lengths_dev receives the u16
 * per-symbol length table (build_code_lengths). */
int actc_huffman_plan(actc_ctx *ctx, const uint32_t *symbols_dev, uint64_t n, uint64_t alphabet,
                      uint16_t *lengths_dev, actc_plan_t *plan_host, actc_stream s);
int actc_huffman_encode(actc_ctx *ctx, const uint32_t *symbols_dev, const actc_plan_t *plan,
                        uint8_t *payload_dev, uint32_t *canon_syms_dev, uint32_t *len_counts_dev,
                        uint64_t *chunk_offsets_dev, actc_stream s);
/* huffman_decode (huffman.py:210-236): symbols out as u32 */
int actc_huffman_decode(actc_ctx *ctx, const actc_stream_t *stream, uint32_t *symbols_dev,
                        actc_decode_result_t *result_host, actc_stream s);
/* build_code_lengths (huffman.py:37-75) from a u64 frequency table */
int actc_code_lengths(actc_ctx *ctx, const uint64_t *freqs_dev, uint64_t alphabet,
                      uint16_t *lengths_dev, actc_plan_t *plan_host, actc_stream s);

/* ---- per-layer statistics (controller inputs) ---- */

/* count_nonzero (tensor.py:181, training.py:352); out_host pinned */
int actc_count_nonzero(const void *x_dev, int dtype, uint64_t n, uint64_t *out_host, actc_stream s);
/* mean(|x|) with numpy's pairwise summation order (tensor.py:182,
 * nn.py:249-253): fp32 input -> f32(f64(sum_f32)/n) */
int actc_mean_abs(actc_ctx *ctx, const void *x_dev, int dtype, uint64_t n, double *out_host,
                  actc_stream s);
/* np.abs(g).reshape(N,-1).max(axis=1).mean() (training.py:358-361);
 * per_sample_max_dev optional [N] output in the input dtype */
int actc_lbar(actc_ctx *ctx, const void *g_dev, int dtype, uint64_t N, uint64_t per_sample,
              void *per_sample_max_dev, double *out_host, actc_stream s);

/* inject_uniform_error (errorprop.py:127-139): out = f64(x) + U[-eb, eb]
 * noise (zeros keep 0 noise when preserve_zeros), bit-identical to numpy's
 * default_rng(seed).uniform draws.  pcg_state = {state_hi, state_lo, inc_hi,
 * inc_lo}: the PCG64 state numpy derives from the seed (host SeedSequence).
 * x is fp32 or fp64 (dtype), out is fp64[n]. */
int actc_inject_uniform(actc_ctx *ctx, const void *x_dev, int dtype, uint64_t n, double eb,
                        int preserve_zeros, const uint64_t *pcg_state, double *out_dev, actc_stream s);

/* ---- instrumentation (not part of the reference interface) ----
 * Every kernel launch the library makes is counted per kind; with timing
 * enabled each launch is also bracketed by CUDA events recorded on the
 * stream it is launched on.  actc_kernel_stats synchronizes the pending
 * events, writes per-kind totals (launches, summed kernel ms) for up to
 * `nkinds` kinds and resets the accumulators.  Process-wide. */
enum {
  ACTC_KIND_QUANT = 0,    /* K1 quantize + Lorenzo + histogram */
  ACTC_KIND_CODEBOOK = 1, /* K2 Huffman codebook */
  ACTC_KIND_COUNT = 2,    /* K3 per-CTA bit count */
  ACTC_KIND_SCAN = 3,     /* exclusive scans of per-CTA totals */
  ACTC_KIND_PACK = 4,     /* K3 bit packing + outlier extraction */
  ACTC_KIND_FIXUP = 5,    /* K3 boundary-word fixup */
  ACTC_KIND_LUT = 6,      /* decoder prefix table */
  ACTC_KIND_DECODE = 7,   /* K4 decode + inverse Lorenzo + recon */
  ACTC_KIND_INDEX = 8,    /* chunk-index rebuild (from_bytes streams) */
  ACTC_KIND_STATS = 9,    /* K5 statistics */
  ACTC_KIND_DEBUG = 10,   /* conformance entry points */
  ACTC_KIND_CRC = 11,     /* K6 CRC-32 */
  ACTC_KIND_INJECT = 12,  /* K7 uniform error injection */
  ACTC_KIND_NKINDS = 13
};
int actc_timing_enable(int on);
int actc_kernel_stats(uint64_t *launches, double *ms, int nkinds);

#ifdef __cplusplus
}
#endif
#endif /* ACTC_H */
