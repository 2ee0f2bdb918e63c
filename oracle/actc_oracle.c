/*
 * actc_oracle.c -- CPU restatement of the COMET activation codec.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the parity oracle for the CUDA
 * path in paper_2111_09562_b200/csrc.  Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline / --impl reference leg may load it; the
 * product path never links or calls it.
 *
 * It restates, in plain C, the algorithm of the reference package
 * /root/reference/pkg/src/actcomp (pure Python/numpy):
 *   prequantize          codec.py:238-251
 *   bound check          codec.py:311-312
 *   lorenzo_encode       codec.py:254-272
 *   bincount             huffman.py:183
 *   build_code_lengths   huffman.py:37-75   (heapq order (freq, tiebreak))
 *   canonical_codes      huffman.py:78-94
 *   huffman_encode       huffman.py:171-207 (MSB-first, np.packbits)
 *   _decode_tables       huffman.py:97-117
 *   _decode_bits         huffman.py:120-142
 *   lorenzo_decode       codec.py:275-293
 *   decompress           codec.py:343-369
 *   to_bytes/from_bytes  codec.py:95-179, _rle_* codec.py:201-235
 *   compute_stats        tensor.py:171-192 (numpy pairwise summation)
 *
 * Parity pinning: the fixtures in tests/golden were produced by running the reference
 * itself (tests/golden/make_golden.py); tests/test_oracle_golden.py checks
 * this restatement against every one of them.
 *
 * Build: see oracle/Makefile (gcc -O2 -ffp-contract=off, no fast-math: the
 * fp64 arithmetic must be IEEE round-to-nearest with no FMA contraction).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define ORC_OK 0
#define ORC_EPARAM 1
#define ORC_EDATA 2
#define ORC_EFORMAT 3
#define ORC_ENOMEM 4

#define LATTICE_LIMIT 2305843009213693952.0 /* 2^61, codec.py:37 */
#define MAX_CODE_LENGTH 63                   /* huffman.py:34 */

static char g_err[256];
const char *orc_last_error(void) { return g_err; }
static int fail(int code, const char *msg) {
  strncpy(g_err, msg, sizeof(g_err) - 1);
  g_err[sizeof(g_err) - 1] = 0;
  return code;
}

/* ------------------------------------------------------------------ */
/* prequantize: codec.py:248-251                                        */
/*   v = f64(x) / (2 eb); q = sign(v) * floor(|v| + 0.5); clip +-2^61    */
/* ------------------------------------------------------------------ */
static inline int64_t prequantize1(double x, double two_eb) {
  double v = x / two_eb;
  double f = floor(fabs(v) + 0.5);
  double s = (v > 0.0) ? 1.0 : ((v < 0.0) ? -1.0 : 0.0); /* np.sign */
  double q = s * f;
  if (q < -LATTICE_LIMIT) q = -LATTICE_LIMIT; /* np.clip */
  if (q > LATTICE_LIMIT) q = LATTICE_LIMIT;
  return (int64_t)q; /* astype(int64); q is integral */
}

void orc_prequantize_f64(const double *x, uint64_t n, double eb, int64_t *q) {
  double two_eb = 2.0 * eb;
  for (uint64_t i = 0; i < n; i++) q[i] = prequantize1(x[i], two_eb);
}

void orc_prequantize_f32(const float *x, uint64_t n, double eb, int64_t *q) {
  double two_eb = 2.0 * eb;
  for (uint64_t i = 0; i < n; i++) q[i] = prequantize1((double)x[i], two_eb);
}

/* ------------------------------------------------------------------ */
/* lorenzo_encode: codec.py:254-272 (with the forced-outlier mask that  */
/* compress() builds at codec.py:311-315)                               */
/* ------------------------------------------------------------------ */
/* returns number of outliers; symbols[i] = 0 marks an outlier */
uint64_t orc_lorenzo_encode(const int64_t *lattice, uint64_t n, uint64_t radius,
                            const uint8_t *force, uint64_t *symbols) {
  int64_t prev = 0;
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; i++) {
    int64_t d = lattice[i] - prev;
    prev = lattice[i];
    uint64_t ad = (uint64_t)(d < 0 ? -d : d);
    int out = ad >= radius || (force && force[i]);
    symbols[i] = out ? 0 : (uint64_t)(d + (int64_t)radius);
    k += out;
  }
  return k;
}

/* lorenzo_decode: codec.py:275-293.  outlier_lattice holds the lattice
 * value of each outlier in position order.  Returns ORC_EFORMAT on a
 * marker/value count mismatch (codec.py:281-285). */
int orc_lorenzo_decode(const uint64_t *symbols, uint64_t n,
                       const int64_t *outlier_lattice, uint64_t k,
                       uint64_t radius, int64_t *out) {
  uint64_t markers = 0;
  for (uint64_t i = 0; i < n; i++) markers += symbols[i] == 0;
  if (markers != k) return fail(ORC_EFORMAT, "outlier count mismatch");
  int64_t acc = 0;
  uint64_t j = 0;
  for (uint64_t i = 0; i < n; i++) {
    if (symbols[i] == 0) {
      acc = outlier_lattice[j++]; /* rebase chain (codec.py:291-292) */
    } else {
      acc += (int64_t)symbols[i] - (int64_t)radius;
    }
    out[i] = acc;
  }
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* build_code_lengths: huffman.py:37-75.                                */
/* heapq pops in (freq, tiebreak) order; leaves have tiebreak = symbol, */
/* internal nodes a counter starting at the alphabet size.  Any binary  */
/* heap keyed on the (unique) pair reproduces the pop sequence.         */
/* ------------------------------------------------------------------ */
typedef struct {
  uint64_t f, tb;
  int64_t node; /* >=0 leaf symbol; <0: -(internal index)-1 */
} hent;

static inline int hless(const hent *a, const hent *b) {
  return a->f < b->f || (a->f == b->f && a->tb < b->tb);
}
static void hpush(hent *h, uint64_t *sz, hent e) {
  uint64_t i = (*sz)++;
  h[i] = e;
  while (i > 0) {
    uint64_t p = (i - 1) / 2;
    if (!hless(&h[i], &h[p])) break;
    hent t = h[i]; h[i] = h[p]; h[p] = t;
    i = p;
  }
}
static hent hpop(hent *h, uint64_t *sz) {
  hent top = h[0];
  h[0] = h[--(*sz)];
  uint64_t i = 0, n = *sz;
  for (;;) {
    uint64_t l = 2 * i + 1, r = l + 1, m = i;
    if (l < n && hless(&h[l], &h[m])) m = l;
    if (r < n && hless(&h[r], &h[m])) m = r;
    if (m == i) break;
    hent t = h[i]; h[i] = h[m]; h[m] = t;
    i = m;
  }
  return top;
}

int orc_build_code_lengths(const uint64_t *freqs, uint64_t A, uint16_t *lengths) {
  memset(lengths, 0, A * sizeof(uint16_t));
  uint64_t live = 0, last = 0;
  for (uint64_t s = 0; s < A; s++)
    if (freqs[s]) { live++; last = s; }
  if (live == 0) return ORC_OK;
  if (live == 1) { lengths[last] = 1; return ORC_OK; } /* huffman.py:50-52 */
  hent *heap = malloc(live * sizeof(hent));
  int64_t *kids = malloc(2 * (live - 1) * sizeof(int64_t));
  if (!heap || !kids) { free(heap); free(kids); return fail(ORC_ENOMEM, "oom"); }
  uint64_t sz = 0;
  for (uint64_t s = 0; s < A; s++)
    if (freqs[s]) hpush(heap, &sz, (hent){freqs[s], s, (int64_t)s});
  uint64_t counter = A, ni = 0;
  while (sz > 1) {
    hent a = hpop(heap, &sz), b = hpop(heap, &sz);
    kids[2 * ni] = a.node;
    kids[2 * ni + 1] = b.node;
    hpush(heap, &sz, (hent){a.f + b.f, counter++, -(int64_t)ni - 1});
    ni++;
  }
  /* depth: internal node i's parent has a larger index; walk top-down. */
  uint32_t *depth = calloc(ni, sizeof(uint32_t));
  int rc = ORC_OK;
  for (uint64_t ii = ni; ii-- > 0;) {
    for (int c = 0; c < 2; c++) {
      int64_t node = kids[2 * ii + c];
      uint32_t d = depth[ii] + 1;
      if (node >= 0) {
        if (d > MAX_CODE_LENGTH) rc = ORC_EPARAM;
        lengths[node] = (uint16_t)(d > 0xFFFF ? 0xFFFF : d);
      } else {
        depth[-node - 1] = d;
      }
    }
  }
  free(depth); free(kids); free(heap);
  if (rc) return fail(rc, "Huffman code length exceeds 63 bits");
  return ORC_OK;
}

/* canonical_codes: huffman.py:78-94; codes in (length, symbol) order */
void orc_canonical_codes(const uint16_t *lengths, uint64_t A, uint64_t *codes) {
  memset(codes, 0, A * sizeof(uint64_t));
  uint64_t code = 0;
  int first = 1;
  unsigned prev = 0;
  for (unsigned len = 1; len <= MAX_CODE_LENGTH; len++) {
    for (uint64_t s = 0; s < A; s++) {
      if (lengths[s] != len) continue;
      if (first) { prev = len; first = 0; }
      code <<= (len - prev);
      codes[s] = code;
      code += 1;
      prev = len;
    }
  }
}

/* ------------------------------------------------------------------ */
/* bit packing, MSB first per byte (huffman.py:192-206, np.packbits)   */
/* ------------------------------------------------------------------ */
static uint64_t encode_bits(const uint64_t *symbols, uint64_t n,
                            const uint16_t *lengths, const uint64_t *codes,
                            uint8_t *payload) {
  uint64_t pos = 0;
  uint64_t acc = 0; /* right-aligned pending bits */
  unsigned nacc = 0;
  for (uint64_t i = 0; i < n; i++) {
    unsigned len = lengths[symbols[i]];
    uint64_t code = codes[symbols[i]];
    /* push len bits, MSB first, in pieces that fit the accumulator */
    while (len) {
      unsigned take = len > 32 ? 32 : len;
      uint64_t piece = (code >> (len - take)) & ((1ull << take) - 1);
      acc = (acc << take) | piece;
      nacc += take;
      len -= take;
      while (nacc >= 8) {
        payload[pos >> 3] = (uint8_t)(acc >> (nacc - 8));
        nacc -= 8;
        pos += 8;
      }
    }
  }
  if (nacc) {
    payload[pos >> 3] = (uint8_t)(acc << (8 - nacc));
    pos += nacc;
  }
  return pos;
}

/* _decode_tables + _decode_bits: huffman.py:97-142.
 * Returns bits consumed, -1 exhausted, -2 invalid code. */
int64_t orc_decode_bits(const uint8_t *payload, uint64_t bit_length, uint64_t count,
                        const uint16_t *lengths, uint64_t A, uint64_t *out) {
  unsigned max_len = 0;
  for (uint64_t s = 0; s < A; s++)
    if (lengths[s] > max_len) max_len = lengths[s];
  int64_t counts[MAX_CODE_LENGTH + 2] = {0}, first_code[MAX_CODE_LENGTH + 2] = {0},
          base[MAX_CODE_LENGTH + 2] = {0};
  if (max_len > MAX_CODE_LENGTH + 1) max_len = MAX_CODE_LENGTH + 1;
  for (uint64_t s = 0; s < A; s++)
    if (lengths[s] && lengths[s] <= max_len) counts[lengths[s]]++;
  uint64_t *syms = malloc((A ? A : 1) * sizeof(uint64_t));
  int64_t code = 0, idx = 0;
  for (unsigned l = 1; l <= max_len; l++) {
    code <<= 1;
    first_code[l] = code;
    base[l] = idx;
    code += counts[l];
    idx += counts[l];
  }
  {
    int64_t fill[MAX_CODE_LENGTH + 2];
    memcpy(fill, base, sizeof(fill));
    for (uint64_t s = 0; s < A; s++)
      if (lengths[s] && lengths[s] <= max_len) syms[fill[lengths[s]]++] = s;
  }
  int64_t c = 0;
  unsigned length = 0;
  uint64_t emitted = 0;
  int64_t result = -1;
  for (uint64_t pos = 0; pos < bit_length; pos++) {
    unsigned bit = (payload[pos >> 3] >> (7 - (pos & 7))) & 1;
    c = (c << 1) | bit;
    length++;
    if (length > max_len) { result = -2; break; }
    int64_t off = c - first_code[length];
    if (off >= 0 && off < counts[length]) {
      out[emitted++] = syms[base[length] + off];
      if (emitted == count) { result = (int64_t)pos + 1; break; }
      c = 0;
      length = 0;
    }
  }
  free(syms);
  return result;
}

/* ------------------------------------------------------------------ */
/* CRC-32 (zlib polynomial, reflected), used by to_bytes/from_bytes     */
/* ------------------------------------------------------------------ */
static uint32_t crc_table[256];
static int crc_ready = 0;
static void crc_init(void) {
  for (uint32_t i = 0; i < 256; i++) {
    uint32_t c = i;
    for (int k = 0; k < 8; k++) c = (c & 1) ? 0xEDB88320u ^ (c >> 1) : c >> 1;
    crc_table[i] = c;
  }
  crc_ready = 1;
}
uint32_t orc_crc32(const uint8_t *p, uint64_t n) {
  if (!crc_ready) crc_init();
  uint32_t c = 0xFFFFFFFFu;
  for (uint64_t i = 0; i < n; i++) c = crc_table[(c ^ p[i]) & 0xFF] ^ (c >> 8);
  return c ^ 0xFFFFFFFFu;
}

/* ------------------------------------------------------------------ */
/* compress (codec.py:296-340) producing the CMTZ blob (codec.py:95-119)*/
/* ------------------------------------------------------------------ */
typedef struct {
  uint64_t n, k, A;
  uint64_t *symbols;   /* n */
  uint64_t *hist;      /* A */
  uint16_t *lengths;   /* A */
  uint64_t *outlier_idx;
  float *outlier_val;
  uint8_t *payload;
  uint64_t payload_bits;
  uint8_t *blob;
  uint64_t blob_len;
  uint64_t rle_runs;
} orc_result;

void orc_free(orc_result *r) {
  if (!r) return;
  free(r->symbols); free(r->hist); free(r->lengths); free(r->outlier_idx);
  free(r->outlier_val); free(r->payload); free(r->blob); free(r);
}

static void put_u8(uint8_t **p, uint8_t v) { *(*p)++ = v; }
static void put_u16(uint8_t **p, uint16_t v) { memcpy(*p, &v, 2); *p += 2; }
static void put_u32(uint8_t **p, uint32_t v) { memcpy(*p, &v, 4); *p += 4; }
static void put_u64(uint8_t **p, uint64_t v) { memcpy(*p, &v, 8); *p += 8; }
static void put_f64(uint8_t **p, double v) { memcpy(*p, &v, 8); *p += 8; }

/* number of (u16 run, u16 len) records incl. splitting (codec.py:201-226) */
static uint64_t rle_count(const uint16_t *len, uint64_t A) {
  if (A == 0) return 0;
  uint64_t runs = 0, i = 0;
  while (i < A) {
    uint64_t j = i;
    while (j < A && len[j] == len[i]) j++;
    uint64_t rl = j - i;
    runs += (rl + 0xFFFE) / 0xFFFF;
    i = j;
  }
  return runs;
}

int orc_compress(const float *x, const uint64_t *dims, int rank, double eb,
                 uint64_t radius, int preserve_zeros, orc_result **out) {
  *out = NULL;
  if (!(eb > 0 && isfinite(eb))) return fail(ORC_EPARAM, "eb must be a positive finite real");
  if (radius < 2) return fail(ORC_EPARAM, "radius must be >= 2");
  if (rank < 1 || rank > 255) return fail(ORC_EPARAM, "bad rank");
  uint64_t n = 1;
  for (int d = 0; d < rank; d++) n *= dims[d];
  for (uint64_t i = 0; i < n; i++)
    if (!isfinite(x[i])) return fail(ORC_EDATA, "tensor contains NaN or Inf");
  orc_result *r = calloc(1, sizeof(orc_result));
  uint64_t A = 2 * radius;
  r->n = n; r->A = A;
  r->symbols = malloc((n ? n : 1) * sizeof(uint64_t));
  r->hist = calloc(A, sizeof(uint64_t));
  r->lengths = calloc(A, sizeof(uint16_t));
  if (!r->symbols || !r->hist || !r->lengths) { orc_free(r); return fail(ORC_ENOMEM, "oom"); }
  double two_eb = 2.0 * eb;
  int64_t prev = 0;
  uint64_t k = 0;
  for (uint64_t i = 0; i < n; i++) {
    double v = (double)x[i];
    int64_t q = prequantize1(v, two_eb);                  /* codec.py:310 */
    double recon = (double)q * two_eb;                    /* codec.py:311 */
    int viol = fabs(v - recon) > eb;                      /* codec.py:312 */
    int64_t d = q - prev;                                 /* codec.py:267 */
    prev = q;
    uint64_t ad = (uint64_t)(d < 0 ? -d : d);
    int o = ad >= radius || viol;                         /* codec.py:268-270 */
    uint64_t s = o ? 0 : (uint64_t)(d + (int64_t)radius); /* codec.py:271 */
    r->symbols[i] = s;
    r->hist[s]++;
    k += o;
  }
  r->k = k;
  r->outlier_idx = malloc((k ? k : 1) * sizeof(uint64_t));
  r->outlier_val = malloc((k ? k : 1) * sizeof(float));
  for (uint64_t i = 0, j = 0; i < n && j < k; i++)
    if (r->symbols[i] == 0) { r->outlier_idx[j] = i; r->outlier_val[j] = x[i]; j++; }
  int rc = orc_build_code_lengths(r->hist, A, r->lengths);
  if (rc) { orc_free(r); return rc; }
  uint64_t *codes = malloc(A * sizeof(uint64_t));
  orc_canonical_codes(r->lengths, A, codes);
  uint64_t bits = 0;
  for (uint64_t s = 0; s < A; s++) bits += r->hist[s] * r->lengths[s];
  uint64_t pbytes = (bits + 7) / 8;
  r->payload = calloc(pbytes + 8, 1);
  r->payload_bits = encode_bits(r->symbols, n, r->lengths, codes, r->payload);
  free(codes);
  /* CMTZ blob, codec.py:95-119; size = 53 + 8r + 12k + 4m + ceil(bits/8) */
  r->rle_runs = rle_count(r->lengths, A);
  r->blob_len = 53 + 8ull * rank + 12ull * k + 4ull * r->rle_runs + pbytes;
  r->blob = malloc(r->blob_len);
  uint8_t *p = r->blob;
  memcpy(p, "CMTZ", 4); p += 4;
  put_u8(&p, 1);
  put_f64(&p, eb);
  put_u32(&p, (uint32_t)radius);
  put_u8(&p, 1); /* lorenzo-1d */
  put_u8(&p, preserve_zeros ? 1 : 0);
  put_u8(&p, 4); /* precision */
  put_u8(&p, (uint8_t)rank);
  for (int d = 0; d < rank; d++) put_u64(&p, dims[d]);
  put_u64(&p, k);
  for (uint64_t j = 0; j < k; j++) {
    put_u64(&p, r->outlier_idx[j]);
    memcpy(p, &r->outlier_val[j], 4); p += 4;
  }
  put_u64(&p, n);
  put_u32(&p, (uint32_t)r->rle_runs);
  for (uint64_t i = 0; i < A;) {
    uint64_t j = i;
    while (j < A && r->lengths[j] == r->lengths[i]) j++;
    uint64_t rl = j - i;
    while (rl > 0xFFFF) { put_u16(&p, 0xFFFF); put_u16(&p, r->lengths[i]); rl -= 0xFFFF; }
    put_u16(&p, (uint16_t)rl); put_u16(&p, r->lengths[i]);
    i = j;
  }
  put_u64(&p, r->payload_bits);
  memcpy(p, r->payload, pbytes); p += pbytes;
  put_u32(&p, orc_crc32(r->blob, (uint64_t)(p - r->blob)));
  *out = r;
  return ORC_OK;
}

uint64_t orc_result_n(const orc_result *r) { return r->n; }
uint64_t orc_result_k(const orc_result *r) { return r->k; }
uint64_t orc_result_blob_len(const orc_result *r) { return r->blob_len; }
uint64_t orc_result_payload_bits(const orc_result *r) { return r->payload_bits; }
uint64_t orc_result_rle_runs(const orc_result *r) { return r->rle_runs; }
void orc_result_copy(const orc_result *r, uint8_t *blob, uint64_t *symbols,
                     uint64_t *hist, uint16_t *lengths) {
  if (blob) memcpy(blob, r->blob, r->blob_len);
  if (symbols) memcpy(symbols, r->symbols, r->n * sizeof(uint64_t));
  if (hist) memcpy(hist, r->hist, r->A * sizeof(uint64_t));
  if (lengths) memcpy(lengths, r->lengths, r->A * sizeof(uint16_t));
}

/* ------------------------------------------------------------------ */
/* from_bytes (codec.py:121-179) + decompress (codec.py:343-369)        */
/* ------------------------------------------------------------------ */
typedef struct { const uint8_t *b; uint64_t len, pos; } cur_t;
static int take(cur_t *c, uint64_t n, const uint8_t **out) {
  if (c->pos + n > c->len || c->pos + n < c->pos) return fail(ORC_EFORMAT, "truncated compressed stream");
  *out = c->b + c->pos;
  c->pos += n;
  return 0;
}
#define TAKE(c, n, p) do { if (take(c, n, &p)) return ORC_EFORMAT; } while (0)

/* Parses a blob; on success fills header fields.  out_dims must hold 255. */
int orc_parse_header(const uint8_t *blob, uint64_t len, uint64_t *out_dims, int *out_rank,
                     uint64_t *n_out, double *eb_out, uint64_t *radius_out, int *preserve_out) {
  if (len < 4 + 1 + 8 + 4 + 2 + 2 + 4) return fail(ORC_EFORMAT, "compressed stream too short");
  uint32_t stored;
  memcpy(&stored, blob + len - 4, 4);
  if (orc_crc32(blob, len - 4) != stored) return fail(ORC_EFORMAT, "checksum mismatch");
  cur_t c = {blob, len - 4, 0};
  const uint8_t *p;
  TAKE(&c, 4, p);
  if (memcmp(p, "CMTZ", 4)) return fail(ORC_EFORMAT, "bad magic");
  TAKE(&c, 15, p);
  uint8_t version = p[0];
  double eb; memcpy(&eb, p + 1, 8);
  uint32_t radius; memcpy(&radius, p + 9, 4);
  uint8_t pred = p[13], flags = p[14];
  if (version != 1) return fail(ORC_EFORMAT, "unsupported version");
  if (pred != 1) return fail(ORC_EFORMAT, "unknown predictor id");
  if (!(eb > 0 && isfinite(eb)) || radius < 2) return fail(ORC_EFORMAT, "invalid codec params in header");
  TAKE(&c, 2, p);
  int rank = p[1];
  if (rank == 0) return fail(ORC_EFORMAT, "rank must be >= 1");
  TAKE(&c, 8ull * rank, p);
  for (int d = 0; d < rank; d++) {
    memcpy(&out_dims[d], p + 8 * d, 8);
    if (out_dims[d] < 1) return fail(ORC_EFORMAT, "bad extents");
  }
  *out_rank = rank; *eb_out = eb; *radius_out = radius; *preserve_out = flags & 1;
  TAKE(&c, 8, p);
  uint64_t k; memcpy(&k, p, 8);
  if (k > (len / 12) + 1) return fail(ORC_EFORMAT, "truncated compressed stream");
  TAKE(&c, 12 * k, p);
  *n_out = k;
  return ORC_OK;
}

/* decompress a blob into fp64 output (n elements).  Full validation. */
int orc_decompress_blob(const uint8_t *blob, uint64_t len, double *out, uint64_t n_cap) {
  uint64_t dims[255]; int rank; uint64_t k; double eb; uint64_t radius; int preserve;
  int rc = orc_parse_header(blob, len, dims, &rank, &k, &eb, &radius, &preserve);
  if (rc) return rc;
  cur_t c = {blob, len - 4, 21 + 8ull * rank + 8};
  const uint8_t *p;
  TAKE(&c, 12 * k, p);
  const uint8_t *pairs = p;
  TAKE(&c, 8, p);
  uint64_t symbol_count; memcpy(&symbol_count, p, 8);
  TAKE(&c, 4, p);
  uint32_t runs; memcpy(&runs, p, 4);
  TAKE(&c, 4ull * runs, p);
  const uint8_t *rle = p;
  uint64_t A = 2 * radius, tot = 0;
  for (uint32_t i = 0; i < runs; i++) { uint16_t rl; memcpy(&rl, rle + 4 * i, 2); tot += rl; }
  if (tot != A) return fail(ORC_EFORMAT, "code-length table does not cover alphabet");
  TAKE(&c, 8, p);
  uint64_t bits; memcpy(&bits, p, 8);
  uint64_t pbytes = bits / 8 + ((bits & 7) != 0);
  TAKE(&c, pbytes, p);
  const uint8_t *payload = p;
  if (c.pos != c.len) return fail(ORC_EFORMAT, "trailing bytes in compressed stream");
  uint64_t n = 1;
  for (int d = 0; d < rank; d++) n *= dims[d];
  if (n > n_cap) return fail(ORC_EPARAM, "output too small");
  if (symbol_count != n) return fail(ORC_EFORMAT, "symbol count != element count");
  uint16_t *lengths = malloc(A * sizeof(uint16_t));
  for (uint32_t i = 0, o = 0; i < runs; i++) {
    uint16_t rl, v; memcpy(&rl, rle + 4 * i, 2); memcpy(&v, rle + 4 * i + 2, 2);
    for (uint16_t j = 0; j < rl; j++) lengths[o++] = v;
  }
  uint64_t *symbols = malloc((n ? n : 1) * sizeof(uint64_t));
  int any = 0;
  for (uint64_t s = 0; s < A; s++) any |= lengths[s] > 0;
  if (n > 0) {
    if (!any) { rc = fail(ORC_EFORMAT, "empty code table with nonzero symbol count"); goto done; }
    if (bits > pbytes * 8) { rc = fail(ORC_EFORMAT, "payload shorter than declared bit length"); goto done; }
    int64_t consumed = orc_decode_bits(payload, bits, n, lengths, A, symbols);
    if (consumed == -1) { rc = fail(ORC_EFORMAT, "bitstream exhausted before all symbols decoded"); goto done; }
    if (consumed == -2) { rc = fail(ORC_EFORMAT, "invalid code in bitstream"); goto done; }
    if ((uint64_t)consumed != bits) { rc = fail(ORC_EFORMAT, "bitstream length mismatch"); goto done; }
  }
  /* marker positions must equal stored indices (codec.py:356-359) */
  {
    uint64_t j = 0;
    for (uint64_t i = 0; i < n; i++) {
      if (symbols[i] == 0) {
        uint64_t idx; memcpy(&idx, pairs + 12 * j, 8);
        if (j >= k || idx != i) { rc = fail(ORC_EFORMAT, "outlier markers disagree with stored indices"); goto done; }
        j++;
      }
    }
    if (j != k) { rc = fail(ORC_EFORMAT, "outlier markers disagree with stored indices"); goto done; }
  }
  {
    double two_eb = 2.0 * eb;
    int64_t acc = 0;
    uint64_t j = 0;
    for (uint64_t i = 0; i < n; i++) {
      double r;
      if (symbols[i] == 0) {
        float fv; memcpy(&fv, pairs + 12 * j + 8, 4);
        acc = prequantize1((double)fv, two_eb); /* codec.py:361-362 */
        r = (double)fv;                         /* splice, codec.py:365-366 */
        j++;
      } else {
        acc += (int64_t)symbols[i] - (int64_t)radius;
        r = (double)acc * two_eb;               /* codec.py:364 */
      }
      if (preserve && fabs(r) <= eb) r = 0.0;   /* re-zero, codec.py:367-368 */
      out[i] = r;
    }
  }
done:
  free(lengths); free(symbols);
  return rc;
}

/* Huffman-only helpers for tests (huffman_encode / huffman_decode). */
int orc_huffman_encode(const uint64_t *symbols, uint64_t n, uint64_t A,
                       uint16_t *lengths, uint8_t *payload, uint64_t *bits_out) {
  uint64_t *hist = calloc(A ? A : 1, sizeof(uint64_t));
  for (uint64_t i = 0; i < n; i++) {
    if (symbols[i] >= A) { free(hist); return fail(ORC_EPARAM, "symbol out of alphabet range"); }
    hist[symbols[i]]++;
  }
  int rc = orc_build_code_lengths(hist, A, lengths);
  free(hist);
  if (rc) return rc;
  if (n == 0) { *bits_out = 0; return ORC_OK; }
  uint64_t *codes = malloc(A * sizeof(uint64_t));
  orc_canonical_codes(lengths, A, codes);
  *bits_out = encode_bits(symbols, n, lengths, codes, payload);
  free(codes);
  return ORC_OK;
}

/* ------------------------------------------------------------------ */
/* statistics: tensor.py:171-192, training.py:351-361, nn.py:249-253    */
/* numpy add.reduce = pairwise summation (8 accumulators, 128 leaves,   */
/* split n2 = n/2 - (n/2) % 8).                                         */
/* ------------------------------------------------------------------ */
static float pw_f32(const float *a, uint64_t n) {
  if (n < 8) {
    float r = 0.0f; /* identity init; exact for |x| inputs */
    for (uint64_t i = 0; i < n; i++) r += a[i];
    return r;
  }
  if (n <= 128) {
    float r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    uint64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    float res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  }
  uint64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pw_f32(a, n2) + pw_f32(a + n2, n - n2);
}
static double pw_f64(const double *a, uint64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (uint64_t i = 0; i < n; i++) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; j++) r[j] = a[j];
    uint64_t i;
    for (i = 8; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; j++) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; i++) res += a[i];
    return res;
  }
  uint64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pw_f64(a, n2) + pw_f64(a + n2, n - n2);
}
float orc_pairwise_sum_f32(const float *a, uint64_t n) { return pw_f32(a, n); }
double orc_pairwise_sum_f64(const double *a, uint64_t n) { return pw_f64(a, n); }

/* mean(|a|) exactly as numpy: f32 path = f32(f64(sum_f32)/n) */
double orc_mean_abs_f32(const float *a, uint64_t n) {
  float *t = malloc(n * sizeof(float));
  for (uint64_t i = 0; i < n; i++) t[i] = fabsf(a[i]);
  float s = pw_f32(t, n);
  free(t);
  return (double)(float)((double)s / (double)n);
}
double orc_mean_abs_f64(const double *a, uint64_t n) {
  double *t = malloc(n * sizeof(double));
  for (uint64_t i = 0; i < n; i++) t[i] = fabs(a[i]);
  double s = pw_f64(t, n);
  free(t);
  return s / (double)n;
}
uint64_t orc_count_nonzero_f64(const double *a, uint64_t n) {
  uint64_t c = 0;
  for (uint64_t i = 0; i < n; i++) c += a[i] != 0.0;
  return c;
}
uint64_t orc_count_nonzero_f32(const float *a, uint64_t n) {
  uint64_t c = 0;
  for (uint64_t i = 0; i < n; i++) c += a[i] != 0.0f;
  return c;
}
/* training.py:360: np.abs(g).reshape(N,-1).max(axis=1).mean() for fp32 g */
double orc_lbar_f32(const float *g, uint64_t N, uint64_t per) {
  float *m = malloc(N * sizeof(float));
  for (uint64_t s = 0; s < N; s++) {
    float mx = 0.0f;
    for (uint64_t i = 0; i < per; i++) { float v = fabsf(g[s * per + i]); if (v > mx) mx = v; }
    m[s] = mx;
  }
  float sum = pw_f32(m, N);
  free(m);
  return (double)(float)((double)sum / (double)N);
}
double orc_lbar_f64(const double *g, uint64_t N, uint64_t per) {
  double *m = malloc(N * sizeof(double));
  for (uint64_t s = 0; s < N; s++) {
    double mx = 0.0;
    for (uint64_t i = 0; i < per; i++) { double v = fabs(g[s * per + i]); if (v > mx) mx = v; }
    m[s] = mx;
  }
  double sum = pw_f64(m, N);
  free(m);
  return sum / (double)N;
}
