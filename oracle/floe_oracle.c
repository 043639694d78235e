/*
 * floe_oracle.c -- CPU restatement of the FloE reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY (see floe_oracle.h).  Never linked by the product.
 * Reference paths are relative to /root/reference/proj/.
 */
#include "floe_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ------------------------------------------------------------------ */
/* tiny fork-join helper: split [0, n) into `threads` contiguous chunks  */

typedef void (*fo_task)(void *ctx, size_t begin, size_t end);
typedef struct {
  fo_task fn;
  void *ctx;
  size_t begin, end;
} fo_chunk;

static void *fo_chunk_main(void *p) {
  fo_chunk *c = (fo_chunk *)p;
  c->fn(c->ctx, c->begin, c->end);
  return NULL;
}

static void fo_parallel(size_t n, int threads, fo_task fn, void *ctx) {
  if (threads <= 1 || n < 2) {
    fn(ctx, 0, n);
    return;
  }
  if ((size_t)threads > n) threads = (int)n;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  fo_chunk ch[256];
  for (int t = 0; t < threads; ++t) {
    ch[t].fn = fn;
    ch[t].ctx = ctx;
    ch[t].begin = n * (size_t)t / (size_t)threads;
    ch[t].end = n * (size_t)(t + 1) / (size_t)threads;
  }
  for (int t = 1; t < threads; ++t)
    pthread_create(&tid[t], NULL, fo_chunk_main, &ch[t]);
  fo_chunk_main(&ch[0]);
  for (int t = 1; t < threads; ++t) pthread_join(tid[t], NULL);
}

/* ------------------------------------------------------------------ */
/* rng: core/src/rng.cpp:12-64                                          */

uint64_t fo_mix64(uint64_t x) { /* rng.cpp:12-17 */
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

void fo_rng_init(fo_rng *r, uint64_t seed, uint64_t stream) { /* rng.cpp:19-25 */
  r->gamma = fo_mix64(stream * 2 + 1) | 1ULL;
  r->state = fo_mix64(seed ^ fo_mix64(stream + 0x632BE59BD9B4E019ULL));
  r->has_spare = 0;
  r->spare = 0.0;
}

uint64_t fo_rng_next(fo_rng *r) { /* rng.cpp:27-30 */
  r->state += r->gamma;
  return fo_mix64(r->state);
}

double fo_rng_uniform(fo_rng *r) { /* rng.cpp:32-34 */
  return (double)(fo_rng_next(r) >> 11) * 0x1.0p-53;
}

double fo_rng_uniform_pos(fo_rng *r) { /* rng.cpp:36-38 */
  return ((double)(fo_rng_next(r) >> 11) + 0.5) * 0x1.0p-53;
}

/* Box-Muller pair from two consecutive draws (rng.cpp:40-52): cos first,
 * sin kept as the spare. */
static void fo_box_muller(uint64_t d1, uint64_t d2, double *c, double *s) {
  double u1 = ((double)(d1 >> 11) + 0.5) * 0x1.0p-53;
  double u2 = (double)(d2 >> 11) * 0x1.0p-53;
  double r = sqrt(-2.0 * log(u1));
  double theta = 2.0 * 3.14159265358979323846 * u2;
  *s = r * sin(theta);
  *c = r * cos(theta);
}

double fo_rng_normal(fo_rng *r) { /* rng.cpp:40-52 */
  if (r->has_spare) {
    r->has_spare = 0;
    return r->spare;
  }
  uint64_t d1 = fo_rng_next(r);
  uint64_t d2 = fo_rng_next(r);
  double c, s;
  fo_box_muller(d1, d2, &c, &s);
  r->spare = s;
  r->has_spare = 1;
  return c;
}

uint64_t fo_rng_below(fo_rng *r, uint64_t n) { /* rng.cpp:60-64 */
  return fo_rng_next(r) % n;
}

typedef struct {
  uint64_t state0, gamma;
  float scale;
  float *out;
  size_t n;
} fo_normals_ctx;

/* Normal i of a fresh stream belongs to Box-Muller pair p = i/2, which
 * consumes draws 2p+1 and 2p+2; the SplitMix state after m draws is
 * state0 + m*gamma, so any pair can be produced independently. */
static void fo_normals_task(void *p, size_t b, size_t e) {
  fo_normals_ctx *c = (fo_normals_ctx *)p;
  size_t p0 = b, p1 = e; /* pair range */
  for (size_t q = p0; q < p1; ++q) {
    uint64_t s1 = c->state0 + (uint64_t)(2 * q + 1) * c->gamma;
    uint64_t s2 = s1 + c->gamma;
    double cv, sv;
    fo_box_muller(fo_mix64(s1), fo_mix64(s2), &cv, &sv);
    size_t i = 2 * q;
    c->out[i] = (float)cv * c->scale;
    if (i + 1 < c->n) c->out[i + 1] = (float)sv * c->scale;
  }
}

void fo_normals(uint64_t seed, uint64_t stream, float scale, size_t n,
                float *out, int threads) {
  fo_rng r;
  fo_rng_init(&r, seed, stream);
  fo_normals_ctx c = {r.state, r.gamma, scale, out, n};
  size_t pairs = (n + 1) / 2;
  fo_parallel(pairs, threads, fo_normals_task, &c);
}

uint64_t fo_weight_stream(uint64_t layer, uint64_t kind, uint64_t expert) {
  return ((layer * 5 + kind) * 65536 + expert) * 64; /* model.cpp:25-28 */
}

typedef struct {
  float *out;
  size_t n;
  uint64_t seed, base;
  float sigma;
} fo_fill_ctx;

static void fo_fill_task(void *p, size_t b, size_t e) {
  fo_fill_ctx *c = (fo_fill_ctx *)p;
  for (size_t s = b; s < e; ++s) {
    size_t lo = c->n * s / 64, hi = c->n * (s + 1) / 64;
    fo_rng r;
    fo_rng_init(&r, c->seed, c->base + s);
    /* model.cpp:37: out[i] = sigma * rng.normal_f() */
    for (size_t i = lo; i < hi; ++i)
      c->out[i] = c->sigma * (float)fo_rng_normal(&r);
  }
}

void fo_fill_gaussian(float *out, size_t n, uint64_t seed, uint64_t base_stream,
                      float sigma, int threads) { /* model.cpp:31-39 */
  fo_fill_ctx c = {out, n, seed, base_stream, sigma};
  fo_parallel(64, threads, fo_fill_task, &c);
}

void fo_token_input(uint64_t seed, uint64_t t, uint32_t d_hidden, float *out) {
  fo_rng r; /* model.cpp:76-81, kTokenStreamBase = 1<<40 (model.cpp:23) */
  fo_rng_init(&r, seed, (1ULL << 40) + t);
  for (uint32_t i = 0; i < d_hidden; ++i) out[i] = (float)fo_rng_normal(&r);
}

/* ------------------------------------------------------------------ */
/* io: core/src/io.cpp:19-78                                            */

uint16_t fo_f32_to_f16(float f) { /* io.cpp:19-51 */
  uint32_t x;
  memcpy(&x, &f, 4);
  uint32_t sign = (x >> 16) & 0x8000u;
  uint32_t mant = x & 0x007FFFFFu;
  int exp = (int)((x >> 23) & 0xFF) - 127;
  if (exp == 128) {
    uint32_t m = mant ? 0x0200u | (mant >> 13) : 0u;
    return (uint16_t)(sign | 0x7C00u | m);
  }
  if (exp > 15) return (uint16_t)(sign | 0x7C00u);
  if (exp >= -14) {
    uint32_t half = ((uint32_t)(exp + 15) << 10) | (mant >> 13);
    uint32_t rem = mant & 0x1FFFu;
    if (rem > 0x1000u || (rem == 0x1000u && (half & 1u))) half++;
    return (uint16_t)(sign | half);
  }
  if (exp >= -25) {
    uint32_t m = mant | 0x00800000u;
    int drop = -exp - 1;
    uint32_t half = m >> drop;
    uint32_t rem = m & ((1u << drop) - 1);
    uint32_t tie = 1u << (drop - 1);
    if (rem > tie || (rem == tie && (half & 1u))) half++;
    return (uint16_t)(sign | half);
  }
  return (uint16_t)sign;
}

float fo_f16_to_f32(uint16_t h) { /* io.cpp:53-78 */
  uint32_t sign = ((uint32_t)h & 0x8000u) << 16;
  uint32_t exp = (h >> 10) & 0x1Fu;
  uint32_t mant = h & 0x3FFu;
  uint32_t out;
  if (exp == 0) {
    if (mant == 0) {
      out = sign;
    } else {
      int e = -1;
      do {
        mant <<= 1;
        e++;
      } while (!(mant & 0x400u));
      out = sign | ((uint32_t)(112 - e) << 23) | ((mant & 0x3FFu) << 13);
    }
  } else if (exp == 31) {
    out = sign | 0x7F800000u | (mant << 13);
  } else {
    out = sign | ((exp + 112) << 23) | (mant << 13);
  }
  float f;
  memcpy(&f, &out, 4);
  return f;
}

typedef struct {
  const float *in;
  uint16_t *out;
} fo_h_ctx;
static void fo_h_task(void *p, size_t b, size_t e) {
  fo_h_ctx *c = (fo_h_ctx *)p;
  for (size_t i = b; i < e; ++i) c->out[i] = fo_f32_to_f16(c->in[i]);
}
void fo_f32_to_f16_array(const float *in, size_t n, uint16_t *out, int threads) {
  fo_h_ctx c = {in, out};
  fo_parallel(n, threads, fo_h_task, &c);
}
void fo_f16_to_f32_array(const uint16_t *in, size_t n, float *out) {
  for (size_t i = 0; i < n; ++i) out[i] = fo_f16_to_f32(in[i]);
}

/* ------------------------------------------------------------------ */
/* quant: core/src/quant.cpp                                            */

static int fo_bits_ok(unsigned bits) { /* quant.cpp:11-14 */
  return bits == 1 || bits == 2 || bits == 3 || bits == 4 || bits == 8;
}

size_t fo_packed_code_bytes(size_t n, unsigned bits) { /* quant.cpp:16-18 */
  return (n * bits + 7) / 8;
}

static void fo_put_code(uint8_t *codes, unsigned bits, size_t i, uint32_t c) {
  size_t bit = i * bits; /* quant.cpp:27-33 */
  size_t idx = bit / 8, off = bit % 8;
  codes[idx] |= (uint8_t)(c << off);
  if (off + bits > 8) codes[idx + 1] |= (uint8_t)(c >> (8 - off));
}

uint32_t fo_get_code(const uint8_t *codes, unsigned bits, size_t i) {
  size_t bit = i * bits; /* quant.cpp:35-41 */
  size_t idx = bit / 8, off = bit % 8;
  uint32_t v = (uint32_t)codes[idx] >> off;
  if (off + bits > 8) v |= (uint32_t)codes[idx + 1] << (8 - off);
  return v & ((1u << bits) - 1);
}

typedef struct {
  const float *x;
  unsigned bits;
  uint32_t g;
  uint8_t *codes;
  uint16_t *scales, *zeros;
} fo_q_ctx;

/* One group of quantize (quant.cpp:59-84). */
static void fo_quant_groups(void *p, size_t gb, size_t ge) {
  fo_q_ctx *c = (fo_q_ctx *)p;
  const float levels = (float)((1u << c->bits) - 1);
  for (size_t g = gb; g < ge; ++g) {
    const float *src = c->x + g * c->g;
    float lo = src[0], hi = src[0];
    for (size_t k = 1; k < c->g; ++k) {
      lo = (src[k] < lo) ? src[k] : lo; /* std::min(lo, src[k]) */
      hi = (hi < src[k]) ? src[k] : hi; /* std::max(hi, src[k]) */
    }
    uint16_t zero16 = fo_f32_to_f16(lo);
    uint16_t scale16 = fo_f32_to_f16((hi - lo) / levels);
    if (fo_f16_to_f32(scale16) <= 0.0f) scale16 = fo_f32_to_f16(1.0f);
    c->zeros[g] = zero16;
    c->scales[g] = scale16;
    float zero = fo_f16_to_f32(zero16);
    float scale = fo_f16_to_f32(scale16);
    for (size_t k = 0; k < c->g; ++k) {
      float t = nearbyintf((src[k] - zero) / scale);
      float cl = t < 0.0f ? 0.0f : (levels < t ? levels : t); /* std::clamp */
      fo_put_code(c->codes, c->bits, g * c->g + k, (uint32_t)cl);
    }
  }
}

int fo_quantize(const float *x, size_t n, unsigned bits, uint32_t group_size,
                uint8_t *codes, uint16_t *scales, uint16_t *zeros, int threads) {
  if (!fo_bits_ok(bits)) return -1; /* quant.cpp:44 */
  if (group_size == 0 || n % group_size != 0) return -2; /* quant.cpp:45-46 */
  for (size_t i = 0; i < n; ++i)
    if (!isfinite(x[i])) return -3; /* quant.cpp:47-48 */
  memset(codes, 0, fo_packed_code_bytes(n, bits));
  fo_q_ctx c = {x, bits, group_size, codes, scales, zeros};
  /* Groups write disjoint code bytes only when a group ends on a byte
   * boundary; otherwise run sequentially (put_code ORs into shared bytes). */
  if (((size_t)group_size * bits) % 8 != 0) threads = 1;
  fo_parallel(n / group_size, threads, fo_quant_groups, &c);
  return 0;
}

float fo_dequantize_at(const uint8_t *codes, const uint16_t *scales,
                       const uint16_t *zeros, unsigned bits,
                       uint32_t group_size, size_t i) { /* quant.cpp:104-109 */
  size_t g = i / group_size;
  float scale = fo_f16_to_f32(scales[g]);
  float zero = fo_f16_to_f32(zeros[g]);
  return (float)fo_get_code(codes, bits, i) * scale + zero;
}

typedef struct {
  const uint8_t *codes;
  const uint16_t *scales, *zeros;
  unsigned bits;
  uint32_t g;
  float *out;
} fo_dq_ctx;
static void fo_dq_task(void *p, size_t b, size_t e) {
  fo_dq_ctx *c = (fo_dq_ctx *)p;
  for (size_t i = b; i < e; ++i)
    c->out[i] = fo_dequantize_at(c->codes, c->scales, c->zeros, c->bits, c->g, i);
}

int fo_dequantize(const uint8_t *codes, const uint16_t *scales,
                  const uint16_t *zeros, size_t n, unsigned bits,
                  uint32_t group_size, float *out, int threads) {
  size_t used = n * bits; /* validate_packing, quant.cpp:94-102 */
  size_t nb = fo_packed_code_bytes(n, bits);
  if (used % 8 != 0 && nb > 0) {
    uint8_t tail = codes[nb - 1] >> (used % 8);
    if (tail != 0) return -1;
  }
  fo_dq_ctx c = {codes, scales, zeros, bits, group_size, out};
  fo_parallel(n, threads, fo_dq_task, &c);
  return 0;
}

typedef struct {
  const uint8_t *codes;
  const uint16_t *scales, *zeros;
  unsigned bits;
  uint32_t g;
  size_t ch_len;
  const float *x;
  float *y;
} fo_qg_ctx;

static void fo_qgemv_task(void *p, size_t cb, size_t ce) {
  fo_qg_ctx *c = (fo_qg_ctx *)p;
  for (size_t ch = cb; ch < ce; ++ch) { /* quant.cpp:128-135 */
    float acc = 0.0f;
    size_t base = ch * c->ch_len;
    for (size_t k = 0; k < c->ch_len; ++k) {
      float w = fo_dequantize_at(c->codes, c->scales, c->zeros, c->bits, c->g,
                                 base + k);
      acc += w * c->x[k];
    }
    c->y[ch] = acc;
  }
}

/* Fast path for byte-aligned groups: identical arithmetic, the f16
 * metadata decoded once per group instead of once per element. */
static void fo_qgemv_task_fast(void *p, size_t cb, size_t ce) {
  fo_qg_ctx *c = (fo_qg_ctx *)p;
  const unsigned bits = c->bits;
  const uint32_t mask = (1u << bits) - 1;
  for (size_t ch = cb; ch < ce; ++ch) {
    float acc = 0.0f;
    size_t base = ch * c->ch_len;
    for (size_t k0 = 0; k0 < c->ch_len; k0 += c->g) {
      size_t i0 = base + k0;
      size_t gi = i0 / c->g;
      float scale = fo_f16_to_f32(c->scales[gi]);
      float zero = fo_f16_to_f32(c->zeros[gi]);
      for (size_t k = 0; k < c->g; ++k) {
        size_t bit = (i0 + k) * bits;
        uint32_t code = ((uint32_t)c->codes[bit >> 3] >> (bit & 7)) & mask;
        float w = (float)code * scale + zero;
        acc += w * c->x[k0 + k];
      }
    }
    c->y[ch] = acc;
  }
}

int fo_qgemv_channels(const uint8_t *codes, const uint16_t *scales,
                      const uint16_t *zeros, size_t n, unsigned bits,
                      uint32_t group_size, size_t ch_len, const float *x,
                      float *y, int threads) {
  if (ch_len == 0 || n % ch_len != 0) return -1; /* quant.cpp:124-125 */
  fo_qg_ctx c = {codes, scales, zeros, bits, group_size, ch_len, x, y};
  int fast = (bits == 1 || bits == 2 || bits == 4 || bits == 8) &&
             ch_len % group_size == 0;
  fo_parallel(n / ch_len, threads, fast ? fo_qgemv_task_fast : fo_qgemv_task,
              &c);
  return 0;
}

double fo_compression_ratio(size_t d_hidden, size_t d_intermediate,
                            unsigned bits, uint32_t group_size,
                            double hot_density, int include_metadata) {
  size_t n = d_hidden * d_intermediate; /* quant.cpp:138-152 */
  double dense = 3.0 * (double)n * 2.0;
  double compressed = (double)fo_packed_code_bytes(n, bits);
  if (include_metadata) compressed += 4.0 * (double)(n / group_size);
  double hot = (double)llround(hot_density * (double)d_intermediate);
  compressed += 2.0 * hot * (double)d_hidden * 2.0;
  return dense / compressed;
}

/* ------------------------------------------------------------------ */
/* la: core/src/la.cpp                                                  */

void fo_gemv(size_t rows, size_t cols, const float *a, const float *x,
             float *y) { /* la.cpp:10-17 */
  for (size_t r = 0; r < rows; ++r) {
    const float *row = a + r * cols;
    float acc = 0.0f;
    for (size_t c = 0; c < cols; ++c) acc += row[c] * x[c];
    y[r] = acc;
  }
}

float fo_dot_f32(const float *a, const float *b, size_t n) { /* la.cpp:25-29 */
  float acc = 0.0f;
  for (size_t i = 0; i < n; ++i) acc += a[i] * b[i];
  return acc;
}

float fo_silu(float x) { return x / (1.0f + expf(-x)); } /* la.cpp:31 */

void fo_softmax_inplace(float *v, size_t n) { /* la.cpp:37-46 */
  if (n == 0) return;
  float mx = v[0];
  for (size_t i = 1; i < n; ++i)
    if (mx < v[i]) mx = v[i]; /* std::max_element keeps the first max */
  float sum = 0.0f;
  for (size_t i = 0; i < n; ++i) {
    v[i] = expf(v[i] - mx);
    sum += v[i];
  }
  for (size_t i = 0; i < n; ++i) v[i] /= sum;
}

static int fo_better(const float *v, uint32_t a, uint32_t b) {
  if (v[a] != v[b]) return v[a] > v[b]; /* la.cpp:52-55 */
  return a < b;
}

int fo_top_k(const float *v, size_t n, size_t k, uint32_t *out) {
  if (k == 0 || k > n) return -1; /* la.cpp:49 */
  /* k selection rounds under the same strict order partial_sort uses. */
  uint8_t *taken = (uint8_t *)calloc(n, 1);
  for (size_t r = 0; r < k; ++r) {
    uint32_t best = 0;
    int have = 0;
    for (uint32_t i = 0; i < n; ++i) {
      if (taken[i]) continue;
      if (!have || fo_better(v, i, best)) {
        best = i;
        have = 1;
      }
    }
    taken[best] = 1;
    out[r] = best;
  }
  free(taken);
  /* ascending index order (la.cpp:59) */
  for (size_t i = 1; i < k; ++i)
    for (size_t j = i; j > 0 && out[j - 1] > out[j]; --j) {
      uint32_t t = out[j];
      out[j] = out[j - 1];
      out[j - 1] = t;
    }
  return 0;
}

/* ------------------------------------------------------------------ */
/* sparsify: core/src/sparsify.cpp                                      */

void fo_sparsity_mask(const float *v, size_t n, float t, uint8_t *mask) {
  for (size_t i = 0; i < n; ++i) /* sparsify.cpp:11-17 */
    mask[i] = fabsf(v[i]) >= t ? 1 : 0;
}

static int fo_cmp_float(const void *a, const void *b) {
  float x = *(const float *)a, y = *(const float *)b;
  return (x > y) - (x < y);
}

float fo_calibrate_threshold(float *mags, size_t n, double k) {
  if (k < 0.0 || k > 1.0) return NAN; /* sparsify.cpp:42-54 */
  if (k == 0.0) return 0.0f;
  if (n == 0) return NAN;
  qsort(mags, n, sizeof(float), fo_cmp_float);
  size_t rank = (size_t)ceil(k * (double)n);
  if (rank == 0) rank = 1;
  if (rank > n) rank = n;
  return mags[rank - 1];
}

/* ------------------------------------------------------------------ */
/* model: core/src/model.cpp                                            */

void fo_expert_forward_sparse(uint32_t dh, uint32_t di, unsigned bits,
                              uint32_t group_size, const uint8_t *codes,
                              const uint16_t *scales, const uint16_t *zeros,
                              const float *gate, const float *down_t,
                              float threshold, const float *x, float *y,
                              float *v_out, uint8_t *mask_out, int threads) {
  /* model.cpp:128-142 */
  size_t n = (size_t)dh * di;
  float *v = v_out ? v_out : (float *)malloc(sizeof(float) * di);
  fo_qgemv_channels(codes, scales, zeros, n, bits, group_size, dh, x, v,
                    threads);
  for (uint32_t j = 0; j < dh; ++j) y[j] = 0.0f;
  for (uint32_t i = 0; i < di; ++i) {
    int keep = !(fabsf(v[i]) < threshold); /* model.cpp:135 */
    if (mask_out) mask_out[i] = (uint8_t)keep;
    if (!keep) continue;
    float g = fo_silu(fo_dot_f32(gate + (size_t)i * dh, x, dh));
    float a = g * v[i];
    const float *d = down_t + (size_t)i * dh;
    for (uint32_t j = 0; j < dh; ++j) y[j] += a * d[j];
  }
  if (!v_out) free(v);
}

void fo_expert_forward_dense(uint32_t dh, uint32_t di, const float *gate,
                             const float *up, const float *down_t,
                             const float *x, float *y) { /* model.cpp:95-107 */
  for (uint32_t j = 0; j < dh; ++j) y[j] = 0.0f;
  for (uint32_t i = 0; i < di; ++i) {
    float g = fo_silu(fo_dot_f32(gate + (size_t)i * dh, x, dh));
    float v = fo_dot_f32(up + (size_t)i * dh, x, dh);
    float a = g * v;
    const float *d = down_t + (size_t)i * dh;
    for (uint32_t j = 0; j < dh; ++j) y[j] += a * d[j];
  }
}

int fo_route(const float *router, uint32_t experts, uint32_t dh,
             const float *u, uint32_t top_k, uint32_t *sel, float *weights) {
  float logits[1024]; /* model.cpp:83-93 */
  if (experts > 1024) return -1;
  fo_gemv(experts, dh, router, u, logits);
  if (fo_top_k(logits, experts, top_k, sel) != 0) return -1;
  for (uint32_t i = 0; i < top_k; ++i) weights[i] = logits[sel[i]];
  fo_softmax_inplace(weights, top_k);
  return 0;
}

int fo_layer_forward(const fo_layer *L, const float *h, float *y, float *u_out,
                     uint32_t *sel_out, float *w_out, uint8_t *masks,
                     int threads) {
  /* block_forward (model.cpp:145-169) with drift_scale = 1 as used by
   * layer_forward(CompressedModel) (model.cpp:182-190). */
  const uint32_t dh = L->d_hidden, di = L->d_intermediate;
  float *mixed = (float *)malloc(sizeof(float) * dh);
  float *u = (float *)malloc(sizeof(float) * dh);
  float *out = (float *)malloc(sizeof(float) * dh);
  uint32_t sel[64];
  float w[64];
  if (L->top_k > 64) return -1;
  fo_gemv(dh, dh, L->mixing, h, mixed);
  const float drift = 1.0f;
  for (uint32_t i = 0; i < dh; ++i) u[i] = h[i] + drift * mixed[i];
  if (fo_route(L->router, L->n_experts, dh, u, L->top_k, sel, w) != 0) return -1;
  for (uint32_t i = 0; i < dh; ++i) y[i] = u[i];
  for (uint32_t j = 0; j < L->top_k; ++j) {
    uint32_t e = sel[j];
    fo_expert_forward_sparse(dh, di, L->bits, L->group_size, L->codes[e],
                             L->scales[e], L->zeros[e], L->gate[e],
                             L->down_t[e], L->thresholds[e], u, out, NULL,
                             masks ? masks + (size_t)j * di : NULL, threads);
    for (uint32_t i = 0; i < dh; ++i) y[i] += drift * w[j] * out[i];
  }
  if (u_out) memcpy(u_out, u, sizeof(float) * dh);
  if (sel_out) memcpy(sel_out, sel, sizeof(uint32_t) * L->top_k);
  if (w_out) memcpy(w_out, w, sizeof(float) * L->top_k);
  free(mixed);
  free(u);
  free(out);
  return 0;
}

/* ------------------------------------------------------------------ */
/* predictor: core/src/predictor.cpp                                    */

int fo_predict_mask(const uint8_t *codes, const uint16_t *scales,
                    const uint16_t *zeros, size_t n, unsigned bits,
                    uint32_t group_size, uint32_t d_hidden,
                    const float *x_prev, float t, uint8_t *mask, int threads) {
  if (d_hidden == 0 || n % d_hidden != 0) return -1; /* predictor.cpp:179-189 */
  size_t ch = n / d_hidden;
  float *v = (float *)malloc(sizeof(float) * ch);
  fo_qgemv_channels(codes, scales, zeros, n, bits, group_size, d_hidden, x_prev,
                    v, threads);
  fo_sparsity_mask(v, ch, t, mask);
  free(v);
  return 0;
}

int fo_predict_experts(const float *w, const float *b, uint32_t experts,
                       uint32_t d_hidden, const float *x,
                       uint32_t prefetch_count, uint32_t *out) {
  float scores[1024]; /* predictor.cpp:164-177 */
  if (experts > 1024) return -1;
  fo_gemv(experts, d_hidden, w, x, scores);
  for (uint32_t e = 0; e < experts; ++e) scores[e] += b[e];
  return fo_top_k(scores, experts, prefetch_count, out);
}

/* ------------------------------------------------------------------ */
/* offload: core/src/offload.cpp                                        */

uint64_t fo_channel_record_bytes(uint32_t d_hidden, uint32_t element_bytes) {
  return 2ull * d_hidden * element_bytes; /* offload.cpp:165-168 */
}

long fo_pack_compact(uint32_t dh, uint32_t di, const float *gate,
                     const float *down_t, const uint8_t *mask,
                     uint32_t element_bytes, uint32_t *channels,
                     uint8_t *payload) { /* offload.cpp:27-53 */
  if (element_bytes != 2 && element_bytes != 4) return -1;
  long nch = 0;
  uint8_t *w = payload;
  for (uint32_t i = 0; i < di; ++i) {
    if (!mask[i]) continue;
    channels[nch++] = i;
    const float *g = gate + (size_t)i * dh;
    const float *d = down_t + (size_t)i * dh;
    if (element_bytes == 4) {
      memcpy(w, g, 4u * dh); /* little-endian host, as ByteWriter::f32 */
      w += 4u * dh;
      memcpy(w, d, 4u * dh);
      w += 4u * dh;
    } else {
      for (uint32_t j = 0; j < dh; ++j) {
        uint16_t hv = fo_f32_to_f16(g[j]);
        *w++ = (uint8_t)hv;
        *w++ = (uint8_t)(hv >> 8);
      }
      for (uint32_t j = 0; j < dh; ++j) {
        uint16_t hv = fo_f32_to_f16(d[j]);
        *w++ = (uint8_t)hv;
        *w++ = (uint8_t)(hv >> 8);
      }
    }
  }
  return nch;
}
