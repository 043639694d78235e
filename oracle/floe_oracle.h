/*
 * floe_oracle.h -- CPU restatement of the FloE reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This header and floe_oracle.c restate, in plain
 * C, the reference algorithms that the B200 path must match.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load the
 * resulting library (oracle/liboracle.so); the product never links it.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/proj/).  Parity of this restatement against the
 * reference itself is pinned two ways (tests/test_oracle_vs_ref.py and
 * tests/test_oracle_golden.py): bit-for-bit against oracle/_ref/libfloe_ref.so
 * (the reference core compiled from its own sources by oracle/Makefile) and
 * against the golden fixtures in tests/golden/ generated from that library.
 *
 * Floating-point discipline: compiled with -O2 -ffp-contract=off and no
 * -march flags, like the reference's default Release build, so every
 * product and sum rounds exactly as the reference's does.
 */
#ifndef FLOE_ORACLE_H
#define FLOE_ORACLE_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- core/rng: SplitMix64 counter streams (core/src/rng.cpp:12-64) ---- */
uint64_t fo_mix64(uint64_t x);
typedef struct {
  uint64_t state;
  uint64_t gamma;
  int has_spare;
  double spare;
} fo_rng;
void fo_rng_init(fo_rng *r, uint64_t seed, uint64_t stream);
uint64_t fo_rng_next(fo_rng *r);
double fo_rng_uniform(fo_rng *r);
double fo_rng_uniform_pos(fo_rng *r);
double fo_rng_normal(fo_rng *r);
uint64_t fo_rng_below(fo_rng *r, uint64_t n);

/* out[i] = (float)normal_i * scale for the first n normals of (seed, stream).
 * Parallel by SplitMix skip-ahead; bit-identical to the sequential stream. */
void fo_normals(uint64_t seed, uint64_t stream, float scale, size_t n,
                float *out, int threads);
/* gen_model's fill_gaussian (core/src/model.cpp:31-39): 64 logical shards,
 * shard s uses stream base+s, out[i] = sigma * normal. */
void fo_fill_gaussian(float *out, size_t n, uint64_t seed, uint64_t base_stream,
                      float sigma, int threads);
/* weight_stream (core/src/model.cpp:25-28) */
uint64_t fo_weight_stream(uint64_t layer, uint64_t kind, uint64_t expert);
/* token_input (core/src/model.cpp:76-81) */
void fo_token_input(uint64_t seed, uint64_t t, uint32_t d_hidden, float *out);

/* ---- core/io: IEEE binary16 (core/src/io.cpp:19-78) ---- */
uint16_t fo_f32_to_f16(float f);
float fo_f16_to_f32(uint16_t h);
void fo_f32_to_f16_array(const float *in, size_t n, uint16_t *out, int threads);
void fo_f16_to_f32_array(const uint16_t *in, size_t n, float *out);

/* ---- core/quant (core/src/quant.cpp) ---- */
size_t fo_packed_code_bytes(size_t n, unsigned bits);
/* returns 0, or -1 bad bits, -2 bad group, -3 non-finite input */
int fo_quantize(const float *x, size_t n, unsigned bits, uint32_t group_size,
                uint8_t *codes, uint16_t *scales, uint16_t *zeros, int threads);
uint32_t fo_get_code(const uint8_t *codes, unsigned bits, size_t i);
float fo_dequantize_at(const uint8_t *codes, const uint16_t *scales,
                       const uint16_t *zeros, unsigned bits,
                       uint32_t group_size, size_t i);
/* returns 0 or -1 on corrupt packing (validate_packing, quant.cpp:94-102) */
int fo_dequantize(const uint8_t *codes, const uint16_t *scales,
                  const uint16_t *zeros, size_t n, unsigned bits,
                  uint32_t group_size, float *out, int threads);
/* qgemv_channels (quant.cpp:122-136): bit-equal sequential sums per channel;
 * threads split channels only.  returns 0 or -1 if ch_len does not divide n */
int fo_qgemv_channels(const uint8_t *codes, const uint16_t *scales,
                      const uint16_t *zeros, size_t n, unsigned bits,
                      uint32_t group_size, size_t ch_len, const float *x,
                      float *y, int threads);
double fo_compression_ratio(size_t d_hidden, size_t d_intermediate,
                            unsigned bits, uint32_t group_size,
                            double hot_density, int include_metadata);

/* ---- core/la (core/src/la.cpp) ---- */
void fo_gemv(size_t rows, size_t cols, const float *a, const float *x,
             float *y);
float fo_dot_f32(const float *a, const float *b, size_t n);
float fo_silu(float x);
void fo_softmax_inplace(float *v, size_t n);
/* top_k (la.cpp:48-61): ties toward the lower index, output ascending.
 * returns 0 or -1 if k out of range */
int fo_top_k(const float *v, size_t n, size_t k, uint32_t *out);

/* ---- core/sparsify (core/src/sparsify.cpp) ---- */
void fo_sparsity_mask(const float *v, size_t n, float t, uint8_t *mask);
/* calibrate_threshold (sparsify.cpp:42-54); sorts `mags` in place */
float fo_calibrate_threshold(float *mags, size_t n, double k);

/* ---- core/model ---- */
/* expert_forward_sparse(const CompressedExpert&, const Vec&)
 * (core/src/model.cpp:128-142).  gate/down_t are f32, channel-major
 * [di][dh].  v_out / mask_out optional (NULL).  threads only parallelise the
 * qgemv stage (per-channel order is unchanged, so results are identical). */
void fo_expert_forward_sparse(uint32_t dh, uint32_t di, unsigned bits,
                              uint32_t group_size, const uint8_t *codes,
                              const uint16_t *scales, const uint16_t *zeros,
                              const float *gate, const float *down_t,
                              float threshold, const float *x, float *y,
                              float *v_out, uint8_t *mask_out, int threads);
/* expert_forward over float weights (model.cpp:95-107) */
void fo_expert_forward_dense(uint32_t dh, uint32_t di, const float *gate,
                             const float *up, const float *down_t,
                             const float *x, float *y);
/* route (model.cpp:83-93). returns 0 or -1 */
int fo_route(const float *router, uint32_t experts, uint32_t dh,
             const float *u, uint32_t top_k, uint32_t *sel, float *weights);

/* One compressed MoE block (block_forward + layer_forward(CompressedModel),
 * model.cpp:145-169,182-190).  experts are described by parallel pointer
 * arrays of length n_experts; u_out (block input), sel/weights (routing) and
 * masks (top_k x di) are optional trace outputs (layer_forward_traced,
 * model.cpp:192-208). */
typedef struct {
  uint32_t d_hidden, d_intermediate, n_experts, top_k;
  unsigned bits;
  uint32_t group_size;
  const float *router; /* [E][dh] */
  const float *mixing; /* [dh][dh] */
  const uint8_t *const *codes;
  const uint16_t *const *scales;
  const uint16_t *const *zeros;
  const float *const *gate;
  const float *const *down_t;
  const float *thresholds; /* [E] */
} fo_layer;
int fo_layer_forward(const fo_layer *L, const float *h, float *y, float *u_out,
                     uint32_t *sel, float *weights, uint8_t *masks,
                     int threads);

/* ---- core/predictor ---- */
/* predict_mask (core/src/predictor.cpp:179-189) */
int fo_predict_mask(const uint8_t *codes, const uint16_t *scales,
                    const uint16_t *zeros, size_t n, unsigned bits,
                    uint32_t group_size, uint32_t d_hidden,
                    const float *x_prev, float t, uint8_t *mask, int threads);
/* predict_experts (predictor.cpp:164-177): scores = W x + b, top_k */
int fo_predict_experts(const float *w, const float *b, uint32_t experts,
                       uint32_t d_hidden, const float *x,
                       uint32_t prefetch_count, uint32_t *out);

/* ---- core/offload ---- */
/* pack_compact (core/src/offload.cpp:27-53).  Writes ascending kept channel
 * ids to channels[] and records of 2*dh elements (gate ‖ down) to payload
 * (f16 when element_bytes == 2, raw f32 when 4).  Returns #channels, or -1. */
long fo_pack_compact(uint32_t dh, uint32_t di, const float *gate,
                     const float *down_t, const uint8_t *mask,
                     uint32_t element_bytes, uint32_t *channels,
                     uint8_t *payload);
uint64_t fo_channel_record_bytes(uint32_t d_hidden, uint32_t element_bytes);

#ifdef __cplusplus
}
#endif
#endif
