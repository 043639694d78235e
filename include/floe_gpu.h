/*
 * floe_gpu.h -- C ABI of the B200-native FloE compressed-expert FFN path.
 *
 * This is the drop-in boundary.  Everything here is plain C: raw pointers,
 * sizes, status codes, opaque handles.  No torch or C++ types cross it.  The
 * C++ header include/floe_b200.hpp restores the reference's value-type API
 * (floe::expert_forward_sparse, floe::layer_forward, floe::predict_mask,
 * floe::predict_experts, floe::qgemv_channels) on top of these calls, and
 * INTEGRATION.md shows the bindings a reference maintainer would add.
 *
 * Reference interfaces each entry point replaces (paths relative to
 * /root/reference/proj/):
 *   floe_gpu_expert_create          CompressedExpert construction/upload:
 *                                   compress_expert   core/src/model.cpp:210-220
 *                                   load_compressed   core/src/model.cpp:434-474
 *   floe_gpu_expert_forward_sparse  Vec expert_forward_sparse(const CompressedExpert&,
 *                                   const Vec&)       core/include/floe/model.hpp:111,
 *                                                     core/src/model.cpp:128-142
 *   floe_gpu_qgemv_channels         qgemv_channels    core/include/floe/quant.hpp:50-51,
 *                                                     core/src/quant.cpp:122-136
 *   floe_gpu_dequantize_up          dequantize        core/src/quant.cpp:111-120
 *   floe_gpu_predict_mask           predict_mask      core/include/floe/predictor.hpp:80-82,
 *                                                     core/src/predictor.cpp:179-189
 *   floe_gpu_predict_experts        predict_experts   core/include/floe/predictor.hpp:75-77,
 *                                                     core/src/predictor.cpp:164-177
 *   floe_gpu_layer_forward          layer_forward(CompressedModel) / layer_forward_traced
 *                                   core/include/floe/model.hpp:118,128-129,
 *                                   core/src/model.cpp:145-208
 *
 * Conventions
 *   - Every function returns FLOE_OK (0) or a nonzero floe_status.  The
 *     message of the last failure on the calling thread is returned by
 *     floe_gpu_last_error(); it keeps the reference's "<fn>: <reason>"
 *     prefixes (e.g. "expert_forward_sparse: dimension mismatch").
 *   - *_dev pointers are device pointers; *_host pointers are host memory.
 *   - Compute calls are stream-ordered on the cudaStream_t passed as `stream`
 *     (NULL = legacy default stream) and never synchronise the host, except
 *     the *_host convenience calls, which return host results.
 *   - Handles (experts, layers, predictors) are immutable after creation and
 *     may be read concurrently from several streams.  A workspace holds the
 *     per-call scratch (v, kept-channel lists, counters) and must not be used
 *     by two streams at the same time.
 *   - There is no CPU fallback: without a usable sm_100 device every compute
 *     call fails with FLOE_ERR_CUDA.
 *   - The fast path is one persistent grid (one CTA per SM) with grid-wide
 *     barriers, launched with programmatic dependent launch so consecutive
 *     calls overlap.  Do not run fast-path calls on two streams at the same
 *     time (their grids would compete for SMs; a barrier watchdog traps after
 *     4 s), or set FLOE_COOP=1 to launch cooperatively (no launch overlap).
 */
#ifndef FLOE_GPU_H
#define FLOE_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FLOE_GPU_ABI_VERSION 1

typedef enum floe_status {
  FLOE_OK = 0,
  FLOE_ERR_INVALID = 1,     /* argument/dimension error (reference: runtime_error) */
  FLOE_ERR_CUDA = 2,        /* CUDA runtime/launch failure or no sm_100 device */
  FLOE_ERR_OOM = 3,         /* device or pinned host allocation failed */
  FLOE_ERR_UNSUPPORTED = 4  /* valid but not implemented on this path */
} floe_status;

typedef void *floe_stream_t; /* a cudaStream_t */

typedef struct floe_gpu_expert floe_gpu_expert;
typedef struct floe_gpu_workspace floe_gpu_workspace;
typedef struct floe_gpu_layer floe_gpu_layer;
typedef struct floe_gpu_predictor floe_gpu_predictor;

/* Host view of one compressed expert: the fields of floe::CompressedExpert
 * (core/include/floe/model.hpp:60-70) as raw arrays.  At most one of
 * {gate_f32 + down_f32} or {records_f16} may be given; with neither, the
 * handle holds only the up projection (qgemv_channels / predict_mask /
 * dequantize_up on a bare QuantizedTensor) and forward calls fail:
 *   gate_f32 / down_f32: f32 [d_intermediate][d_hidden] channel-major, as the
 *       reference stores them; converted to f16 on the device with IEEE RNE
 *       (identical to floe::f32_to_f16, core/src/io.cpp:19-51).
 *   records_f16: the compact wire format of pack_compact(element_bytes=2)
 *       (core/src/offload.cpp:27-53) for ALL channels: [di][gate|down][dh]. */
typedef struct floe_expert_host_view {
  uint32_t d_hidden;
  uint32_t d_intermediate;
  uint32_t bits;       /* 1,2,3,4,8 (quant.cpp:11-14) */
  uint32_t group_size; /* must divide d_hidden*d_intermediate */
  const uint8_t *codes;   /* packed_code_bytes(n, bits) bytes, LE in-byte */
  const uint16_t *scales; /* f16 bit patterns, n/group_size */
  const uint16_t *zeros;  /* f16 bit patterns, n/group_size */
  const float *gate_f32;
  const float *down_f32;
  const uint16_t *records_f16;
  float threshold; /* keep channel c iff |v[c]| >= threshold (model.cpp:135) */
  uint32_t flags;  /* FLOE_VIEW_DEVICE: every pointer above is a device pointer */
} floe_expert_host_view;

#define FLOE_VIEW_DEVICE 1u
/* keep the gate|down records host-resident (pinned, mapped): the kernels
 * read the kept channels' records directly over PCIe (SURVEY config 3) */
#define FLOE_VIEW_HOST_RECORDS 2u

typedef struct floe_expert_info {
  uint32_t d_hidden, d_intermediate, bits, group_size;
  float threshold;
  uint64_t code_bytes;     /* packed up-projection codes */
  uint64_t meta_bytes;     /* f16 scales + zeros */
  uint64_t record_bytes;   /* one gate|down f16 channel record (4*d_hidden) */
  int fast_path;           /* 1 when the specialised sm_100a kernels apply */
} floe_expert_info;

/* ---------------------------------------------------------------- runtime */
const char *floe_gpu_last_error(void);
int floe_gpu_abi_version(void);
/* Device properties of the current device; fails if it is not sm_100. */
int floe_gpu_device_info(int *sm_count, int *cc_major, int *cc_minor,
                         size_t *total_mem);

/* Device memory and copies for callers that do not link the CUDA runtime
 * (the C++ value-type API, FFI bindings).  floe_gpu_copy is cudaMemcpyDefault
 * on `stream` followed by a synchronisation of that stream. */
int floe_gpu_device_malloc(void **ptr, size_t bytes);
int floe_gpu_device_free(void *ptr);
int floe_gpu_copy(void *dst, const void *src, size_t bytes, floe_stream_t stream);

/* ---------------------------------------------------------------- experts */
int floe_gpu_expert_create(const floe_expert_host_view *view,
                           floe_gpu_expert **out);
int floe_gpu_expert_destroy(floe_gpu_expert *e);
int floe_gpu_expert_info(const floe_gpu_expert *e, floe_expert_info *info);
/* Thresholds are per expert (ThresholdTable, core/src/model.cpp:237). */
int floe_gpu_expert_set_threshold(floe_gpu_expert *e, float threshold);
/* The quantized up projection in the reference packing (codes
 * ceil(n*bits/8) bytes, f16 scales / zeros n/g each; quant.hpp:20-31) and
 * the threshold, copied to host memory -- the inverse of expert_create's
 * upload (record-cache / FLOQ writers).  Synchronous. */
int floe_gpu_expert_download(const floe_gpu_expert *e, uint8_t *codes_host,
                             uint16_t *scales_host, uint16_t *zeros_host,
                             float *threshold);

/* Placement of an expert's gate|down records: resident = 1 -> HBM,
 * 0 -> pinned host memory read in place over PCIe by the kernels.  Stream
 * ordered on `stream` (copy, descriptor switch in the expert and in every
 * layer holding it, release of the old copy).  The host copy, once made, is
 * kept for later promotions.  Mirrors ExpertCache residency
 * (core/src/offload.cpp:89-159) at expert granularity. */
int floe_gpu_expert_set_resident(floe_gpu_expert *e, int resident, floe_stream_t stream);
int floe_gpu_expert_residency(const floe_gpu_expert *e, int *resident, uint64_t *device_bytes);

/* -------------------------------------------------------------- workspace */
/* Scratch for calls on experts of at most d_intermediate channels and
 * d_hidden inputs, up to max_slots experts per call (top_k for layers). */
int floe_gpu_workspace_create(uint32_t d_hidden, uint32_t d_intermediate,
                              uint32_t max_slots, floe_gpu_workspace **out);
int floe_gpu_workspace_destroy(floe_gpu_workspace *ws);

/* --------------------------------------------------------------- hot path */
/* y = expert_forward_sparse(e, x) (model.cpp:128-142):
 *   v = qgemv_channels(up_q, x); keep c iff |v[c]| >= threshold;
 *   y = sum_{kept c} silu(gate_c . x) * v[c] * down_c.
 * x_dev/y_dev: f32[d_hidden].  Optional outputs (NULL to skip):
 *   v_dev       f32[d_intermediate]   the up-projection activations
 *   mask_dev    u8 [d_intermediate]   sparsity_mask(v, threshold)
 *   kept_dev    u32[d_intermediate]   kept channel ids, UNORDERED
 *   n_kept_dev  u32[1]                number of kept channels          */
int floe_gpu_expert_forward_sparse(const floe_gpu_expert *e,
                                   floe_gpu_workspace *ws, const float *x_dev,
                                   float *y_dev, float *v_dev,
                                   uint8_t *mask_dev, uint32_t *kept_dev,
                                   uint32_t *n_kept_dev, floe_stream_t stream);

/* Same computation from/to HOST memory (the reference's value-type call):
 * copies x in through pinned staging, runs the path, copies y back and
 * synchronises `stream`.  v_host / mask_host optional. */
int floe_gpu_expert_forward_sparse_host(const floe_gpu_expert *e,
                                        floe_gpu_workspace *ws,
                                        const float *x_host, float *y_host,
                                        float *v_host, uint8_t *mask_host,
                                        floe_stream_t stream);

/* v = qgemv_channels(up_q, d_hidden, x) (quant.cpp:122-136). */
int floe_gpu_qgemv_channels(const floe_gpu_expert *e, floe_gpu_workspace *ws,
                            const float *x_dev, float *v_dev,
                            floe_stream_t stream);

/* Batched up projection (SURVEY config 4): v_dev[t][c] = qgemv_channels(up_q,
 * d_hidden, x_dev[t]) for n_tokens <= 64 tokens, x_dev [n_tokens][d_hidden],
 * v_dev [n_tokens][d_intermediate].  One pass over the codes on the tcgen05
 * tensor cores (exact integer group sums); fast-layout experts only
 * (FLOE_ERR_UNSUPPORTED otherwise).  A token with a non-finite x gets NaN. */
int floe_gpu_qgemv_channels_batched(const floe_gpu_expert *e, const float *x_dev,
                                    uint32_t n_tokens, float *v_dev, floe_stream_t stream);

/* Batched expert_forward_sparse (SURVEY config 4): y_dev[t] =
 * expert_forward_sparse(e, x_dev[t]) for n_tokens <= 64 tokens (model.cpp:128-142;
 * each token keeps its own channels, !(|v| < threshold)).  The up projection
 * runs once for the batch on the tensor cores, and the gate/down records of the
 * union of kept channels are read once.  x_dev [n][d_hidden], y_dev
 * [n][d_hidden], v_dev nullable [n][d_intermediate].  Fast-layout experts with
 * gate/down records only. */
int floe_gpu_expert_forward_batched(const floe_gpu_expert *e, const float *x_dev,
                                    uint32_t n_tokens, float *y_dev, float *v_dev,
                                    floe_stream_t stream);

/* expert_forward_sparse (model.cpp:128-142) for many tokens (config 5
 * prefill, large config-4 batches): y_dev[t] = expert_forward_sparse(e,
 * x_dev[t]), any n_tokens.  Three dense f16 tensor-core GEMMs with f32
 * accumulation after a power-of-two scale per token: the up projection with
 * x and the dequantized weights split into f16 hi + lo (v to ~22 bits: the
 * masks), the gate and down products with the f16-rounded activations and
 * SwiGLU coefficients against the f16 records; the per-token mask
 * !(|v| < threshold) is applied to the coefficients.  Reads the expert's codes
 * and records once per call.  Fast-layout experts with records. */
int floe_gpu_expert_forward_prefill(const floe_gpu_expert *e, const float *x_dev,
                                    uint32_t n_tokens, float *y_dev, floe_stream_t stream);

/* pack_compact (core/src/offload.cpp:27-53) on the device: the channels c with
 * mask_dev[c] != 0 in ascending order -> channels_dev [n] and their records,
 * f16 gate row | f16 down row (element_bytes 2: 4*d_hidden bytes each, the
 * wire format of the host-resident decode and of records_f16), into payload
 * (device or pinned, mapped host memory: the H2D/D2H wire path); *n_out_dev =
 * n.  element_bytes 4 is FLOE_ERR_UNSUPPORTED (the device keeps f16 records).
 * Byte-identical to the reference for element_bytes 2. */
int floe_gpu_pack_compact(const floe_gpu_expert *e, const uint8_t *mask_dev,
                          uint32_t element_bytes, uint32_t *channels_dev, uint8_t *payload,
                          uint32_t *n_out_dev, floe_stream_t stream);

/* out = dequantize(up_q) in f32, bit-exact with floe::dequantize. */
int floe_gpu_dequantize_up(const floe_gpu_expert *e, float *out_dev,
                           floe_stream_t stream);

/* Reuse predictor (predictor.cpp:179-189): mask = |qgemv(up_next, x_prev)| >= t
 * with an explicit threshold t.  Same optional outputs as forward. */
int floe_gpu_predict_mask(const floe_gpu_expert *next, floe_gpu_workspace *ws,
                          const float *x_prev_dev, float t, uint8_t *mask_dev,
                          uint32_t *kept_dev, uint32_t *n_kept_dev,
                          floe_stream_t stream);

/* ---------------------------------------------------------------- layers */
/* One compressed MoE block (floe::CompressedLayer + cfg.top_k).  router and
 * mixing are f32 row-major ([E][dh], [dh][dh]) as in the reference;
 * mixing_f16 != 0 stores the mixing matrix as f16 on the device (IEEE RNE),
 * halving its bytes.  `experts` are borrowed (not owned) and must outlive
 * the layer; all must share d_hidden/d_intermediate. */
typedef struct floe_layer_host_view {
  uint32_t d_hidden;
  uint32_t n_experts;
  uint32_t top_k;
  const float *router;
  const float *mixing;
  int mixing_f16;
  floe_gpu_expert *const *experts;
} floe_layer_host_view;

typedef struct floe_gpu_layer_trace {
  float *block_input_dev;   /* f32[d_hidden]  (u)                        */
  uint32_t *experts_dev;    /* u32[top_k]     ascending expert ids       */
  float *weights_dev;       /* f32[top_k]     softmax routing weights    */
  uint8_t *masks_dev;       /* u8[top_k][d_intermediate]                 */
} floe_gpu_layer_trace;

int floe_gpu_layer_create(const floe_layer_host_view *view,
                          floe_gpu_layer **out);
int floe_gpu_layer_destroy(floe_gpu_layer *l);
/* y = layer_forward(m, layer, h): u = h + mixing.h; route(router, u, top_k);
 * y = u + sum_j w_j * expert_forward_sparse(E_j, u).  trace may be NULL. */
int floe_gpu_layer_forward(const floe_gpu_layer *l, floe_gpu_workspace *ws,
                           const float *h_dev, float *y_dev,
                           const floe_gpu_layer_trace *trace,
                           floe_stream_t stream);

/* block_forward (model.cpp:145-169) for n_tokens tokens at once (SURVEY
 * configs 4 and 5): h_dev [n][dh] -> y_dev [n][dh].  The mixing matrix is
 * streamed once for up to 64 tokens, the tokens are routed and grouped by
 * expert on the device, and every routed expert runs over its tokens: up to
 * 4 tokens through floe_gpu_expert_forward_batched (one pass over its codes,
 * the union of the kept channels' records read once), more through
 * floe_gpu_expert_forward_prefill (tensor-core GEMMs).  With a workspace (`ws`
 * nullable: then always the batched path), batches of up to 10 tokens run
 * token by token through the fused layer kernel, which is faster there.
 * The experts run concurrently on up to 8 internal side streams (their up
 * projections first, in order on `stream`); the call joins them back into
 * `stream` before it returns.
 * Synchronises `stream` once (the per-expert token counts decide the
 * launches). */
int floe_gpu_layer_forward_batched(const floe_gpu_layer *l, floe_gpu_workspace *ws,
                                   const float *h_dev, uint32_t n_tokens, float *y_dev,
                                   floe_stream_t stream);

/* Host-buffer layer call (the reference's value-type layer_forward): h in,
 * y out, through pinned staging; synchronises `stream`. */
int floe_gpu_layer_forward_host(const floe_gpu_layer *l, floe_gpu_workspace *ws,
                                const float *h_host, float *y_host,
                                floe_stream_t stream);

/* ------------------------------------------------ host-resident decode */
/* Config 3 of SURVEY.md: a stack of layers whose experts' gate|down records
 * stay in pinned host memory (the kernels read kept channels of non-resident
 * experts over PCIe), with an LRU of whole experts in HBM under
 * `vram_budget` bytes, promoted from the routing of earlier tokens by copies
 * on a side stream (the reference's simulate_decode / ExpertCache,
 * core/src/offload.cpp:89-159,299-464, as a real engine).  decode runs one
 * token through every layer (h_dev -> y_dev) on `stream`. */
typedef struct floe_gpu_offload floe_gpu_offload;
typedef struct floe_offload_stats {
  uint64_t tokens;
  uint64_t records_from_hbm;     /* kept channel records served from resident experts */
  uint64_t records_over_pcie;    /* ... read in place from pinned host memory        */
  uint64_t record_bytes;         /* bytes per record (4 * d_hidden)                   */
  uint64_t up_bytes_per_expert;  /* codes + f16 meta, always resident in HBM          */
  uint64_t promotions, evictions, bytes_promoted;
  uint64_t device_record_bytes;  /* records resident in HBM now                       */
  /* DecodeTimeline (core/include/floe/offload.hpp:128-157) over the decoded
   * tokens.  demanded == from_cache + prefetch_used + sync; the bytes moved
   * (promotions + sync) == prefetch_used + prefetch_wasted + sync +
   * prefetch_pending (promotions not yet demanded or evicted).  Up projections
   * are HBM-resident (cache); a promotion is one prefetch batch. */
  uint64_t bytes_demanded, bytes_from_cache, bytes_prefetch_used, bytes_sync;
  uint64_t bytes_prefetch_wasted, bytes_prefetch_pending;
  uint64_t requests_up, requests_channel;
  /* predictor scores on the decode path (eval on; predictor.cpp:206-254):
   * reuse masks (predict_mask of layer l's experts from layer l-1's block
   * input) and, with a predictor attached, predict_experts sets. */
  double mask_precision, mask_recall;
  uint64_t mask_samples;
  double set_precision, set_recall;
  uint64_t set_samples;
} floe_offload_stats;
int floe_gpu_offload_create(floe_gpu_layer *const *layers, uint32_t n_layers,
                            uint64_t vram_budget, floe_gpu_offload **out);
int floe_gpu_offload_destroy(floe_gpu_offload *o);
int floe_gpu_offload_decode(floe_gpu_offload *o, floe_gpu_workspace *ws, const float *h_dev,
                            float *y_dev, floe_stream_t stream);
/* decode_replay: every layer l reads its own block input h_dev[l*d_hidden ..]
 * and writes y_dev[l*d_hidden ..] (replay of recorded hidden states,
 * predictor.cpp:60-85) -- same placement policy and accounting as decode. */
int floe_gpu_offload_decode_replay(floe_gpu_offload *o, floe_gpu_workspace *ws,
                                   const float *h_dev, float *y_dev, floe_stream_t stream);
int floe_gpu_offload_stats(floe_gpu_offload *o, floe_offload_stats *out, floe_stream_t stream);
/* Score the predictors on the decode path (reuse masks always; expert sets
 * when `predictor` is non-NULL, top `count` of W x + b).  Adds one K1-only
 * pass over a layer's experts per layer (replaces
 * predictor.cpp:reuse_mask_metrics / eval_sets offline scoring). */
int floe_gpu_offload_set_eval(floe_gpu_offload *o, int enable, const floe_gpu_predictor *predictor,
                              uint32_t count);

/* ------------------------------------------------------ record-cache file */
/* The device-friendly counterpart of FLOQ (load_compressed,
 * core/src/model.cpp:414-474, which stores gate/down as f32: 488 MB per
 * Mixtral expert): "FLOR" keeps the up projection in the reference packing
 * and every channel's gate|down record in the f16 pack_compact wire format
 * (offload.cpp:27-53), 253 MB per expert, uploaded as-is.  Little-endian,
 * every section 64-B aligned:
 *   header (64 B): "FLOR", u32 version = 1, layers, experts, top_k, d_hidden,
 *                  d_intermediate, bits, group_size, mixing_f16, 6 x u32 0
 *   per layer:  router f32[E*dh]; mixing (f16 if mixing_f16 else f32)[dh*dh]
 *   per expert: 64 B {f32 threshold, 15 x u32 0}; codes; f16 scales[n/g];
 *               f16 zeros[n/g]; f16 records[di][2*dh]
 * load creates the experts (flags: FLOE_VIEW_HOST_RECORDS keeps the records
 * in pinned host memory, config 3) and the layers; the caller owns both and
 * destroys the layers before the experts. */
typedef struct floe_record_cache_info {
  uint32_t layers, experts, top_k, d_hidden, d_intermediate, bits, group_size, mixing_f16;
  uint64_t file_bytes;
} floe_record_cache_info;
int floe_gpu_record_cache_save(floe_gpu_layer *const *layers, uint32_t n_layers,
                               const char *path);
int floe_gpu_record_cache_info(const char *path, floe_record_cache_info *info);
int floe_gpu_record_cache_load(const char *path, uint32_t flags,
                               floe_gpu_layer **layers_out,
                               floe_gpu_expert **experts_out);

/* ----------------------------------------------------- counters / profile */
/* Device-side running totals kept by a workspace: calls (K1 launches) and
 * kept channels summed over all slots -- the byte-accounting identity
 * bytes = calls*(codes+meta) + kept*record_bytes uses them.  Stream-ordered
 * reset; the read synchronises `stream`. */
int floe_gpu_workspace_reset_counters(floe_gpu_workspace *ws, floe_stream_t stream);
int floe_gpu_workspace_read_counters(floe_gpu_workspace *ws, uint64_t *calls,
                                     uint64_t *kept_total, floe_stream_t stream);
/* Per-stage CUDA-event timing: when enabled, forward calls record an event
 * before and after every kernel on the launching stream and accumulate the
 * elapsed device time per stage.  Stages: 0 mixing, 1 route, 2 K1 (up GEMV +
 * threshold), 3 K2 (gate/down), 4 the fused persistent kernel (whole
 * expert/layer call in one launch).  read synchronises; ms[5], launches[5]. */
int floe_gpu_workspace_set_profiling(floe_gpu_workspace *ws, int enable);
int floe_gpu_workspace_read_profile(floe_gpu_workspace *ws, double *ms,
                                    uint64_t *launches);

/* Diagnostics: per-CTA %globaltimer marks of the fused kernel's phases
 * (0 start, 1 mixing done, 2 routed, 3 K1 done, 4 after barrier, 5 K2 done),
 * 8 u64 slots per CTA.  read copies min(cap, grid*8) values and synchronises. */
int floe_gpu_workspace_set_phase_trace(floe_gpu_workspace *ws, int enable);
int floe_gpu_workspace_read_phase_trace(floe_gpu_workspace *ws, uint64_t *out, uint32_t cap,
                                        uint32_t *grid);

/* ----------------------------------------------------------------- models */
/* A stack of HBM-resident compressed layers (floe::CompressedModel) decoded
 * token by token: the reference's `run` loop, h = layer_forward(m, l, h) for
 * l = 0..L-1 (tools/cli.cpp:86-107).  Layers are borrowed. */
typedef struct floe_gpu_model floe_gpu_model;
int floe_gpu_model_create(floe_gpu_layer *const *layers, uint32_t n_layers,
                          floe_gpu_model **out);
int floe_gpu_model_destroy(floe_gpu_model *m);
/* replay == 0: h_dev [dh] through every layer into y_dev [dh].
 * replay != 0: layer l reads h_dev[l*dh ..] and writes y_dev[l*dh ..] (the
 * recorded block inputs of predictor.cpp:60-85); each layer still waits for
 * the previous one, as a chained decode does.  Stream-ordered. */
int floe_gpu_model_decode(floe_gpu_model *m, floe_gpu_workspace *ws, const float *h_dev,
                          float *y_dev, int replay, floe_stream_t stream);
/* 1 if decode runs every layer of a token in ONE launch of the multi-layer
 * kernel (fast-path layers of one shape, f16 mixing, <= 8 experts; FLOE_MULTI=0
 * turns it off), 0 if it launches the fused kernel once per layer. */
int floe_gpu_model_multi_layer(const floe_gpu_model *m);
/* The same from/to HOST memory through pinned staging; synchronises `stream`. */
int floe_gpu_model_decode_host(floe_gpu_model *m, floe_gpu_workspace *ws, const float *h_host,
                               float *y_host, int replay, floe_stream_t stream);

/* ------------------------------------------------------------ calibration */
/* Threshold calibration on the device, bit-exact with the reference's
 * collect_stats + calibrate_model (core/src/model.cpp:242-330) and
 * SampleReservoir / calibrate / calibrate_threshold
 * (core/src/sparsify.cpp:42-64,128-142).  A run keeps one reservoir per
 * (layer, expert): SampleReservoir(sample_cap, seed ^ 0x5eedca11,
 * layer*experts + expert); `seed` is collect_stats' seed (the calibration
 * token stream's).  The caller drives the layers (the float model of a
 * Mixtral stack does not fit in HBM at once): for each layer, calib_layer runs
 * the DENSE float layer over the tokens' block inputs and returns the next
 * layer's inputs, exactly as collect_stats chains them. */
typedef struct floe_gpu_calib floe_gpu_calib;
typedef struct floe_float_layer_view { /* f32 DEVICE pointers, reference layouts */
  const float *router;        /* [E][dh] row-major                         */
  const float *mixing;        /* [dh][dh] row-major                        */
  const float *const *gate;   /* host array of E device pointers, [di][dh] */
  const float *const *up;     /* channel-major (ExpertWeights::gate/up)    */
  const float *const *down_t; /* [di][dh] (ExpertWeights::down_t)          */
} floe_float_layer_view;
int floe_gpu_calib_create(uint32_t layers, uint32_t experts, uint32_t d_hidden,
                          uint32_t d_intermediate, uint64_t seed, uint64_t sample_cap,
                          floe_gpu_calib **out);
int floe_gpu_calib_destroy(floe_gpu_calib *c);
/* One layer of collect_stats over `tokens` block inputs h_dev [tokens][dh]
 * (in token-stream order): u = h + drift_scale*mixing h, route, and for every
 * routed expert the dense SwiGLU forward; |up_c . u| of every channel goes to
 * the (layer, expert) reservoir in token order; h_next_dev [tokens][dh]
 * (nullable) receives the layer outputs.  Several calls per layer append in
 * call order.  Synchronises `stream` once (routing readback). */
int floe_gpu_calib_layer(floe_gpu_calib *c, uint32_t layer, const floe_float_layer_view *w,
                         uint32_t top_k, float drift_scale, const float *h_dev,
                         float *h_next_dev, uint32_t tokens, floe_stream_t stream);
/* calibrate(samples, k): thresholds_host[layer*E + expert] (host, L*E floats).
 * Fails with "calibrate: no samples for layer L expert E" like the reference
 * when an expert was never routed (k > 0). */
int floe_gpu_calib_thresholds(floe_gpu_calib *c, double k, float *thresholds_host);

/* ------------------------------------------------------- synthetic model */
/* Reference random streams on the device (rng.cpp:12-64): out[i] =
 * sigma * (float)normal_i.  sharded = 1 reproduces gen_model's fill_gaussian
 * (model.cpp:31-39: 64 shards, shard s on stream base+s); sharded = 0 is one
 * sequential stream (acceptance_test.cpp seeded_expert / token_input).
 * Double-precision Box-Muller: equal to the host stream except for rare
 * last-ulp differences of the device libm (tests count them). */
int floe_gpu_gen_normals(uint64_t seed, uint64_t stream_id, uint64_t n, float sigma,
                         int sharded, float *out_dev, floe_stream_t stream);
/* quantize (quant.cpp:43-86) on the device, bit-exact: codes must hold
 * ceil(n*bits/8) bytes, scales/zeros n/group_size f16 patterns. */
int floe_gpu_quantize(const float *x_dev, uint64_t n, uint32_t bits,
                      uint32_t group_size, uint8_t *codes_dev,
                      uint16_t *scales_dev, uint16_t *zeros_dev,
                      floe_stream_t stream);

/* ------------------------------------------------------------- predictor */
/* InterExpertPredictor (predictor.hpp:20-33): maps w[target-1] (E x dh,
 * row-major) and biases b[target-1] (E) for targets 1..layers-1. */
int floe_gpu_predictor_create(uint32_t layers, uint32_t experts,
                              uint32_t d_hidden, const float *w_host,
                              const float *b_host, floe_gpu_predictor **out);
int floe_gpu_predictor_destroy(floe_gpu_predictor *p);
/* out_dev = predict_experts(p, x, layer, count): top_k of W x + b, ascending,
 * ties toward the lower index.  layer 0 is an error, as in the reference. */
int floe_gpu_predict_experts(const floe_gpu_predictor *p, const float *x_dev,
                             uint32_t layer, uint32_t count, uint32_t *out_dev,
                             floe_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* FLOE_GPU_H */
