// ref_shim.cpp -- extern "C" entry points over the UNMODIFIED reference core.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// the reference's own sources (/root/reference/proj/core/src/*.cpp, read in
// place, never copied) into oracle/_ref/libfloe_ref.so.  Python tests load it
// with ctypes to (a) pin the C restatement in oracle/floe_oracle.c bit for bit
// and (b) generate the golden fixtures in tests/golden/.  bench.py's
// cpu_baseline leg and `--impl reference` time the reference's own
// expert_forward_sparse / layer_forward through it.
//
// Every function only marshals plain buffers into the reference's value types
// and calls the reference API; no arithmetic lives here.

#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>
#include <thread>
#include <vector>

#include "floe/io.hpp"
#include "floe/la.hpp"
#include "floe/model.hpp"
#include "floe/offload.hpp"
#include "floe/predictor.hpp"
#include "floe/quant.hpp"
#include "floe/rng.hpp"
#include "floe/sparsify.hpp"

using namespace floe;

namespace {
thread_local std::string g_err;

template <typename F>
int guarded(F &&f) {
  try {
    f();
    return 0;
  } catch (const std::exception &e) {
    g_err = e.what();
    return -1;
  }
}

QuantizedTensor make_q(const std::uint8_t *codes, const std::uint16_t *scales,
                       const std::uint16_t *zeros, std::size_t n, unsigned bits,
                       std::uint32_t g) {
  QuantizedTensor q;
  q.n = n;
  q.bits = bits;
  q.group_size = g;
  q.codes.assign(codes, codes + packed_code_bytes(n, bits));
  q.scales.assign(scales, scales + n / g);
  q.zeros.assign(zeros, zeros + n / g);
  return q;
}
}  // namespace

extern "C" {

const char *ref_last_error() { return g_err.c_str(); }

// ---- rng / io ----
void ref_normals(std::uint64_t seed, std::uint64_t stream, std::size_t n,
                 float *out) {
  Rng r(seed, stream);
  for (std::size_t i = 0; i < n; ++i) out[i] = r.normal_f();
}

void ref_uniforms(std::uint64_t seed, std::uint64_t stream, std::size_t n,
                  double *out) {
  Rng r(seed, stream);
  for (std::size_t i = 0; i < n; ++i) out[i] = r.uniform();
}

// acceptance_test.cpp:38-53 / test_model.cpp:27-43 seeded_expert.
void ref_seeded_expert(std::uint32_t dh, std::uint32_t di, std::uint64_t seed,
                       float *gate, float *up, float *down) {
  const float sd = 1.0f / std::sqrt(static_cast<float>(dh));
  float *dst[3] = {gate, up, down};
  for (int s = 0; s < 3; ++s) {
    Rng rng(seed, static_cast<std::uint64_t>(s + 1));
    std::size_t n = static_cast<std::size_t>(dh) * di;
    for (std::size_t i = 0; i < n; ++i) dst[s][i] = rng.normal_f() * sd;
  }
}

void ref_token_input(std::uint64_t seed, std::uint64_t t, std::uint32_t dh,
                     float *out) {
  Vec x = token_input(seed, t, dh);
  std::memcpy(out, x.data(), sizeof(float) * dh);
}

void ref_f32_to_f16(const float *in, std::size_t n, std::uint16_t *out) {
  for (std::size_t i = 0; i < n; ++i) out[i] = f32_to_f16(in[i]);
}
void ref_f16_to_f32(const std::uint16_t *in, std::size_t n, float *out) {
  for (std::size_t i = 0; i < n; ++i) out[i] = f16_to_f32(in[i]);
}

// ---- quant ----
std::size_t ref_packed_code_bytes(std::size_t n, unsigned bits) {
  return packed_code_bytes(n, bits);
}

int ref_quantize(const float *x, std::size_t n, unsigned bits, std::uint32_t g,
                 std::uint8_t *codes, std::uint16_t *scales,
                 std::uint16_t *zeros) {
  return guarded([&] {
    QuantizedTensor q = quantize(x, n, bits, g);
    std::memcpy(codes, q.codes.data(), q.codes.size());
    std::memcpy(scales, q.scales.data(), 2 * q.scales.size());
    std::memcpy(zeros, q.zeros.data(), 2 * q.zeros.size());
  });
}

int ref_dequantize(const std::uint8_t *codes, const std::uint16_t *scales,
                   const std::uint16_t *zeros, std::size_t n, unsigned bits,
                   std::uint32_t g, float *out) {
  return guarded([&] {
    QuantizedTensor q = make_q(codes, scales, zeros, n, bits, g);
    dequantize(q, out);
  });
}

int ref_qgemv_channels(const std::uint8_t *codes, const std::uint16_t *scales,
                       const std::uint16_t *zeros, std::size_t n, unsigned bits,
                       std::uint32_t g, std::size_t ch_len, const float *x,
                       float *y) {
  return guarded([&] {
    QuantizedTensor q = make_q(codes, scales, zeros, n, bits, g);
    qgemv_channels(q, ch_len, x, y);
  });
}

double ref_compression_ratio(std::size_t dh, std::size_t di, unsigned bits,
                             std::uint32_t g, double hot, int meta) {
  return compression_ratio(dh, di, bits, g, hot, meta != 0);
}

// ---- la / sparsify ----
int ref_top_k(const float *v, std::size_t n, std::size_t k, std::uint32_t *out) {
  return guarded([&] {
    Vec vv(v, v + n);
    auto idx = top_k(vv, k);
    std::memcpy(out, idx.data(), sizeof(std::uint32_t) * idx.size());
  });
}

void ref_softmax(float *v, std::size_t n) {
  Vec vv(v, v + n);
  softmax_inplace(vv);
  std::memcpy(v, vv.data(), sizeof(float) * n);
}

float ref_silu(float x) { return silu(x); }

float ref_calibrate_threshold(const float *mags, std::size_t n, double k) {
  return calibrate_threshold(std::vector<float>(mags, mags + n), k);
}

int ref_route(const float *router, std::uint32_t experts, std::uint32_t dh,
              const float *u, std::uint32_t top_k_n, std::uint32_t *sel,
              float *w) {
  return guarded([&] {
    Matrix m(experts, dh);
    std::memcpy(m.data.data(), router, sizeof(float) * experts * dh);
    RouteResult r = route(m, Vec(u, u + dh), top_k_n);
    std::memcpy(sel, r.experts.data(), 4 * r.experts.size());
    std::memcpy(w, r.weights.data(), 4 * r.weights.size());
  });
}

// ---- compressed expert handles ----
void *ref_expert_create(std::uint32_t dh, std::uint32_t di, unsigned bits,
                        std::uint32_t g, const std::uint8_t *codes,
                        const std::uint16_t *scales, const std::uint16_t *zeros,
                        const float *gate, const float *down, float threshold) {
  auto *e = new CompressedExpert();
  std::size_t n = static_cast<std::size_t>(dh) * di;
  e->d_hidden = dh;
  e->d_intermediate = di;
  e->up_q = make_q(codes, scales, zeros, n, bits, g);
  e->gate.assign(gate, gate + n);
  e->down_t.assign(down, down + n);
  e->threshold = threshold;
  return e;
}

// compress_expert (model.cpp:210-220) straight from float weights.
void *ref_expert_compress(std::uint32_t dh, std::uint32_t di,
                          const float *gate, const float *up, const float *down,
                          unsigned bits, std::uint32_t g, float threshold) {
  ExpertWeights w;
  std::size_t n = static_cast<std::size_t>(dh) * di;
  w.d_hidden = dh;
  w.d_intermediate = di;
  w.gate.assign(gate, gate + n);
  w.up.assign(up, up + n);
  w.down_t.assign(down, down + n);
  try {
    return new CompressedExpert(compress_expert(w, bits, g, threshold));
  } catch (const std::exception &e) {
    g_err = e.what();
    return nullptr;
  }
}

void ref_expert_destroy(void *h) { delete static_cast<CompressedExpert *>(h); }

void ref_expert_set_threshold(void *h, float t) {
  static_cast<CompressedExpert *>(h)->threshold = t;
}

// Raw views into a handle (valid while the handle lives).
void ref_expert_view(void *h, const std::uint8_t **codes,
                     const std::uint16_t **scales, const std::uint16_t **zeros,
                     const float **gate, const float **down, float *threshold) {
  auto *e = static_cast<CompressedExpert *>(h);
  *codes = e->up_q.codes.data();
  *scales = e->up_q.scales.data();
  *zeros = e->up_q.zeros.data();
  *gate = e->gate.data();
  *down = e->down_t.data();
  *threshold = e->threshold;
}

int ref_expert_forward(void *h, const float *x, float *y) {
  return guarded([&] {
    auto *e = static_cast<CompressedExpert *>(h);
    Vec out = expert_forward_sparse(*e, Vec(x, x + e->d_hidden));
    std::memcpy(y, out.data(), sizeof(float) * out.size());
  });
}

// Replica throughput: `threads` host threads each run `iters` independent
// expert_forward_sparse calls on the shared read-only expert.  Returns the
// wall time in seconds (steady_clock), or a negative value on error.
double ref_expert_forward_replicas(void *h, const float *x, unsigned threads,
                                   unsigned iters) {
  auto *e = static_cast<CompressedExpert *>(h);
  Vec xv(x, x + e->d_hidden);
  std::vector<std::thread> pool;
  auto t0 = std::chrono::steady_clock::now();
  for (unsigned t = 0; t < threads; ++t)
    pool.emplace_back([&] {
      for (unsigned i = 0; i < iters; ++i) {
        Vec out = expert_forward_sparse(*e, xv);
        if (out.empty()) std::terminate();
      }
    });
  for (auto &t : pool) t.join();
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double>(t1 - t0).count();
}

int ref_expert_forward_dense(std::uint32_t dh, std::uint32_t di,
                             const float *gate, const float *up,
                             const float *down, const float *x, float *y) {
  return guarded([&] {
    ExpertWeights w;
    std::size_t n = static_cast<std::size_t>(dh) * di;
    w.d_hidden = dh;
    w.d_intermediate = di;
    w.gate.assign(gate, gate + n);
    w.up.assign(up, up + n);
    w.down_t.assign(down, down + n);
    Vec out = expert_forward(w, Vec(x, x + dh));
    std::memcpy(y, out.data(), sizeof(float) * dh);
  });
}

int ref_pack_compact(void *h, const std::uint8_t *mask, std::uint32_t eb,
                     std::uint32_t *channels, std::uint8_t *payload,
                     std::uint64_t *n_channels) {
  return guarded([&] {
    auto *e = static_cast<CompressedExpert *>(h);
    std::vector<std::uint8_t> m(mask, mask + e->d_intermediate);
    CompactSelection s = pack_compact(*e, m, eb);
    std::memcpy(channels, s.channels.data(), 4 * s.channels.size());
    std::memcpy(payload, s.payload.data(), s.payload.size());
    *n_channels = s.channels.size();
  });
}

int ref_predict_mask(const std::uint8_t *codes, const std::uint16_t *scales,
                     const std::uint16_t *zeros, std::size_t n, unsigned bits,
                     std::uint32_t g, std::uint32_t dh, const float *x_prev,
                     float t, std::uint8_t *mask) {
  return guarded([&] {
    QuantizedTensor q = make_q(codes, scales, zeros, n, bits, g);
    auto m = predict_mask(q, dh, Vec(x_prev, x_prev + dh), t);
    std::memcpy(mask, m.data(), m.size());
  });
}

// predict_experts through a one-target InterExpertPredictor (layers = 2).
int ref_predict_experts(const float *w, const float *b, std::uint32_t experts,
                        std::uint32_t dh, const float *x, std::uint32_t count,
                        std::uint32_t *out) {
  return guarded([&] {
    InterExpertPredictor p;
    p.layers = 2;
    p.experts = experts;
    p.d_hidden = dh;
    p.w.emplace_back(experts, dh);
    std::memcpy(p.w[0].data.data(), w, sizeof(float) * experts * dh);
    p.b.emplace_back(b, b + experts);
    auto sel = predict_experts(p, Vec(x, x + dh), 1, count);
    std::memcpy(out, sel.data(), 4 * sel.size());
  });
}

// ---- compressed models (gen_model -> calibrate_model -> compress_model) ----
void *ref_cmodel_build(std::uint32_t layers, std::uint32_t experts,
                       std::uint32_t top_k_n, std::uint32_t dh,
                       std::uint32_t di, std::uint64_t seed,
                       std::uint64_t calib_seed, std::uint64_t calib_tokens,
                       double k, unsigned bits, std::uint32_t g,
                       unsigned workers) {
  try {
    MoEConfig cfg;
    cfg.layers = layers;
    cfg.experts = experts;
    cfg.top_k = top_k_n;
    cfg.d_hidden = dh;
    cfg.d_intermediate = di;
    cfg.seed = seed;
    MoEModel m = gen_model(cfg, workers);
    ThresholdTable t =
        calibrate_model(m, calib_seed, calib_tokens, k, kReservoirCap, workers);
    return new CompressedModel(compress_model(m, t, bits, g));
  } catch (const std::exception &e) {
    g_err = e.what();
    return nullptr;
  }
}

// gen_model -> compress_model with a caller-supplied ThresholdTable (L*E
// thresholds), skipping calibrate_model's dense passes (bench setup).
void *ref_cmodel_build_thresholds(std::uint32_t layers, std::uint32_t experts,
                                  std::uint32_t top_k_n, std::uint32_t dh,
                                  std::uint32_t di, std::uint64_t seed,
                                  const float *thresholds, unsigned bits,
                                  std::uint32_t g, unsigned workers) {
  try {
    MoEConfig cfg;
    cfg.layers = layers;
    cfg.experts = experts;
    cfg.top_k = top_k_n;
    cfg.d_hidden = dh;
    cfg.d_intermediate = di;
    cfg.seed = seed;
    ThresholdTable t(layers, experts);
    for (std::uint32_t l = 0; l < layers; ++l)
      for (std::uint32_t e = 0; e < experts; ++e)
        t.set(l, e, thresholds[l * experts + e], 0.0f);
    CompressedModel *out = nullptr;
    {
      MoEModel m = gen_model(cfg, workers);
      out = new CompressedModel(compress_model(m, t, bits, g));
    }
    return out;
  } catch (const std::exception &e) {
    g_err = e.what();
    return nullptr;
  }
}

// gen_model(seed) with `layers` layers; every layer calibrated as a 1-layer
// model (calibrate_model on layer l's weights alone: the replayed block
// inputs the decode bench feeds each layer) -> compress_model.  The
// thresholds go to out[L*E].
void *ref_cmodel_build_replay(std::uint32_t layers, std::uint32_t experts, std::uint32_t top_k_n,
                              std::uint32_t dh, std::uint32_t di, std::uint64_t seed,
                              std::uint64_t calib_seed, std::uint64_t calib_tokens, double k,
                              unsigned bits, std::uint32_t g, unsigned workers, float *out) {
  try {
    MoEConfig cfg;
    cfg.layers = layers;
    cfg.experts = experts;
    cfg.top_k = top_k_n;
    cfg.d_hidden = dh;
    cfg.d_intermediate = di;
    cfg.seed = seed;
    MoEModel m = gen_model(cfg, workers);
    ThresholdTable t(layers, experts);
    for (std::uint32_t l = 0; l < layers; ++l) {
      MoEModel one;
      one.cfg = cfg;
      one.cfg.layers = 1;
      one.layers.push_back(std::move(m.layers[l]));
      ThresholdTable tl = calibrate_model(one, calib_seed, calib_tokens, k, kReservoirCap, workers);
      m.layers[l] = std::move(one.layers[0]);
      for (std::uint32_t e = 0; e < experts; ++e) {
        t.set(l, e, tl.at(0, e), static_cast<float>(k));
        out[l * experts + e] = tl.at(0, e);
      }
    }
    return new CompressedModel(compress_model(m, t, bits, g));
  } catch (const std::exception &e) {
    g_err = e.what();
    return nullptr;
  }
}

// calibrate_model (model.cpp:323-330) on a float model given as arrays:
// router [L][E][dh], mixing [L][dh][dh], gate/up/down_t [L][E][di][dh]; the
// thresholds go to out[L*E].  Returns 0 or -1 (ref_last_error).
int ref_calibrate_weights(std::uint32_t layers, std::uint32_t experts, std::uint32_t top_k_n,
                          std::uint32_t dh, std::uint32_t di, const float *router,
                          const float *mixing, const float *gate, const float *up,
                          const float *down, std::uint64_t calib_seed, std::uint64_t tokens,
                          double k, std::uint64_t cap, unsigned workers, float drift,
                          float *out) {
  return guarded([&] {
    MoEModel m;
    m.cfg.layers = layers;
    m.cfg.experts = experts;
    m.cfg.top_k = top_k_n;
    m.cfg.d_hidden = dh;
    m.cfg.d_intermediate = di;
    m.layers.resize(layers);
    const std::size_t n = (std::size_t)dh * di;
    for (std::uint32_t l = 0; l < layers; ++l) {
      MoELayer &L = m.layers[l];
      L.router = Matrix(experts, dh);
      std::memcpy(L.router.data.data(), router + (std::size_t)l * experts * dh,
                  sizeof(float) * experts * dh);
      L.mixing = Matrix(dh, dh);
      std::memcpy(L.mixing.data.data(), mixing + (std::size_t)l * dh * dh, sizeof(float) * dh * dh);
      for (std::uint32_t e = 0; e < experts; ++e) {
        ExpertWeights w;
        w.d_hidden = dh;
        w.d_intermediate = di;
        const std::size_t o = ((std::size_t)l * experts + e) * n;
        w.gate.assign(gate + o, gate + o + n);
        w.up.assign(up + o, up + o + n);
        w.down_t.assign(down + o, down + o + n);
        L.experts.push_back(std::move(w));
      }
    }
    ThresholdTable t = calibrate_model(m, calib_seed, tokens, k, cap, workers, drift);
    for (std::uint32_t l = 0; l < layers; ++l)
      for (std::uint32_t e = 0; e < experts; ++e) out[l * experts + e] = t.at(l, e);
  });
}

// Replica throughput of layer_forward(CompressedModel): `threads` host threads
// split n_tokens independent tokens (hs: n_tokens x dh) round-robin.  Returns
// wall seconds (steady_clock), negative on error.
double ref_layer_forward_replicas(void *cm, std::uint32_t layer, const float *hs,
                                  std::uint32_t n_tokens, unsigned threads) {
  auto *m = static_cast<CompressedModel *>(cm);
  const std::uint32_t dh = m->cfg.d_hidden;
  std::vector<std::thread> pool;
  bool failed = false;
  auto t0 = std::chrono::steady_clock::now();
  for (unsigned t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      try {
        for (std::uint32_t i = t; i < n_tokens; i += threads) {
          Vec out = layer_forward(*m, layer, Vec(hs + (std::size_t)i * dh,
                                                 hs + (std::size_t)(i + 1) * dh));
          if (out.size() != dh) failed = true;
        }
      } catch (...) {
        failed = true;
      }
    });
  for (auto &t : pool) t.join();
  auto t1 = std::chrono::steady_clock::now();
  return failed ? -1.0 : std::chrono::duration<double>(t1 - t0).count();
}

// `threads` host threads split n independent layer_forward calls: call i runs
// layer i % n_layers on input hs[i].  Returns wall seconds, negative on error.
double ref_layer_calls_replicas(void *cm, std::uint32_t n_layers, const float *hs,
                                std::uint32_t n, unsigned threads) {
  auto *m = static_cast<CompressedModel *>(cm);
  const std::uint32_t dh = m->cfg.d_hidden;
  std::vector<std::thread> pool;
  bool failed = false;
  auto t0 = std::chrono::steady_clock::now();
  for (unsigned t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      try {
        for (std::uint32_t i = t; i < n; i += threads) {
          Vec out = layer_forward(*m, i % n_layers,
                                  Vec(hs + (std::size_t)i * dh, hs + (std::size_t)(i + 1) * dh));
          if (out.size() != dh) failed = true;
        }
      } catch (...) {
        failed = true;
      }
    });
  for (auto &t : pool) t.join();
  auto t1 = std::chrono::steady_clock::now();
  return failed ? -1.0 : std::chrono::duration<double>(t1 - t0).count();
}

void *ref_cmodel_load(const char *path) {
  try {
    return new CompressedModel(load_compressed(path));
  } catch (const std::exception &e) {
    g_err = e.what();
    return nullptr;
  }
}

int ref_cmodel_save(void *cm, const char *path) {
  return guarded([&] { save_compressed(*static_cast<CompressedModel *>(cm), path); });
}

void ref_cmodel_destroy(void *cm) { delete static_cast<CompressedModel *>(cm); }

void ref_cmodel_dims(void *cm, std::uint32_t *out6, unsigned *bits,
                     std::uint32_t *g) {
  auto *m = static_cast<CompressedModel *>(cm);
  out6[0] = m->cfg.layers;
  out6[1] = m->cfg.experts;
  out6[2] = m->cfg.top_k;
  out6[3] = m->cfg.d_hidden;
  out6[4] = m->cfg.d_intermediate;
  out6[5] = static_cast<std::uint32_t>(m->cfg.seed);
  *bits = m->bits;
  *g = m->group_size;
}

void ref_cmodel_layer_view(void *cm, std::uint32_t layer, const float **router,
                           const float **mixing) {
  auto *m = static_cast<CompressedModel *>(cm);
  *router = m->layers[layer].router.data.data();
  *mixing = m->layers[layer].mixing.data.data();
}

void *ref_cmodel_expert(void *cm, std::uint32_t layer, std::uint32_t e) {
  auto *m = static_cast<CompressedModel *>(cm);
  return &m->layers[layer].experts[e];
}

int ref_layer_forward(void *cm, std::uint32_t layer, const float *h, float *y) {
  return guarded([&] {
    auto *m = static_cast<CompressedModel *>(cm);
    Vec out = layer_forward(*m, layer, Vec(h, h + m->cfg.d_hidden));
    std::memcpy(y, out.data(), sizeof(float) * out.size());
  });
}

// layer_forward_traced: u[dh], sel[top_k], w[top_k], masks[top_k][di], y[dh].
int ref_layer_forward_traced(void *cm, std::uint32_t layer, const float *h,
                             float *u, std::uint32_t *sel, float *w,
                             std::uint8_t *masks, float *y) {
  return guarded([&] {
    auto *m = static_cast<CompressedModel *>(cm);
    LayerTrace t = layer_forward_traced(*m, layer, Vec(h, h + m->cfg.d_hidden));
    std::memcpy(u, t.block_input.data(), 4 * t.block_input.size());
    std::memcpy(sel, t.experts.data(), 4 * t.experts.size());
    std::memcpy(w, t.weights.data(), 4 * t.weights.size());
    for (std::size_t j = 0; j < t.masks.size(); ++j)
      std::memcpy(masks + j * m->cfg.d_intermediate, t.masks[j].data(),
                  t.masks[j].size());
    std::memcpy(y, t.out.data(), 4 * t.out.size());
  });
}

}  // extern "C"
