// floe_b200.hpp -- the reference's value-type C++ API over the C ABI.
//
// A drop-in for the FloE hot path of the reference core (namespace floe,
// /root/reference/proj/core/include/floe/{quant,model,predictor}.hpp): the
// same function names, argument meaning and error behaviour
// (std::runtime_error with the reference's "<fn>: <reason>" messages), with
// the arithmetic running on the B200 through include/floe_gpu.h.  Header-only
// C++17; link with -lfloe_b200.
//
//   reference                                          here (namespace floe::gpu)
//   void qgemv_channels(const QuantizedTensor&, ...)   qgemv_channels       quant.hpp:50-51
//   Vec  expert_forward_sparse(const CompressedExpert&, const Vec&)          model.hpp:111
//   Vec  layer_forward(const CompressedModel&, uint32_t, const Vec&)        model.hpp:118
//   LayerTrace layer_forward_traced(...)                                    model.hpp:128-129
//   CompressedModel load_compressed(const std::string&)                     model.hpp:163
//   std::vector<uint8_t> predict_mask(const QuantizedTensor&, uint32_t, const Vec&, float)
//                                                                           predictor.hpp:80-82
//   std::vector<uint32_t> predict_experts(const InterExpertPredictor&, const Vec&, uint32_t,
//                                         uint32_t)                         predictor.hpp:75-77
//
// Two ways to use it:
//   * inside the reference build: #include the reference's
//     floe/model.hpp and floe/predictor.hpp first and define
//     FLOE_B200_REFERENCE_TYPES; floe::gpu then takes the reference's own
//     floe::CompressedExpert / CompressedModel / QuantizedTensor /
//     InterExpertPredictor objects, zero copy (the upload reads their vectors
//     in place);
//   * standalone: floe::gpu defines the same types with the same field names
//     AND storage order as the reference (quant.hpp:20-31, la.hpp:19-32,
//     model.hpp:26-35,60-83,121-129, predictor.hpp:20-33).
// The entry points are templates over those types (field names only), so both
// compile to the same code.
//
// Upload cache: the free functions keep the device copy of each expert/layer/
// predictor they were called with, keyed by the object's address AND a
// content fingerprint (sizes, threshold and 64 sampled words of every weight
// buffer), so a freed-and-reallocated or replaced object at the same address
// is uploaded again; at most kCacheEntries objects are kept (least recently
// used evicted); clear_cache() drops everything (call it after editing
// weights in place: sampled fingerprints do not see every element).
// Threads: every host thread gets its own workspace (pinned staging, device
// scratch), and all value-type calls run on the legacy default stream, so
// concurrent calls from several threads serialise on the device and never
// share buffers -- thread-compatible like the reference.
// DeviceExpert / DeviceLayer / Workspace give explicit control (stream-ordered
// device calls, no hidden synchronisation) for callers that manage their own
// device memory.
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstring>
#include <list>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "floe_gpu.h"

namespace floe {
namespace gpu {

// ---------------------------------------------------------------- types
#ifdef FLOE_B200_REFERENCE_TYPES
using floe::CompressedExpert;
using floe::CompressedLayer;
using floe::CompressedModel;
using floe::InterExpertPredictor;
using floe::LayerTrace;
using floe::Matrix;
using floe::MoEConfig;
using floe::QuantizedTensor;
using floe::Vec;
#else
using Vec = std::vector<float>;

struct QuantizedTensor {
  std::size_t n = 0;                  // element count
  unsigned bits = 0;                  // one of {1, 2, 3, 4, 8}
  std::uint32_t group_size = 0;       // consecutive elements per metadata group
  std::vector<std::uint8_t> codes;    // ceil(n*bits/8), LE in byte, first code in LSBs
  std::vector<std::uint16_t> scales;  // f16 bits, n / group_size
  std::vector<std::uint16_t> zeros;   // f16 bits, n / group_size
};

struct Matrix {  // row-major
  std::size_t rows = 0, cols = 0;
  Vec data;
  Matrix() = default;
  Matrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0f) {}
};

struct MoEConfig {
  std::uint32_t layers = 0, experts = 0, top_k = 0, d_hidden = 0, d_intermediate = 0;
  std::uint64_t seed = 0;
};

struct CompressedExpert {
  std::uint32_t d_hidden = 0, d_intermediate = 0;
  QuantizedTensor up_q;  // channel-major [di][dh]
  Vec gate;              // f32 channel-major [di][dh]
  Vec down_t;            // f32 channel-major [di][dh]
  float threshold = 0.0f;
};

struct CompressedLayer {
  Matrix router;  // [E][dh]
  Matrix mixing;  // [dh][dh]
  std::vector<CompressedExpert> experts;
};

struct CompressedModel {
  MoEConfig cfg;
  unsigned bits = 0;
  std::uint32_t group_size = 0;
  std::vector<CompressedLayer> layers;
};

struct LayerTrace {
  Vec block_input;
  std::vector<std::uint32_t> experts;
  Vec weights;
  std::vector<std::vector<std::uint8_t>> masks;
  Vec out;
};

struct InterExpertPredictor {
  std::uint32_t layers = 0, experts = 0, d_hidden = 0;
  std::vector<Matrix> w;  // [target-1] -> experts x d_hidden
  std::vector<Vec> b;     // [target-1] -> experts
};
#endif

// ------------------------------------------------------------ plumbing
inline void check(int rc) {
  if (rc != FLOE_OK) throw std::runtime_error(floe_gpu_last_error());
}

class Workspace {
 public:
  Workspace(std::uint32_t d_hidden, std::uint32_t d_intermediate, std::uint32_t max_slots = 1) {
    check(floe_gpu_workspace_create(d_hidden, d_intermediate, max_slots, &ws_));
  }
  ~Workspace() { floe_gpu_workspace_destroy(ws_); }
  Workspace(const Workspace &) = delete;
  Workspace &operator=(const Workspace &) = delete;
  floe_gpu_workspace *get() const { return ws_; }

 private:
  floe_gpu_workspace *ws_ = nullptr;
};

// A compressed expert resident in HBM (the upload reads the host object's
// buffers in place).  With with_ffn = false only the up projection is
// uploaded (qgemv_channels / predict_mask on a bare tensor).
class DeviceExpert {
 public:
  template <class Q>
  DeviceExpert(const Q &up_q, std::uint32_t d_hidden, std::uint32_t d_intermediate,
               const float *gate, const float *down_t, float threshold) {
    floe_expert_host_view v{};
    v.d_hidden = d_hidden;
    v.d_intermediate = d_intermediate;
    v.bits = up_q.bits;
    v.group_size = up_q.group_size;
    v.codes = up_q.codes.data();
    v.scales = up_q.scales.data();
    v.zeros = up_q.zeros.data();
    v.gate_f32 = gate;
    v.down_f32 = down_t;
    v.threshold = threshold;
    check(floe_gpu_expert_create(&v, &h_));
    dh_ = d_hidden;
    di_ = d_intermediate;
  }
  template <class Expert>
  explicit DeviceExpert(const Expert &e, bool with_ffn = true)
      : DeviceExpert(e.up_q, e.d_hidden, e.d_intermediate, with_ffn ? ffn_ptr(e, e.gate) : nullptr,
                     with_ffn ? ffn_ptr(e, e.down_t) : nullptr, e.threshold) {}
  ~DeviceExpert() { floe_gpu_expert_destroy(h_); }
  DeviceExpert(const DeviceExpert &) = delete;
  DeviceExpert &operator=(const DeviceExpert &) = delete;
  floe_gpu_expert *get() const { return h_; }
  std::uint32_t d_hidden() const { return dh_; }
  std::uint32_t d_intermediate() const { return di_; }

 private:
  template <class Expert>
  static const float *ffn_ptr(const Expert &e, const Vec &v) {
    if (v.size() != (std::size_t)e.d_hidden * e.d_intermediate)
      throw std::runtime_error("expert_forward_sparse: dimension mismatch");
    return v.data();
  }
  floe_gpu_expert *h_ = nullptr;
  std::uint32_t dh_ = 0, di_ = 0;
};

class DeviceLayer {
 public:
  template <class Layer>
  DeviceLayer(const Layer &l, std::uint32_t top_k, bool mixing_f16 = false) {
    std::vector<floe_gpu_expert *> hs;
    for (const auto &e : l.experts) {
      experts_.push_back(std::make_unique<DeviceExpert>(e));
      hs.push_back(experts_.back()->get());
    }
    if (hs.empty()) throw std::runtime_error("model config: all dimensions must be >= 1");
    floe_layer_host_view v{};
    v.d_hidden = experts_[0]->d_hidden();
    v.n_experts = (std::uint32_t)hs.size();
    v.top_k = top_k;
    v.router = l.router.data.data();
    v.mixing = l.mixing.data.data();
    v.mixing_f16 = mixing_f16 ? 1 : 0;
    v.experts = hs.data();
    check(floe_gpu_layer_create(&v, &h_));
    top_k_ = top_k;
  }
  ~DeviceLayer() { floe_gpu_layer_destroy(h_); }
  DeviceLayer(const DeviceLayer &) = delete;
  DeviceLayer &operator=(const DeviceLayer &) = delete;
  floe_gpu_layer *get() const { return h_; }
  std::uint32_t d_hidden() const { return experts_[0]->d_hidden(); }
  std::uint32_t d_intermediate() const { return experts_[0]->d_intermediate(); }
  std::uint32_t top_k() const { return top_k_; }

 private:
  std::vector<std::unique_ptr<DeviceExpert>> experts_;
  floe_gpu_layer *h_ = nullptr;
  std::uint32_t top_k_ = 0;
};

namespace detail {

// ---- content fingerprints (sizes + 64 sampled 8-byte words per buffer)
inline std::uint64_t mix(std::uint64_t h, std::uint64_t v) {
  v *= 0x9E3779B97F4A7C15ull;
  return (h ^ (v ^ (v >> 29))) * 0xBF58476D1CE4E5B9ull;
}
inline std::uint64_t sample(std::uint64_t h, const void *p, std::size_t bytes) {
  h = mix(h, bytes);
  const auto *b = static_cast<const std::uint8_t *>(p);
  if (!b) return h;
  if (bytes < 8) {
    for (std::size_t i = 0; i < bytes; ++i) h = mix(h, b[i]);
    return h;
  }
  for (std::size_t i = 0; i < 64; ++i) {
    std::uint64_t w;
    std::memcpy(&w, b + (bytes - 8) * i / 63, 8);
    h = mix(h, w);
  }
  return h;
}
template <class V>
std::uint64_t sample_vec(std::uint64_t h, const V &v) {
  return sample(h, v.data(), v.size() * sizeof(v[0]));
}
template <class Q>
std::uint64_t fp_q(const Q &q) {
  std::uint64_t h = mix(mix(mix(0, q.n), q.bits), q.group_size);
  return sample_vec(sample_vec(sample_vec(h, q.codes), q.scales), q.zeros);
}
template <class Expert>
std::uint64_t fp_expert(const Expert &e) {
  std::uint32_t tb;
  std::memcpy(&tb, &e.threshold, 4);
  std::uint64_t h = mix(mix(fp_q(e.up_q), e.d_hidden), e.d_intermediate);
  return mix(sample_vec(sample_vec(h, e.gate), e.down_t), tb);
}

// ---- the upload cache: (address, fingerprint) -> device object, bounded LRU
constexpr std::size_t kCacheEntries = 512;
struct Cache {
  std::mutex mu;
  using Key = std::pair<const void *, std::uint64_t>;
  std::list<std::pair<Key, std::shared_ptr<void>>> lru;  // most recent first
  std::map<Key, decltype(lru)::iterator> index;
};
inline Cache &cache() {
  static Cache c;
  return c;
}

template <typename T, typename Make>
std::shared_ptr<T> cached(const void *key, std::uint64_t f, Make make) {
  Cache &c = cache();
  std::lock_guard<std::mutex> g(c.mu);
  const Cache::Key k{key, f};
  auto it = c.index.find(k);
  if (it != c.index.end()) {
    c.lru.splice(c.lru.begin(), c.lru, it->second);
    return std::static_pointer_cast<T>(it->second->second);
  }
  std::shared_ptr<T> obj = make();
  c.lru.emplace_front(k, obj);
  c.index[k] = c.lru.begin();
  while (c.lru.size() > kCacheEntries) {  // in-flight users keep their shared_ptr
    c.index.erase(c.lru.back().first);
    c.lru.pop_back();
  }
  return obj;
}

// ---- one workspace per (host thread, shape)
inline std::shared_ptr<Workspace> workspace(std::uint32_t dh, std::uint32_t di,
                                            std::uint32_t slots) {
  thread_local std::map<std::tuple<std::uint32_t, std::uint32_t, std::uint32_t>,
                        std::shared_ptr<Workspace>>
      ws;
  auto &w = ws[{dh, di, slots}];
  if (!w) w = std::make_shared<Workspace>(dh, di, slots);
  return w;
}

// Device-side scratch vectors of one call (the value-type calls copy through
// the workspace's pinned staging; these hold extra outputs).
struct DevBuf {
  void *p = nullptr;
  explicit DevBuf(std::size_t bytes) {
    if (floe_gpu_device_malloc(&p, bytes) != FLOE_OK) throw std::runtime_error(floe_gpu_last_error());
  }
  ~DevBuf() { floe_gpu_device_free(p); }
};

}  // namespace detail

// Drop every cached device copy (after editing host weights in place).
inline void clear_cache() {
  detail::Cache &c = detail::cache();
  std::lock_guard<std::mutex> g(c.mu);
  c.index.clear();
  c.lru.clear();
}

// ------------------------------------------------------- reference API
// y = expert_forward_sparse(e, h)  (model.cpp:128-142)
template <class Expert>
Vec expert_forward_sparse(const Expert &e, const Vec &h) {
  if (h.size() != e.d_hidden) throw std::runtime_error("expert_forward_sparse: dimension mismatch");
  auto dev = detail::cached<DeviceExpert>(&e, detail::fp_expert(e),
                                          [&] { return std::make_shared<DeviceExpert>(e); });
  auto ws = detail::workspace(e.d_hidden, e.d_intermediate, 1);
  Vec y(e.d_hidden);
  check(floe_gpu_expert_forward_sparse_host(dev->get(), ws->get(), h.data(), y.data(), nullptr,
                                            nullptr, nullptr));
  return y;
}

// y[c] = sum_k dequant(q)[c*ch_len + k] * x[k]  (quant.cpp:122-136)
template <class Q>
void qgemv_channels(const Q &q, std::size_t ch_len, const float *x, float *y) {
  if (ch_len == 0 || q.n % ch_len != 0)
    throw std::runtime_error("qgemv_channels: ch_len must divide element count");
  const auto dh = (std::uint32_t)ch_len, di = (std::uint32_t)(q.n / ch_len);
  auto dev = detail::cached<DeviceExpert>(&q, detail::fp_q(q) ^ 0x71u, [&] {
    return std::make_shared<DeviceExpert>(q, dh, di, nullptr, nullptr, 0.0f);
  });
  auto ws = detail::workspace(dh, di, 1);
  detail::DevBuf dx(4 * ch_len), dy(4ull * di);
  check(floe_gpu_copy(dx.p, x, 4 * ch_len, nullptr));
  check(floe_gpu_qgemv_channels(dev->get(), ws->get(), static_cast<const float *>(dx.p),
                                static_cast<float *>(dy.p), nullptr));
  check(floe_gpu_copy(y, dy.p, 4ull * di, nullptr));
}

// mask[c] = |qgemv(up_next, x_prev)[c]| >= t  (predictor.cpp:179-189)
template <class Q>
std::vector<std::uint8_t> predict_mask(const Q &up_next, std::uint32_t d_hidden, const Vec &x_prev,
                                       float t) {
  if (x_prev.size() != d_hidden) throw std::runtime_error("predict_mask: dimension mismatch");
  if (d_hidden == 0 || up_next.n % d_hidden != 0)
    throw std::runtime_error("predict_mask: tensor not channel-divisible");
  const auto di = (std::uint32_t)(up_next.n / d_hidden);
  auto dev = detail::cached<DeviceExpert>(&up_next, detail::fp_q(up_next) ^ 0x71u, [&] {
    return std::make_shared<DeviceExpert>(up_next, d_hidden, di, nullptr, nullptr, 0.0f);
  });
  auto ws = detail::workspace(d_hidden, di, 1);
  detail::DevBuf dx(4ull * d_hidden), dm(di);
  check(floe_gpu_copy(dx.p, x_prev.data(), 4ull * d_hidden, nullptr));
  check(floe_gpu_predict_mask(dev->get(), ws->get(), static_cast<const float *>(dx.p), t,
                              static_cast<std::uint8_t *>(dm.p), nullptr, nullptr, nullptr));
  std::vector<std::uint8_t> m(di);
  check(floe_gpu_copy(m.data(), dm.p, m.size(), nullptr));
  return m;
}

namespace detail {
template <class Model>
std::shared_ptr<DeviceLayer> layer_of(const Model &m, std::uint32_t layer) {
  if (layer >= m.cfg.layers || layer >= m.layers.size())
    throw std::runtime_error("layer_forward: bad layer");
  const auto &l = m.layers[layer];
  std::uint64_t f = sample_vec(sample_vec(mix(0, m.cfg.top_k), l.router.data), l.mixing.data);
  for (const auto &e : l.experts) f = mix(f, fp_expert(e));
  return cached<DeviceLayer>(&l, f, [&] { return std::make_shared<DeviceLayer>(l, m.cfg.top_k); });
}
}  // namespace detail

// layer_forward(CompressedModel) (model.cpp:182-190)
template <class Model>
Vec layer_forward(const Model &m, std::uint32_t layer, const Vec &h) {
  auto L = detail::layer_of(m, layer);
  if (h.size() != L->d_hidden()) throw std::runtime_error("gemv: dimension mismatch");
  auto ws = detail::workspace(L->d_hidden(), L->d_intermediate(), L->top_k());
  Vec y(h.size());
  check(floe_gpu_layer_forward_host(L->get(), ws->get(), h.data(), y.data(), nullptr));
  return y;
}

// layer_forward_traced (model.cpp:192-208)
template <class Model>
LayerTrace layer_forward_traced(const Model &m, std::uint32_t layer, const Vec &h) {
  auto L = detail::layer_of(m, layer);
  const std::uint32_t dh = L->d_hidden(), di = L->d_intermediate(), k = L->top_k();
  if (h.size() != dh) throw std::runtime_error("gemv: dimension mismatch");
  auto ws = detail::workspace(dh, di, k);
  detail::DevBuf dh_in(4ull * dh), dy(4ull * dh), du(4ull * dh), de(4ull * k), dw(4ull * k),
      dm((std::size_t)k * di);
  floe_gpu_layer_trace tr{static_cast<float *>(du.p), static_cast<std::uint32_t *>(de.p),
                          static_cast<float *>(dw.p), static_cast<std::uint8_t *>(dm.p)};
  check(floe_gpu_copy(dh_in.p, h.data(), 4ull * dh, nullptr));
  check(floe_gpu_layer_forward(L->get(), ws->get(), static_cast<const float *>(dh_in.p),
                               static_cast<float *>(dy.p), &tr, nullptr));
  LayerTrace t;
  t.block_input.resize(dh);
  t.out.resize(dh);
  t.experts.resize(k);
  t.weights.resize(k);
  std::vector<std::uint8_t> masks((std::size_t)k * di);
  check(floe_gpu_copy(t.block_input.data(), du.p, 4ull * dh, nullptr));
  check(floe_gpu_copy(t.out.data(), dy.p, 4ull * dh, nullptr));
  check(floe_gpu_copy(t.experts.data(), de.p, 4ull * k, nullptr));
  check(floe_gpu_copy(t.weights.data(), dw.p, 4ull * k, nullptr));
  check(floe_gpu_copy(masks.data(), dm.p, masks.size(), nullptr));
  for (std::uint32_t j = 0; j < k; ++j)
    t.masks.emplace_back(masks.begin() + (std::size_t)j * di, masks.begin() + (std::size_t)(j + 1) * di);
  return t;
}

// predict_experts (predictor.cpp:164-177)
template <class Predictor>
std::vector<std::uint32_t> predict_experts(const Predictor &p, const Vec &x, std::uint32_t layer,
                                           std::uint32_t prefetch_count) {
  if (layer == 0) throw std::runtime_error("predict_experts: layer 0 has no lookahead predictor");
  if (layer >= p.layers) throw std::runtime_error("predict_experts: bad layer");
  if (x.size() != p.d_hidden) throw std::runtime_error("predict_experts: dimension mismatch");
  if (prefetch_count == 0 || prefetch_count > p.experts)
    throw std::runtime_error("top_k: k out of range");
  std::uint64_t f = detail::mix(detail::mix(detail::mix(0, p.layers), p.experts), p.d_hidden);
  for (const auto &m : p.w) f = detail::sample_vec(f, m.data);
  for (const auto &v : p.b) f = detail::sample_vec(f, v);
  auto dev = detail::cached<floe_gpu_predictor>(&p, f, [&] {
    std::vector<float> w, b;
    for (const auto &m : p.w) w.insert(w.end(), m.data.begin(), m.data.end());
    for (const auto &v : p.b) b.insert(b.end(), v.begin(), v.end());
    floe_gpu_predictor *h = nullptr;
    check(floe_gpu_predictor_create(p.layers, p.experts, p.d_hidden, w.data(), b.data(), &h));
    return std::shared_ptr<floe_gpu_predictor>(h, [](floe_gpu_predictor *q) {
      floe_gpu_predictor_destroy(q);
    });
  });
  detail::DevBuf dx(4ull * x.size()), dout(4ull * prefetch_count);
  check(floe_gpu_copy(dx.p, x.data(), 4ull * x.size(), nullptr));
  check(floe_gpu_predict_experts(dev.get(), static_cast<const float *>(dx.p), layer,
                                 prefetch_count, static_cast<std::uint32_t *>(dout.p), nullptr));
  std::vector<std::uint32_t> out(prefetch_count);
  check(floe_gpu_copy(out.data(), dout.p, 4ull * prefetch_count, nullptr));
  return out;
}

// ----------------------------------------------------------- FLOQ loader
// load_compressed (model.cpp:434-474): magic "FLOQ", u32 version = 1,
// layers/experts/top_k/d_hidden/d_intermediate u32, seed u64, bits u8,
// group_size u32; per layer router f32[E*dh], mixing f32[dh*dh]; per expert
// packed codes, f16 scales, f16 zeros, f32 gate, f32 down_t, f32 threshold.
// Little-endian throughout; same validation and messages as the reference.
inline CompressedModel load_compressed(const std::string &path) {
  std::FILE *f = std::fopen(path.c_str(), "rb");
  if (!f) throw std::runtime_error("read_file: cannot open " + path);
  std::vector<std::uint8_t> buf;
  {
    std::uint8_t chunk[1 << 16];
    std::size_t got;
    while ((got = std::fread(chunk, 1, sizeof chunk, f)) > 0) buf.insert(buf.end(), chunk, chunk + got);
    std::fclose(f);
  }
  std::size_t pos = 0;
  auto need = [&](std::size_t n) {
    if (buf.size() - pos < n) throw std::runtime_error("ByteReader: truncated input");
  };
  auto rd = [&](void *dst, std::size_t n) {
    need(n);
    std::memcpy(dst, buf.data() + pos, n);
    pos += n;
  };
  auto u8 = [&] { std::uint8_t v; rd(&v, 1); return v; };
  auto u32 = [&] { std::uint32_t v; rd(&v, 4); return v; };
  auto u64 = [&] { std::uint64_t v; rd(&v, 8); return v; };
  char magic[4];
  rd(magic, 4);
  if (std::memcmp(magic, "FLOQ", 4) != 0) throw std::runtime_error("model file: bad magic");
  const std::uint32_t version = u32();
  if (version != 1)
    throw std::runtime_error("model file: unsupported version " + std::to_string(version));
  CompressedModel m;
  m.cfg.layers = u32();
  m.cfg.experts = u32();
  m.cfg.top_k = u32();
  m.cfg.d_hidden = u32();
  m.cfg.d_intermediate = u32();
  m.cfg.seed = u64();
  if (!m.cfg.layers || !m.cfg.experts || !m.cfg.top_k || !m.cfg.d_hidden || !m.cfg.d_intermediate)
    throw std::runtime_error("model config: all dimensions must be >= 1");
  if (m.cfg.top_k > m.cfg.experts) throw std::runtime_error("model config: need 1 <= top_k <= experts");
  m.bits = u8();
  m.group_size = u32();
  const std::size_t dh = m.cfg.d_hidden, di = m.cfg.d_intermediate, n = dh * di;
  if (m.group_size == 0 || n % m.group_size != 0)
    throw std::runtime_error("compressed file: bad group size");
  const std::size_t code_bytes = (n * m.bits + 7) / 8;
  m.layers.resize(m.cfg.layers);
  for (auto &layer : m.layers) {
    layer.router = Matrix(m.cfg.experts, dh);
    rd(layer.router.data.data(), 4 * layer.router.data.size());
    layer.mixing = Matrix(dh, dh);
    rd(layer.mixing.data.data(), 4 * layer.mixing.data.size());
    layer.experts.resize(m.cfg.experts);
    for (auto &e : layer.experts) {
      e.d_hidden = m.cfg.d_hidden;
      e.d_intermediate = m.cfg.d_intermediate;
      e.up_q.n = n;
      e.up_q.bits = m.bits;
      e.up_q.group_size = m.group_size;
      e.up_q.codes.resize(code_bytes);
      rd(e.up_q.codes.data(), code_bytes);
      e.up_q.scales.resize(n / m.group_size);
      rd(e.up_q.scales.data(), 2 * e.up_q.scales.size());
      e.up_q.zeros.resize(n / m.group_size);
      rd(e.up_q.zeros.data(), 2 * e.up_q.zeros.size());
      e.gate.resize(n);
      e.down_t.resize(n);
      rd(e.gate.data(), 4 * n);
      rd(e.down_t.data(), 4 * n);
      rd(&e.threshold, 4);
    }
  }
  if (pos != buf.size()) throw std::runtime_error("compressed file: trailing bytes in " + path);
  return m;
}

}  // namespace gpu
}  // namespace floe
