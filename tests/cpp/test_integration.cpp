// test_integration.cpp -- the INTEGRATION.md binding, compiled the way a
// maintainer would build the reference with FLOE_WITH_B200: the reference's
// own headers and sources (compiled in place from /root/reference by
// tests/cpp/Makefile), this repository's include/floe_b200.hpp in reference-
// type mode, linked with libfloe_b200.so.
//
// The reference builds, calibrates and compresses a model (gen_model ->
// calibrate_model -> compress_model); floe::gpu:: then runs on the
// reference's OWN floe::CompressedModel / CompressedExpert objects (no copy,
// no parallel types) from one thread and from two concurrent threads; the
// outputs must equal the single-thread ones and the reference's
// floe::layer_forward / floe::expert_forward_sparse, and the error messages
// must be the reference's.
//
//   test_integration            (exit 0 = pass; prints a summary line)
#include <cmath>
#include <cstdio>
#include <string>
#include <thread>
#include <vector>

#include "floe/model.hpp"
#include "floe/predictor.hpp"
#include "floe/quant.hpp"
#include "floe/sparsify.hpp"

#define FLOE_B200_REFERENCE_TYPES
#include "floe_b200.hpp"

using floe::Vec;

static double rel_l2(const Vec &a, const Vec &b) {
  double num = 0, den = 0;
  for (std::size_t i = 0; i < a.size(); ++i) {
    num += (double)(a[i] - b[i]) * (a[i] - b[i]);
    den += (double)b[i] * b[i];
  }
  return std::sqrt(num / (den > 0 ? den : 1));
}

template <class F>
static std::string message_of(F &&f) {
  try {
    f();
  } catch (const std::exception &e) {
    return e.what();
  }
  return "(no exception)";
}

int main() {
  floe::MoEConfig cfg;
  cfg.layers = 2;
  cfg.experts = 4;
  cfg.top_k = 2;
  cfg.d_hidden = 2048;
  cfg.d_intermediate = 512;
  cfg.seed = 7;
  floe::MoEModel fm = floe::gen_model(cfg, 8);
  floe::ThresholdTable tt = floe::calibrate_model(fm, 3, 64, 0.8, floe::kReservoirCap, 8);
  const floe::CompressedModel cm = floe::compress_model(fm, tt, 2, 64);

  const std::uint32_t NT = 8;
  std::vector<Vec> toks;
  for (std::uint32_t t = 0; t < NT; ++t) toks.push_back(floe::token_input(1, t, cfg.d_hidden));
  int bad = 0;
  auto expect = [&](bool ok, const std::string &what) {
    if (!ok) {
      std::fprintf(stderr, "FAIL %s\n", what.c_str());
      ++bad;
    }
  };

  // one thread: the reference's own objects straight into floe::gpu
  std::vector<Vec> y1(NT * cfg.layers), ye1(NT);
  for (std::uint32_t t = 0; t < NT; ++t) {
    for (std::uint32_t l = 0; l < cfg.layers; ++l) {
      y1[t * cfg.layers + l] = floe::gpu::layer_forward(cm, l, toks[t]);
      const Vec ref = floe::layer_forward(cm, l, toks[t]);
      expect(rel_l2(y1[t * cfg.layers + l], ref) <= 1e-2, "layer_forward vs reference");
    }
    ye1[t] = floe::gpu::expert_forward_sparse(cm.layers[0].experts[t % cfg.experts], toks[t]);
    const Vec ref = floe::expert_forward_sparse(cm.layers[0].experts[t % cfg.experts], toks[t]);
    expect(rel_l2(ye1[t], ref) <= 1e-2, "expert_forward_sparse vs reference");
  }
  // two concurrent threads, interleaved tokens
  std::vector<Vec> y2(NT * cfg.layers), ye2(NT);
  std::vector<std::string> errs(2);
  auto worker = [&](std::uint32_t k) {
    try {
      for (int rep = 0; rep < 3; ++rep)
        for (std::uint32_t t = k; t < NT; t += 2) {
          for (std::uint32_t l = 0; l < cfg.layers; ++l)
            y2[t * cfg.layers + l] = floe::gpu::layer_forward(cm, l, toks[t]);
          ye2[t] = floe::gpu::expert_forward_sparse(cm.layers[0].experts[t % cfg.experts], toks[t]);
        }
    } catch (const std::exception &e) {
      errs[k] = e.what();
    }
  };
  std::thread a(worker, 0u), b(worker, 1u);
  a.join();
  b.join();
  expect(errs[0].empty() && errs[1].empty(), "threads raised: " + errs[0] + " / " + errs[1]);
  // the only difference between runs is the order of the cross-CTA f32 reductions into y
  for (std::uint32_t i = 0; i < NT * cfg.layers; ++i)
    expect(rel_l2(y2[i], y1[i]) <= 1e-6, "2 threads == 1 thread (layer) " + std::to_string(i));
  for (std::uint32_t t = 0; t < NT; ++t)
    expect(rel_l2(ye2[t], ye1[t]) <= 1e-6, "2 threads == 1 thread (expert) " + std::to_string(t));

  // qgemv_channels and predict_mask on the reference's QuantizedTensor
  {
    const auto &q = cm.layers[1].experts[0].up_q;
    Vec v(q.n / cfg.d_hidden), vr(q.n / cfg.d_hidden);
    floe::gpu::qgemv_channels(q, cfg.d_hidden, toks[0].data(), v.data());
    floe::qgemv_channels(q, cfg.d_hidden, toks[0].data(), vr.data());
    expect(rel_l2(v, vr) <= 1e-5, "qgemv_channels vs reference");
    const float t = cm.layers[1].experts[0].threshold;
    auto m = floe::gpu::predict_mask(q, cfg.d_hidden, toks[0], t);
    auto mr = floe::predict_mask(q, cfg.d_hidden, toks[0], t);
    for (std::size_t c = 0; c < m.size(); ++c)
      if (m[c] != mr[c]) expect(std::fabs(std::fabs(vr[c]) - t) <= 1e-3, "predict_mask tie rule");
  }

  // the reference's error contract, message for message
  auto same = [&](const std::string &what, auto &&ours, auto &&theirs) {
    const std::string a1 = message_of(ours), b1 = message_of(theirs);
    expect(a1 == b1, what + ": '" + a1 + "' vs '" + b1 + "'");
  };
  same("bad layer", [&] { floe::gpu::layer_forward(cm, 7, toks[0]); },
       [&] { floe::layer_forward(cm, 7, toks[0]); });
  same("expert dim", [&] { floe::gpu::expert_forward_sparse(cm.layers[0].experts[0], Vec(3)); },
       [&] { floe::expert_forward_sparse(cm.layers[0].experts[0], Vec(3)); });
  floe::QuantizedTensor odd = floe::quantize(Vec(96, 0.5f), 2, 32);
  same("predict_mask divisible", [&] { floe::gpu::predict_mask(odd, 64, Vec(64), 0.1f); },
       [&] { floe::predict_mask(odd, 64, Vec(64), 0.1f); });
  same("qgemv ch_len", [&] { Vec y(2); floe::gpu::qgemv_channels(odd, 64, Vec(64).data(), y.data()); },
       [&] { Vec y(2); floe::qgemv_channels(odd, 64, Vec(64).data(), y.data()); });
  floe::InterExpertPredictor p;
  p.layers = 2;
  p.experts = cfg.experts;
  p.d_hidden = cfg.d_hidden;
  p.w.push_back(cm.layers[0].router);
  p.b.push_back(Vec(cfg.experts, 0.0f));
  same("predict_experts layer 0", [&] { floe::gpu::predict_experts(p, toks[0], 0, 2); },
       [&] { floe::predict_experts(p, toks[0], 0, 2); });
  same("predict_experts bad layer", [&] { floe::gpu::predict_experts(p, toks[0], 2, 2); },
       [&] { floe::predict_experts(p, toks[0], 2, 2); });
  expect(floe::gpu::predict_experts(p, toks[0], 1, 2) == floe::predict_experts(p, toks[0], 1, 2),
         "predict_experts vs reference");

  // an object edited in place is uploaded again (content fingerprint)
  {
    floe::CompressedExpert e = cm.layers[0].experts[1];
    const Vec y0 = floe::gpu::expert_forward_sparse(e, toks[0]);
    e.threshold = INFINITY;  // nothing kept -> exact zeros (test_model.cpp:129-134)
    const Vec yz = floe::gpu::expert_forward_sparse(e, toks[0]);
    bool zero = true;
    for (float f : yz) zero = zero && f == 0.0f;
    expect(zero && rel_l2(y0, Vec(y0.size(), 0.0f)) > 0, "threshold edit re-uploads");
  }
  std::printf("test_integration: %u tokens x %u layers, 2 threads, %d failures\n", NT, cfg.layers,
              bad);
  return bad ? 1 : 0;
}
