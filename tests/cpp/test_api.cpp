// test_api.cpp -- the C++ value-type API (include/floe_b200.hpp) driven the
// way the reference's own tests drive floe:: (test_model.cpp, test_cli.cpp
// `run`): load a FLOQ file written by the reference's save_compressed, chain
// layer_forward_traced over the layers for each token (cmd_run, cli.cpp:86-107),
// and call expert_forward_sparse / qgemv_channels / predict_mask /
// predict_experts on the loaded objects.  Outputs go to raw little-endian
// files that tests/test_cpp_api.py compares with the reference core.
//
//   test_api <model.floq> <tokens.f32> <n_tokens> <out_dir>
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "floe_b200.hpp"

using namespace floe::gpu;

template <typename T>
static void dump(const std::string &path, const std::vector<T> &v) {
  std::ofstream f(path, std::ios::binary | std::ios::app);
  f.write(reinterpret_cast<const char *>(v.data()), sizeof(T) * v.size());
}

static int expect_error(const char *what, const char *needle, void (*fn)()) {
  try {
    fn();
  } catch (const std::runtime_error &e) {
    if (std::string(e.what()).find(needle) != std::string::npos) return 0;
    std::fprintf(stderr, "%s: wrong message '%s'\n", what, e.what());
    return 1;
  }
  std::fprintf(stderr, "%s: no exception\n", what);
  return 1;
}

static CompressedModel *g_model = nullptr;

int main(int argc, char **argv) {
  if (argc != 5) {
    std::fprintf(stderr, "usage: test_api <model.floq> <tokens.f32> <n_tokens> <out_dir>\n");
    return 2;
  }
  const std::string out = argv[4];
  CompressedModel m = load_compressed(argv[1]);
  g_model = &m;
  const std::uint32_t dh = m.cfg.d_hidden, nt = (std::uint32_t)std::stoul(argv[3]);
  std::vector<float> toks((std::size_t)nt * dh);
  {
    std::ifstream f(argv[2], std::ios::binary);
    f.read(reinterpret_cast<char *>(toks.data()), 4 * toks.size());
    if (!f) return 3;
  }
  // decode: h -> layer 0 -> layer 1 -> ...  (cmd_run)
  for (std::uint32_t t = 0; t < nt; ++t) {
    Vec h(toks.begin() + (std::size_t)t * dh, toks.begin() + (std::size_t)(t + 1) * dh);
    for (std::uint32_t l = 0; l < m.cfg.layers; ++l) {
      LayerTrace tr = layer_forward_traced(m, l, h);
      Vec y = layer_forward(m, l, h);  // untraced == traced (test_model.cpp:263-279)
      dump(out + "/u.f32", tr.block_input);
      dump(out + "/sel.u32", tr.experts);
      dump(out + "/w.f32", tr.weights);
      for (const auto &mk : tr.masks) dump(out + "/masks.u8", mk);
      dump(out + "/y.f32", tr.out);
      dump(out + "/y_untraced.f32", y);
      h = tr.out;
    }
  }
  // one expert, its up projection, and the reuse predictor on the next layer
  const CompressedExpert &e = m.layers[0].experts[0];
  Vec x(toks.begin(), toks.begin() + dh);
  dump(out + "/expert_y.f32", expert_forward_sparse(e, x));
  Vec v(e.d_intermediate);
  qgemv_channels(e.up_q, dh, x.data(), v.data());
  dump(out + "/qgemv_v.f32", v);
  if (m.cfg.layers > 1)
    dump(out + "/predict_mask.u8", predict_mask(m.layers[1].experts[0].up_q, dh, x,
                                                m.layers[1].experts[0].threshold));
  InterExpertPredictor p;
  p.layers = 2;
  p.experts = m.cfg.experts;
  p.d_hidden = dh;
  p.w.push_back(m.layers[0].router);  // any E x dh map
  p.b.push_back(Vec(m.cfg.experts, 0.0f));
  dump(out + "/predict_experts.u32", predict_experts(p, x, 1, m.cfg.top_k));
  // the reference's error contract
  int bad = 0;
  bad += expect_error("dimension", "expert_forward_sparse: dimension mismatch", [] {
    expert_forward_sparse(g_model->layers[0].experts[0], Vec(3, 0.0f));
  });
  bad += expect_error("layer0", "predict_experts: layer 0 has no lookahead predictor", [] {
    InterExpertPredictor q;
    q.layers = 2;
    q.experts = 2;
    q.d_hidden = 3;
    predict_experts(q, Vec(3, 0.0f), 0, 1);
  });
  bad += expect_error("magic", "model file: bad magic", [] {
    std::ofstream("/tmp/floe_bad_magic.bin") << "FLOEjunk";
    load_compressed("/tmp/floe_bad_magic.bin");
  });
  std::printf("test_api: %u tokens x %u layers, %d contract failures\n", nt, m.cfg.layers, bad);
  return bad ? 1 : 0;
}
