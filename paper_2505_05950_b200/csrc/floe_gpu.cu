// floe_gpu.cu -- C ABI (include/floe_gpu.h) over the sm_100a kernels.
//
// Host-side responsibilities: device residency of compressed experts in the
// layout DESIGN.md documents, per-stream workspaces, launch configuration,
// stage profiling and the reference's error contract ("<fn>: <reason>"
// messages).  There is deliberately no CPU fallback anywhere in this file.
#include <cublasLt.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <new>
#include <string>
#include <vector>

#include "../../include/floe_gpu.h"
#include "floe_gen.cuh"
#include "floe_v2.cuh"
#include "floe_v3.cuh"
#include "floe_tc.cuh"
#include "floe_calib.cuh"
#include "floe_blayer.cuh"
#include "floe_prefill.cuh"
#include "floe_k1b.cuh"
#include <map>
#include <tuple>

#include <cub/device/device_segmented_radix_sort.cuh>
#include <cub/device/device_select.cuh>
#include <cub/iterator/counting_input_iterator.cuh>

using floe_k::ExpertDesc;
using floe_k::K1Args;
using floe_k::K2Args;

namespace {

thread_local std::string g_err;

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  std::vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(call)                                                                   \
  do {                                                                             \
    cudaError_t e_ = (call);                                                       \
    if (e_ != cudaSuccess)                                                         \
      return fail(e_ == cudaErrorMemoryAllocation ? FLOE_ERR_OOM : FLOE_ERR_CUDA,  \
                  "%s: %s (%s)", __func__, cudaGetErrorString(e_), #call);         \
  } while (0)

#define CK_LAUNCH()                                                                \
  do {                                                                             \
    cudaError_t e_ = cudaGetLastError();                                           \
    if (e_ != cudaSuccess)                                                         \
      return fail(FLOE_ERR_CUDA, "%s: kernel launch failed: %s", __func__,         \
                  cudaGetErrorString(e_));                                         \
  } while (0)

struct DeviceInfo {
  int ok = 0, sm = 0, major = 0, minor = 0;
  size_t mem = 0;
  std::string err;
};

const DeviceInfo &device_info() {
  static DeviceInfo info;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaError_t e = cudaGetDevice(&dev);
    cudaDeviceProp p{};
    if (e == cudaSuccess) e = cudaGetDeviceProperties(&p, dev);
    if (e != cudaSuccess) {
      info.err = std::string("no usable CUDA device: ") + cudaGetErrorString(e);
      return;
    }
    info.sm = p.multiProcessorCount;
    info.major = p.major;
    info.minor = p.minor;
    info.mem = p.totalGlobalMem;
    if (p.major != 10) {
      info.err = "device is sm_" + std::to_string(p.major * 10 + p.minor) +
                 "; this library carries sm_100a code only";
      return;
    }
    info.ok = 1;
  });
  return info;
}

int require_device(const char *fn) {
  const DeviceInfo &d = device_info();
  if (!d.ok) return fail(FLOE_ERR_CUDA, "%s: %s", fn, d.err.c_str());
  return FLOE_OK;
}

bool bits_ok(uint32_t b) { return b == 1 || b == 2 || b == 3 || b == 4 || b == 8; }

uint64_t packed_code_bytes(uint64_t n, uint32_t bits) { return (n * bits + 7) / 8; }

// The sm_100a fast path (floe_v2.cuh): INT2 codes, d_hidden 2048 or 4096,
// quantisation groups made of whole 64-element spans.
bool fast_shape(uint32_t dh, uint32_t bits, uint32_t g) {
  return bits == 2 && (dh == 4096 || dh == 2048) && g % 64 == 0 && dh % g == 0;
}

cudaStream_t S(floe_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

uint64_t up256(uint64_t x) { return (x + 255) & ~uint64_t(255); }

constexpr uint32_t kMaxSeg = 1024;  // K1 CTAs (segments) per slot

}  // namespace

// ---------------------------------------------------------------------------
struct floe_gpu_expert {
  uint32_t dh = 0, di = 0, bits = 0, g = 0;
  float threshold = 0.0f;
  uint64_t code_bytes = 0, n_groups = 0;
  void *block = nullptr;  // one device allocation for everything
  ExpertDesc host_desc{};
  ExpertDesc *dev_desc = nullptr;
  bool fast = false;  // tile-fragment layout + fused kernel
  bool up_only = false;  // no gate/down records (qgemv_channels / predict_mask only)
  // gate|down records: in HBM (rec_dev) or host-resident in pinned, mapped
  // memory (rec_host) that the kernels read directly over PCIe
  __half *rec_dev = nullptr;
  __half *rec_host = nullptr;
  bool resident = true;
  std::vector<ExpertDesc *> tables;  // device layer-table entries copying host_desc
};

enum { kStageMixing = 0, kStageRoute = 1, kStageK1 = 2, kStageK2 = 3, kStageFused = 4, kStages = 5 };

struct floe_gpu_workspace {
  uint32_t dh = 0, di = 0, slots = 0;
  void *block = nullptr;
  uint32_t *kept_idx = nullptr;
  float *kept_v = nullptr;
  uint32_t *seg_count = nullptr;  // [slots][kMaxSeg]
  uint32_t g1 = 0;                // K1 grid.x of the last K1 launch (segments per slot)
  float *mix_partial = nullptr;   // [dh/8][32] partial router logits
  uint32_t *mix_done = nullptr;
  unsigned long long *stats = nullptr;
  unsigned long long *bar = nullptr;  // fused kernel's grid barrier (monotonic)
  unsigned long long *tick = nullptr;    // fused kernel: monotonic CTA ticket
  unsigned long long *y_flag = nullptr;  // fused kernel, expert mode: y-zeroed flag + CTA count
  uint32_t *kcount = nullptr;            // fused kernel: per-call kept counts per slot
  unsigned long long *pcnt = nullptr;    // fused kernel: published predicted partials
  unsigned long long *pf_tick = nullptr; // fused kernel: next-mixing prefetch tickets
  unsigned long long *lbar = nullptr;    // multi-layer decode: end-of-layer arrivals (tickets)
  float *pred_partial = nullptr;         // fused kernel: [32][kMaxGrid] predicted partials
  unsigned long long *phase_ns = nullptr;  // diagnostics: [grid][8] phase marks
  uint32_t *sel = nullptr;
  float *weights = nullptr, *u = nullptr, *x = nullptr, *y = nullptr, *v = nullptr;
  uint8_t *mask = nullptr;
  // pinned host staging for the *_host calls
  float *hx = nullptr, *hy = nullptr, *hv = nullptr;
  uint8_t *hmask = nullptr;
  unsigned long long *hstats = nullptr;
  // stage profiling (CUDA events on the launching stream)
  bool profiling = false;
  std::vector<cudaEvent_t> pool;  // free events
  struct Pending {
    int stage;
    cudaEvent_t a, b;
  };
  std::vector<Pending> pending;
  double ms[kStages] = {};
  uint64_t launches[kStages] = {};
};

struct floe_gpu_layer {
  uint32_t dh = 0, di = 0, E = 0, top_k = 0, bits = 0, g = 0;
  bool mix_f16 = false, fast = false;
  float *router = nullptr;
  void *mixing = nullptr;
  float *router_pred = nullptr;  // fused path: router + router * mixing (routing predictor)
  ExpertDesc *table = nullptr;
  std::vector<floe_gpu_expert *> experts;  // borrowed (offload engine)
};

struct floe_gpu_predictor {
  uint32_t layers = 0, experts = 0, dh = 0;
  float *w = nullptr, *b = nullptr;
};

namespace {

// ---- stage profiling --------------------------------------------------------
cudaEvent_t take_event(floe_gpu_workspace *ws) {
  if (!ws->pool.empty()) {
    cudaEvent_t e = ws->pool.back();
    ws->pool.pop_back();
    return e;
  }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

struct StageScope {  // records [a, b] around one kernel when profiling is on
  floe_gpu_workspace *ws;
  int stage;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  StageScope(floe_gpu_workspace *w, int s, cudaStream_t stream) : ws(w), stage(s), st(stream) {
    if (ws && ws->profiling) {
      a = take_event(ws);
      cudaEventRecord(a, st);
    }
  }
  ~StageScope() {
    if (a) {
      cudaEvent_t b = take_event(ws);
      cudaEventRecord(b, st);
      ws->pending.push_back({stage, a, b});
    }
  }
};

// ---- launch helpers -------------------------------------------------------
// Keep freed stream-ordered memory cached in the default pool (the batched and
// prefill paths allocate their scratch per call; without this every host sync
// returns it to the driver and the next call maps it again).
void keep_pool() {
  static const bool ready = [] {
    cudaMemPool_t pool;
    int dev = 0;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t thr = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
    }
    return true;
  }();
  (void)ready;
}

template <typename F>
int set_smem(F *fn, uint32_t bytes) {
  cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess)
    return fail(FLOE_ERR_CUDA, "set_smem: cudaFuncSetAttribute(%u B): %s", bytes,
                cudaGetErrorString(e));
  return FLOE_OK;
}

struct K1Launch {
  const ExpertDesc *table;
  const uint32_t *sel;
  uint32_t slots, dh, di, bits, g;
  int use_thr;
  float thr;
  const float *x;
  float *v_out;
  uint8_t *mask_out;
  float *y_zero;
};

// Generic-path K1 (any bits / group / d_hidden): segments per slot = grid.x.
int launch_k1(const K1Launch &L, floe_gpu_workspace *ws, cudaStream_t st) {
  K1Args a{};
  a.table = L.table;
  a.sel = L.sel;
  a.x = L.x;
  a.dh = L.dh;
  a.di = L.di;
  a.bits = L.bits;
  a.group_size = L.g;
  a.use_threshold = L.use_thr;
  a.threshold = L.thr;
  a.v_out = L.v_out;
  a.mask_out = L.mask_out;
  a.kept_idx = ws->kept_idx;
  a.kept_v = ws->kept_v;
  a.seg_count = ws->seg_count;
  a.y_zero = L.y_zero;
  const uint32_t sm = (uint32_t)device_info().sm;
  const uint32_t g1 = std::min<uint32_t>(
      {std::max<uint32_t>(1, std::min<uint32_t>((L.di + 63) / 64, 4u * sm)), kMaxSeg});
  ws->g1 = g1;
  StageScope prof(ws, kStageK1, st);
  floe_k::k1_generic<<<dim3(g1, L.slots), 256, 0, st>>>(a);
  CK_LAUNCH();
  return FLOE_OK;
}

struct K2Launch {
  const ExpertDesc *table;
  const uint32_t *sel;
  const float *weights;
  uint32_t slots, dh, di;
  const float *x;
  float *y;  // nullptr: finalize only (n_kept / kept ids of a K1-only call)
  uint32_t *n_kept_out, *kept_out;
};

int launch_k2(const K2Launch &L, floe_gpu_workspace *ws, cudaStream_t st) {
  K2Args a{};
  a.table = L.table;
  a.sel = L.sel;
  a.weights = L.weights;
  a.x = L.x;
  a.dh = L.dh;
  a.di = L.di;
  a.slots = L.slots;
  a.g1 = ws->g1;
  a.kept_idx = ws->kept_idx;
  a.kept_v = ws->kept_v;
  a.seg_count = ws->seg_count;
  a.y = L.y;
  a.n_kept_out = L.n_kept_out;
  a.kept_out = L.kept_out;
  a.stats = L.y ? ws->stats : nullptr;
  const int sm = device_info().sm;
  const uint32_t prefix_bytes = 4u * (L.slots * ws->g1 + 1);
  if (!L.y && !L.n_kept_out && !L.kept_out) return FLOE_OK;
  StageScope prof(ws, kStageK2, st);
  if (int rc = set_smem(floe_k::k2_generic, prefix_bytes)) return rc;
  floe_k::k2_generic<<<(L.y ? 4 : 1) * sm, 128, prefix_bytes, st>>>(a);
  CK_LAUNCH();
  return FLOE_OK;
}

// The fast path: one cooperative persistent launch of floe_v2::fused.
struct FusedLaunch {
  // layer mode (mixing != nullptr) or single-expert mode
  const void *mixing;
  bool mix_f16;
  const float *h, *router, *router_pred;
  uint32_t n_experts, top_k;
  const floe_gpu_layer_trace *trace;
  // experts
  const ExpertDesc *table;
  uint32_t slots, dh, di;
  bool k1_only;
  int use_thr;
  float thr;
  const float *x;
  float *u, *y, *v_out;
  uint8_t *mask_out;
  uint32_t *n_kept_out, *kept_out;
  unsigned long long *place_acc;  // nullable: offload engine's HBM / PCIe record counts
  const void *next_mixing = nullptr;  // nullable: the next layer's mixing (L2 prefetch)
  uint64_t next_mixing_bytes = 0;
};

template <int DH>
int launch_v2_dh(const FusedLaunch &L, floe_gpu_workspace *ws, cudaStream_t st) {
  namespace V = floe_v2;
  const uint32_t G = std::min<uint32_t>((uint32_t)device_info().sm, V::kMaxGrid);
  const uint32_t tps = V::tiles_per_expert(L.di);
  const uint32_t NT = L.slots * tps;
  const uint32_t max_tiles = std::max<uint32_t>(1, (NT + G - 1) / G);
  static int optin = [] {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
    return v;
  }();
  static size_t static_smem = [] {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, V::fused<DH>);
    return fa.sharedSizeBytes;
  }();
  // ring stages: fixed per d_hidden (a multiple of the consumer warp pairs:
  // stage ownership in phases A/B)
  const uint32_t ns = V::ring_stages(DH);
  const uint32_t smem = V::smem_layout(DH, ns, max_tiles, G).total;
  if ((int64_t)smem + (int64_t)static_smem + 1024 > (int64_t)optin)
    return fail(FLOE_ERR_UNSUPPORTED, "fused path: shared memory too small for the ring");

  V::FusedArgs a{};
  a.has_mixing = L.mixing != nullptr;
  a.k1_only = L.k1_only;
  a.mixing = L.mixing;
  a.mix_f16 = L.mix_f16;
  a.h = L.h;
  a.router = L.router;
  a.router_pred = L.router_pred;
  a.n_experts = L.n_experts;
  a.top_k = L.top_k;
  a.partial = ws->mix_partial;
  a.u_trace = L.trace ? L.trace->block_input_dev : nullptr;
  a.sel_trace = L.trace ? L.trace->experts_dev : nullptr;
  a.w_trace = L.trace ? L.trace->weights_dev : nullptr;
  a.sel_out = ws->sel;
  a.w_out = ws->weights;
  a.x = L.x;
  a.u = L.u;
  a.y = L.y;
  a.di = L.di;
  a.slots = L.slots;
  a.table = L.table;
  a.use_threshold = L.use_thr;
  a.threshold = L.thr;
  a.v_out = L.v_out;
  a.mask_out = L.mask_out ? L.mask_out : (L.trace ? L.trace->masks_dev : nullptr);
  a.kcount = ws->kcount;
  a.tick = ws->tick;
  a.bar = ws->bar;
  a.y_flag = ws->y_flag;
  a.pred_partial = ws->pred_partial;
  a.pcnt = ws->pcnt;
  a.next_mixing = L.next_mixing;
  a.next_mixing_bytes = L.next_mixing_bytes;
  a.pf_tick = ws->pf_tick;

  a.n_kept_out = L.n_kept_out;
  a.kept_out = L.kept_out;
  a.stats = L.k1_only ? nullptr : ws->stats;
  a.place_acc = L.place_acc;
  a.phase_ns = ws->phase_ns;
  a.ns = ns;
  a.max_tiles = max_tiles;
  // test hook (tests/test_gpu_spec.py): invert the predicted logits so the
  // misprediction path of the layer kernel runs
  static const uint32_t dbg = [] {
    const char *d = std::getenv("FLOE_TEST_MISPREDICT");
    return (d && std::strcmp(d, "1") == 0) ? 8u : 0u;
  }();
  a.debug = dbg;
  static const uint32_t early_env = [] {
    const char *p = std::getenv("FLOE_EARLY");
    return p ? (uint32_t)std::atoi(p) : (uint32_t)V::kEarly;
  }();
  a.early = early_env;

  if (int rc = set_smem(V::fused<DH>, smem)) return rc;
  void *kargs[] = {&a};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(V::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[3];
  attr[0].id = cudaLaunchAttributeCooperative;  // grid barriers need co-residency
  attr[0].val.cooperative = 1;
  // programmatic dependent launch: back-to-back calls overlap the next
  // grid's prologue and weight prefetch with this one's drain
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  static const bool pdl_env = [] {
    const char *p = std::getenv("FLOE_PDL");
    return !(p && std::strcmp(p, "0") == 0);
  }();
  // Cooperative launch guarantees the co-residency the grid barriers need,
  // but the driver then does not overlap a launch with its predecessor (PDL
  // is ignored: 55.3 vs 52.5 us per layer, 32.8 vs 29.3 us per expert).
  // Without it the grid (one CTA per SM, G <= SMs, ~200 KB smem each) is
  // still co-resident: a PDL dependent only launches once EVERY CTA of its
  // primary has executed griddepcontrol.launch_dependents (issued at kernel
  // start), so a fused grid never competes for SMs with its successor.  What
  // the driver no longer rules out is another grid-barrier kernel holding SMs
  // concurrently (two fused launches on two streams, or an MPS SM limit):
  // there the barrier watchdog traps instead of hanging.  FLOE_COOP=1, or an
  // MPS client with an active-thread limit, keeps the cooperative launch.
  static const bool coop_env = [] {
    const char *p = std::getenv("FLOE_COOP");
    if (p) return std::strcmp(p, "0") != 0;
    return std::getenv("CUDA_MPS_ACTIVE_THREAD_PERCENTAGE") != nullptr;
  }();
  const bool use_pdl = pdl_env && !ws->profiling;
  cfg.attrs = coop_env ? attr : attr + 1;
  cfg.numAttrs = coop_env ? (use_pdl ? 2 : 1) : (use_pdl ? 1 : 0);
  // CTA pairs (clusters of 2) balance phase C over distributed shared memory;
  // 148 SMs hold 74 pairs at one CTA per SM.  FLOE_PAIRS=0 turns it off.
  static const bool pairs_env = [] {
    const char *p = std::getenv("FLOE_PAIRS");
    return !(p && std::strcmp(p, "0") == 0);
  }();
  a.paired = (pairs_env && !coop_env && (G % 2) == 0) ? 1 : 0;
  if (a.paired) {
    attr[cfg.numAttrs + 1].id = cudaLaunchAttributeClusterDimension;
    attr[cfg.numAttrs + 1].val.clusterDim.x = 2;
    attr[cfg.numAttrs + 1].val.clusterDim.y = 1;
    attr[cfg.numAttrs + 1].val.clusterDim.z = 1;
    ++cfg.numAttrs;
  }
  StageScope prof(ws, kStageFused, st);
  const cudaError_t e =
      cudaLaunchKernelExC(&cfg, reinterpret_cast<const void *>(V::fused<DH>), kargs);
  if (e != cudaSuccess)
    return fail(FLOE_ERR_CUDA, "fused launch failed: %s", cudaGetErrorString(e));
  CK_LAUNCH();
  return FLOE_OK;
}

int launch_v2(const FusedLaunch &L, floe_gpu_workspace *ws, cudaStream_t st) {
  if (L.slots > (uint32_t)floe_k::kMaxSlots || (L.mixing && L.n_experts > 32))
    return fail(FLOE_ERR_UNSUPPORTED, "fused path: at most 32 experts and 8 slots");
  if (L.dh == 4096) return launch_v2_dh<4096>(L, ws, st);
  if (L.dh == 2048) return launch_v2_dh<2048>(L, ws, st);
  return fail(FLOE_ERR_UNSUPPORTED, "fused path: d_hidden %u", L.dh);
}

int check_ws(const char *fn, const floe_gpu_workspace *ws, uint32_t dh, uint32_t di,
             uint32_t slots) {
  if (!ws) return fail(FLOE_ERR_INVALID, "%s: null workspace", fn);
  if (ws->dh < dh || ws->di < di || ws->slots < slots)
    return fail(FLOE_ERR_INVALID,
                "%s: workspace too small (have dh=%u di=%u slots=%u, need %u/%u/%u)", fn,
                ws->dh, ws->di, ws->slots, dh, di, slots);
  return FLOE_OK;
}

}  // namespace

// ===========================================================================
extern "C" {

const char *floe_gpu_last_error(void) { return g_err.c_str(); }
int floe_gpu_abi_version(void) { return FLOE_GPU_ABI_VERSION; }

int floe_gpu_device_info(int *sm_count, int *cc_major, int *cc_minor, size_t *total_mem) {
  const DeviceInfo &d = device_info();
  if (sm_count) *sm_count = d.sm;
  if (cc_major) *cc_major = d.major;
  if (cc_minor) *cc_minor = d.minor;
  if (total_mem) *total_mem = d.mem;
  if (!d.ok) return fail(FLOE_ERR_CUDA, "floe_gpu_device_info: %s", d.err.c_str());
  return FLOE_OK;
}

int floe_gpu_device_malloc(void **ptr, size_t bytes) {
  if (!ptr) return fail(FLOE_ERR_INVALID, "device_malloc: null argument");
  *ptr = nullptr;
  if (int rc = require_device("device_malloc")) return rc;
  if (bytes == 0) return FLOE_OK;
  CK(cudaMalloc(ptr, bytes));
  return FLOE_OK;
}

int floe_gpu_device_free(void *ptr) {
  if (ptr) CK(cudaFree(ptr));
  return FLOE_OK;
}

int floe_gpu_copy(void *dst, const void *src, size_t bytes, floe_stream_t stream) {
  if (bytes == 0) return FLOE_OK;
  if (!dst || !src) return fail(FLOE_ERR_INVALID, "copy: null argument");
  if (int rc = require_device("copy")) return rc;
  CK(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, S(stream)));
  CK(cudaStreamSynchronize(S(stream)));
  return FLOE_OK;
}

// ---------------------------------------------------------------- experts --
int floe_gpu_expert_create(const floe_expert_host_view *v, floe_gpu_expert **out) {
  if (!v || !out) return fail(FLOE_ERR_INVALID, "expert_create: null argument");
  *out = nullptr;
  if (int rc = require_device("expert_create")) return rc;
  if (v->d_hidden == 0 || v->d_intermediate == 0)
    return fail(FLOE_ERR_INVALID, "expert_create: all dimensions must be >= 1");
  if (!bits_ok(v->bits))
    return fail(FLOE_ERR_INVALID, "quantize: bits must be one of {1,2,3,4,8}");
  const uint64_t n = (uint64_t)v->d_hidden * v->d_intermediate;
  if (v->group_size == 0 || n % v->group_size != 0)
    return fail(FLOE_ERR_INVALID, "quantize: group_size must divide element count");
  if (!v->codes || !v->scales || !v->zeros)
    return fail(FLOE_ERR_INVALID, "expert_create: codes/scales/zeros required");
  const bool have_f32 = v->gate_f32 && v->down_f32;
  if (have_f32 && v->records_f16)
    return fail(FLOE_ERR_INVALID,
                "expert_create: give at most one of gate_f32+down_f32 or records_f16");
  if ((v->gate_f32 != nullptr) != (v->down_f32 != nullptr))
    return fail(FLOE_ERR_INVALID, "expert_create: gate_f32 and down_f32 go together");
  const bool up_only = !have_f32 && !v->records_f16;  // qgemv / predict_mask only
  const bool on_device = (v->flags & FLOE_VIEW_DEVICE) != 0;
  // Device-resident inputs may still be in flight on the caller's streams
  // (e.g. quantize just launched): creation is not a hot path, so wait.
  if (on_device) CK(cudaDeviceSynchronize());

  auto *e = new (std::nothrow) floe_gpu_expert();
  if (!e) return fail(FLOE_ERR_OOM, "expert_create: host allocation failed");
  e->dh = v->d_hidden;
  e->di = v->d_intermediate;
  e->bits = v->bits;
  e->g = v->group_size;
  e->threshold = v->threshold;
  e->code_bytes = packed_code_bytes(n, v->bits);
  e->n_groups = n / v->group_size;
  e->fast = fast_shape(e->dh, e->bits, e->g);

  // One allocation, 256-B aligned sections:
  //   fast:    [desc][tiles: ceil(di/16) x 5*dh B][records]
  //   generic: [desc][codes][scales][zeros][records]
  const uint64_t o_codes = up256(sizeof(ExpertDesc));
  const uint64_t tile_total = (uint64_t)floe_v2::tiles_per_expert(e->di) * floe_v2::tile_bytes(e->dh);
  const uint64_t o_scales = up256(o_codes + e->code_bytes);
  const uint64_t o_zeros = up256(o_scales + 2 * e->n_groups);
  const uint64_t o_rec = e->fast ? up256(o_codes + tile_total) : up256(o_zeros + 2 * e->n_groups);
  e->up_only = up_only;
  const uint64_t total = o_rec;  // records live in their own allocation (residency)
  cudaError_t ce = cudaMalloc(&e->block, total);
  if (ce != cudaSuccess) {
    delete e;
    return fail(FLOE_ERR_OOM, "expert_create: cudaMalloc(%llu) failed: %s",
                (unsigned long long)total, cudaGetErrorString(ce));
  }
  char *base = static_cast<char *>(e->block);
  e->dev_desc = reinterpret_cast<ExpertDesc *>(base);
  if (e->fast) {
    e->host_desc.tiles = reinterpret_cast<const uint32_t *>(base + o_codes);
  } else {
    e->host_desc.codes = reinterpret_cast<const uint8_t *>(base + o_codes);
    e->host_desc.scales = reinterpret_cast<const uint16_t *>(base + o_scales);
    e->host_desc.zeros = reinterpret_cast<const uint16_t *>(base + o_zeros);
  }
  if (!up_only) {
    ce = cudaMalloc(reinterpret_cast<void **>(&e->rec_dev), 4 * n);
    if (ce != cudaSuccess) {
      cudaFree(e->block);
      delete e;
      return fail(FLOE_ERR_OOM, "expert_create: cudaMalloc(records, %llu) failed: %s",
                  (unsigned long long)(4 * n), cudaGetErrorString(ce));
    }
  }
  e->host_desc.records = e->rec_dev;
  e->host_desc.host_records = 0;
  e->host_desc.threshold = v->threshold;

  auto cleanup = [&](int rc) {
    cudaFree(e->block);
    if (e->rec_dev) cudaFree(e->rec_dev);
    delete e;
    return rc;
  };
  cudaStream_t st;
  if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess)
    return cleanup(fail(FLOE_ERR_CUDA, "expert_create: stream creation failed"));
  cudaError_t err = cudaSuccess;
  auto cp = [&](void *dst, const void *src, size_t bytes) {
    if (err == cudaSuccess) err = cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDefault, st);
  };
  cp(e->dev_desc, &e->host_desc, sizeof(ExpertDesc));
  if (e->fast) {
    // stage the reference arrays on the device (unless they are there), then
    // build the tile-fragment layout
    const uint8_t *dc = v->codes;
    const uint16_t *dsc = v->scales, *dz = v->zeros;
    void *tmp = nullptr;
    if (!on_device && err == cudaSuccess) {
      const uint64_t tb = up256(e->code_bytes) + 2 * up256(2 * e->n_groups);
      err = cudaMalloc(&tmp, tb);
      if (err == cudaSuccess) {
        char *tc = static_cast<char *>(tmp);
        cp(tc, v->codes, e->code_bytes);
        cp(tc + up256(e->code_bytes), v->scales, 2 * e->n_groups);
        cp(tc + up256(e->code_bytes) + up256(2 * e->n_groups), v->zeros, 2 * e->n_groups);
        dc = reinterpret_cast<const uint8_t *>(tc);
        dsc = reinterpret_cast<const uint16_t *>(tc + up256(e->code_bytes));
        dz = reinterpret_cast<const uint16_t *>(tc + up256(e->code_bytes) + up256(2 * e->n_groups));
      }
    }
    if (err == cudaSuccess) {
      floe_v2::tile_up<<<1024, 256, 0, st>>>(dc, dsc, dz, e->dh, e->di, e->g,
                                             reinterpret_cast<uint32_t *>(base + o_codes));
      err = cudaGetLastError();
    }
    if (tmp) {
      if (err == cudaSuccess) err = cudaStreamSynchronize(st);
      cudaFree(tmp);
    }
  } else {
    cp(base + o_codes, v->codes, e->code_bytes);
    cp(base + o_scales, v->scales, 2 * e->n_groups);
    cp(base + o_zeros, v->zeros, 2 * e->n_groups);
  }
  __half *rec = e->rec_dev;
  if (up_only) {
    // nothing to upload
  } else if (v->records_f16) {
    cp(rec, v->records_f16, 4 * n);
  } else if (on_device) {
    if (err == cudaSuccess) {
      floe_k::pack_records<<<4096, 256, 0, st>>>(v->gate_f32, v->down_f32, e->dh, e->di, rec);
      err = cudaGetLastError();
    }
  } else {
    // Stage host f32 gate/down through a bounded device buffer, convert with RNE.
    const uint64_t chunk_ch = std::max<uint64_t>(1, (64ull << 20) / (8ull * e->dh));
    const uint64_t tmp_ch = std::min<uint64_t>(chunk_ch, e->di);
    float *tmp = nullptr;
    if (err == cudaSuccess) err = cudaMalloc(&tmp, 8ull * e->dh * tmp_ch);
    for (uint64_t c0 = 0; c0 < e->di && err == cudaSuccess; c0 += tmp_ch) {
      const uint64_t nc = std::min<uint64_t>(tmp_ch, e->di - c0);
      cp(tmp, v->gate_f32 + c0 * e->dh, 4ull * e->dh * nc);
      cp(tmp + (uint64_t)e->dh * tmp_ch, v->down_f32 + c0 * e->dh, 4ull * e->dh * nc);
      if (err == cudaSuccess) {
        floe_k::pack_records<<<1024, 256, 0, st>>>(tmp, tmp + (uint64_t)e->dh * tmp_ch, e->dh,
                                                   nc, rec + c0 * 2 * e->dh);
        err = cudaGetLastError();
      }
      if (err == cudaSuccess) err = cudaStreamSynchronize(st);  // tmp reused next chunk
    }
    if (tmp) cudaFree(tmp);
  }
  if (err == cudaSuccess) err = cudaStreamSynchronize(st);
  cudaStreamDestroy(st);
  if (err != cudaSuccess)
    return cleanup(fail(FLOE_ERR_CUDA, "expert_create: upload failed: %s",
                        cudaGetErrorString(err)));
  *out = e;
  if ((v->flags & FLOE_VIEW_HOST_RECORDS) && !up_only) {
    if (int rc = floe_gpu_expert_set_resident(e, 0, nullptr)) {
      *out = nullptr;
      floe_gpu_expert_destroy(e);
      return rc;
    }
    if (cudaDeviceSynchronize() != cudaSuccess)
      return fail(FLOE_ERR_CUDA, "expert_create: host-resident demotion failed");
  }
  return FLOE_OK;
}

// Residency of the gate|down records (the host-resident decode of SURVEY
// config 3; ExpertCache entries of core/src/offload.cpp:89-159 at expert
// granularity).  Stream-ordered: the copy, the descriptor switch (expert and
// every layer table holding it) and the release of the old copy all run on
// `stream`, so kernels on `stream` see either placement consistently.
int floe_gpu_expert_set_resident(floe_gpu_expert *e, int resident, floe_stream_t stream) {
  if (!e) return fail(FLOE_ERR_INVALID, "expert_set_resident: null expert");
  if (e->up_only) return fail(FLOE_ERR_INVALID, "expert_set_resident: expert has no gate/down");
  const bool want = resident != 0;
  if (want == e->resident) return FLOE_OK;
  cudaStream_t st = S(stream);
  const uint64_t bytes = 4ull * e->dh * e->di;
  if (!want) {
    if (!e->rec_host) {
      CK(cudaHostAlloc(reinterpret_cast<void **>(&e->rec_host), bytes,
                       cudaHostAllocMapped | cudaHostAllocPortable));
      CK(cudaMemcpyAsync(e->rec_host, e->rec_dev, bytes, cudaMemcpyDeviceToHost, st));
    }
    void *dptr = nullptr;
    CK(cudaHostGetDevicePointer(&dptr, e->rec_host, 0));
    e->host_desc.records = static_cast<const __half *>(dptr);
    e->host_desc.host_records = 1;
  } else {
    CK(cudaMallocAsync(reinterpret_cast<void **>(&e->rec_dev), bytes, st));
    CK(cudaMemcpyAsync(e->rec_dev, e->rec_host, bytes, cudaMemcpyHostToDevice, st));
    e->host_desc.records = e->rec_dev;
    e->host_desc.host_records = 0;
  }
  CK(cudaMemcpyAsync(e->dev_desc, &e->host_desc, sizeof(ExpertDesc), cudaMemcpyHostToDevice, st));
  for (ExpertDesc *t : e->tables)
    CK(cudaMemcpyAsync(t, &e->host_desc, sizeof(ExpertDesc), cudaMemcpyHostToDevice, st));
  if (!want) {
    CK(cudaFreeAsync(e->rec_dev, st));
    e->rec_dev = nullptr;
  }
  e->resident = want;
  return FLOE_OK;
}

int floe_gpu_expert_residency(const floe_gpu_expert *e, int *resident, uint64_t *device_bytes) {
  if (!e) return fail(FLOE_ERR_INVALID, "expert_residency: null expert");
  if (resident) *resident = e->resident ? 1 : 0;
  if (device_bytes)
    *device_bytes = (e->resident && !e->up_only) ? 4ull * e->dh * e->di : 0ull;
  return FLOE_OK;
}

int floe_gpu_expert_destroy(floe_gpu_expert *e) {
  if (!e) return FLOE_OK;
  cudaDeviceSynchronize();  // stream-ordered residency changes may be in flight
  cudaFree(e->block);
  if (e->rec_dev) cudaFree(e->rec_dev);
  if (e->rec_host) cudaFreeHost(e->rec_host);
  delete e;
  return FLOE_OK;
}

int floe_gpu_expert_info(const floe_gpu_expert *e, floe_expert_info *info) {
  if (!e || !info) return fail(FLOE_ERR_INVALID, "expert_info: null argument");
  info->d_hidden = e->dh;
  info->d_intermediate = e->di;
  info->bits = e->bits;
  info->group_size = e->g;
  info->threshold = e->threshold;
  info->code_bytes = e->code_bytes;
  info->meta_bytes = 4 * e->n_groups;
  info->record_bytes = 4ull * e->dh;
  info->fast_path = e->fast ? 1 : 0;
  return FLOE_OK;
}

int floe_gpu_expert_set_threshold(floe_gpu_expert *e, float t) {
  if (!e) return fail(FLOE_ERR_INVALID, "expert_set_threshold: null expert");
  // Not a hot-path call: drain every stream first (kernels in flight may read
  // the descriptors), then update the expert's own descriptor AND every layer
  // table entry that copies it, so layer_forward and expert_forward_sparse
  // see the same threshold (ThresholdTable is per expert, model.cpp:237).
  CK(cudaDeviceSynchronize());
  e->threshold = t;
  e->host_desc.threshold = t;
  CK(cudaMemcpy(e->dev_desc, &e->host_desc, sizeof(ExpertDesc), cudaMemcpyHostToDevice));
  for (ExpertDesc *tab : e->tables)
    CK(cudaMemcpy(tab, &e->host_desc, sizeof(ExpertDesc), cudaMemcpyHostToDevice));
  return FLOE_OK;
}

// The expert's quantized up projection in the reference packing (the tile
// layout re-packed on the device) and its threshold: what a record-cache file
// or a FLOQ writer needs.  Synchronous.
int floe_gpu_expert_download(const floe_gpu_expert *e, uint8_t *codes_host, uint16_t *scales_host,
                             uint16_t *zeros_host, float *threshold) {
  if (!e || !codes_host || !scales_host || !zeros_host)
    return fail(FLOE_ERR_INVALID, "expert_download: null argument");
  if (int rc = require_device("expert_download")) return rc;
  if (threshold) *threshold = e->threshold;
  if (!e->fast) {
    CK(cudaMemcpy(codes_host, e->host_desc.codes, e->code_bytes, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(scales_host, e->host_desc.scales, 2 * e->n_groups, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(zeros_host, e->host_desc.zeros, 2 * e->n_groups, cudaMemcpyDeviceToHost));
    return FLOE_OK;
  }
  uint8_t *buf = nullptr;
  const uint64_t nb = e->code_bytes + 4 * e->n_groups;
  CK(cudaMalloc(&buf, nb));
  uint16_t *sc = reinterpret_cast<uint16_t *>(buf + e->code_bytes), *zr = sc + e->n_groups;
  floe_v2::untile_up<<<1184, 256>>>(e->host_desc.tiles, e->dh, e->di, e->g, buf, sc, zr);
  cudaError_t ce = cudaGetLastError();
  if (ce == cudaSuccess) ce = cudaMemcpy(codes_host, buf, e->code_bytes, cudaMemcpyDeviceToHost);
  if (ce == cudaSuccess) ce = cudaMemcpy(scales_host, sc, 2 * e->n_groups, cudaMemcpyDeviceToHost);
  if (ce == cudaSuccess) ce = cudaMemcpy(zeros_host, zr, 2 * e->n_groups, cudaMemcpyDeviceToHost);
  cudaFree(buf);
  if (ce != cudaSuccess) return fail(FLOE_ERR_CUDA, "expert_download: %s", cudaGetErrorString(ce));
  return FLOE_OK;
}

// -------------------------------------------------------------- workspace --
int floe_gpu_workspace_create(uint32_t dh, uint32_t di, uint32_t slots,
                              floe_gpu_workspace **out) {
  if (!out) return fail(FLOE_ERR_INVALID, "workspace_create: null argument");
  *out = nullptr;
  if (int rc = require_device("workspace_create")) return rc;
  if (dh == 0 || di == 0 || slots == 0 || slots > (uint32_t)floe_k::kMaxSlots)
    return fail(FLOE_ERR_INVALID, "workspace_create: need dh, di >= 1 and 1 <= slots <= %d",
                floe_k::kMaxSlots);
  auto *w = new (std::nothrow) floe_gpu_workspace();
  if (!w) return fail(FLOE_ERR_OOM, "workspace_create: host allocation failed");
  w->dh = dh;
  w->di = di;
  w->slots = slots;
  const uint64_t sd = (uint64_t)slots * di;
  const int MS = floe_k::kMaxSlots;
  uint64_t o = 0;
  const uint64_t o_idx = o;   o = up256(o + 4 * sd);
  const uint64_t o_kv = o;    o = up256(o + 4 * sd);
  const uint64_t o_cnt = o;   o = up256(o + 4ull * MS * kMaxSeg);
  const uint64_t o_mp = o;    o = up256(o + 4ull * 32 * std::max<uint64_t>(1024, (dh + 7) / 8));
  const uint64_t o_md = o;    o = up256(o + 16);
  const uint64_t o_st = o;    o = up256(o + 32);  // stats[2], grid barrier counter
  const uint64_t o_fk = o;    o = up256(o + 40 + 4ull * MS);  // tick, y flag[2], pcnt, pf_tick, kcount[MS]
  const uint64_t o_pp = o;    o = up256(o + 4ull * 32 * floe_v2::kMaxGrid);
  const uint64_t o_sel = o;   o = up256(o + 4 * MS);
  const uint64_t o_w = o;     o = up256(o + 4 * MS);
  const uint64_t o_u = o;     o = up256(o + 4ull * dh);
  const uint64_t o_x = o;     o = up256(o + 4ull * dh);
  const uint64_t o_y = o;     o = up256(o + 4ull * dh);
  const uint64_t o_v = o;     o = up256(o + 4 * sd);
  const uint64_t o_m = o;     o = up256(o + sd);
  cudaError_t ce = cudaMalloc(&w->block, o);
  if (ce != cudaSuccess) {
    delete w;
    return fail(FLOE_ERR_OOM, "workspace_create: cudaMalloc failed: %s", cudaGetErrorString(ce));
  }
  char *b = static_cast<char *>(w->block);
  w->kept_idx = reinterpret_cast<uint32_t *>(b + o_idx);
  w->kept_v = reinterpret_cast<float *>(b + o_kv);
  w->seg_count = reinterpret_cast<uint32_t *>(b + o_cnt);
  w->mix_partial = reinterpret_cast<float *>(b + o_mp);
  w->mix_done = reinterpret_cast<uint32_t *>(b + o_md);
  w->stats = reinterpret_cast<unsigned long long *>(b + o_st);
  w->bar = w->stats + 2;
  w->lbar = w->stats + 3;
  w->tick = reinterpret_cast<unsigned long long *>(b + o_fk);
  w->y_flag = w->tick + 1;
  w->pcnt = w->tick + 3;
  w->pf_tick = w->tick + 4;
  w->kcount = reinterpret_cast<uint32_t *>(w->tick + 5);
  w->pred_partial = reinterpret_cast<float *>(b + o_pp);
  w->sel = reinterpret_cast<uint32_t *>(b + o_sel);
  w->weights = reinterpret_cast<float *>(b + o_w);
  w->u = reinterpret_cast<float *>(b + o_u);
  w->x = reinterpret_cast<float *>(b + o_x);
  w->y = reinterpret_cast<float *>(b + o_y);
  w->v = reinterpret_cast<float *>(b + o_v);
  w->mask = reinterpret_cast<uint8_t *>(b + o_m);
  ce = cudaMemset(w->block, 0, o);
  if (ce == cudaSuccess) ce = cudaMallocHost(&w->hx, 4ull * dh);
  if (ce == cudaSuccess) ce = cudaMallocHost(&w->hy, 4ull * dh);
  if (ce == cudaSuccess) ce = cudaMallocHost(&w->hv, 4 * sd);
  if (ce == cudaSuccess) ce = cudaMallocHost(reinterpret_cast<void **>(&w->hmask), sd);
  if (ce == cudaSuccess) ce = cudaMallocHost(reinterpret_cast<void **>(&w->hstats), 16);
  if (ce == cudaSuccess) ce = cudaDeviceSynchronize();
  if (ce != cudaSuccess) {
    floe_gpu_workspace_destroy(w);
    return fail(FLOE_ERR_OOM, "workspace_create: %s", cudaGetErrorString(ce));
  }
  *out = w;
  return FLOE_OK;
}

int floe_gpu_workspace_destroy(floe_gpu_workspace *w) {
  if (!w) return FLOE_OK;
  for (auto &p : w->pending) {
    cudaEventDestroy(p.a);
    cudaEventDestroy(p.b);
  }
  for (auto e : w->pool) cudaEventDestroy(e);
  if (w->block) cudaFree(w->block);
  if (w->hx) cudaFreeHost(w->hx);
  if (w->hy) cudaFreeHost(w->hy);
  if (w->hv) cudaFreeHost(w->hv);
  if (w->hmask) cudaFreeHost(w->hmask);
  if (w->hstats) cudaFreeHost(w->hstats);
  if (w->phase_ns) cudaFree(w->phase_ns);
  delete w;
  return FLOE_OK;
}

int floe_gpu_workspace_reset_counters(floe_gpu_workspace *w, floe_stream_t stream) {
  if (!w) return fail(FLOE_ERR_INVALID, "workspace_reset_counters: null workspace");
  CK(cudaMemsetAsync(w->stats, 0, 16, S(stream)));
  return FLOE_OK;
}

int floe_gpu_workspace_read_counters(floe_gpu_workspace *w, uint64_t *calls,
                                     uint64_t *kept_total, floe_stream_t stream) {
  if (!w) return fail(FLOE_ERR_INVALID, "workspace_read_counters: null workspace");
  CK(cudaMemcpyAsync(w->hstats, w->stats, 16, cudaMemcpyDeviceToHost, S(stream)));
  CK(cudaStreamSynchronize(S(stream)));
  if (calls) *calls = w->hstats[0];
  if (kept_total) *kept_total = w->hstats[1];
  return FLOE_OK;
}

int floe_gpu_workspace_set_phase_trace(floe_gpu_workspace *w, int enable) {
  if (!w) return fail(FLOE_ERR_INVALID, "workspace_set_phase_trace: null workspace");
  if (enable && !w->phase_ns) {
    CK(cudaMalloc(&w->phase_ns, 8ull * floe_v2::kTraceSlots * device_info().sm));
    CK(cudaMemset(w->phase_ns, 0, 8ull * floe_v2::kTraceSlots * device_info().sm));
  } else if (!enable && w->phase_ns) {
    cudaFree(w->phase_ns);
    w->phase_ns = nullptr;
  }
  return FLOE_OK;
}

int floe_gpu_workspace_read_phase_trace(floe_gpu_workspace *w, uint64_t *out, uint32_t cap,
                                        uint32_t *grid) {
  if (!w || !out) return fail(FLOE_ERR_INVALID, "workspace_read_phase_trace: null argument");
  const uint32_t n = std::min<uint32_t>(cap, (uint32_t)floe_v2::kTraceSlots * device_info().sm);
  if (grid) *grid = device_info().sm;
  if (!w->phase_ns) return fail(FLOE_ERR_INVALID, "workspace_read_phase_trace: tracing is off");
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out, w->phase_ns, 8ull * n, cudaMemcpyDeviceToHost));
  CK(cudaMemset(w->phase_ns, 0, 8ull * floe_v2::kTraceSlots * device_info().sm));  // fresh marks
  return FLOE_OK;
}

int floe_gpu_workspace_set_profiling(floe_gpu_workspace *w, int enable) {
  if (!w) return fail(FLOE_ERR_INVALID, "workspace_set_profiling: null workspace");
  w->profiling = enable != 0;
  return FLOE_OK;
}

int floe_gpu_workspace_read_profile(floe_gpu_workspace *w, double *ms, uint64_t *launches) {
  if (!w) return fail(FLOE_ERR_INVALID, "workspace_read_profile: null workspace");
  for (auto &p : w->pending) {
    CK(cudaEventSynchronize(p.b));
    float t = 0.0f;
    CK(cudaEventElapsedTime(&t, p.a, p.b));
    w->ms[p.stage] += t;
    w->launches[p.stage] += 1;
    w->pool.push_back(p.a);
    w->pool.push_back(p.b);
  }
  w->pending.clear();
  for (int s = 0; s < kStages; ++s) {
    if (ms) ms[s] = w->ms[s];
    if (launches) launches[s] = w->launches[s];
    w->ms[s] = 0.0;
    w->launches[s] = 0;
  }
  return FLOE_OK;
}

// --------------------------------------------------------------- hot path --
int floe_gpu_expert_forward_sparse(const floe_gpu_expert *e, floe_gpu_workspace *ws,
                                   const float *x, float *y, float *v_out,
                                   uint8_t *mask_out, uint32_t *kept_out,
                                   uint32_t *n_kept_out, floe_stream_t stream) {
  if (!e || !x || !y) return fail(FLOE_ERR_INVALID, "expert_forward_sparse: null argument");
  if (e->up_only)
    return fail(FLOE_ERR_INVALID, "expert_forward_sparse: expert was created without gate/down");
  if (int rc = check_ws("expert_forward_sparse", ws, e->dh, e->di, 1)) return rc;
  if (e->fast) {
    FusedLaunch f{};
    f.table = e->dev_desc;
    f.slots = 1;
    f.dh = e->dh;
    f.di = e->di;
    f.x = x;
    f.y = y;
    f.v_out = v_out;
    f.mask_out = mask_out;
    f.n_kept_out = n_kept_out;
    f.kept_out = kept_out;
    return launch_v2(f, ws, S(stream));
  }
  K1Launch k1{e->dev_desc, nullptr, 1, e->dh, e->di, e->bits, e->g, 0, 0.0f,
              x, v_out, mask_out, y};
  if (int rc = launch_k1(k1, ws, S(stream))) return rc;
  K2Launch k2{e->dev_desc, nullptr, nullptr, 1, e->dh, e->di, x, y, n_kept_out, kept_out};
  return launch_k2(k2, ws, S(stream));
}

int floe_gpu_expert_forward_sparse_host(const floe_gpu_expert *e, floe_gpu_workspace *ws,
                                        const float *x_host, float *y_host, float *v_host,
                                        uint8_t *mask_host, floe_stream_t stream) {
  if (!e || !x_host || !y_host)
    return fail(FLOE_ERR_INVALID, "expert_forward_sparse: null argument");
  if (int rc = check_ws("expert_forward_sparse", ws, e->dh, e->di, 1)) return rc;
  cudaStream_t st = S(stream);
  std::memcpy(ws->hx, x_host, 4ull * e->dh);
  CK(cudaMemcpyAsync(ws->x, ws->hx, 4ull * e->dh, cudaMemcpyHostToDevice, st));
  if (int rc = floe_gpu_expert_forward_sparse(e, ws, ws->x, ws->y, v_host ? ws->v : nullptr,
                                              mask_host ? ws->mask : nullptr, nullptr,
                                              nullptr, stream))
    return rc;
  CK(cudaMemcpyAsync(ws->hy, ws->y, 4ull * e->dh, cudaMemcpyDeviceToHost, st));
  if (v_host) CK(cudaMemcpyAsync(ws->hv, ws->v, 4ull * e->di, cudaMemcpyDeviceToHost, st));
  if (mask_host) CK(cudaMemcpyAsync(ws->hmask, ws->mask, e->di, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::memcpy(y_host, ws->hy, 4ull * e->dh);
  if (v_host) std::memcpy(v_host, ws->hv, 4ull * e->di);
  if (mask_host) std::memcpy(mask_host, ws->hmask, e->di);
  return FLOE_OK;
}

int floe_gpu_qgemv_channels(const floe_gpu_expert *e, floe_gpu_workspace *ws,
                            const float *x, float *v_out, floe_stream_t stream) {
  if (!e || !x || !v_out) return fail(FLOE_ERR_INVALID, "qgemv_channels: null argument");
  if (int rc = check_ws("qgemv_channels", ws, e->dh, e->di, 1)) return rc;
  if (e->fast) {
    FusedLaunch f{};
    f.table = e->dev_desc;
    f.slots = 1;
    f.dh = e->dh;
    f.di = e->di;
    f.k1_only = true;
    f.use_thr = 1;
    f.thr = __builtin_inff();  // nothing kept: v only
    f.x = x;
    f.v_out = v_out;
    return launch_v2(f, ws, S(stream));
  }
  K1Launch k1{e->dev_desc, nullptr, 1, e->dh, e->di, e->bits, e->g, 1,
              __builtin_inff(), x, v_out, nullptr, nullptr};
  return launch_k1(k1, ws, S(stream));
}

}  // extern "C"
namespace {
template <int DH>
int launch_batched(const floe_tc::BatchedArgs &a, cudaStream_t st) {
  const floe_tc::BatchedSmem L = floe_tc::batched_smem(DH, a.B);
  if (int rc = set_smem(floe_tc::k1_batched<DH>, L.total)) return rc;
  const uint32_t blocks = (a.di + floe_tc::kRows - 1) / floe_tc::kRows;
  floe_tc::k1_batched<DH><<<blocks, floe_tc::kBThreads, L.total, st>>>(a);
  CK_LAUNCH();
  return FLOE_OK;
}
// Small batches (<= floe_k1b::kMaxTokens): the IMMA kernel, 8 tokens per pass.
// Returns FLOE_ERR_UNSUPPORTED (nothing launched) when the layout does not fit
// shared memory; the caller then takes the tcgen05 kernel.
size_t k1b_smem(uint32_t dh, uint32_t di, uint32_t *grid) {
  const uint32_t NI = (di + 15u) / 16u * floe_k1b::kItems;
  const uint32_t G = std::min<uint32_t>((uint32_t)device_info().sm, NI);
  if (grid) *grid = G;
  return floe_k1b::smem_layout(dh, floe_k1b::tiles_per_cta(di, G)).total;
}
constexpr size_t kK1bSmemMax = 220u * 1024u;
template <int DH>
int launch_k1b(const floe_gpu_expert *e, const float *x, uint32_t B, float *v_out, float *invS,
               uint8_t *xt, float *xs, cudaStream_t st) {
  uint32_t G = 0;
  const size_t sm = k1b_smem(DH, e->di, &G);
  if (int rc = set_smem(floe_k1b::k1<DH>, sm)) return rc;
  for (uint32_t p0 = 0; p0 < B; p0 += floe_k1b::kTok) {
    const uint32_t nb = std::min<uint32_t>(floe_k1b::kTok, B - p0);
    floe_k1b::limbs<DH><<<DH / 64, 256, 0, st>>>(x + (size_t)p0 * DH, nb, invS + p0, xt, xs,
                                             v_out + (size_t)p0 * e->di, e->di, G);
    floe_k1b::Args a{e->host_desc.tiles, e->di, nb, xt, xs, invS + p0, v_out + (size_t)p0 * e->di,
                     nullptr};
    static const bool trace = std::getenv("FLOE_K1B_TRACE") != nullptr;
    if (trace) {
      CK(cudaMalloc(&a.trace, 8ull * 8 * G));
      CK(cudaMemsetAsync(a.trace, 0, 8ull * 8 * G, st));
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(G);
    cfg.blockDim = dim3(floe_k1b::kThreads);
    cfg.dynamicSmemBytes = sm;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;  // tiles stream during limbs()
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, floe_k1b::k1<DH>, a));
    if (trace) {  // diagnostics: per-CTA marks (us) from the first CTA start
      std::vector<unsigned long long> h(8ull * G);
      CK(cudaStreamSynchronize(st));
      CK(cudaMemcpy(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost));
      unsigned long long t0 = ~0ull;
      for (uint32_t b = 0; b < G; ++b) t0 = std::min(t0, h[8ull * b]);
      for (uint32_t b : {0u, G / 3, G / 2, G - 1}) {
        std::fprintf(stderr, "[k1b] cta %u:", b);
        for (int k = 0; k < 6; ++k) std::fprintf(stderr, " %d:%.2f", k, (h[8ull * b + k] - t0) / 1e3);
        std::fprintf(stderr, "\n");
      }
      double mx[6] = {0};
      for (uint32_t b = 0; b < G; ++b)
        for (int k = 0; k < 6; ++k) mx[k] = std::max(mx[k], (h[8ull * b + k] - t0) / 1e3);
      std::fprintf(stderr, "[k1b] max: %.2f %.2f %.2f %.2f %.2f %.2f\n", mx[0], mx[1], mx[2], mx[3], mx[4], mx[5]);
      cudaFree(a.trace);
    }
  }
  CK_LAUNCH();
  return FLOE_OK;
}
// Gate/down stage of the batched expert forward (after the batched K1 wrote
// v): union of kept channels, gate dots (tcgen05 GEMM or CUDA-core warps),
// down product (tcgen05 GEMM or CUDA-core tiles) into y.  Scratch layout as
// floe_gpu_expert_forward_batched documents.
template <int DH>
int batched_gate_down(const floe_gpu_expert *e, const float *x, uint32_t B, float *y_out,
                      const float *v, uint8_t *scratch, size_t o_xh, size_t o_g, bool tc_gate,
                      bool tc_down, uint32_t gate_split, cudaStream_t st) {
  const uint32_t di = e->di;
  const size_t o_v = 256, o_uc = o_v + ((4ull * B * di + 255) & ~size_t(255));
  const size_t o_um = o_uc + ((4ull * di + 255) & ~size_t(255));
  const size_t o_a = o_um + 8ull * di;
  uint32_t *count = reinterpret_cast<uint32_t *>(scratch);
  uint32_t *uc = reinterpret_cast<uint32_t *>(scratch + o_uc);
  unsigned long long *um = reinterpret_cast<unsigned long long *>(scratch + o_um);
  float *A = reinterpret_cast<float *>(scratch + o_a);
  uint8_t *xh = scratch + o_xh;
  float *Gp = reinterpret_cast<float *>(scratch + o_g);
  float *xsc = reinterpret_cast<float *>(scratch + o_g + 4ull * di * B);
  float *inv_xsc = xsc + floe_tc::kMaxTokens;
  uint32_t *amax = reinterpret_cast<uint32_t *>(inv_xsc + floe_tc::kMaxTokens);
  const int sm = device_info().sm;
  CK(cudaMemsetAsync(count, 0, 4, st));
  // <= 4 tokens on the CUDA cores: the fused union kernel (one pass over the
  // records through a bulk-copy ring; FLOE_UNION_FUSED=0 keeps the two-kernel
  // coeffs + down_accum path)
  static const bool union_fused = [] {
    const char *p = std::getenv("FLOE_UNION_FUSED");
    return !(p && std::strcmp(p, "0") == 0);
  }();
  // up to 8 tokens in groups of <= 4, each group over its own union (a group's
  // union is smaller than the batch's: 4 tokens keep ~59% of the channels at
  // k = 0.8, 8 tokens ~83%)
  const bool fused = union_fused && !tc_gate && !tc_down && B <= 2u * floe_tc::kUTok &&
                     di <= (uint32_t)sm * floe_tc::kUMaxRows;
  if (fused) {
    const __half *rec = e->host_desc.records;
    const uint32_t usm = floe_tc::kUStages * 4u * DH;
    // records per barrier batch: 8 (FLOE_UNION_UR=4: 4; 16 tokens per layer
    // call 0.65 -> 0.64 ms with 8)
    static const bool ur8 = [] {
      const char *p = std::getenv("FLOE_UNION_UR");
      return !(p && std::atoi(p) == 4);
    }();
    auto kern = ur8 ? floe_tc::union_ffn<DH, 8> : floe_tc::union_ffn<DH, 4>;
    if (int rc = set_smem(kern, usm)) return rc;
    CK(cudaMemsetAsync(y_out, 0, 4ull * B * DH, st));
    for (uint32_t g0 = 0; g0 < B; g0 += floe_tc::kUTok) {
      const uint32_t nb = std::min<uint32_t>(floe_tc::kUTok, B - g0);
      if (g0) CK(cudaMemsetAsync(count, 0, 4, st));
      floe_tc::union_masks<<<(di + 255) / 256, 256, 0, st>>>(v + (size_t)g0 * di, nb, di,
                                                             e->host_desc.threshold, count, uc, um);
      kern<<<sm, floe_tc::kUThreads, usm, st>>>(
          rec, x + (size_t)g0 * DH, v + (size_t)g0 * di, nb, di, count, uc, um, y_out + (size_t)g0 * DH);
      CK_LAUNCH();
    }
    return FLOE_OK;
  }
  floe_tc::hilo_token_scale<<<B, 256, 0, st>>>(x, DH, xsc, inv_xsc, amax);
  CK_LAUNCH();
  floe_tc::union_masks<<<(di + 255) / 256, 256, 0, st>>>(v, B, di, e->host_desc.threshold, count,
                                                         uc, um);
  CK_LAUNCH();
  const __half *rec = e->host_desc.records;
  if (tc_gate) {
    floe_tc::x_hilo<<<DH / 64, 256, 0, st>>>(x, DH, B, xsc, xh);
    CK_LAUNCH();
    const uint32_t gsm = floe_tc::kGemmStages * (16384u + floe_tc::gemm_n(B) * 128u);
    if (int rc = set_smem(floe_tc::gate_gemm<DH>, gsm)) return rc;
    CK(cudaMemsetAsync(Gp, 0, 4ull * di * B, st));
    floe_tc::gate_gemm<DH><<<dim3((di + 127) / 128, gate_split), 128, gsm, st>>>(
        rec, xh, v, B, di, count, uc, um, A, Gp, inv_xsc, amax);
    CK_LAUNCH();
    floe_tc::gate_finish<<<4 * sm, 256, 0, st>>>(Gp, v, B, di, count, uc, um, A, amax);
    CK_LAUNCH();
  } else {
    floe_tc::coeffs<DH><<<4 * sm, 256, 0, st>>>(rec, x, v, B, di, count, uc, um, A,
                                                tc_down ? amax : nullptr);
    CK_LAUNCH();
  }
  CK(cudaMemsetAsync(y_out, 0, 4ull * B * DH, st));
  if (tc_down) {
    const uint32_t gsm = floe_tc::kDownStages * (128u * floe_tc::kDownKChunk * 2u +
                                                 floe_tc::kDownKChunk * 256u * 2u);
    if (int rc = set_smem(floe_tc::down_gemm<DH>, gsm)) return rc;
    floe_tc::down_gemm<DH><<<dim3(DH / 256, (di + floe_tc::kDownKRange - 1) / floe_tc::kDownKRange),
                             128, gsm, st>>>(rec, B, count, uc, A, y_out, amax);
  } else {
    // row chunks of <= kDownRowCap union rows (the union is at most di)
    const uint32_t chunks = (di + floe_tc::kDownRowCap - 1) / floe_tc::kDownRowCap;
    const uint32_t dsm = 4u * floe_tc::kDownRowCap * ((B + 3u) & ~3u);
    if (int rc = set_smem(floe_tc::down_accum<DH>, dsm)) return rc;
    floe_tc::down_accum<DH><<<dim3(DH / 1024, chunks), 256, dsm, st>>>(rec, B, count, uc, A, y_out);
  }
  CK_LAUNCH();
  return FLOE_OK;
}

}  // namespace
extern "C" {

int floe_gpu_qgemv_channels_batched(const floe_gpu_expert *e, const float *x, uint32_t n_tokens,
                                    float *v_out, floe_stream_t stream) {
  if (!e || !x || !v_out) return fail(FLOE_ERR_INVALID, "qgemv_channels_batched: null argument");
  if (n_tokens == 0) return FLOE_OK;
  if (n_tokens > (uint32_t)floe_tc::kMaxTokens)
    return fail(FLOE_ERR_INVALID, "qgemv_channels_batched: at most %d tokens", floe_tc::kMaxTokens);
  if (!e->fast)
    return fail(FLOE_ERR_UNSUPPORTED,
                "qgemv_channels_batched: needs the tile layout (bits 2, d_hidden 2048/4096, g %% 64 == 0)");
  if (int rc = require_device("qgemv_channels_batched")) return rc;
  cudaStream_t st = S(stream);
  // up to 16 tokens: the IMMA kernel (floe_k1b.cuh); FLOE_K1_IMMA_MAX moves
  // the switch (0: always the tcgen05 kernel)
  static const uint32_t imma_max = [] {
    const char *p = std::getenv("FLOE_K1_IMMA_MAX");
    return p ? (uint32_t)std::atoi(p) : (uint32_t)floe_k1b::kDefaultMax;
  }();
  if (n_tokens <= std::min<uint32_t>(imma_max, floe_k1b::kMaxTokens) &&
      k1b_smem(e->dh, e->di, nullptr) <= kK1bSmemMax) {
    keep_pool();
    const size_t o_xs = 256, o_xt = (o_xs + floe_k1b::xs_bytes(e->dh) + 1023) & ~size_t(1023);
    uint8_t *scratch = nullptr;  // invS | xs | xt (stream-ordered)
    CK(cudaMallocAsync(reinterpret_cast<void **>(&scratch), o_xt + floe_k1b::xt_bytes(e->dh), st));
    float *invS = reinterpret_cast<float *>(scratch);
    const int rc = e->dh == 4096
                       ? launch_k1b<4096>(e, x, n_tokens, v_out, invS, scratch + o_xt,
                                          reinterpret_cast<float *>(scratch + o_xs), st)
                       : launch_k1b<2048>(e, x, n_tokens, v_out, invS, scratch + o_xt,
                                          reinterpret_cast<float *>(scratch + o_xs), st);
    cudaFreeAsync(scratch, st);
    return rc;
  }
  const uint32_t Bp = floe_tc::padded_tokens(n_tokens), spans = e->dh / 64;
  const size_t xl_bytes = (size_t)spans * floe_tc::xl_span_bytes(n_tokens);
  const size_t xs_bytes = 4ull * spans * Bp;
  keep_pool();
  uint8_t *scratch = nullptr;  // S | invS | xs | xl (stream-ordered)
  const size_t o_inv = 256, o_xs = 512, o_xl = (o_xs + xs_bytes + 1023) & ~size_t(1023);
  CK(cudaMallocAsync(reinterpret_cast<void **>(&scratch), o_xl + xl_bytes, st));
  float *Sv = reinterpret_cast<float *>(scratch), *invS = reinterpret_cast<float *>(scratch + o_inv);
  float *xs = reinterpret_cast<float *>(scratch + o_xs);
  uint8_t *xl = scratch + o_xl;
  floe_tc::token_scale<<<n_tokens, 256, 0, st>>>(x, e->dh, invS, Sv);
  floe_tc::token_limbs<<<spans, 256, 0, st>>>(x, e->dh, n_tokens, Sv, xl, xs);
  if (cudaError_t le = cudaGetLastError(); le != cudaSuccess) {
    cudaFreeAsync(scratch, st);
    return fail(FLOE_ERR_CUDA, "qgemv_channels_batched: launch failed: %s", cudaGetErrorString(le));
  }
  floe_tc::BatchedArgs a{};
  a.tiles = e->host_desc.tiles;
  a.dh = e->dh;
  a.di = e->di;
  a.B = n_tokens;
  a.xl = xl;
  a.xs = xs;
  a.invS = invS;
  a.v = v_out;
  static const bool tc_trace = std::getenv("FLOE_TC_TRACE") != nullptr;
  const uint32_t blocks = (e->di + floe_tc::kRows - 1) / floe_tc::kRows;
  if (tc_trace) CK(cudaMalloc(&a.trace, 8ull * 32 * blocks));
  if (tc_trace) CK(cudaMemset(a.trace, 0, 8ull * 32 * blocks));
  const int rc = e->dh == 4096 ? launch_batched<4096>(a, st) : launch_batched<2048>(a, st);
  CK(cudaFreeAsync(scratch, st));
  if (tc_trace && rc == FLOE_OK) {  // diagnostics: per-CTA marks relative to the first start
    std::vector<unsigned long long> h(32ull * blocks);
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(h.data(), a.trace, h.size() * 8, cudaMemcpyDeviceToHost));
    unsigned long long t0 = ~0ull;
    for (uint32_t b = 0; b < blocks; ++b) t0 = std::min(t0, h[32ull * b]);
    for (uint32_t b : {0u, blocks / 2, blocks - 1}) {
      std::fprintf(stderr, "[tc] B=%u cta %u:", n_tokens, b);
      for (int k = 0; k < 32; ++k)
        if (h[32ull * b + k]) std::fprintf(stderr, " %d:%.2f", k, (h[32ull * b + k] - t0) / 1e3);
      std::fprintf(stderr, "\n");
    }
    cudaFree(a.trace);
  }
  return rc;
}

}  // extern "C"

// ------------------------------------------------------------ prefill path ---
// Dense f16 tensor-core GEMMs (cuBLASLt, f32 accumulation) for experts that
// receive many tokens (floe_prefill.cuh).  Plain library GEMMs; the dequant,
// the hi/lo splits with per-row scales, the mask and SwiGLU are this library's
// kernels.
namespace {
struct Lt {
  cublasLtHandle_t h = nullptr;
  void *ws = nullptr;
  size_t ws_bytes = 64ull << 20;
  std::mutex mu;
  std::map<std::tuple<int, int, int, int, int, int, int, int, int>, cublasLtMatmulAlgo_t> algos;
  // the batched layer's side streams run GEMMs concurrently: each has its own
  // workspace (lt_reserve); every other stream uses ws, as before
  std::map<cudaStream_t, void *> stream_ws;
};
Lt *lt_get() {
  static Lt *L = [] {
    Lt *x = new Lt();
    if (cublasLtCreate(&x->h) != CUBLAS_STATUS_SUCCESS || cudaMalloc(&x->ws, x->ws_bytes) != cudaSuccess) {
      x->h = nullptr;
    }
    return x;
  }();
  return L;
}

// C (m x n, column-major, ldc, f32) = op(A) op(B) + beta C; A, B f16
// tokens up to which the prefill path computes v with the exact batched K1
const uint32_t kExactK1Max = [] {
  const char *p = std::getenv("FLOE_EXACT_K1_MAX");
  return p ? (uint32_t)std::atoi(p) : 64u;
}();

// Give side stream `st` its own cuBLASLt workspace (at stream creation, so no
// cudaMalloc -- a device-wide synchronisation -- happens inside a layer call).
// Returns false when it cannot be allocated.
bool lt_reserve(cudaStream_t st) {
  Lt *L = lt_get();
  if (!L->h) return true;  // no cuBLASLt: lt_gemm fails loudly on use
  std::lock_guard<std::mutex> g(L->mu);
  if (L->stream_ws.count(st)) return true;
  void *w = nullptr;
  if (cudaMalloc(&w, L->ws_bytes) != cudaSuccess) return false;
  L->stream_ws[st] = w;
  return true;
}

int lt_gemm(bool ta, bool tb, int m, int n, int k, const __half *A, int lda, const __half *B, int ldb,
            float beta, float *C, int ldc, cudaStream_t st) {
  Lt *L = lt_get();
  if (!L->h) return fail(FLOE_ERR_CUDA, "prefill: cuBLASLt unavailable");
  cublasLtMatmulDesc_t op = nullptr;
  cublasLtMatrixLayout_t la = nullptr, lb = nullptr, lc = nullptr;
  const cublasOperation_t oa = ta ? CUBLAS_OP_T : CUBLAS_OP_N, ob = tb ? CUBLAS_OP_T : CUBLAS_OP_N;
  bool ok = cublasLtMatmulDescCreate(&op, CUBLAS_COMPUTE_32F, CUDA_R_32F) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSA, &oa, sizeof(oa)) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatmulDescSetAttribute(op, CUBLASLT_MATMUL_DESC_TRANSB, &ob, sizeof(ob)) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatrixLayoutCreate(&la, CUDA_R_16F, ta ? k : m, ta ? m : k, lda) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatrixLayoutCreate(&lb, CUDA_R_16F, tb ? n : k, tb ? k : n, ldb) == CUBLAS_STATUS_SUCCESS;
  ok = ok && cublasLtMatrixLayoutCreate(&lc, CUDA_R_32F, m, n, ldc) == CUBLAS_STATUS_SUCCESS;
  cublasLtMatmulAlgo_t algo{};
  // algorithms are cached per shape class; the token count (a GEMM dimension
  // that changes with every routing) only by its power-of-two bucket: a
  // heuristic query costs far more than the GEMMs of a small expert
  int nb = 1;
  while (nb < n) nb <<= 1;
  if (ok) {
    const auto key = std::make_tuple((int)ta, (int)tb, m, nb, k, lda, ldb, ldc, beta != 0.0f ? 1 : 0);
    std::lock_guard<std::mutex> g(L->mu);
    auto it = L->algos.find(key);
    if (it != L->algos.end()) {
      algo = it->second;
    } else {
      cublasLtMatmulPreference_t pref = nullptr;
      cublasLtMatmulHeuristicResult_t res{};
      int got = 0;
      ok = cublasLtMatmulPreferenceCreate(&pref) == CUBLAS_STATUS_SUCCESS &&
           cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES,
                                                &L->ws_bytes, sizeof(L->ws_bytes)) == CUBLAS_STATUS_SUCCESS &&
           cublasLtMatmulAlgoGetHeuristic(L->h, op, la, lb, lc, lc, pref, 1, &res, &got) ==
               CUBLAS_STATUS_SUCCESS && got > 0;
      if (pref) cublasLtMatmulPreferenceDestroy(pref);
      if (ok) {
        algo = res.algo;
        L->algos[key] = algo;
      }
    }
  }
  const float alpha = 1.0f;
  if (ok) {
    cublasLtMatmulHeuristicResult_t chk{};
    if (cublasLtMatmulAlgoCheck(L->h, op, la, lb, lc, lc, &algo, &chk) != CUBLAS_STATUS_SUCCESS ||
        chk.workspaceSize > L->ws_bytes) {  // not valid at this n: a fresh heuristic
      cublasLtMatmulPreference_t pref = nullptr;
      cublasLtMatmulHeuristicResult_t res{};
      int got = 0;
      ok = cublasLtMatmulPreferenceCreate(&pref) == CUBLAS_STATUS_SUCCESS &&
           cublasLtMatmulPreferenceSetAttribute(pref, CUBLASLT_MATMUL_PREF_MAX_WORKSPACE_BYTES,
                                                &L->ws_bytes, sizeof(L->ws_bytes)) == CUBLAS_STATUS_SUCCESS &&
           cublasLtMatmulAlgoGetHeuristic(L->h, op, la, lb, lc, lc, pref, 1, &res, &got) ==
               CUBLAS_STATUS_SUCCESS && got > 0;
      if (pref) cublasLtMatmulPreferenceDestroy(pref);
      if (ok) algo = res.algo;
    }
  }
  void *wsp = L->ws;
  if (ok) {
    std::lock_guard<std::mutex> g(L->mu);
    auto it = L->stream_ws.find(st);
    if (it != L->stream_ws.end()) wsp = it->second;
  }
  if (ok)
    ok = cublasLtMatmul(L->h, op, &alpha, A, la, B, lb, &beta, C, lc, C, lc, &algo, wsp, L->ws_bytes,
                        st) == CUBLAS_STATUS_SUCCESS;
  if (lc) cublasLtMatrixLayoutDestroy(lc);
  if (lb) cublasLtMatrixLayoutDestroy(lb);
  if (la) cublasLtMatrixLayoutDestroy(la);
  if (op) cublasLtMatmulDescDestroy(op);
  return ok ? FLOE_OK : fail(FLOE_ERR_CUDA, "prefill: cuBLASLt matmul failed (%d x %d x %d)", m, n, k);
}
}  // namespace

extern "C" {

}  // extern "C"
namespace {
// v_pre: v [n][di] already computed by the exact batched K1 (n <= kExactK1Max)
int prefill_impl(const floe_gpu_expert *e, const float *x, uint32_t n_tokens, float *y,
                 floe_stream_t stream, const float *v_pre);
}  // namespace
extern "C" {

int floe_gpu_expert_forward_prefill(const floe_gpu_expert *e, const float *x, uint32_t n_tokens,
                                    float *y, floe_stream_t stream) {
  return prefill_impl(e, x, n_tokens, y, stream, nullptr);
}

}  // extern "C"
namespace {
int prefill_impl(const floe_gpu_expert *e, const float *x, uint32_t n_tokens, float *y,
                 floe_stream_t stream, const float *v_pre) {
  if (!e || !x || !y) return fail(FLOE_ERR_INVALID, "expert_forward_sparse: null argument");
  if (n_tokens == 0) return FLOE_OK;
  if (!e->fast || e->up_only || !e->host_desc.records)
    return fail(FLOE_ERR_UNSUPPORTED, "expert_forward_prefill: needs the tile layout and records");
  if (int rc = require_device("expert_forward_prefill")) return rc;
  cudaStream_t st = S(stream);
  keep_pool();
  const uint32_t dh = e->dh, di = e->di, n = n_tokens;
  // scratch: Wb [di][3dh] f16 (large n) | Xa [n][3dh] f16 | v, g [n][di] f32 | Ah [n][di] f16 | inv, ainv [n]
  const size_t wb_bytes = n <= kExactK1Max ? 0 : 2ull * di * 3 * dh;
  const size_t o_wb = 0, o_xa = o_wb + wb_bytes, o_v = o_xa + 2ull * n * 3 * dh;
  const size_t o_g = o_v + 4ull * n * di, o_a = o_g + 4ull * n * di, o_inv = o_a + 2ull * n * di;
  const size_t o_ainv = o_inv + 4ull * n, total = o_ainv + 4ull * n;
  uint8_t *sc = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void **>(&sc), total, st));
  __half *Wb = reinterpret_cast<__half *>(sc + o_wb), *Xa = reinterpret_cast<__half *>(sc + o_xa);
  float *v = reinterpret_cast<float *>(sc + o_v), *g = reinterpret_cast<float *>(sc + o_g);
  __half *Ac = reinterpret_cast<__half *>(sc + o_a);
  float *inv = reinterpret_cast<float *>(sc + o_inv), *ainv = reinterpret_cast<float *>(sc + o_ainv);
  auto done = [&](int rc) {
    cudaFreeAsync(sc, st);
    return rc;
  };
  const int sm = device_info().sm;
  // Up to kExactK1Max tokens the exact batched K1 (tcgen05 kind::i8 on the
  // codes, no dequantized copy) computes v; above, the dequantized f16 hi/lo
  // GEMM (its fixed cost -- writing and reading the 352 MB copy -- amortised)
  const bool exact_k1 = n <= kExactK1Max;
  floe_pf::xcat<<<n, 1024, 0, st>>>(x, dh, Xa, inv);
  if (!exact_k1) {
    if (dh == 4096) floe_pf::wcat_tiled<4096><<<sm * 8, 256, 0, st>>>(e->host_desc.tiles, di, Wb);
    else floe_pf::wcat_tiled<2048><<<sm * 8, 256, 0, st>>>(e->host_desc.tiles, di, Wb);
  }
  if (cudaGetLastError() != cudaSuccess) return done(fail(FLOE_ERR_CUDA, "prefill: launch failed"));
  const __half *rec = e->host_desc.records;  // [di][gate row | down row]
  const int D = (int)dh, I = (int)di, N = (int)n;
  if (exact_k1 && v_pre) {
    v = const_cast<float *>(v_pre);
  } else if (exact_k1) {
    if (int rc = floe_gpu_qgemv_channels_batched(e, x, n, v, stream)) return done(rc);
  } else {
    // v (n x di row-major == di x n column-major) = Wb^T-view . Xa, K = 3 dh
    if (int rc = lt_gemm(true, false, I, N, 3 * D, Wb, 3 * D, Xa, 3 * D, 0.0f, v, I, st)) return done(rc);
  }
  // g = gate . x_hi  (gate rows: ld 2 dh)
  if (int rc = lt_gemm(true, false, I, N, D, rec, 2 * D, Xa, 3 * D, 0.0f, g, I, st)) return done(rc);
  if (di <= 16u * 1024u)
    floe_pf::coeffs_reg<16><<<n, 1024, 0, st>>>(v, g, inv, di, e->host_desc.threshold, Ac, ainv,
                                                exact_k1 ? 1 : 0);
  else
    floe_pf::coeffs<<<n, 256, 0, st>>>(v, g, inv, di, e->host_desc.threshold, Ac, ainv, exact_k1 ? 1 : 0);
  // y (n x dh row-major == dh x n column-major) = down^T-view . a_hi
  if (int rc = lt_gemm(false, false, D, N, I, rec + dh, 2 * D, Ac, I, 0.0f, y, D, st)) return done(rc);
  floe_pf::unscale_rows<<<n, 1024, 0, st>>>(y, dh, ainv);
  if (cudaGetLastError() != cudaSuccess) return done(fail(FLOE_ERR_CUDA, "prefill: launch failed"));
  return done(FLOE_OK);
}
}  // namespace
extern "C" {

}  // extern "C"
namespace {
// v_pre: v [n][di] already computed (the batched layer's up-projection stage)
int batched_impl(const floe_gpu_expert *e, const float *x, uint32_t n_tokens, float *y_out,
                 float *v_out, floe_stream_t stream, const float *v_pre);
}  // namespace
extern "C" {

int floe_gpu_expert_forward_batched(const floe_gpu_expert *e, const float *x, uint32_t n_tokens,
                                    float *y_out, float *v_out, floe_stream_t stream) {
  return batched_impl(e, x, n_tokens, y_out, v_out, stream, nullptr);
}

}  // extern "C"
namespace {
int batched_impl(const floe_gpu_expert *e, const float *x, uint32_t n_tokens, float *y_out,
                 float *v_out, floe_stream_t stream, const float *v_pre) {
  if (!e || !x || !y_out) return fail(FLOE_ERR_INVALID, "expert_forward_batched: null argument");
  if (n_tokens == 0) return FLOE_OK;
  if (e->up_only)
    return fail(FLOE_ERR_INVALID, "expert_forward_batched: expert has no gate/down records");
  if (!e->fast)
    return fail(FLOE_ERR_UNSUPPORTED, "expert_forward_batched: needs the tile layout");
  if (n_tokens > (uint32_t)floe_tc::kMaxTokens)
    return fail(FLOE_ERR_INVALID, "expert_forward_batched: at most %d tokens", floe_tc::kMaxTokens);
  cudaStream_t st = S(stream);
  const uint32_t B = n_tokens, di = e->di, dh = e->dh;
  // scratch: count | v [B][di] | uc [di] | um [di] | A [di][B] | x hi/lo table
  const size_t o_v = 256, o_uc = o_v + ((4ull * B * di + 255) & ~size_t(255));
  const size_t o_um = o_uc + ((4ull * di + 255) & ~size_t(255));
  const size_t o_a = o_um + 8ull * di;
  const size_t o_xh = (o_a + 4ull * di * B + 1023) & ~size_t(1023);
  const size_t o_g = o_xh + (((size_t)(dh / 64) * floe_tc::gemm_n(B) * 128u + 255) & ~size_t(255));
  // G: split-K partial gate dots; then x scale | 1/x scale | max|A| per token
  const size_t total = o_g + 4ull * di * B + 3ull * 4 * floe_tc::kMaxTokens;
  uint8_t *scratch = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void **>(&scratch), total, st));
  uint32_t *count = reinterpret_cast<uint32_t *>(scratch);
  float *v = v_pre ? const_cast<float *>(v_pre) : v_out ? v_out : reinterpret_cast<float *>(scratch + o_v);
  uint32_t *uc = reinterpret_cast<uint32_t *>(scratch + o_uc);
  unsigned long long *um = reinterpret_cast<unsigned long long *>(scratch + o_um);
  // K parts of the gate GEMM per 128-channel block: more CTAs in flight at
  // small batches, fewer partial-sum atomics at large ones
  const uint32_t kGateSplit = B <= 16 ? 8u : 4u;
  // gate dots: a tcgen05 GEMM (128-channel blocks, K split in 4-8) pays off from
  // about 16 tokens; fewer tokens use the CUDA-core warps.
  // FLOE_GATE_TC=0/1 forces either.
  static const int gate_env = [] {
    const char *p = std::getenv("FLOE_GATE_TC");
    return p ? std::atoi(p) : -1;
  }();
  const bool tc_gate = gate_env >= 0 ? gate_env != 0 : B >= 16;
  // down product: the tcgen05 GEMM (MN-major gathered down rows, 256-channel
  // ranges per CTA) wins from about 16 tokens (207 vs 215 us at B=16, 358 vs
  // 451 at B=64); FLOE_DOWN_TC=0/1 forces either
  static const int down_env = [] {
    const char *p = std::getenv("FLOE_DOWN_TC");
    return p ? std::atoi(p) : -1;
  }();
  const bool tc_down = down_env >= 0 ? down_env != 0 : B >= 16;
  int rc = v_pre ? FLOE_OK : floe_gpu_qgemv_channels_batched(e, x, B, v, stream);
  if (rc == FLOE_OK)
    rc = dh == 4096 ? batched_gate_down<4096>(e, x, B, y_out, v, scratch, o_xh, o_g, tc_gate,
                                              tc_down, kGateSplit, st)
                    : batched_gate_down<2048>(e, x, B, y_out, v, scratch, o_xh, o_g, tc_gate,
                                              tc_down, kGateSplit, st);
  // the scratch is released on every path (stream-ordered)
  const cudaError_t fe = cudaFreeAsync(scratch, st);
  if (rc == FLOE_OK && fe != cudaSuccess)
    return fail(FLOE_ERR_CUDA, "expert_forward_batched: %s", cudaGetErrorString(fe));
  return rc;
}
}  // namespace
extern "C" {

int floe_gpu_dequantize_up(const floe_gpu_expert *e, float *out, floe_stream_t stream) {
  if (!e || !out) return fail(FLOE_ERR_INVALID, "dequantize: null argument");
  const uint64_t n = (uint64_t)e->dh * e->di;
  if (e->fast)
    floe_v2::dequant_tiled<<<4 * device_info().sm, 256, 0, S(stream)>>>(e->host_desc.tiles, e->dh,
                                                                        e->di, out);
  else
    floe_k::dequant_up<<<4 * device_info().sm, 256, 0, S(stream)>>>(e->dev_desc, n, e->bits,
                                                                     e->g, out);
  CK_LAUNCH();
  return FLOE_OK;
}

int floe_gpu_predict_mask(const floe_gpu_expert *next, floe_gpu_workspace *ws,
                          const float *x_prev, float t, uint8_t *mask_out,
                          uint32_t *kept_out, uint32_t *n_kept_out, floe_stream_t stream) {
  if (!next || !x_prev) return fail(FLOE_ERR_INVALID, "predict_mask: null argument");
  if (int rc = check_ws("predict_mask", ws, next->dh, next->di, 1)) return rc;
  if (next->fast) {
    FusedLaunch f{};
    f.table = next->dev_desc;
    f.slots = 1;
    f.dh = next->dh;
    f.di = next->di;
    f.k1_only = true;
    f.use_thr = 1;
    f.thr = t;
    f.x = x_prev;
    f.mask_out = mask_out;
    f.kept_out = kept_out;
    f.n_kept_out = n_kept_out;
    return launch_v2(f, ws, S(stream));
  }
  K1Launch k1{next->dev_desc, nullptr, 1, next->dh, next->di, next->bits, next->g, 1, t,
              x_prev, nullptr, mask_out, nullptr};
  if (int rc = launch_k1(k1, ws, S(stream))) return rc;
  K2Launch fin{next->dev_desc, nullptr, nullptr, 1, next->dh, next->di, x_prev, nullptr,
               n_kept_out, kept_out};
  return launch_k2(fin, ws, S(stream));
}

// ----------------------------------------------------------------- layers --
int floe_gpu_layer_create(const floe_layer_host_view *v, floe_gpu_layer **out) {
  if (!v || !out) return fail(FLOE_ERR_INVALID, "layer_create: null argument");
  *out = nullptr;
  if (int rc = require_device("layer_create")) return rc;
  if (v->n_experts == 0 || v->d_hidden == 0)
    return fail(FLOE_ERR_INVALID, "model config: all dimensions must be >= 1");
  if (v->top_k == 0 || v->top_k > v->n_experts)
    return fail(FLOE_ERR_INVALID, "model config: need 1 <= top_k <= experts");
  if (v->n_experts > 32 || v->top_k > (uint32_t)floe_k::kMaxSlots)
    return fail(FLOE_ERR_UNSUPPORTED, "layer_create: at most 32 experts and top_k <= %d",
                floe_k::kMaxSlots);
  if (!v->router || !v->mixing || !v->experts)
    return fail(FLOE_ERR_INVALID, "layer_create: router, mixing and experts required");
  const floe_gpu_expert *e0 = v->experts[0];
  if (!e0) return fail(FLOE_ERR_INVALID, "layer_create: null expert");
  for (uint32_t i = 0; i < v->n_experts; ++i) {
    const floe_gpu_expert *e = v->experts[i];
    if (!e || e->dh != v->d_hidden || e->di != e0->di || e->bits != e0->bits || e->g != e0->g)
      return fail(FLOE_ERR_INVALID, "layer_create: expert %u shape differs from the layer", i);
    if (e->up_only) return fail(FLOE_ERR_INVALID, "layer_create: expert %u has no gate/down", i);
  }
  auto *l = new (std::nothrow) floe_gpu_layer();
  if (!l) return fail(FLOE_ERR_OOM, "layer_create: host allocation failed");
  if (cudaDeviceSynchronize() != cudaSuccess) {  // router/mixing may be device tensors in flight
    delete l;
    return fail(FLOE_ERR_CUDA, "layer_create: device synchronisation failed");
  }
  l->dh = v->d_hidden;
  l->di = e0->di;
  l->E = v->n_experts;
  l->top_k = v->top_k;
  l->bits = e0->bits;
  l->g = e0->g;
  l->mix_f16 = v->mixing_f16 != 0;
  l->fast = e0->fast;
  const uint64_t dh = l->dh;
  std::vector<ExpertDesc> table(l->E);
  for (uint32_t i = 0; i < l->E; ++i) table[i] = v->experts[i]->host_desc;
  cudaError_t ce = cudaMalloc(&l->router, 4ull * l->E * dh);
  if (ce == cudaSuccess) ce = cudaMalloc(&l->mixing, (l->mix_f16 ? 2ull : 4ull) * dh * dh);
  if (ce == cudaSuccess) ce = cudaMalloc(&l->table, sizeof(ExpertDesc) * l->E);
  if (ce == cudaSuccess)
    ce = cudaMemcpy(l->router, v->router, 4ull * l->E * dh, cudaMemcpyDefault);
  if (ce == cudaSuccess)
    ce = cudaMemcpy(l->table, table.data(), sizeof(ExpertDesc) * l->E, cudaMemcpyHostToDevice);
  if (ce == cudaSuccess)
    for (uint32_t i = 0; i < l->E; ++i) {
      v->experts[i]->tables.push_back(l->table + i);
      l->experts.push_back(v->experts[i]);
    }
  if (ce == cudaSuccess) {
    if (!l->mix_f16) {
      ce = cudaMemcpy(l->mixing, v->mixing, 4ull * dh * dh, cudaMemcpyDefault);
    } else {
      float *tmp = nullptr;
      ce = cudaMalloc(&tmp, 4ull * dh * dh);
      if (ce == cudaSuccess) ce = cudaMemcpy(tmp, v->mixing, 4ull * dh * dh, cudaMemcpyDefault);
      if (ce == cudaSuccess) {
        floe_k::f32_to_f16_rn<<<1024, 256>>>(tmp, dh * dh, static_cast<__half *>(l->mixing));
        ce = cudaGetLastError();
      }
      if (ce == cudaSuccess) ce = cudaDeviceSynchronize();
      if (tmp) cudaFree(tmp);
    }
  }
  // Routing predictor of the fused layer kernel: router * (h + mixing h) =
  // (router + router * mixing) h, with the mixing weights exactly as the
  // kernel reads them (f16 or f32), accumulated in f64.  The kernel streams
  // the predicted experts' K1 tiles during the mixing GEMV and verifies the
  // prediction against the exact routing of u before any record is read.
  if (ce == cudaSuccess && l->fast && l->E <= 32) {
    ce = cudaMalloc(&l->router_pred, 4ull * l->E * dh);
    if (ce == cudaSuccess) {
      const uint32_t blocks = (dh + 127) / 128;
      if (l->mix_f16)
        floe_k::router_pred<__half><<<blocks, 128>>>(l->router, static_cast<const __half *>(l->mixing),
                                                      l->E, dh, l->router_pred);
      else
        floe_k::router_pred<float><<<blocks, 128>>>(l->router, static_cast<const float *>(l->mixing),
                                                     l->E, dh, l->router_pred);
      ce = cudaGetLastError();
      if (ce == cudaSuccess) ce = cudaDeviceSynchronize();
    }
  }
  if (ce != cudaSuccess) {
    floe_gpu_layer_destroy(l);
    return fail(FLOE_ERR_OOM, "layer_create: %s", cudaGetErrorString(ce));
  }
  *out = l;
  return FLOE_OK;
}

int floe_gpu_layer_destroy(floe_gpu_layer *l) {
  if (!l) return FLOE_OK;
  cudaDeviceSynchronize();  // kernels in flight may still read the table
  // unregister this layer's table entries from its (borrowed) experts, so a
  // later residency or threshold change does not write into freed memory
  for (size_t i = 0; i < l->experts.size(); ++i) {
    auto &tabs = l->experts[i]->tables;
    tabs.erase(std::remove(tabs.begin(), tabs.end(), l->table + i), tabs.end());
  }
  if (l->router) cudaFree(l->router);
  if (l->mixing) cudaFree(l->mixing);
  if (l->router_pred) cudaFree(l->router_pred);
  if (l->table) cudaFree(l->table);
  delete l;
  return FLOE_OK;
}

namespace {
// place_acc (nullable, fast path only): the fused kernel adds each slot's kept
// record count to [0] (records in HBM) or [1] (pinned host records over PCIe).
int layer_forward_impl(const floe_gpu_layer *l, floe_gpu_workspace *ws, const float *h, float *y,
                       const floe_gpu_layer_trace *tr, unsigned long long *place_acc,
                       cudaStream_t st, const floe_gpu_layer *next = nullptr,
                       uint32_t *n_kept_out = nullptr);
}  // namespace

int floe_gpu_layer_forward(const floe_gpu_layer *l, floe_gpu_workspace *ws, const float *h,
                           float *y, const floe_gpu_layer_trace *tr, floe_stream_t stream) {
  if (!l || !h || !y) return fail(FLOE_ERR_INVALID, "layer_forward: null argument");
  if (int rc = check_ws("layer_forward", ws, l->dh, l->di, l->top_k)) return rc;
  return layer_forward_impl(l, ws, h, y, tr, nullptr, S(stream));
}

namespace {
bool layer_fused(const floe_gpu_layer *l) { return l->fast && l->E <= 32; }

int layer_forward_impl(const floe_gpu_layer *l, floe_gpu_workspace *ws, const float *h, float *y,
                       const floe_gpu_layer_trace *tr, unsigned long long *place_acc,
                       cudaStream_t st, const floe_gpu_layer *next, uint32_t *n_kept_out) {
  if (layer_fused(l)) {
    FusedLaunch f{};
    f.n_kept_out = n_kept_out;  // per routed slot (ascending expert order)
    if (next && next->fast) {  // the decode loop's next layer: its mixing goes to L2 early
      f.next_mixing = next->mixing;
      f.next_mixing_bytes = (uint64_t)next->dh * next->dh * (next->mix_f16 ? 2u : 4u);
    }
    f.mixing = l->mixing;
    f.mix_f16 = l->mix_f16;
    f.h = h;
    f.router = l->router;
    f.router_pred = l->router_pred;
    f.n_experts = l->E;
    f.top_k = l->top_k;
    f.trace = tr;
    f.table = l->table;
    f.slots = l->top_k;
    f.dh = l->dh;
    f.di = l->di;
    f.x = ws->u;
    f.u = ws->u;
    f.y = y;
    f.place_acc = place_acc;
    return launch_v2(f, ws, st);
  }
  float *u_tr = tr ? tr->block_input_dev : nullptr;
  {
    // mixing GEMV + residual + router logits + top-k + softmax in one launch
    StageScope prof(ws, kStageMixing, st);
    floe_k::MixArgs m{};
    m.m = l->mixing;
    m.h = h;
    m.dh = l->dh;
    m.router = l->router;
    m.E = l->E;
    m.k = l->top_k;
    m.u = ws->u;
    m.y_init = y;
    m.u_trace = u_tr;
    m.partial = ws->mix_partial;
    m.done = ws->mix_done;
    m.sel = ws->sel;
    m.weights = ws->weights;
    m.sel_trace = tr ? tr->experts_dev : nullptr;
    m.w_trace = tr ? tr->weights_dev : nullptr;
    const dim3 grid((l->dh + 7) / 8);
    const size_t smem = 4ull * l->dh;
    if (smem > 48 * 1024) {
      if (int rc = set_smem(l->mix_f16 ? (void (*)(floe_k::MixArgs))floe_k::mixing_route<__half>
                                       : floe_k::mixing_route<float>, (uint32_t)smem))
        return rc;
    }
    if (l->mix_f16)
      floe_k::mixing_route<__half><<<grid, 256, smem, st>>>(m);
    else
      floe_k::mixing_route<float><<<grid, 256, smem, st>>>(m);
    CK_LAUNCH();
  }
  K1Launch k1{l->table, ws->sel, l->top_k, l->dh, l->di, l->bits, l->g, 0, 0.0f,
              ws->u, nullptr, tr ? tr->masks_dev : nullptr, nullptr};
  if (int rc = launch_k1(k1, ws, st)) return rc;
  K2Launch k2{l->table, ws->sel, ws->weights, l->top_k, l->dh, l->di, ws->u, y, nullptr, nullptr};
  return launch_k2(k2, ws, st);
}
}  // namespace

int floe_gpu_layer_forward_host(const floe_gpu_layer *l, floe_gpu_workspace *ws,
                                const float *h_host, float *y_host, floe_stream_t stream) {
  if (!l || !h_host || !y_host) return fail(FLOE_ERR_INVALID, "layer_forward: null argument");
  if (int rc = check_ws("layer_forward", ws, l->dh, l->di, l->top_k)) return rc;
  cudaStream_t st = S(stream);
  std::memcpy(ws->hx, h_host, 4ull * l->dh);
  CK(cudaMemcpyAsync(ws->x, ws->hx, 4ull * l->dh, cudaMemcpyHostToDevice, st));
  if (int rc = floe_gpu_layer_forward(l, ws, ws->x, ws->y, nullptr, stream)) return rc;
  CK(cudaMemcpyAsync(ws->hy, ws->y, 4ull * l->dh, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  std::memcpy(y_host, ws->hy, 4ull * l->dh);
  return FLOE_OK;
}

// ----------------------------------------------------------- offload engine --
// Host-resident decode (SURVEY config 3; the reference's simulate_decode /
// ExpertCache, core/src/offload.cpp:89-159,299-464, made real).  Every
// expert's gate|down records live in pinned host memory; the fused kernel
// reads the kept channels of non-resident experts in place over PCIe (the
// simulator's "sync" bytes, fetched on demand at exactly channel
// granularity, no host round trip).  An LRU of whole experts under a VRAM
// budget holds recently routed experts in HBM: the routing of token t
// (read back asynchronously) promotes missing experts with copies on a side
// stream; a promoted copy is switched in, and an evicted one switched out and
// freed, on the decode stream between tokens, so every kernel sees one
// consistent placement and the byte accounting is exact.
namespace {
__global__ void offload_account(const uint32_t *seg_count, uint32_t G, uint32_t slots,
                                const uint32_t *sel, const uint8_t *resident,
                                unsigned long long *acc /* [2]: from HBM, over PCIe */) {
  const uint32_t lane = threadIdx.x;
  for (uint32_t s = 0; s < slots; ++s) {
    uint32_t n = 0;
    for (uint32_t b = lane; b < G; b += 32) n += seg_count[s * G + b];
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
    if (lane == 0) atomicAdd(&acc[resident[sel[s]] ? 0 : 1], (unsigned long long)n);
  }
}
}  // namespace

// eval_masks / eval_sets (predictor.cpp:206-254): per sample precision
// inter/|pred| (1 if both empty, 0 if only the prediction is) and recall
// inter/|truth| (1 for an empty truth), summed for the macro average.
__device__ __forceinline__ void accumulate_pr(uint32_t inter, uint32_t pn, uint32_t tn,
                                              double *psum, double *rsum) {
  atomicAdd(psum, pn == 0 ? (tn == 0 ? 1.0 : 0.0) : (double)inter / (double)pn);
  atomicAdd(rsum, tn == 0 ? 1.0 : (double)inter / (double)tn);
}

// block k: predicted mask of routed expert sel[k] vs the layer's true mask k
__global__ void score_masks(const uint8_t *__restrict__ pmask, const uint8_t *__restrict__ tmask,
                            const uint32_t *__restrict__ sel, uint32_t di, double *acc,
                            unsigned long long *samples) {
  const uint32_t k = blockIdx.x;
  const uint8_t *p = pmask + (size_t)sel[k] * di, *t = tmask + (size_t)k * di;
  uint32_t inter = 0, pn = 0, tn = 0;
  for (uint32_t i = threadIdx.x; i < di; i += blockDim.x) {
    const bool a = p[i] != 0, b = t[i] != 0;
    pn += a;
    tn += b;
    inter += a && b;
  }
  __shared__ uint32_t red[3][32];
  for (int o = 16; o >= 1; o >>= 1) {
    inter += __shfl_xor_sync(0xffffffffu, inter, o);
    pn += __shfl_xor_sync(0xffffffffu, pn, o);
    tn += __shfl_xor_sync(0xffffffffu, tn, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = inter;
    red[1][threadIdx.x >> 5] = pn;
    red[2][threadIdx.x >> 5] = tn;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t I = 0, P = 0, T = 0;
    for (uint32_t w = 0; w < blockDim.x / 32; ++w) {
      I += red[0][w];
      P += red[1][w];
      T += red[2][w];
    }
    accumulate_pr(I, P, T, acc, acc + 1);
    atomicAdd(samples, 1ull);
  }
}

// predicted expert set (count ids) vs the routed set (K ids)
__global__ void score_sets(const uint32_t *__restrict__ pred, uint32_t count,
                           const uint32_t *__restrict__ sel, uint32_t K, double *acc,
                           unsigned long long *samples) {
  uint32_t inter = 0;
  for (uint32_t i = 0; i < count; ++i)
    for (uint32_t j = 0; j < K; ++j) inter += pred[i] == sel[j];
  accumulate_pr(inter, count, K, acc, acc + 1);
  atomicAdd(samples, 1ull);
}

struct floe_gpu_offload {
  std::vector<floe_gpu_layer *> layers;
  uint32_t L = 0, E = 0, K = 0, dh = 0;
  uint64_t budget = 0, rec_bytes = 0, committed = 0;  // bytes of HBM copies (ready + in flight)
  enum State : uint8_t { kHost = 0, kCopying = 1, kResident = 2 };
  std::vector<uint8_t> state;                 // [L*E]
  std::vector<__half *> pending;              // [L*E] device copy in flight
  std::vector<cudaEvent_t> copy_done;         // [L*E]
  std::vector<uint64_t> last_use;             // [L*E] token of last routing
  std::vector<float> freq;                    // [L*E] decayed routing count
  uint8_t *resident_dev = nullptr;            // [L*E] for the byte accounting
  std::vector<uint8_t> resident_host;
  uint32_t *sel_dev = nullptr;                // [L][K] routing of the last token
  uint32_t *sel_host = nullptr;               // pinned
  float *buf = nullptr;                       // 2 x dh ping-pong
  unsigned long long *acc = nullptr;          // [2] kept records from HBM / over PCIe
  cudaEvent_t sel_ready = nullptr;
  bool sel_pending = false;  // generic path: a routing readback is in flight
  bool sel_fresh = false;    // sel_host holds a routing the policy has not used
  cudaStream_t side = nullptr;
  uint64_t tokens = 0, promotions = 0, evictions = 0, bytes_promoted = 0;
  uint64_t up_bytes = 0;
  // DecodeTimeline (offload.hpp:128-157), classified per completed token from
  // its routing, kept counts and the placement its kernels saw: up projections
  // are HBM-resident (cache); records of resident experts are cache hits, or
  // prefetch_used on an expert's first demand after its promotion landed (the
  // rest of that promotion is wasted, as in simulate_decode: it stays cached);
  // records of host-resident experts are sync (read in place over PCIe).
  uint32_t *nkept_dev = nullptr;  // [L][K] kept records per routed slot, this token
  struct Readback {
    uint32_t *sel = nullptr, *nkept = nullptr;  // pinned [L][K]
    cudaEvent_t ev = nullptr;
    std::vector<uint8_t> resident, fresh;      // placement the token's kernels saw
    bool busy = false;
  };
  std::vector<Readback> ring;  // tokens in flight (in order)
  uint32_t ring_head = 0, ring_n = 0;
  std::vector<uint8_t> fresh;  // promoted, landed, not yet demanded
  uint64_t t_demanded = 0, t_cache = 0, t_used = 0, t_sync = 0, t_wasted = 0, t_req_ch = 0,
           t_req_up = 0, t_tokens = 0;
  // prediction scoring on the decode path (predictor.cpp:164-254): reuse
  // masks of layer l's routed experts from layer l-1's block input, and the
  // learned predictor's expert sets when one is attached
  bool eval = false;
  floe_gpu_workspace *ews = nullptr;  // E slots: every expert of a layer in one K1-only pass
  uint8_t *pmask_dev = nullptr;       // [E][di]
  uint8_t *tmask_dev = nullptr;       // [L][K][di]
  float *u_dev = nullptr;             // [L][dh] block inputs
  double *pr_dev = nullptr;           // [4]: mask precision/recall sums, set precision/recall sums
  unsigned long long *pn_dev = nullptr;  // [2]: mask samples, set samples
  const floe_gpu_predictor *pred = nullptr;
  uint32_t pred_count = 0;
  uint32_t *pexp_dev = nullptr;       // [E]
};

namespace {
int offload_switch(floe_gpu_offload *o, uint32_t i, bool to_hbm, cudaStream_t st) {
  floe_gpu_expert *e = o->layers[i / o->E]->experts[i % o->E];
  if (to_hbm) {
    e->rec_dev = o->pending[i];
    o->pending[i] = nullptr;
    e->host_desc.records = e->rec_dev;
    e->host_desc.host_records = 0;
  } else {
    void *dptr = nullptr;
    CK(cudaHostGetDevicePointer(&dptr, e->rec_host, 0));
    e->host_desc.records = static_cast<const __half *>(dptr);
    e->host_desc.host_records = 1;
  }
  CK(cudaMemcpyAsync(e->dev_desc, &e->host_desc, sizeof(ExpertDesc), cudaMemcpyHostToDevice, st));
  for (ExpertDesc *t : e->tables)
    CK(cudaMemcpyAsync(t, &e->host_desc, sizeof(ExpertDesc), cudaMemcpyHostToDevice, st));
  if (!to_hbm) {  // kernels already enqueued on st may still read the old copy: free after them
    CK(cudaFreeAsync(e->rec_dev, st));
    e->rec_dev = nullptr;
  }
  e->resident = to_hbm;
  o->resident_host[i] = to_hbm ? 1 : 0;
  CK(cudaMemcpyAsync(o->resident_dev + i, &o->resident_host[i], 1, cudaMemcpyHostToDevice, st));
  return FLOE_OK;
}

// Between tokens: switch in finished copies; read the previous token's routing
// (if it is done) and promote its missing experts into free budget, or in
// place of a resident expert routed clearly less often (ExpertCache's LRU,
// offload.cpp:89-159, with frequency-aware admission: see below).
constexpr float kFreqDecay = 0.98f;   // per token: a ~50-token memory of routing counts
constexpr float kAdmitMargin = 3.0f;  // extra routings (decayed) to displace a resident expert

// Timeline classification of one completed token (see floe_gpu_offload).
void offload_classify(floe_gpu_offload *o, const floe_gpu_offload::Readback &r) {
  const uint64_t rb = 4ull * o->dh;
  for (uint32_t l = 0; l < o->L; ++l)
    for (uint32_t k = 0; k < o->K; ++k) {
      const uint32_t i = l * o->E + r.sel[l * o->K + k];
      const uint64_t bytes = (uint64_t)r.nkept[l * o->K + k] * rb;
      o->t_demanded += o->up_bytes + bytes;
      o->t_cache += o->up_bytes;
      if (!r.resident[i]) {
        o->t_sync += bytes;
        o->t_req_ch += r.nkept[l * o->K + k];  // one bulk copy per record
      } else if (r.fresh[i] && o->fresh[i]) {
        o->t_used += bytes;
        o->t_wasted += o->rec_bytes - bytes;
        o->fresh[i] = 0;
      } else {
        o->t_cache += bytes;
      }
    }
  ++o->t_tokens;
}

// Completed tokens in order; `block` waits for the oldest one.
int offload_drain(floe_gpu_offload *o, bool block) {
  while (o->ring_n) {
    floe_gpu_offload::Readback &r = o->ring[o->ring_head];
    if (block) {
      CK(cudaEventSynchronize(r.ev));
      block = false;
    } else if (cudaEventQuery(r.ev) != cudaSuccess) {
      break;
    }
    offload_classify(o, r);
    std::memcpy(o->sel_host, r.sel, 4ull * o->L * o->K);  // the newest routing
    o->sel_fresh = true;
    r.busy = false;
    o->ring_head = (o->ring_head + 1) % (uint32_t)o->ring.size();
    --o->ring_n;
  }
  return FLOE_OK;
}

int offload_policy(floe_gpu_offload *o, cudaStream_t st) {
  const uint32_t N = o->L * o->E;
  for (uint32_t i = 0; i < N; ++i)
    if (o->state[i] == floe_gpu_offload::kCopying && cudaEventQuery(o->copy_done[i]) == cudaSuccess) {
      if (int rc = offload_switch(o, i, true, st)) return rc;
      o->state[i] = floe_gpu_offload::kResident;
      o->fresh[i] = 1;
    }
  if (int rc = offload_drain(o, o->ring_n == o->ring.size())) return rc;
  if (o->sel_pending && cudaEventQuery(o->sel_ready) == cudaSuccess) {
    o->sel_pending = false;
    o->sel_fresh = true;
  }
  if (!o->sel_fresh) return FLOE_OK;
  o->sel_fresh = false;
  std::vector<uint32_t> want;
  for (float &f : o->freq) f *= kFreqDecay;
  for (uint32_t l = 0; l < o->L; ++l)
    for (uint32_t k = 0; k < o->K; ++k) {
      const uint32_t i = l * o->E + o->sel_host[l * o->K + k];
      o->last_use[i] = o->tokens;
      o->freq[i] += 1.0f;
      if (o->state[i] == floe_gpu_offload::kHost) want.push_back(i);
    }
  for (uint32_t i : want) {
    while (o->committed + o->rec_bytes > o->budget) {  // the budget is full: pick a victim
      // least frequently routed resident expert, ties to the least recently used
      int64_t victim = -1;
      for (uint32_t j = 0; j < N; ++j)
        if (o->state[j] == floe_gpu_offload::kResident &&
            (victim < 0 || o->freq[j] < o->freq[victim] ||
             (o->freq[j] == o->freq[victim] && o->last_use[j] < o->last_use[victim])))
          victim = j;
      if (victim < 0 || o->last_use[victim] >= o->tokens) break;  // nothing evictable
      // Admission: a promotion moves the whole record block (~1/keep-fraction
      // times what one routing reads in place), so replace a resident expert
      // only for one routed clearly more often; otherwise a budget smaller
      // than the working set thrashes and pays more PCIe than it saves.
      if (o->freq[i] < o->freq[victim] + kAdmitMargin) break;
      if (int rc = offload_switch(o, (uint32_t)victim, false, st)) return rc;
      if (o->fresh[victim]) {  // promoted, never demanded: the whole batch was wasted
        o->t_wasted += o->rec_bytes;
        o->fresh[victim] = 0;
      }
      o->state[victim] = floe_gpu_offload::kHost;
      o->committed -= o->rec_bytes;
      ++o->evictions;
    }
    if (o->committed + o->rec_bytes > o->budget) break;
    floe_gpu_expert *e = o->layers[i / o->E]->experts[i % o->E];
    CK(cudaMallocAsync(reinterpret_cast<void **>(&o->pending[i]), o->rec_bytes, o->side));
    CK(cudaMemcpyAsync(o->pending[i], e->rec_host, o->rec_bytes, cudaMemcpyHostToDevice, o->side));
    CK(cudaEventRecord(o->copy_done[i], o->side));
    o->state[i] = floe_gpu_offload::kCopying;
    o->committed += o->rec_bytes;
    o->bytes_promoted += o->rec_bytes;
    ++o->promotions;
  }
  return FLOE_OK;
}
}  // namespace

extern "C" {

int floe_gpu_offload_create(floe_gpu_layer *const *layers, uint32_t n_layers,
                            uint64_t vram_budget, floe_gpu_offload **out) {
  if (!layers || !out || n_layers == 0) return fail(FLOE_ERR_INVALID, "offload_create: bad arguments");
  *out = nullptr;
  if (int rc = require_device("offload_create")) return rc;
  auto o = std::make_unique<floe_gpu_offload>();
  for (uint32_t l = 0; l < n_layers; ++l) {
    const floe_gpu_layer *ly = layers[l];
    if (!ly || ly->dh != layers[0]->dh || ly->E != layers[0]->E || ly->top_k != layers[0]->top_k ||
        ly->di != layers[0]->di)
      return fail(FLOE_ERR_INVALID, "offload_create: layer %u shape differs", l);
    o->layers.push_back(const_cast<floe_gpu_layer *>(ly));
  }
  o->L = n_layers;
  o->E = layers[0]->E;
  o->K = layers[0]->top_k;
  o->dh = layers[0]->dh;
  o->budget = vram_budget;
  o->rec_bytes = 4ull * o->dh * layers[0]->di;
  const uint32_t N = o->L * o->E;
  o->state.assign(N, floe_gpu_offload::kHost);
  o->pending.assign(N, nullptr);
  o->copy_done.assign(N, nullptr);
  o->last_use.assign(N, 0);
  o->freq.assign(N, 0.0f);
  o->resident_host.assign(N, 0);
  CK(cudaStreamCreateWithFlags(&o->side, cudaStreamNonBlocking));
  for (auto &ev : o->copy_done) CK(cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&o->sel_ready, cudaEventDisableTiming));
  CK(cudaMalloc(&o->resident_dev, N));
  CK(cudaMalloc(&o->sel_dev, 4ull * o->L * o->K));
  CK(cudaMallocHost(&o->sel_host, 4ull * o->L * o->K));
  CK(cudaMalloc(&o->buf, 8ull * o->dh));
  CK(cudaMalloc(&o->acc, 16));
  CK(cudaMemset(o->acc, 0, 16));
  CK(cudaMalloc(&o->nkept_dev, 4ull * o->L * o->K));
  o->fresh.assign(N, 0);
  o->ring.resize(4);
  for (auto &r : o->ring) {
    CK(cudaMallocHost(&r.sel, 4ull * o->L * o->K));
    CK(cudaMallocHost(&r.nkept, 4ull * o->L * o->K));
    CK(cudaEventCreateWithFlags(&r.ev, cudaEventDisableTiming));
  }
  // every expert starts host-resident (records in pinned host memory)
  for (uint32_t i = 0; i < N; ++i) {
    floe_gpu_expert *e = o->layers[i / o->E]->experts[i % o->E];
    if (e->up_only) return fail(FLOE_ERR_INVALID, "offload_create: expert without gate/down");
    if (e->resident)
      if (int rc = floe_gpu_expert_set_resident(e, 0, nullptr)) return rc;
    o->up_bytes = e->code_bytes + 4 * e->n_groups;
  }
  CK(cudaMemset(o->resident_dev, 0, N));
  CK(cudaDeviceSynchronize());
  *out = o.release();
  return FLOE_OK;
}

int floe_gpu_offload_destroy(floe_gpu_offload *o) {
  if (!o) return FLOE_OK;
  cudaDeviceSynchronize();
  for (uint32_t i = 0; i < o->L * o->E; ++i) {
    if (o->pending[i]) cudaFree(o->pending[i]);
    if (o->copy_done[i]) cudaEventDestroy(o->copy_done[i]);
  }
  if (o->sel_ready) cudaEventDestroy(o->sel_ready);
  for (auto &r : o->ring) {
    cudaFreeHost(r.sel);
    cudaFreeHost(r.nkept);
    if (r.ev) cudaEventDestroy(r.ev);
  }
  cudaFree(o->nkept_dev);
  if (o->ews) floe_gpu_workspace_destroy(o->ews);
  cudaFree(o->pmask_dev);
  cudaFree(o->tmask_dev);
  cudaFree(o->u_dev);
  cudaFree(o->pr_dev);
  cudaFree(o->pn_dev);
  cudaFree(o->pexp_dev);
  if (o->side) cudaStreamDestroy(o->side);
  cudaFree(o->resident_dev);
  cudaFree(o->sel_dev);
  cudaFreeHost(o->sel_host);
  cudaFree(o->buf);
  cudaFree(o->acc);
  delete o;
  return FLOE_OK;
}

namespace {
// One token through every layer.  replay == false: the layers chain
// (h -> layer 0 -> ... -> y, as predictor.cpp:66-83 drives layer_forward).
// replay == true: layer l reads its own recorded block input h[l] and writes
// y[l] (the traces the reference pairs with routing decisions,
// predictor.cpp:60-85), so a benchmark can hold every layer at its calibrated
// sparsity instead of following a random-weight stack's growing activations.
int offload_token(floe_gpu_offload *o, floe_gpu_workspace *ws, const float *h_dev, float *y_dev,
                  bool replay, cudaStream_t st) {
  if (int rc = offload_policy(o, st)) return rc;
  // the placement this token's kernels see (switches happen between tokens)
  floe_gpu_offload::Readback &rb = o->ring[(o->ring_head + o->ring_n) % o->ring.size()];
  rb.resident = o->resident_host;
  rb.fresh = o->fresh;
  const float *in = h_dev;
  const uint32_t di = o->layers[0]->di;
  for (uint32_t l = 0; l < o->L; ++l) {
    float *outp = replay ? y_dev + (size_t)l * o->dh
                         : (l + 1 == o->L ? y_dev : o->buf + (l & 1) * o->dh);
    if (replay) in = h_dev + (size_t)l * o->dh;
    floe_gpu_layer_trace tr{o->eval ? o->u_dev + (size_t)l * o->dh : nullptr, o->sel_dev + l * o->K,
                            nullptr, o->eval ? o->tmask_dev + (size_t)l * o->K * di : nullptr};
    const floe_gpu_layer *ly = o->layers[l];
    if (int rc = check_ws("offload_decode", ws, ly->dh, ly->di, ly->top_k)) return rc;
    if (layer_fused(ly)) {  // the fused kernel does the record accounting itself
      if (int rc = layer_forward_impl(ly, ws, in, outp, &tr, o->acc, st, nullptr,
                                      o->nkept_dev + l * o->K))
        return rc;
      if (o->eval && l > 0) {
        // reuse predictor: every expert of layer l against layer l-1's block
        // input (one K1-only pass, each expert's own threshold), scored on
        // the experts layer l routed to
        for (uint32_t e0 = 0; e0 < o->E; e0 += 2) {  // two experts per pass (smem lists)
          FusedLaunch f{};
          f.table = ly->table + e0;
          f.slots = std::min<uint32_t>(2, o->E - e0);
          f.dh = ly->dh;
          f.di = ly->di;
          f.k1_only = true;
          f.x = o->u_dev + (size_t)(l - 1) * o->dh;
          f.mask_out = o->pmask_dev + (size_t)e0 * di;
          if (int rc = launch_v2(f, o->ews, st)) return rc;
        }
        score_masks<<<o->K, 256, 0, st>>>(o->pmask_dev, o->tmask_dev + (size_t)l * o->K * di,
                                          o->sel_dev + l * o->K, di, o->pr_dev, o->pn_dev);
        CK_LAUNCH();
        if (o->pred && l < o->pred->layers) {
          if (int rc = floe_gpu_predict_experts(o->pred, o->u_dev + (size_t)(l - 1) * o->dh, l,
                                                o->pred_count, o->pexp_dev, st))
            return rc;
          score_sets<<<1, 1, 0, st>>>(o->pexp_dev, o->pred_count, o->sel_dev + l * o->K, o->K,
                                      o->pr_dev + 2, o->pn_dev + 1);
          CK_LAUNCH();
        }
      }
    } else {
      if (int rc = layer_forward_impl(ly, ws, in, outp, &tr, nullptr, st)) return rc;
      offload_account<<<1, 32, 0, st>>>(ws->seg_count, (uint32_t)device_info().sm, o->K,
                                        o->sel_dev + l * o->K, o->resident_dev + l * o->E,
                                        o->acc);
      CK_LAUNCH();
    }
    in = outp;
  }
  // every token's routing and kept counts come back (timeline, promotions)
  if (layer_fused(o->layers[0])) {
    CK(cudaMemcpyAsync(rb.sel, o->sel_dev, 4ull * o->L * o->K, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(rb.nkept, o->nkept_dev, 4ull * o->L * o->K, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(rb.ev, st));
    rb.busy = true;
    ++o->ring_n;
  } else if (!o->sel_pending) {
    CK(cudaMemcpyAsync(o->sel_host, o->sel_dev, 4ull * o->L * o->K, cudaMemcpyDeviceToHost, st));
    CK(cudaEventRecord(o->sel_ready, st));
    o->sel_pending = true;
  }
  ++o->tokens;
  return FLOE_OK;
}
}  // namespace

int floe_gpu_offload_decode(floe_gpu_offload *o, floe_gpu_workspace *ws, const float *h_dev,
                            float *y_dev, floe_stream_t stream) {
  if (!o || !ws || !h_dev || !y_dev) return fail(FLOE_ERR_INVALID, "offload_decode: null argument");
  return offload_token(o, ws, h_dev, y_dev, false, S(stream));
}

int floe_gpu_offload_decode_replay(floe_gpu_offload *o, floe_gpu_workspace *ws,
                                   const float *h_dev, float *y_dev, floe_stream_t stream) {
  if (!o || !ws || !h_dev || !y_dev)
    return fail(FLOE_ERR_INVALID, "offload_decode_replay: null argument");
  return offload_token(o, ws, h_dev, y_dev, true, S(stream));
}

int floe_gpu_offload_stats(floe_gpu_offload *o, floe_offload_stats *out, floe_stream_t stream) {
  if (!o || !out) return fail(FLOE_ERR_INVALID, "offload_stats: null argument");
  unsigned long long acc[2];
  CK(cudaStreamSynchronize(S(stream)));
  CK(cudaMemcpy(acc, o->acc, 16, cudaMemcpyDeviceToHost));
  std::memset(out, 0, sizeof *out);
  out->tokens = o->tokens;
  out->records_from_hbm = acc[0];
  out->records_over_pcie = acc[1];
  out->record_bytes = 4ull * o->dh;
  out->up_bytes_per_expert = o->up_bytes;
  out->promotions = o->promotions;
  out->evictions = o->evictions;
  out->bytes_promoted = o->bytes_promoted;
  uint64_t dev = 0;
  for (uint32_t i = 0; i < o->L * o->E; ++i)
    if (o->state[i] == floe_gpu_offload::kResident) dev += o->rec_bytes;
  out->device_record_bytes = dev;
  if (int rc = offload_drain(o, false)) return rc;  // the stream is idle: every token completes
  out->bytes_demanded = o->t_demanded;
  out->bytes_from_cache = o->t_cache;
  out->bytes_prefetch_used = o->t_used;
  out->bytes_sync = o->t_sync;
  out->bytes_prefetch_wasted = o->t_wasted;
  out->bytes_prefetch_pending = o->bytes_promoted - o->t_used - o->t_wasted;
  out->requests_up = 0;
  out->requests_channel = o->t_req_ch + o->promotions;
  if (o->eval) {
    double pr[4];
    unsigned long long pn[2];
    CK(cudaMemcpy(pr, o->pr_dev, sizeof pr, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(pn, o->pn_dev, sizeof pn, cudaMemcpyDeviceToHost));
    out->mask_samples = pn[0];
    out->set_samples = pn[1];
    out->mask_precision = pn[0] ? pr[0] / pn[0] : 0.0;
    out->mask_recall = pn[0] ? pr[1] / pn[0] : 0.0;
    out->set_precision = pn[1] ? pr[2] / pn[1] : 0.0;
    out->set_recall = pn[1] ? pr[3] / pn[1] : 0.0;
  }
  return FLOE_OK;
}

int floe_gpu_offload_set_eval(floe_gpu_offload *o, int enable, const floe_gpu_predictor *predictor,
                              uint32_t count) {
  if (!o) return fail(FLOE_ERR_INVALID, "offload_set_eval: null argument");
  if (predictor && (predictor->experts != o->E || predictor->dh != o->dh ||
                    count == 0 || count > o->E))
    return fail(FLOE_ERR_INVALID, "offload_set_eval: predictor shape mismatch");
  if (enable && !layer_fused(o->layers[0]))
    return fail(FLOE_ERR_UNSUPPORTED, "offload_set_eval: needs the fused layer path");
  if (enable && o->E > (uint32_t)floe_k::kMaxSlots)
    return fail(FLOE_ERR_UNSUPPORTED, "offload_set_eval: at most %d experts", floe_k::kMaxSlots);
  CK(cudaDeviceSynchronize());
  if (enable && !o->ews) {
    const uint32_t di = o->layers[0]->di;
    if (int rc = floe_gpu_workspace_create(o->dh, di, o->E, &o->ews)) return rc;
    CK(cudaMalloc(&o->pmask_dev, (size_t)o->E * di));
    CK(cudaMalloc(&o->tmask_dev, (size_t)o->L * o->K * di));
    CK(cudaMalloc(&o->u_dev, 4ull * o->L * o->dh));
    CK(cudaMalloc(&o->pr_dev, 4 * sizeof(double)));
    CK(cudaMalloc(&o->pn_dev, 2 * sizeof(unsigned long long)));
    CK(cudaMalloc(&o->pexp_dev, 4ull * o->E));
  }
  if (enable) {
    CK(cudaMemset(o->pr_dev, 0, 4 * sizeof(double)));
    CK(cudaMemset(o->pn_dev, 0, 2 * sizeof(unsigned long long)));
  }
  o->eval = enable != 0;
  o->pred = predictor;
  o->pred_count = count;
  return FLOE_OK;
}

}  // extern "C"

// ------------------------------------------------------------ compact pack ---
namespace {
// record c of the expert (f16 gate row | f16 down row) -> slot i of the payload
__global__ void gather_records(const __half *__restrict__ rec, const uint32_t *__restrict__ ch,
                               const uint32_t *__restrict__ n, uint32_t dh,
                               uint8_t *__restrict__ payload) {
  const uint32_t i = blockIdx.x;
  if (i >= *n) return;
  const uint4 *src = reinterpret_cast<const uint4 *>(rec + (size_t)ch[i] * 2 * dh);
  uint4 *dst = reinterpret_cast<uint4 *>(payload + (size_t)i * 4 * dh);
  for (uint32_t k = threadIdx.x; k < dh / 4; k += blockDim.x) dst[k] = src[k];
}
}  // namespace

extern "C" {

int floe_gpu_pack_compact(const floe_gpu_expert *e, const uint8_t *mask, uint32_t element_bytes,
                          uint32_t *channels, uint8_t *payload, uint32_t *n_out,
                          floe_stream_t stream) {
  if (!e || !mask || !channels || !payload || !n_out)
    return fail(FLOE_ERR_INVALID, "pack_compact: null argument");
  if (element_bytes != 2 && element_bytes != 4)
    return fail(FLOE_ERR_INVALID, "pack_compact: element_bytes must be 2 or 4");
  if (element_bytes == 4)
    return fail(FLOE_ERR_UNSUPPORTED, "pack_compact: the device holds f16 records (element_bytes 2)");
  if (e->up_only) return fail(FLOE_ERR_INVALID, "pack_compact: expert has no gate/down records");
  if (e->dh % 8) return fail(FLOE_ERR_UNSUPPORTED, "pack_compact: d_hidden must be a multiple of 8");
  cudaStream_t st = S(stream);
  size_t tmp = 0;
  cub::CountingInputIterator<uint32_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, tmp, it, mask, channels, n_out, (int)e->di, st);
  void *t = nullptr;
  CK(cudaMallocAsync(&t, tmp, st));
  cub::DeviceSelect::Flagged(t, tmp, it, mask, channels, n_out, (int)e->di, st);
  gather_records<<<e->di, 256, 0, st>>>(e->host_desc.records, channels, n_out, e->dh, payload);
  const cudaError_t ce = cudaGetLastError();
  cudaFreeAsync(t, st);
  if (ce != cudaSuccess) return fail(FLOE_ERR_CUDA, "pack_compact: %s", cudaGetErrorString(ce));
  return FLOE_OK;
}

}  // extern "C"

// ------------------------------------------------------- batched MoE layer ---
// Experts routed at most this many tokens of a batch run them through the fused
// single-expert kernel (FLOE_BATCHED_SMALL overrides; measured crossover).
static const uint32_t kBatchedSmall = [] {
  const char *p = std::getenv("FLOE_BATCHED_SMALL");
  return p ? (uint32_t)std::atoi(p) : 0u;  // 0: with the experts concurrent, none
}();
// Batches of at most this many tokens run token by token through the fused
// layer kernel (FLOE_LAYER_PER_TOKEN overrides).
// (5 with the experts concurrent: a 5..7-token union pass reads ~the whole
// record set in two 4-token groups; 24 tokens per layer call 0.68 -> 0.59 ms)
static const uint32_t kPrefillMin = [] {  // tokens per expert for the prefill GEMMs
  const char *p = std::getenv("FLOE_PREFILL_MIN");
  return p ? (uint32_t)std::atoi(p) : 5u;
}();
// tokens per call from which f16 mixing runs as the two tensor-core GEMMs
// (measured: 16 tokens 1.115 -> 0.952 ms per layer call; the CUDA-core
// mix_batched re-reads h per 256-column chunk and is latency-bound)
static const uint32_t kMixGemmMin = [] {
  const char *p = std::getenv("FLOE_MIX_GEMM_MIN");
  return p ? (uint32_t)std::atoi(p) : 1u;
}();
// Side streams of the batched layer (per device, created once, non-blocking);
// FLOE_LAYER_STREAMS=1 keeps every expert on the caller's stream.
constexpr int kSideStreams = 8;
static const int kLayerStreams = [] {
  const char *p = std::getenv("FLOE_LAYER_STREAMS");
  return p ? std::atoi(p) : kSideStreams;
}();
// experts routed at least this many tokens stay on the caller's stream (the
// default: those past the exact up projection, whose dequantized-copy scratch
// of 352 MB per expert would be held 8 times over)
static const uint32_t kLayerSerialMin = [] {
  const char *p = std::getenv("FLOE_LAYER_SERIAL_MIN");
  return p ? (uint32_t)std::atoi(p) : 65u;
}();
static cudaStream_t *side_streams() {
  static std::mutex mu;
  static cudaStream_t pool[64][kSideStreams] = {};
  static int state[64] = {};  // 0 untried, 1 ready, -1 failed (serial from then on)
  if (kLayerStreams <= 1) return nullptr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> g(mu);
  if (state[dev] == 0) {
    state[dev] = 1;
    for (auto &s : pool[dev])
      if (cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking) != cudaSuccess || !lt_reserve(s)) {
        state[dev] = -1;  // the layer keeps every expert on the caller's stream
        break;
      }
  }
  return state[dev] == 1 ? pool[dev] : nullptr;
}
static const uint32_t kLayerPerToken = [] {
  const char *p = std::getenv("FLOE_LAYER_PER_TOKEN");
  return p ? (uint32_t)std::atoi(p) : 10u;
}();
extern "C" {

int floe_gpu_layer_forward_batched(const floe_gpu_layer *l, floe_gpu_workspace *ws,
                                   const float *h, uint32_t n_tokens, float *y,
                                   floe_stream_t stream) {
  if (!l || !h || !y) return fail(FLOE_ERR_INVALID, "layer_forward: null argument");
  if (ws)
    if (int rc = check_ws("layer_forward_batched", ws, l->dh, l->di, 1)) return rc;
  if (n_tokens == 0) return FLOE_OK;
  if (!l->fast)
    return fail(FLOE_ERR_UNSUPPORTED, "layer_forward_batched: needs the tile layout");
  if (int rc = require_device("layer_forward_batched")) return rc;
  cudaStream_t st = S(stream);
  const uint32_t T = n_tokens, E = l->E, K = l->top_k, dh = l->dh, P = T * K;
  // Small batches: the fused single-token layer kernel per token is faster
  // (one launch per token, mixing + both experts; tools/bench_blayer.py)
  if (ws && T <= kLayerPerToken && ws->slots >= K) {
    for (uint32_t t = 0; t < T; ++t)
      if (int rc = floe_gpu_layer_forward(l, ws, h + (size_t)t * dh, y + (size_t)t * dh, nullptr,
                                          stream))
        return rc;
    return FLOE_OK;
  }
  // scratch: u [T][dh] | logits [T][E] | sel [P] | w [P] | counts [E] | lists [E][T] |
  //          X [T][dh] (one expert's rows) | Y [T][dh] | out [P][dh] |
  //          mixing GEMM: Ha [T][3dh] f16, inv [T], M.h [T][dh]
  const size_t CH = floe_tc::kMaxTokens;
  const bool mix_tc = l->mix_f16 && T >= kMixGemmMin;
  const size_t o_u = 0, o_lg = o_u + 4ull * T * dh, o_sel = o_lg + 4ull * T * E;
  const size_t o_w = o_sel + 4ull * P, o_cnt = o_w + 4ull * P, o_lst = o_cnt + 4ull * 32;
  const size_t o_x = (o_lst + 4ull * E * T + 255) & ~size_t(255);
  // X and Y hold every expert's rows at its own offset (experts run concurrently)
  const size_t o_y = o_x + 4ull * P * dh, o_out = o_y + 4ull * P * dh;
  const size_t o_ha = o_out + 4ull * P * dh, o_hinv = o_ha + (mix_tc ? 2ull * T * 3 * dh : 0);
  const size_t o_mh = (o_hinv + 4ull * T + 255) & ~size_t(255);
  const size_t total = o_mh + (mix_tc ? 4ull * T * dh : 0);
  uint8_t *sc = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void **>(&sc), total, st));
  float *u = reinterpret_cast<float *>(sc + o_u), *lg = reinterpret_cast<float *>(sc + o_lg);
  uint32_t *sel = reinterpret_cast<uint32_t *>(sc + o_sel);
  float *w = reinterpret_cast<float *>(sc + o_w);
  uint32_t *cnt = reinterpret_cast<uint32_t *>(sc + o_cnt), *lst = reinterpret_cast<uint32_t *>(sc + o_lst);
  float *X = reinterpret_cast<float *>(sc + o_x), *Y = reinterpret_cast<float *>(sc + o_y);
  float *outp = reinterpret_cast<float *>(sc + o_out);
  auto done = [&](int rc) {
    cudaFreeAsync(sc, st);
    return rc;
  };
  // u = h + mixing h (model.cpp:150-152).  Many tokens with f16 mixing: two
  // tensor-core GEMMs over the hi and lo halves of the row-scaled h (f32
  // accumulation); otherwise kMixTok tokens per pass on the CUDA cores.
  const uint32_t mix_smem = 4u * floe_bl::kMixTok * 256u;
  if (mix_tc) {
    keep_pool();
    __half *Ha = reinterpret_cast<__half *>(sc + o_ha);
    float *hinv = reinterpret_cast<float *>(sc + o_hinv), *mh = reinterpret_cast<float *>(sc + o_mh);
    floe_pf::xcat<<<T, 1024, 0, st>>>(h, dh, Ha, hinv);
    const __half *M = static_cast<const __half *>(l->mixing);
    const int D = (int)dh, N = (int)T;
    if (int rc = lt_gemm(true, false, D, N, D, M, D, Ha, 3 * D, 0.0f, mh, D, st)) return done(rc);
    if (int rc = lt_gemm(true, false, D, N, D, M, D, Ha + 2 * dh, 3 * D, 1.0f, mh, D, st)) return done(rc);
    floe_pf::residual<<<T, 1024, 0, st>>>(h, mh, hinv, dh, u);
  }
  for (uint32_t t0 = 0; t0 < (mix_tc ? 0u : T); t0 += floe_bl::kMixTok) {
    const uint32_t nt = std::min<uint32_t>(floe_bl::kMixTok, T - t0);
    if (l->mix_f16) {
      if (int rc = set_smem(floe_bl::mix_batched<__half>, mix_smem)) return done(rc);
      floe_bl::mix_batched<__half><<<(dh + 7) / 8, 256, 4u * nt * 256u, st>>>(
          static_cast<const __half *>(l->mixing), dh, h + (size_t)t0 * dh, nt, u + (size_t)t0 * dh);
    } else {
      if (int rc = set_smem(floe_bl::mix_batched<float>, mix_smem)) return done(rc);
      floe_bl::mix_batched<float><<<(dh + 7) / 8, 256, 4u * nt * 256u, st>>>(
          static_cast<const float *>(l->mixing), dh, h + (size_t)t0 * dh, nt, u + (size_t)t0 * dh);
    }
  }
  // route (model.cpp:83-93) and group the (token, slot) pairs by expert
  if (cudaMemsetAsync(cnt, 0, 4ull * E, st) != cudaSuccess)
    return done(fail(FLOE_ERR_CUDA, "layer_forward_batched: memset failed"));
  floe_bl::router_logits<<<(T * E * 32 + 255) / 256, 256, 0, st>>>(l->router, E, dh, u, T, lg);
  floe_bl::route_batched<<<(T * 32 + 255) / 256, 256, 0, st>>>(lg, T, E, K, sel, w, cnt, lst);
  if (cudaGetLastError() != cudaSuccess)
    return done(fail(FLOE_ERR_CUDA, "layer_forward_batched: launch failed"));
  uint32_t hc[32];
  if (cudaMemcpyAsync(hc, cnt, 4ull * E, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return done(fail(FLOE_ERR_CUDA, "layer_forward_batched: routing readback failed"));
  // every expert over its tokens: a few tokens go one by one through the fused
  // single-expert kernel (one pass over the expert per token, ~15 us), more
  // through the prefill GEMMs (the expert read once) or the batched forward.
  // Experts on the prefill / batched paths run concurrently on side streams
  // (each is a few small kernels that leave SMs idle on its own); the fused
  // single-expert kernel synchronises its grid, so those experts stay on the
  // caller's stream, issued before the fork.
  uint32_t off[33];
  off[0] = 0;
  for (uint32_t e = 0; e < E; ++e) off[e + 1] = off[e] + hc[e];
  auto on_main = [&](uint32_t n) { return ws && n < kPrefillMin && n <= kBatchedSmall; };
  // The exact batched up projections of the concurrent experts run first, one
  // after another on the caller's stream (with the IMMA up projection inside
  // the side streams, a few layer calls in a hundred ended in an unspecified
  // launch failure); v then feeds the concurrent gate/down stage.
  const bool concurrent = side_streams() != nullptr;
  auto pre_k1 = [&](uint32_t n) {
    return concurrent && n && !on_main(n) &&
           (n >= kPrefillMin ? n <= kExactK1Max : n <= (uint32_t)CH);
  };
  uint32_t voff[33];
  voff[0] = 0;
  for (uint32_t e = 0; e < E; ++e) voff[e + 1] = voff[e] + (pre_k1(hc[e]) ? hc[e] : 0u);
  float *V = nullptr;
  if (voff[E]) {
    if (cudaMallocAsync(reinterpret_cast<void **>(&V), 4ull * voff[E] * l->di, st) != cudaSuccess)
      return done(fail(FLOE_ERR_CUDA, "layer_forward_batched: scratch allocation failed"));
    for (uint32_t e = 0; e < E; ++e) {
      if (voff[e + 1] == voff[e]) continue;
      const uint32_t n = hc[e];
      float *Xe = X + (size_t)off[e] * dh;
      floe_bl::gather_rows<<<dim3(4, n), 256, 0, st>>>(u, lst + (size_t)e * T, n, K, dh, Xe);
      if (int rc = floe_gpu_qgemv_channels_batched(l->experts[e], Xe, n,
                                                   V + (size_t)voff[e] * l->di, stream)) {
        cudaFreeAsync(V, st);
        return done(rc);
      }
    }
  }
  auto run_expert = [&](uint32_t e, cudaStream_t es) -> int {
    float *Xe = X + (size_t)off[e] * dh, *Ye = Y + (size_t)off[e] * dh;
    floe_stream_t fs = reinterpret_cast<floe_stream_t>(es);
    if (hc[e] >= kPrefillMin) {  // many tokens: the prefill GEMMs, the expert read once
      const uint32_t n = hc[e];
      const uint32_t *pairs = lst + (size_t)e * T;
      const float *ve = voff[e + 1] > voff[e] ? V + (size_t)voff[e] * l->di : nullptr;
      if (!ve) floe_bl::gather_rows<<<dim3(4, n), 256, 0, es>>>(u, pairs, n, K, dh, Xe);
      if (int rc = prefill_impl(l->experts[e], Xe, n, Ye, fs, ve)) return rc;
      floe_bl::scatter_rows<<<dim3(4, n), 256, 0, es>>>(Ye, pairs, n, dh, outp);
      return FLOE_OK;
    }
    const float *ve = voff[e + 1] > voff[e] ? V + (size_t)voff[e] * l->di : nullptr;  // one chunk
    for (uint32_t c0 = 0; c0 < hc[e]; c0 += (uint32_t)CH) {
      const uint32_t n = std::min<uint32_t>((uint32_t)CH, hc[e] - c0);
      const uint32_t *pairs = lst + (size_t)e * T + c0;
      if (!ve) floe_bl::gather_rows<<<dim3(4, n), 256, 0, es>>>(u, pairs, n, K, dh, Xe);
      if (ve) {
        if (int rc = batched_impl(l->experts[e], Xe, n, Ye, nullptr, fs, ve)) return rc;
      } else if (on_main(n)) {
        for (uint32_t i = 0; i < n; ++i)
          if (int rc = floe_gpu_expert_forward_sparse(l->experts[e], ws, Xe + (size_t)i * dh,
                                                      Ye + (size_t)i * dh, nullptr, nullptr,
                                                      nullptr, nullptr, fs))
            return rc;
      } else if (int rc = floe_gpu_expert_forward_batched(l->experts[e], Xe, n, Ye, nullptr, fs)) {
        return rc;
      }
      floe_bl::scatter_rows<<<dim3(4, n), 256, 0, es>>>(Ye, pairs, n, dh, outp);
    }
    return FLOE_OK;
  };
  // experts with many tokens (>= FLOE_LAYER_SERIAL_MIN) fill the GPU on their
  // own and run one after another on the caller's stream too (8 experts of
  // ~1000 tokens concurrently: 4096-token layer 5.7 -> 12 ms)
  auto serial = [&](uint32_t n) { return on_main(n) || n >= kLayerSerialMin; };
  for (uint32_t e = 0; e < E; ++e)
    if (hc[e] && serial(hc[e]))
      if (int rc = run_expert(e, st)) {
        if (V) cudaFreeAsync(V, st);
        return done(rc);
      }
  cudaStream_t *side = side_streams();
  uint32_t nside = 0;
  for (uint32_t e = 0; e < E; ++e) nside += hc[e] && !serial(hc[e]);
  nside = std::min<uint32_t>(nside, (uint32_t)std::min(kLayerStreams, kSideStreams));
  if (!side) nside = 0;
  if (nside <= 1) {
    for (uint32_t e = 0; e < E; ++e)
      if (hc[e] && !serial(hc[e]))
        if (int rc = run_expert(e, st)) {
          if (V) cudaFreeAsync(V, st);
          return done(rc);
        }
  } else {
    cudaEvent_t fork = nullptr, join[kSideStreams] = {};
    bool ok = cudaEventCreateWithFlags(&fork, cudaEventDisableTiming) == cudaSuccess &&
              cudaEventRecord(fork, st) == cudaSuccess;
    for (uint32_t i = 0; ok && i < nside; ++i)
      ok = cudaEventCreateWithFlags(&join[i], cudaEventDisableTiming) == cudaSuccess &&
           cudaStreamWaitEvent(side[i], fork, 0) == cudaSuccess;
    int rc = ok ? FLOE_OK : fail(FLOE_ERR_CUDA, "layer_forward_batched: stream fork failed");
    // the largest experts first, dealt round-robin over the side streams
    uint32_t order[32], no = 0;
    for (uint32_t e = 0; e < E; ++e)
      if (hc[e] && !serial(hc[e])) order[no++] = e;
    std::stable_sort(order, order + no, [&](uint32_t a, uint32_t b) { return hc[a] > hc[b]; });
    for (uint32_t j = 0; rc == FLOE_OK && j < no; ++j) rc = run_expert(order[j], side[j % nside]);
    // join on every path: the scratch is freed on the caller's stream
    for (uint32_t i = 0; i < nside; ++i) {
      if (!join[i]) continue;
      if (cudaEventRecord(join[i], side[i]) != cudaSuccess ||
          cudaStreamWaitEvent(st, join[i], 0) != cudaSuccess)
        if (rc == FLOE_OK) rc = fail(FLOE_ERR_CUDA, "layer_forward_batched: stream join failed");
      cudaEventDestroy(join[i]);
    }
    if (fork) cudaEventDestroy(fork);
    if (rc != FLOE_OK) {
      if (V) cudaFreeAsync(V, st);
      return done(rc);
    }
  }
  if (V) cudaFreeAsync(V, st);
  floe_bl::combine<<<dim3(4, T), 256, 0, st>>>(u, outp, w, K, dh, y);
  if (cudaGetLastError() != cudaSuccess)
    return done(fail(FLOE_ERR_CUDA, "layer_forward_batched: launch failed"));
  return done(FLOE_OK);
}

}  // extern "C"

// ------------------------------------------------------------------ models ---
// A stack of HBM-resident compressed layers decoded token by token: the
// reference's `run` loop h = layer_forward(m, l, h) over l (cli.cpp:86-107).
struct floe_gpu_model {
  std::vector<const floe_gpu_layer *> layers;
  uint32_t dh = 0;
  float *buf = nullptr;                        // ping-pong [2][dh]
  float *hin = nullptr, *hout = nullptr;       // device staging [L][dh]
  float *pin_in = nullptr, *pin_out = nullptr; // pinned host staging [L][dh]
  floe_v3::LayerDesc *ldesc = nullptr;         // [L] device: the multi-layer decode kernel
  bool multi = false;                          // every layer fits floe_v3::decode
};

extern "C++" {
namespace {

// One launch of floe_v3::decode: the token through every layer of the model.
template <int DH>
int launch_v3_dh(const floe_gpu_model *m, floe_gpu_workspace *ws, const float *h, float *y,
                 int replay, cudaStream_t st) {
  namespace V = floe_v2;
  namespace W = floe_v3;
  const floe_gpu_layer *l0 = m->layers[0];
  const uint32_t G = std::min<uint32_t>((uint32_t)device_info().sm, V::kMaxGrid);
  const uint32_t NT = l0->top_k * V::tiles_per_expert(l0->di);
  const uint32_t max_tiles = std::max<uint32_t>(1, (NT + G - 1) / G);
  static int optin = [] {
    int v = 0;
    cudaDeviceGetAttribute(&v, cudaDevAttrMaxSharedMemoryPerBlockOptin, 0);
    return v;
  }();
  static size_t static_smem = [] {
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, W::decode<DH>);
    return fa.sharedSizeBytes;
  }();
  const uint32_t ns = W::ring_stages(DH);
  const uint32_t smem = V::smem_layout(DH, ns, max_tiles, G).total;
  if ((int64_t)smem + (int64_t)static_smem + 1024 > (int64_t)optin)
    return fail(FLOE_ERR_UNSUPPORTED, "decode: shared memory too small for the ring");
  W::DecodeArgs a{};
  a.layers = m->ldesc;
  a.n_layers = (uint32_t)m->layers.size();
  a.n_experts = l0->E;
  a.top_k = l0->top_k;
  a.di = l0->di;
  a.h = h;
  a.y = y;
  a.buf = m->buf;
  a.replay = replay;
  a.u = ws->u;
  a.partial = ws->mix_partial;
  a.pred_partial = ws->pred_partial;
  a.pcnt = ws->pcnt;
  a.bar = ws->bar;
  a.lbar = ws->lbar;
  a.stats = ws->stats;
  a.place_acc = nullptr;
  a.phase_ns = ws->phase_ns;
  static const uint32_t trace_layer = [] {
    const char *p = std::getenv("FLOE_TRACE_LAYER");
    return p ? (uint32_t)std::atoi(p) : 0xffffffffu;
  }();
  a.trace_layer = trace_layer == 0xffffffffu ? a.n_layers - 1 : trace_layer;
  a.ns = ns;
  a.max_tiles = max_tiles;
  static const uint32_t dbg = [] {
    const char *d = std::getenv("FLOE_TEST_MISPREDICT");
    return (d && std::strcmp(d, "1") == 0) ? 8u : 0u;
  }();
  a.debug = dbg;
  if (int rc = set_smem(W::decode<DH>, smem)) return rc;
  void *kargs[] = {&a};
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(G);
  cfg.blockDim = dim3(V::kThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  // Same launch as floe_v2::fused (see launch_v2_dh): one CTA per SM, PDL,
  // CTA pairs; FLOE_COOP=1 keeps the cooperative launch (no pairs).
  static const bool coop_env = [] {
    const char *p = std::getenv("FLOE_COOP");
    if (p) return std::strcmp(p, "0") != 0;
    return std::getenv("CUDA_MPS_ACTIVE_THREAD_PERCENTAGE") != nullptr;
  }();
  static const bool pairs_env = [] {
    const char *p = std::getenv("FLOE_PAIRS");
    return !(p && std::strcmp(p, "0") == 0);
  }();
  cudaLaunchAttribute attr[3];
  uint32_t na = 0;
  if (coop_env) {
    attr[na].id = cudaLaunchAttributeCooperative;
    attr[na++].val.cooperative = 1;
  } else if (!ws->profiling) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na++].val.programmaticStreamSerializationAllowed = 1;
  }
  a.paired = (pairs_env && !coop_env && (G % 2) == 0) ? 1 : 0;
  if (a.paired) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = 2;
    attr[na].val.clusterDim.y = 1;
    attr[na++].val.clusterDim.z = 1;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  StageScope prof(ws, kStageFused, st);
  const cudaError_t e = cudaLaunchKernelExC(&cfg, reinterpret_cast<const void *>(W::decode<DH>), kargs);
  if (e != cudaSuccess) return fail(FLOE_ERR_CUDA, "decode launch failed: %s", cudaGetErrorString(e));
  CK_LAUNCH();
  return FLOE_OK;
}

bool multi_env() {
  static const bool on = [] {
    const char *p = std::getenv("FLOE_MULTI");
    return !(p && std::strcmp(p, "0") == 0);
  }();
  return on;
}

}  // namespace
}  // extern "C++"

extern "C" {

int floe_gpu_model_create(floe_gpu_layer *const *layers, uint32_t n_layers,
                          floe_gpu_model **out) {
  if (!layers || !out || n_layers == 0) return fail(FLOE_ERR_INVALID, "model_create: bad arguments");
  *out = nullptr;
  if (int rc = require_device("model_create")) return rc;
  auto m = std::make_unique<floe_gpu_model>();
  for (uint32_t l = 0; l < n_layers; ++l) {
    if (!layers[l] || layers[l]->dh != layers[0]->dh)
      return fail(FLOE_ERR_INVALID, "model_create: layer %u shape differs", l);
    m->layers.push_back(layers[l]);
  }
  m->dh = layers[0]->dh;
  const size_t v = 4ull * m->dh * n_layers;
  CK(cudaMalloc(&m->buf, 8ull * m->dh));
  // the multi-layer decode kernel: fast-path layers of one shape, f16 mixing,
  // at most 8 experts
  const floe_gpu_layer *l0 = layers[0];
  bool multi = (l0->dh == 4096 || l0->dh == 2048) && l0->E <= (uint32_t)floe_v3::kMaxE &&
               l0->top_k <= (uint32_t)floe_k::kMaxSlots;
  for (uint32_t l = 0; l < n_layers && multi; ++l) {
    const floe_gpu_layer *ly = layers[l];
    multi = ly->fast && ly->mix_f16 && ly->router_pred && ly->dh == l0->dh && ly->di == l0->di &&
            ly->E == l0->E && ly->top_k == l0->top_k;
  }
  if (multi) {
    std::vector<floe_v3::LayerDesc> ld(n_layers);
    for (uint32_t l = 0; l < n_layers; ++l)
      ld[l] = {static_cast<const __half *>(layers[l]->mixing), layers[l]->router,
               layers[l]->router_pred, layers[l]->table};
    CK(cudaMalloc(&m->ldesc, sizeof(floe_v3::LayerDesc) * n_layers));
    CK(cudaMemcpy(m->ldesc, ld.data(), sizeof(floe_v3::LayerDesc) * n_layers,
                  cudaMemcpyHostToDevice));
    m->multi = true;
  }
  CK(cudaMalloc(&m->hin, v));
  CK(cudaMalloc(&m->hout, v));
  CK(cudaMallocHost(&m->pin_in, v));
  CK(cudaMallocHost(&m->pin_out, v));
  *out = m.release();
  return FLOE_OK;
}

int floe_gpu_model_destroy(floe_gpu_model *m) {
  if (!m) return FLOE_OK;
  cudaDeviceSynchronize();
  cudaFree(m->buf);
  cudaFree(m->ldesc);
  cudaFree(m->hin);
  cudaFree(m->hout);
  cudaFreeHost(m->pin_in);
  cudaFreeHost(m->pin_out);
  delete m;
  return FLOE_OK;
}

// replay == 0: h [dh] -> layer 0 -> ... -> y [dh];  replay != 0: layer l reads
// h[l] and writes y[l] (recorded block inputs, predictor.cpp:60-85): every
// layer's work is that of a decode whose hidden states keep their scale, and
// each launch still waits for the previous layer (stream order + PDL), as a
// chained decode does.
int floe_gpu_model_decode(floe_gpu_model *m, floe_gpu_workspace *ws, const float *h, float *y,
                          int replay, floe_stream_t stream) {
  if (!m || !ws || !h || !y) return fail(FLOE_ERR_INVALID, "model_decode: null argument");
  cudaStream_t st = S(stream);
  const uint32_t L = (uint32_t)m->layers.size();
  if (m->multi && multi_env()) {  // one launch for the whole token
    if (int rc = check_ws("model_decode", ws, m->dh, m->layers[0]->di, m->layers[0]->top_k)) return rc;
    return m->dh == 4096 ? launch_v3_dh<4096>(m, ws, h, y, replay, st)
                         : launch_v3_dh<2048>(m, ws, h, y, replay, st);
  }
  const float *in = h;
  for (uint32_t l = 0; l < L; ++l) {
    const floe_gpu_layer *ly = m->layers[l];
    if (int rc = check_ws("layer_forward", ws, ly->dh, ly->di, ly->top_k)) return rc;
    float *o = replay ? y + (size_t)l * m->dh : (l + 1 == L ? y : m->buf + (l & 1) * m->dh);
    if (replay) in = h + (size_t)l * m->dh;
    const floe_gpu_layer *next = m->layers[(l + 1) % L];  // the next token starts at layer 0
    if (int rc = layer_forward_impl(ly, ws, in, o, nullptr, nullptr, st, next)) return rc;
    in = o;
  }
  return FLOE_OK;
}

int floe_gpu_model_multi_layer(const floe_gpu_model *m) {
  return m && m->multi && multi_env() ? 1 : 0;
}

int floe_gpu_model_decode_host(floe_gpu_model *m, floe_gpu_workspace *ws, const float *h_host,
                               float *y_host, int replay, floe_stream_t stream) {
  if (!m || !ws || !h_host || !y_host) return fail(FLOE_ERR_INVALID, "model_decode: null argument");
  cudaStream_t st = S(stream);
  const size_t bytes = 4ull * m->dh * (replay ? m->layers.size() : 1);
  // page-locked caller buffers are copied directly; pageable ones go through
  // the model's pinned staging buffers (a host memcpy each way)
  auto page_locked = [](const void *p) {
    cudaPointerAttributes at{};
    if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
      cudaGetLastError();
      return false;
    }
    return at.type == cudaMemoryTypeHost;
  };
  const bool direct_in = page_locked(h_host), direct_out = page_locked(y_host);
  if (!direct_in) std::memcpy(m->pin_in, h_host, bytes);
  CK(cudaMemcpyAsync(m->hin, direct_in ? h_host : m->pin_in, bytes, cudaMemcpyHostToDevice, st));
  if (int rc = floe_gpu_model_decode(m, ws, m->hin, m->hout, replay, stream)) return rc;
  CK(cudaMemcpyAsync(direct_out ? y_host : m->pin_out, m->hout, bytes, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (!direct_out) std::memcpy(y_host, m->pin_out, bytes);
  return FLOE_OK;
}

}  // extern "C"

// ------------------------------------------------------------ calibration ---
// collect_stats / calibrate_model on the device (floe_calib.cuh; reference
// core/src/model.cpp:242-330, core/src/sparsify.cpp:42-64,128-142).
struct floe_gpu_calib {
  uint32_t L = 0, E = 0, dh = 0, di = 0;
  uint64_t cap = 0, seed = 0;
  float *samples = nullptr;          // [L*E][cap]
  floe_cal::ResState *st = nullptr;  // [L*E]
  uint32_t *owner = nullptr;         // [cap]
};

extern "C" {

int floe_gpu_calib_create(uint32_t layers, uint32_t experts, uint32_t d_hidden,
                          uint32_t d_intermediate, uint64_t seed, uint64_t sample_cap,
                          floe_gpu_calib **out) {
  if (!out) return fail(FLOE_ERR_INVALID, "calib_create: null argument");
  *out = nullptr;
  if (int rc = require_device("calib_create")) return rc;
  if (layers == 0 || experts == 0 || experts > 32 || d_hidden == 0 || d_intermediate == 0 ||
      sample_cap == 0 || sample_cap > 0xffffffffull)
    return fail(FLOE_ERR_INVALID, "calib_create: need layers, d_hidden, d_intermediate, cap >= 1 "
                                  "and 1 <= experts <= 32");
  auto *c = new (std::nothrow) floe_gpu_calib();
  if (!c) return fail(FLOE_ERR_OOM, "calib_create: host allocation failed");
  c->L = layers;
  c->E = experts;
  c->dh = d_hidden;
  c->di = d_intermediate;
  c->cap = sample_cap;
  c->seed = seed;
  const uint32_t R = layers * experts;
  cudaError_t ce = cudaMalloc(&c->samples, 4ull * R * sample_cap);
  if (ce == cudaSuccess) ce = cudaMalloc(&c->st, sizeof(floe_cal::ResState) * R);
  if (ce == cudaSuccess) ce = cudaMalloc(&c->owner, 4ull * sample_cap);
  if (ce == cudaSuccess) {
    // SampleReservoir(cap, seed ^ 0x5eedca11, layer * E + expert) (model.cpp:300-304)
    floe_cal::reservoir_init<<<(R + 127) / 128, 128>>>(c->st, seed ^ 0x5eedca11ull, 0, R);
    ce = cudaGetLastError();
  }
  if (ce == cudaSuccess) ce = cudaDeviceSynchronize();
  if (ce != cudaSuccess) {
    floe_gpu_calib_destroy(c);
    return fail(FLOE_ERR_OOM, "calib_create: %s", cudaGetErrorString(ce));
  }
  *out = c;
  return FLOE_OK;
}

int floe_gpu_calib_destroy(floe_gpu_calib *c) {
  if (!c) return FLOE_OK;
  cudaDeviceSynchronize();
  if (c->samples) cudaFree(c->samples);
  if (c->st) cudaFree(c->st);
  if (c->owner) cudaFree(c->owner);
  delete c;
  return FLOE_OK;
}

int floe_gpu_calib_layer(floe_gpu_calib *c, uint32_t layer, const floe_float_layer_view *w,
                         uint32_t top_k, float drift_scale, const float *h, float *h_next,
                         uint32_t tokens, floe_stream_t stream) {
  namespace C = floe_cal;
  if (!c || !w || !h) return fail(FLOE_ERR_INVALID, "collect_stats: null argument");
  if (tokens == 0) return fail(FLOE_ERR_INVALID, "collect_stats: empty token stream");
  if (layer >= c->L) return fail(FLOE_ERR_INVALID, "collect_stats: bad layer");
  if (top_k == 0 || top_k > c->E)
    return fail(FLOE_ERR_INVALID, "model config: need 1 <= top_k <= experts");
  if (!w->router || !w->mixing || !w->gate || !w->up || !w->down_t)
    return fail(FLOE_ERR_INVALID, "collect_stats: incomplete layer view");
  cudaStream_t st = S(stream);
  const uint32_t E = c->E, dh = c->dh, di = c->di, T = tokens, K = top_k, P = T * K;
  // scratch (stream-ordered): u, logits, sel, w, pairs, acoef, vals, out, pointer tables
  const size_t o_u = 0, o_lg = o_u + 4ull * T * dh, o_sel = o_lg + 4ull * T * E;
  const size_t o_w = o_sel + 4ull * P, o_pr = (o_w + 4ull * P + 15) & ~size_t(15);
  const size_t o_pof = o_pr + sizeof(C::Pair) * P;
  const size_t o_ac = (o_pof + 4ull * P + 255) & ~size_t(255);
  const size_t o_val = o_ac + 4ull * P * di, o_out = o_val + 4ull * P * di;
  const size_t o_ptr = (o_out + 4ull * P * dh + 15) & ~size_t(15);
  const size_t total = o_ptr + 8ull * 4 * E;
  uint8_t *sc = nullptr;
  CK(cudaMallocAsync(reinterpret_cast<void **>(&sc), total, st));
  float *u = reinterpret_cast<float *>(sc + o_u), *lg = reinterpret_cast<float *>(sc + o_lg);
  uint32_t *sel = reinterpret_cast<uint32_t *>(sc + o_sel);
  float *wt = reinterpret_cast<float *>(sc + o_w);
  C::Pair *pairs = reinterpret_cast<C::Pair *>(sc + o_pr);
  int32_t *pair_of = reinterpret_cast<int32_t *>(sc + o_pof);
  float *acoef = reinterpret_cast<float *>(sc + o_ac), *vals = reinterpret_cast<float *>(sc + o_val);
  float *outp = reinterpret_cast<float *>(sc + o_out);
  const float **ptrs = reinterpret_cast<const float **>(sc + o_ptr);  // up | gate | down | vals
  int rc = FLOE_OK;
  auto done = [&](int r) {
    cudaFreeAsync(sc, st);
    return r;
  };
  // u = h + drift * mixing h; logits = router u; route
  C::gemv_seq<<<dim3((dh + 255) / 256, T), 256, 0, st>>>(w->mixing, dh, dh, h, h, drift_scale, u);
  C::gemv_seq<<<dim3((E + 255) / 256, T), 256, 0, st>>>(w->router, E, dh, u, nullptr, 1.0f, lg);
  C::route_tokens<<<(T + 127) / 128, 128, 0, st>>>(lg, T, E, K, sel, wt);
  if (cudaGetLastError() != cudaSuccess) return done(fail(FLOE_ERR_CUDA, "collect_stats: launch failed"));
  // (token, expert) pairs in token order; position of each token among its
  // expert's tokens (the reservoir's add order: tokens, then channels)
  std::vector<uint32_t> hsel(P);
  if (cudaMemcpyAsync(hsel.data(), sel, 4ull * P, cudaMemcpyDeviceToHost, st) != cudaSuccess ||
      cudaStreamSynchronize(st) != cudaSuccess)
    return done(fail(FLOE_ERR_CUDA, "collect_stats: routing readback failed"));
  std::vector<uint32_t> n_e(E, 0), off(E, 0);
  std::vector<C::Pair> hp(P);
  std::vector<int32_t> hpof(P);
  for (uint32_t t = 0; t < T; ++t)
    for (uint32_t j = 0; j < K; ++j) {
      const uint32_t e = hsel[t * K + j];
      hp[t * K + j] = C::Pair{t, j, e, n_e[e]++};
      hpof[t * K + j] = (int32_t)(t * K + j);
    }
  for (uint32_t e = 1; e < E; ++e) off[e] = off[e - 1] + n_e[e - 1];
  std::vector<const float *> hptr(4 * E);
  for (uint32_t e = 0; e < E; ++e) {
    hptr[e] = w->up[e];
    hptr[E + e] = w->gate[e];
    hptr[2 * E + e] = w->down_t[e];
    hptr[3 * E + e] = vals + (size_t)off[e] * di;
  }
  if (cudaMemcpyAsync(pairs, hp.data(), sizeof(C::Pair) * P, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(pair_of, hpof.data(), 4ull * P, cudaMemcpyHostToDevice, st) != cudaSuccess ||
      cudaMemcpyAsync(ptrs, hptr.data(), 8ull * 4 * E, cudaMemcpyHostToDevice, st) != cudaSuccess)
    return done(fail(FLOE_ERR_CUDA, "collect_stats: upload failed"));
  C::up_gate_seq<<<dim3((di + 127) / 128, P), 128, 0, st>>>(
      ptrs, ptrs + E, u, dh, di, pairs, reinterpret_cast<float *const *>(sc + o_ptr + 8ull * 3 * E),
      acoef);
  if (h_next) {
    C::down_seq<<<dim3((dh + 127) / 128, P), 128, 0, st>>>(ptrs + 2 * E, pairs, acoef, dh, di, outp);
    C::combine_seq<<<dim3((dh + 127) / 128, T), 128, 0, st>>>(u, outp, wt, pair_of, T, K, dh,
                                                              drift_scale, h_next);
  }
  if (cudaGetLastError() != cudaSuccess) return done(fail(FLOE_ERR_CUDA, "collect_stats: launch failed"));
  // reservoir adds, expert by expert (each reservoir sees its values in token order)
  for (uint32_t e = 0; e < E; ++e) {
    if (!n_e[e]) continue;
    const uint64_t n = (uint64_t)n_e[e] * di;
    C::ResState *rs = c->st + (size_t)layer * E + e;
    float *smp = c->samples + ((size_t)layer * E + e) * c->cap;
    if (cudaMemsetAsync(c->owner, 0, 4ull * c->cap, st) != cudaSuccess)
      return done(fail(FLOE_ERR_CUDA, "collect_stats: memset failed"));
    C::reservoir_claim<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(rs, c->cap, n, c->owner);
    C::reservoir_apply<<<(unsigned)((c->cap + 255) / 256), 256, 0, st>>>(c->cap, vals + (size_t)off[e] * di,
                                                                      c->owner, smp);
    C::reservoir_advance<<<1, 1, 0, st>>>(rs, n);
  }
  if (cudaGetLastError() != cudaSuccess) return done(fail(FLOE_ERR_CUDA, "collect_stats: launch failed"));
  return done(rc);
}

int floe_gpu_calib_thresholds(floe_gpu_calib *c, double k, float *thresholds_host) {
  if (!c || !thresholds_host) return fail(FLOE_ERR_INVALID, "calibrate: null argument");
  if (k < 0.0 || k > 1.0) return fail(FLOE_ERR_INVALID, "calibrate_threshold: k must be in [0,1]");
  const uint32_t R = c->L * c->E;
  std::vector<floe_cal::ResState> hs(R);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(hs.data(), c->st, sizeof(floe_cal::ResState) * R, cudaMemcpyDeviceToHost));
  for (uint32_t i = 0; i < R; ++i)
    if (hs[i].seen == 0 && k != 0.0)
      return fail(FLOE_ERR_INVALID, "calibrate: no samples for layer %u expert %u", i / c->E,
                  i % c->E);
  // sort every reservoir's samples (segments [i cap, i cap + min(seen, cap)))
  std::vector<int> begin(R), end(R);
  for (uint32_t i = 0; i < R; ++i) {
    begin[i] = (int)((uint64_t)i * c->cap);
    end[i] = (int)((uint64_t)i * c->cap + std::min<uint64_t>(hs[i].seen, c->cap));
  }
  if ((uint64_t)R * c->cap > 0x7fffffffull)
    return fail(FLOE_ERR_UNSUPPORTED, "calibrate: more than 2^31 samples");
  float *sorted = nullptr, *out = nullptr;
  int *d_off = nullptr;
  void *tmp = nullptr;
  size_t tmp_bytes = 0;
  const int nitems = (int)((uint64_t)R * c->cap);
  CK(cudaMalloc(&sorted, 4ull * nitems));
  CK(cudaMalloc(&d_off, 8ull * R));
  CK(cudaMalloc(&out, 4ull * R));
  CK(cudaMemcpy(d_off, begin.data(), 4ull * R, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(d_off + R, end.data(), 4ull * R, cudaMemcpyHostToDevice));
  cub::DeviceSegmentedRadixSort::SortKeys(nullptr, tmp_bytes, c->samples, sorted, nitems, (int)R,
                                          d_off, d_off + R);
  CK(cudaMalloc(&tmp, tmp_bytes));
  cub::DeviceSegmentedRadixSort::SortKeys(tmp, tmp_bytes, c->samples, sorted, nitems, (int)R,
                                          d_off, d_off + R);
  floe_cal::reservoir_pick<<<(R + 127) / 128, 128>>>(c->st, sorted, c->cap, R, k, out);
  const cudaError_t ce = cudaGetLastError();
  if (ce == cudaSuccess) CK(cudaMemcpy(thresholds_host, out, 4ull * R, cudaMemcpyDeviceToHost));
  cudaFree(tmp);
  cudaFree(sorted);
  cudaFree(d_off);
  cudaFree(out);
  if (ce != cudaSuccess) return fail(FLOE_ERR_CUDA, "calibrate: %s", cudaGetErrorString(ce));
  return FLOE_OK;
}

}  // extern "C"

// ------------------------------------------------------- synthetic model ---
int floe_gpu_gen_normals(uint64_t seed, uint64_t stream_id, uint64_t n, float sigma,
                         int sharded, float *out, floe_stream_t stream) {
  if (!out) return fail(FLOE_ERR_INVALID, "gen_normals: null output");
  if (int rc = require_device("gen_normals")) return rc;
  if (n == 0) return FLOE_OK;
  floe_gen::gen_normals<<<8 * device_info().sm, 256, 0, S(stream)>>>(seed, stream_id, n, sigma,
                                                                     sharded, out);
  CK_LAUNCH();
  return FLOE_OK;
}

int floe_gpu_quantize(const float *x, uint64_t n, uint32_t bits, uint32_t g, uint8_t *codes,
                      uint16_t *scales, uint16_t *zeros, floe_stream_t stream) {
  if (!x || !codes || !scales || !zeros) return fail(FLOE_ERR_INVALID, "quantize: null argument");
  if (int rc = require_device("quantize")) return rc;
  if (!bits_ok(bits)) return fail(FLOE_ERR_INVALID, "quantize: bits must be one of {1,2,3,4,8}");
  if (g == 0 || n % g != 0)
    return fail(FLOE_ERR_INVALID, "quantize: group_size must divide element count");
  cudaStream_t st = S(stream);
  const uint64_t groups = n / g;
  const uint64_t nb = packed_code_bytes(n, bits);
  const bool aligned = (32 % bits == 0) && ((uint64_t)g * bits) % 32 == 0 &&
                       (reinterpret_cast<uintptr_t>(codes) & 3) == 0;
  const int blocks = 8 * device_info().sm;
  if (aligned) {
    floe_gen::quantize_groups<<<blocks, 256, 0, st>>>(x, groups, g, bits, codes, scales, zeros, 1);
    CK_LAUNCH();
    return FLOE_OK;
  }
  // put_code ORs into shared bytes: build in a zeroed, word-padded buffer.
  uint8_t *tmp = nullptr;
  const uint64_t tb = ((nb + 3) & ~uint64_t(3)) + 8;
  CK(cudaMallocAsync(reinterpret_cast<void **>(&tmp), tb, st));
  CK(cudaMemsetAsync(tmp, 0, tb, st));
  floe_gen::quantize_groups<<<blocks, 256, 0, st>>>(x, groups, g, bits, tmp, scales, zeros, 0);
  CK_LAUNCH();
  CK(cudaMemcpyAsync(codes, tmp, nb, cudaMemcpyDeviceToDevice, st));
  CK(cudaFreeAsync(tmp, st));
  return FLOE_OK;
}

// -------------------------------------------------------------- predictor --
int floe_gpu_predictor_create(uint32_t layers, uint32_t experts, uint32_t dh,
                              const float *w, const float *b, floe_gpu_predictor **out) {
  if (!out || !w || !b) return fail(FLOE_ERR_INVALID, "predictor_create: null argument");
  *out = nullptr;
  if (int rc = require_device("predictor_create")) return rc;
  if (layers < 2) return fail(FLOE_ERR_INVALID, "predictor file: needs at least two layers");
  if (experts == 0 || experts > 32 || dh == 0)
    return fail(FLOE_ERR_INVALID, "predictor_create: need 1 <= experts <= 32, d_hidden >= 1");
  auto *p = new (std::nothrow) floe_gpu_predictor();
  if (!p) return fail(FLOE_ERR_OOM, "predictor_create: host allocation failed");
  p->layers = layers;
  p->experts = experts;
  p->dh = dh;
  const uint64_t nw = (uint64_t)(layers - 1) * experts * dh, nb = (uint64_t)(layers - 1) * experts;
  cudaError_t ce = cudaMalloc(&p->w, 4 * nw);
  if (ce == cudaSuccess) ce = cudaMalloc(&p->b, 4 * nb);
  if (ce == cudaSuccess) ce = cudaMemcpy(p->w, w, 4 * nw, cudaMemcpyDefault);
  if (ce == cudaSuccess) ce = cudaMemcpy(p->b, b, 4 * nb, cudaMemcpyDefault);
  if (ce != cudaSuccess) {
    floe_gpu_predictor_destroy(p);
    return fail(FLOE_ERR_OOM, "predictor_create: %s", cudaGetErrorString(ce));
  }
  *out = p;
  return FLOE_OK;
}

int floe_gpu_predictor_destroy(floe_gpu_predictor *p) {
  if (!p) return FLOE_OK;
  if (p->w) cudaFree(p->w);
  if (p->b) cudaFree(p->b);
  delete p;
  return FLOE_OK;
}

int floe_gpu_predict_experts(const floe_gpu_predictor *p, const float *x, uint32_t layer,
                             uint32_t count, uint32_t *out, floe_stream_t stream) {
  if (!p || !x || !out) return fail(FLOE_ERR_INVALID, "predict_experts: null argument");
  if (layer == 0)
    return fail(FLOE_ERR_INVALID, "predict_experts: layer 0 has no lookahead predictor");
  if (layer >= p->layers) return fail(FLOE_ERR_INVALID, "predict_experts: bad layer");
  if (count == 0 || count > p->experts) return fail(FLOE_ERR_INVALID, "top_k: k out of range");
  const uint64_t off = (uint64_t)(layer - 1) * p->experts;
  floe_k::route_topk<<<1, 256, 0, S(stream)>>>(p->w + off * p->dh, p->b + off, x, p->experts,
                                               p->dh, count, 0, out, nullptr, nullptr, nullptr);
  CK_LAUNCH();
  return FLOE_OK;
}

}  // extern "C"

// --------------------------------------------------------- record cache ---
// "FLOR" files (include/floe_gpu.h): the device image of a compressed model,
// f16 records instead of FLOQ's f32 gate/down.
namespace {
constexpr uint32_t kFlorVersion = 1;
constexpr uint64_t kFlorAlign = 64;
uint64_t flor_pad(uint64_t n) { return (n + kFlorAlign - 1) & ~(kFlorAlign - 1); }

struct FlorHeader {
  char magic[4];
  uint32_t version, layers, experts, top_k, dh, di, bits, g, mix_f16, reserved[6];
};
static_assert(sizeof(FlorHeader) == 64, "FLOR header is 64 bytes");

struct File {
  FILE *f = nullptr;
  ~File() {
    if (f) std::fclose(f);
  }
};

uint64_t flor_expert_bytes(uint32_t dh, uint32_t di, uint32_t bits, uint32_t g) {
  const uint64_t n = (uint64_t)dh * di;
  return 64 + flor_pad((n * bits + 7) / 8) + 2 * flor_pad(2 * (n / g)) + flor_pad(4ull * dh * di);
}
uint64_t flor_layer_bytes(const FlorHeader &h) {
  return flor_pad(4ull * h.experts * h.dh) + flor_pad((uint64_t)h.dh * h.dh * (h.mix_f16 ? 2 : 4)) +
         h.experts * flor_expert_bytes(h.dh, h.di, h.bits, h.g);
}

int flor_read_header(const char *path, File &file, FlorHeader &h, uint64_t &size) {
  if (!path) return fail(FLOE_ERR_INVALID, "record_cache: null path");
  file.f = std::fopen(path, "rb");
  if (!file.f) return fail(FLOE_ERR_INVALID, "record_cache: cannot open %s", path);
  std::fseek(file.f, 0, SEEK_END);
  size = (uint64_t)std::ftell(file.f);
  std::fseek(file.f, 0, SEEK_SET);
  if (std::fread(&h, sizeof h, 1, file.f) != 1) return fail(FLOE_ERR_INVALID, "record_cache: truncated file");
  if (std::memcmp(h.magic, "FLOR", 4) != 0) return fail(FLOE_ERR_INVALID, "record_cache: bad magic");
  if (h.version != kFlorVersion) return fail(FLOE_ERR_INVALID, "record_cache: unsupported version");
  if (!h.layers || !h.experts || !h.top_k || h.top_k > h.experts || !h.dh || !h.di || !h.g ||
      ((uint64_t)h.dh * h.di) % h.g)
    return fail(FLOE_ERR_INVALID, "record_cache: bad shape");
  if (size != 64 + (uint64_t)h.layers * flor_layer_bytes(h))
    return fail(FLOE_ERR_INVALID, "record_cache: truncated file");
  return FLOE_OK;
}
}  // namespace

extern "C" {

int floe_gpu_record_cache_save(floe_gpu_layer *const *layers, uint32_t n_layers, const char *path) {
  if (!layers || !n_layers || !path) return fail(FLOE_ERR_INVALID, "record_cache_save: bad arguments");
  if (int rc = require_device("record_cache_save")) return rc;
  const floe_gpu_layer *l0 = layers[0];
  FlorHeader h{};
  std::memcpy(h.magic, "FLOR", 4);
  h.version = kFlorVersion;
  h.layers = n_layers;
  h.experts = l0->E;
  h.top_k = l0->top_k;
  h.dh = l0->dh;
  h.di = l0->di;
  const floe_gpu_expert *e0 = l0->experts[0];
  h.bits = e0->bits;
  h.g = e0->g;
  h.mix_f16 = l0->mix_f16 ? 1 : 0;
  for (uint32_t l = 0; l < n_layers; ++l) {
    const floe_gpu_layer *ly = layers[l];
    if (!ly || ly->E != h.experts || ly->top_k != h.top_k || ly->dh != h.dh || ly->di != h.di ||
        (ly->mix_f16 ? 1u : 0u) != h.mix_f16)
      return fail(FLOE_ERR_INVALID, "record_cache_save: layer %u shape differs", l);
    for (const floe_gpu_expert *e : ly->experts)
      if (e->bits != h.bits || e->g != h.g || e->up_only)
        return fail(FLOE_ERR_INVALID, "record_cache_save: layer %u expert without records or "
                                      "with another quantisation", l);
  }
  File file;
  file.f = std::fopen(path, "wb");
  if (!file.f) return fail(FLOE_ERR_INVALID, "record_cache_save: cannot open %s", path);
  std::vector<uint8_t> buf;
  auto put = [&](const void *p, uint64_t n) {  // one 64-B aligned section
    static const uint8_t zero[kFlorAlign] = {};
    if (n && std::fwrite(p, 1, n, file.f) != n) return false;
    const uint64_t pad = flor_pad(n) - n;
    return pad == 0 || std::fwrite(zero, 1, pad, file.f) == pad;
  };
  if (!put(&h, sizeof h)) return fail(FLOE_ERR_INVALID, "record_cache_save: write failed");
  const uint64_t n = (uint64_t)h.dh * h.di, ng = n / h.g, code_bytes = (n * h.bits + 7) / 8;
  for (uint32_t l = 0; l < n_layers; ++l) {
    const floe_gpu_layer *ly = layers[l];
    const uint64_t rb = 4ull * h.experts * h.dh, mb = (uint64_t)h.dh * h.dh * (h.mix_f16 ? 2 : 4);
    buf.resize(std::max(rb, mb));
    CK(cudaMemcpy(buf.data(), ly->router, rb, cudaMemcpyDeviceToHost));
    if (!put(buf.data(), rb)) return fail(FLOE_ERR_INVALID, "record_cache_save: write failed");
    CK(cudaMemcpy(buf.data(), ly->mixing, mb, cudaMemcpyDeviceToHost));
    if (!put(buf.data(), mb)) return fail(FLOE_ERR_INVALID, "record_cache_save: write failed");
    for (const floe_gpu_expert *e : ly->experts) {
      uint32_t eh[16] = {};
      float thr = 0.0f;
      buf.resize(std::max<uint64_t>(code_bytes + 4 * ng, 4ull * n));
      uint16_t *sc = reinterpret_cast<uint16_t *>(buf.data() + code_bytes);
      if (int rc = floe_gpu_expert_download(e, buf.data(), sc, sc + ng, &thr)) return rc;
      std::memcpy(&eh[0], &thr, 4);
      if (!put(eh, sizeof eh) || !put(buf.data(), code_bytes) || !put(sc, 2 * ng) ||
          !put(sc + ng, 2 * ng))
        return fail(FLOE_ERR_INVALID, "record_cache_save: write failed");
      CK(cudaMemcpy(buf.data(), e->resident ? (const void *)e->rec_dev : (const void *)e->rec_host,
                    4ull * n, cudaMemcpyDefault));
      if (!put(buf.data(), 4ull * n)) return fail(FLOE_ERR_INVALID, "record_cache_save: write failed");
    }
  }
  return FLOE_OK;
}

int floe_gpu_record_cache_info(const char *path, floe_record_cache_info *info) {
  if (!info) return fail(FLOE_ERR_INVALID, "record_cache_info: null argument");
  File file;
  FlorHeader h;
  uint64_t size = 0;
  if (int rc = flor_read_header(path, file, h, size)) return rc;
  *info = floe_record_cache_info{h.layers, h.experts, h.top_k, h.dh, h.di, h.bits, h.g, h.mix_f16, size};
  return FLOE_OK;
}

int floe_gpu_record_cache_load(const char *path, uint32_t flags, floe_gpu_layer **layers_out,
                               floe_gpu_expert **experts_out) {
  if (!layers_out || !experts_out) return fail(FLOE_ERR_INVALID, "record_cache_load: null argument");
  File file;
  FlorHeader h;
  uint64_t size = 0;
  if (int rc = flor_read_header(path, file, h, size)) return rc;
  const uint64_t n = (uint64_t)h.dh * h.di, ng = n / h.g, code_bytes = (n * h.bits + 7) / 8;
  std::vector<floe_gpu_layer *> made_l;
  std::vector<floe_gpu_expert *> made_e;
  auto undo = [&](int rc) {
    for (floe_gpu_layer *l : made_l) floe_gpu_layer_destroy(l);
    for (floe_gpu_expert *e : made_e) floe_gpu_expert_destroy(e);
    return rc;
  };
  auto get = [&](void *p, uint64_t bytes) {  // one 64-B aligned section
    if (bytes && std::fread(p, 1, bytes, file.f) != bytes) return false;
    return std::fseek(file.f, (long)(flor_pad(bytes) - bytes), SEEK_CUR) == 0;
  };
  std::vector<float> router((size_t)h.experts * h.dh), mixing((size_t)h.dh * h.dh);
  std::vector<uint16_t> mix16(h.mix_f16 ? (size_t)h.dh * h.dh : 0);
  std::vector<uint8_t> up(code_bytes + 4 * ng);
  std::vector<uint16_t> rec(2 * n);
  for (uint32_t l = 0; l < h.layers; ++l) {
    if (!get(router.data(), 4ull * router.size())) return undo(fail(FLOE_ERR_INVALID, "record_cache: truncated file"));
    if (h.mix_f16) {
      if (!get(mix16.data(), 2ull * mix16.size())) return undo(fail(FLOE_ERR_INVALID, "record_cache: truncated file"));
      for (size_t i = 0; i < mix16.size(); ++i) {  // exact: f16 -> f32 (re-rounded identically on upload)
        __half_raw r;
        r.x = mix16[i];
        mixing[i] = __half2float(__half(r));
      }
    } else if (!get(mixing.data(), 4ull * mixing.size())) {
      return undo(fail(FLOE_ERR_INVALID, "record_cache: truncated file"));
    }
    std::vector<floe_gpu_expert *> ex(h.experts);
    for (uint32_t e = 0; e < h.experts; ++e) {
      uint32_t eh[16];
      uint16_t *sc = reinterpret_cast<uint16_t *>(up.data() + code_bytes);
      if (!get(eh, sizeof eh) || !get(up.data(), code_bytes) || !get(sc, 2 * ng) || !get(sc + ng, 2 * ng) ||
          !get(rec.data(), 2ull * rec.size()))
        return undo(fail(FLOE_ERR_INVALID, "record_cache: truncated file"));
      floe_expert_host_view v{};
      v.d_hidden = h.dh;
      v.d_intermediate = h.di;
      v.bits = h.bits;
      v.group_size = h.g;
      v.codes = up.data();
      v.scales = sc;
      v.zeros = sc + ng;
      v.records_f16 = rec.data();
      std::memcpy(&v.threshold, &eh[0], 4);
      v.flags = flags & FLOE_VIEW_HOST_RECORDS;
      if (int rc = floe_gpu_expert_create(&v, &ex[e])) return undo(rc);
      made_e.push_back(ex[e]);
    }
    floe_layer_host_view lv{h.dh, h.experts, h.top_k, router.data(), mixing.data(), (int)h.mix_f16,
                            ex.data()};
    floe_gpu_layer *ly = nullptr;
    if (int rc = floe_gpu_layer_create(&lv, &ly)) return undo(rc);
    made_l.push_back(ly);
  }
  for (size_t i = 0; i < made_l.size(); ++i) layers_out[i] = made_l[i];
  for (size_t i = 0; i < made_e.size(); ++i) experts_out[i] = made_e[i];
  return FLOE_OK;
}

}  // extern "C"
