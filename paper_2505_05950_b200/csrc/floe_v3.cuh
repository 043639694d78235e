// floe_v3.cuh -- persistent multi-layer decode: ONE launch runs a token through
// every layer of a model (the reference's `h = layer_forward(m, l, h)` loop,
// tools/cli.cpp:86-107, each layer model.cpp:145-208), with a grid barrier
// between layers instead of a kernel boundary.
//
// Per layer the work is that of floe_v2::fused in layer mode (phase A mixing
// GEMV + router partials, exact routing, phase B K1 on the tensor cores,
// phase C gate/SwiGLU/down over the kept records); the K1 tile math, the K1
// operand setup, the phase-C record math and the CTA-pair balance are the same
// code.  What changes is the layer boundary:
//
//   * The mixing matrix of layer l+1 is cut into row chunks (kChunkRows rows,
//     16 KB items of two f16 rows).  Chunk c of layer l+1 is owned by the CTA
//     that finished phase C of layer l in position c (a ticket from the
//     end-of-layer counter), and that CTA streams the chunk into its record
//     ring right after its last record of layer l -- while slower CTAs are
//     still streaming their records.  The last G - NCH finishers own no chunk.
//     Once every CTA has finished layer l (the end-of-layer counter reaches G),
//     a chunk owner loads h (16 KB) and computes u = h + M h for its rows from
//     shared memory.
//   * Per-chunk partial router logits and predicted logits are indexed by
//     chunk, not by CTA, and summed in chunk order: routing does not depend on
//     which CTA owned which chunk (run-to-run deterministic).
//   * The record ring carries, in order: mixing items of layer 0, records of
//     layer 0, mixing items of layer 1, records of layer 1, ...; the K1 ring
//     (20 KB stages over the same bytes) is used between them.  Every ring and
//     barrier index runs on across layers.
//
// f16 mixing, d_hidden 4096 or 2048, at most 8 experts per layer.
#pragma once

#include "floe_v2.cuh"

namespace floe_v3 {

using floe_k::ExpertDesc;
using namespace floe_v2;

constexpr int kChunkRows = 32;                 // mixing rows per chunk
constexpr int kChunkItems = kChunkRows / 2;    // 16 KB items (2 f16 rows at d_hidden 4096)
constexpr int kMaxE = 8;

struct LayerDesc {
  const __half *mixing;      // [DH][DH] f16
  const float *router;       // [E][DH]
  const float *router_pred;  // [E][DH] router + router * mixing
  const ExpertDesc *table;   // [E]
};

struct DecodeArgs {
  const LayerDesc *layers;  // [n_layers] device
  uint32_t n_layers, n_experts, top_k, di;
  // block inputs/outputs: replay -> layer l reads h + l*DH, writes y + l*DH;
  // chained -> layer 0 reads h, layer l writes buf[l & 1] (y for the last),
  // layer l + 1 reads what layer l wrote
  const float *h;
  float *y;
  float *buf;  // [2][DH] (chained)
  int replay;
  float *u;             // [DH] block input u of the current layer (exchange)
  float *partial;       // [32][kMaxGrid] per-chunk partial router logits
  float *pred_partial;  // [32][kMaxGrid] per-chunk predicted partials
  unsigned long long *pcnt;  // monotonic: G arrivals per layer (predicted partials published)
  unsigned long long *bar;   // monotonic: G arrivals per layer (u and partials complete)
  unsigned long long *lbar;  // monotonic: G arrivals per layer (layer output complete) -> tickets
  unsigned long long *stats;
  unsigned long long *place_acc;  // nullable [2]: kept records read from HBM / over PCIe
  unsigned long long *phase_ns;   // nullable [G][kTraceSlots]: marks of layer trace_layer
  uint32_t trace_layer;
  int paired;
  uint32_t ns, max_tiles;
  uint32_t debug;  // bit 3: invert the predicted logits (misprediction path)
};

// Poll a monotonic counter until it reaches target, with a back-off: many SMs
// spinning on one L2 line slow every other access through that slice.
__device__ __forceinline__ void poll_until(const unsigned long long *p, unsigned long long target,
                                           const char *what, uint32_t tag) {
  const unsigned long long t0 = gtime();
  for (uint32_t it = 1;; ++it) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    if (v >= target) break;
    __nanosleep(200);
    if ((it & 255u) == 0 && gtime() - t0 > floe_ptx::kWatchdogNs)
      floe_ptx::watchdog_fire(what, (uint32_t)target, tag);
  }
}

// Arrive with release semantics (the CTA's writes before the preceding
// bar.sync are ordered before the arrival: release is cumulative) and return
// the previous count.
__device__ __forceinline__ unsigned long long atom_add_release(unsigned long long *p) {
  unsigned long long old;
  asm volatile("atom.release.gpu.global.add.u64 %0, [%1], 1;" : "=l"(old) : "l"(p) : "memory");
  return old;
}

__device__ __forceinline__ void grid_barrier(unsigned long long *bar, uint32_t G) {
  const unsigned long long old = atom_add_release(bar);
  poll_until(bar, (old / G + 1) * G, "grid barrier", (uint32_t)(old % G));  // acquire loads
}

// Item j of chunk c holds rows 2 p, 2 p + 1 of the chunk, p = (j + 5 c) mod
// kChunkItems: the chunks are 2^k bytes apart, so without the rotation every
// CTA would read the same offset of its chunk at the same time (the same DRAM
// channels).
__device__ __forceinline__ uint32_t chunk_item(uint32_t c, uint32_t j) {
  return (j + 5u * c) % (uint32_t)kChunkItems;
}

// Spin on an mbarrier phase without suspending (the producer's control
// waits: its wake-up latency is on the critical path of every layer).
__device__ __forceinline__ void mbar_spin(uint64_t *bar, uint32_t parity, uint32_t tag) {
  if (floe_ptx::mbar_test_wait(bar, parity)) return;
  const unsigned long long t0 = gtime();
  for (uint32_t it = 1;; ++it) {
    if (floe_ptx::mbar_test_wait(bar, parity)) return;
    if ((it & 1023u) == 0 && gtime() - t0 > floe_ptx::kWatchdogNs)
      floe_ptx::watchdog_fire("mbarrier", tag, parity);
  }
}

template <int DH>
__device__ __forceinline__ const float *layer_in(const DecodeArgs &a, uint32_t l) {
  if (a.replay) return a.h + (size_t)l * DH;
  return l == 0 ? a.h : a.buf + ((l - 1) & 1u) * DH;
}
template <int DH>
__device__ __forceinline__ float *layer_out(const DecodeArgs &a, uint32_t l) {
  if (a.replay) return a.y + (size_t)l * DH;
  return l + 1 == a.n_layers ? a.y : a.buf + (l & 1u) * DH;
}


template <int DH>
__global__ void __launch_bounds__(kThreads, 1) decode(const DecodeArgs a) {
  constexpr uint32_t TILE_B = tile_bytes(DH);
  constexpr uint32_t REC_B = 4 * DH;
  constexpr uint32_t ns = ring_stages(DH);
  constexpr uint32_t nsC = rec_stages(DH);
  static_assert(nsC <= (uint32_t)kMaxStages, "record ring");
  constexpr uint32_t SPANS = DH / 64;
  constexpr uint32_t NCH = DH / kChunkRows;  // chunks per mixing matrix
  static_assert(DH == 4096 || DH == 2048, "d_hidden 4096 or 2048");
  static_assert(REC_B == 2 * DH * 2, "a record stage holds two f16 mixing rows");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ uint64_t fullC[kMaxStages], emptyC[kMaxStages];
  __shared__ float stage_scale[kMaxStages];
  // single-use-per-layer barriers: waited with parity (layer & 1)
  __shared__ uint64_t hbar, rbar, predbar, bar1, routebar, ubar, listbar, totbar;
  __shared__ uint64_t peerbar, donebar, tickbar, lpass, parbar;
  __shared__ uint32_t n_pub, n_total, n_list, tau_s, ptaken_s, spec_ok;
  __shared__ __align__(16) LayerDesc ld_s[2];
  __shared__ __align__(16) ExpertDesc table_s[2][kMaxE];
  __shared__ __align__(16) float rsl[2][kMaxE][kChunkRows];  // router / router_pred rows of the chunk
  __shared__ float u_s[kChunkRows];
  __shared__ float pthr_s[floe_k::kMaxSlots], ethr_s[floe_k::kMaxSlots], w_s[floe_k::kMaxSlots];
  __shared__ const uint8_t *ptiles_s[floe_k::kMaxSlots];
  __shared__ const uint8_t *etiles_s[floe_k::kMaxSlots];
  __shared__ const __half *rec_s[floe_k::kMaxSlots];
  __shared__ uint32_t rhost_s[floe_k::kMaxSlots], slot_cnt[floe_k::kMaxSlots];
  __shared__ float redmax[kConsumerWarps];
  __shared__ float2 xch[kConsumerWarps / kQ][2][kQ - 1][8];
  __shared__ float red[2][2][8][4];  // [group][batch parity][warp][value]

  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const bool producer = warp == kConsumerWarps;
  const bool router_warp = warp == kConsumerWarps + 1;
  const SmemLayout L = smem_layout(DH, ns, a.max_tiles, G);
  uint8_t *ring = smem + L.ring;
  float *hs = reinterpret_cast<float *>(smem + L.ubuf);
  uint8_t *xtab = smem + L.uni;
  float *xs = reinterpret_cast<float *>(smem + L.xs);
  uint32_t *lf = reinterpret_cast<uint32_t *>(smem + L.lf);
  float *lv = reinterpret_cast<float *>(smem + L.lv);
  const uint32_t list_cap = kTileCh * a.max_tiles;
  const uint32_t E = a.n_experts;
  const uint64_t l2_stream = floe_ptx::policy_evict_first();

  auto stage = [&](uint32_t u) { return ring + (u % ns) * TILE_B; };
  auto wait_full = [&](uint32_t u) {
    floe_ptx::mbar_wait(&full[u % ns], (u / ns) & 1u, (1u << 28) | (u & 0xffffffu));
  };
  auto wait_empty = [&](uint32_t u) {
    if (u >= ns) floe_ptx::mbar_wait(&empty[u % ns], ((u / ns) + 1) & 1u, (2u << 28) | (u & 0xffffffu));
  };
  auto issue = [&](uint32_t u, const void *src, uint32_t bytes) {
    floe_ptx::mbar_arrive_expect_tx(&full[u % ns], bytes);
    floe_ptx::bulk_g2s_hint(stage(u), src, bytes, &full[u % ns], l2_stream);
  };
  auto stageC = [&](uint32_t k) { return ring + (k % nsC) * REC_B; };
  auto issueC = [&](uint32_t k, const void *src, float scale, uint64_t pol) {
    if (k >= nsC) floe_ptx::mbar_wait(&emptyC[k % nsC], ((k / nsC) + 1) & 1u, (5u << 28) | (k & 0xffffffu));
    stage_scale[k % nsC] = scale;
    floe_ptx::mbar_arrive_expect_tx(&fullC[k % nsC], REC_B);
    floe_ptx::bulk_g2s_hint(stageC(k), src, REC_B, &fullC[k % nsC], pol);
  };
  // phase marks of one layer (diagnostics)
  uint32_t l = 0;
  auto mark = [&](int k) {
    if (a.phase_ns && l == a.trace_layer && k < kTraceSlots) a.phase_ns[b * kTraceSlots + k] = gtime();
  };
  auto mark_prev = [&](int k) {  // end-of-layer events of the layer before the traced one
    if (a.phase_ns && l + 1 == a.trace_layer && k < kTraceSlots) a.phase_ns[b * kTraceSlots + k] = gtime();
  };

  if (t == 0) {
    for (uint32_t s = 0; s < ns; ++s) {
      floe_ptx::mbar_init(&full[s], 1);
      floe_ptx::mbar_init(&empty[s], kConsumerWarps);
    }
    for (uint32_t s = 0; s < nsC; ++s) {
      floe_ptx::mbar_init(&fullC[s], 1);
      floe_ptx::mbar_init(&emptyC[s], 8);  // the 8 warps of the item's group
    }
    floe_ptx::mbar_init(&hbar, 1);
    floe_ptx::mbar_init(&rbar, 1);
    floe_ptx::mbar_init(&predbar, 1);
    floe_ptx::mbar_init(&bar1, 1);
    floe_ptx::mbar_init(&routebar, 1);
    floe_ptx::mbar_init(&ubar, 1);
    floe_ptx::mbar_init(&listbar, 1);
    floe_ptx::mbar_init(&totbar, 1);
    floe_ptx::mbar_init(&peerbar, 1);
    floe_ptx::mbar_init(&donebar, 1);
    floe_ptx::mbar_init(&tickbar, 1);
    floe_ptx::mbar_init(&lpass, 1);
    floe_ptx::mbar_init(&parbar, 1);
    floe_ptx::fence_barrier_init();
    n_list = 0u;
    tau_s = b;  // layer 0: chunk b
    pdl_launch_dependents();
  }
  if (t < (uint32_t)floe_k::kMaxSlots) slot_cnt[t] = 0u;
  if (t == 0) ld_s[0] = a.layers[0];
  if (t < E) table_s[0][t] = a.layers[0].table[t];
  for (uint32_t i = t; i < list_cap; i += kThreads) lf[i] = 0u;
  __syncthreads();
  if (a.paired) floe_ptx::cluster_sync_all();
  else __syncthreads();

  const uint32_t tps = tiles_per_expert(a.di);
  const uint32_t NT = a.top_k * tps;
  const uint32_t tile_lo = (uint32_t)(((uint64_t)NT * b) / G);
  const uint32_t nB = (uint32_t)(((uint64_t)NT * (b + 1)) / G) - tile_lo;

  if (producer) {
    // =================== producer warp (lane 0 issues every copy) ===================
    if (lane != 0) return;
    uint32_t U = 0, K = 0;  // K1-ring uses / record-ring items issued so far
    // hbar / rbar complete once per chunk-owning layer (not every layer)
    // chunk prefetch of layer ln: router slices, then the first nsC items
    // (the rest follow once h is in and consumption frees stages)
    auto chunk_begin = [&](uint32_t ln, uint32_t c) {
      const LayerDesc &D = ld_s[ln & 1u];
      const uint32_t r0 = c * kChunkRows;
      floe_ptx::mbar_arrive_expect_tx(&rbar, 2u * E * kChunkRows * 4u);
      for (uint32_t e = 0; e < E; ++e) {
        floe_ptx::bulk_g2s(&rsl[0][e][0], D.router + (size_t)e * DH + r0, kChunkRows * 4u, &rbar);
        floe_ptx::bulk_g2s(&rsl[1][e][0], D.router_pred + (size_t)e * DH + r0, kChunkRows * 4u, &rbar);
      }
      const uint8_t *m = reinterpret_cast<const uint8_t *>(D.mixing) + (size_t)r0 * DH * 2u;
      const uint32_t pre = min((uint32_t)kChunkItems, nsC);
      for (uint32_t j = 0; j < pre; ++j)
        issueC(K + j, m + (size_t)chunk_item(c, j) * REC_B, 0.0f, l2_stream);
    };
    auto chunk_rest = [&](uint32_t ln, uint32_t c) {
      const LayerDesc &D = ld_s[ln & 1u];
      const uint8_t *m = reinterpret_cast<const uint8_t *>(D.mixing) + (size_t)c * kChunkRows * DH * 2u;
      for (uint32_t j = min((uint32_t)kChunkItems, nsC); j < (uint32_t)kChunkItems; ++j)
        issueC(K + j, m + (size_t)chunk_item(c, j) * REC_B, 0.0f, l2_stream);
      K += kChunkItems;
    };
    uint32_t chunk = b < NCH ? b : 0xffffffffu;
    if (chunk != 0xffffffffu) chunk_begin(0, chunk);
    pdl_wait();
    if (chunk != 0xffffffffu) {
      floe_ptx::mbar_arrive_expect_tx(&hbar, 4u * DH);
      floe_ptx::bulk_g2s(hs, layer_in<DH>(a, 0), 4u * DH, &hbar);
    }
    for (l = 0; l < a.n_layers; ++l) {
      const uint32_t P = l & 1u;
      mark(31);
      if (chunk != 0xffffffffu && a.phase_ns && l == a.trace_layer) {  // diagnostics: prefetch landed
        const uint32_t pre = min((uint32_t)kChunkItems, nsC);
        floe_ptx::mbar_wait(&fullC[K % nsC], (K / nsC) & 1u, 22u << 28);
        mark(11);
        floe_ptx::mbar_wait(&fullC[(K + pre - 1) % nsC], ((K + pre - 1) / nsC) & 1u, 22u << 28);
        mark(15);
      }
      if (chunk != 0xffffffffu) chunk_rest(l, chunk);
      mark(23);
      if (chunk != 0xffffffffu && a.phase_ns && l == a.trace_layer) {  // diagnostics: tail landed
        const uint32_t kl = K - 1;
        floe_ptx::mbar_wait(&fullC[kl % nsC], (kl / nsC) & 1u, 22u << 28);
        mark(53);
      }
      mbar_spin(&predbar, P, 6u << 28);  // predicted routing
      mbar_spin(&bar1, P, 15u << 28);    // u complete
      mark(16);
      asm volatile("fence.proxy.async.global;" ::: "memory");  // u: generic-proxy writes
      mark(35);
      // The K1 ring covers the record ring's bytes.  Every record-ring item
      // issued so far has been released: the consumers released the last
      // ones (this layer's mixing items, or the previous layer's records)
      // before the bar.sync that precedes t0's arrival on bar1.
      mark(32);
      floe_ptx::mbar_arrive_expect_tx(&ubar, 4u * DH);
      floe_ptx::bulk_g2s(hs, a.u, 4u * DH, &ubar);
      mark(33);
      for (uint32_t j = 0; j < nB; ++j) {
        const TileRef tr = tile_ref2(tile_lo + j, a.top_k, a.di);
        wait_empty(U);
        issue(U++, ptiles_s[tr.slot] + (size_t)tr.t * TILE_B, TILE_B);
      }
      mark(17);
      mbar_spin(&routebar, P, 7u << 28);
      const bool ok = spec_ok != 0u;
      if (!ok)
        for (uint32_t j = 0; j < nB; ++j) {
          const TileRef tr = tile_ref2(tile_lo + j, a.top_k, a.di);
          wait_empty(U);
          issue(U++, etiles_s[tr.slot] + (size_t)tr.t * TILE_B, TILE_B);
        }
      // early records (floe_v2::fused): record item r goes to record stage
      // (K + r) % nsC once the K1-ring stages under it have seen their last
      // use released and the K1 epilogues have appended entry r; stages over
      // the x table wait for the end of K1
      uint32_t k_early = 0;
      if (ok) {
        const uint32_t uEnd = U;
        const uint32_t c_lim = ns * TILE_B / REC_B;  // record stages below the x table
        auto stages_free = [&](uint32_t cs) {
          const uint32_t lo = cs * REC_B, hi = lo + REC_B;
          for (uint32_t st = lo / TILE_B; st <= (hi - 1) / TILE_B; ++st)
            if (uEnd > st) {
              const uint32_t us = st + ((uEnd - 1 - st) / ns) * ns;
              if (!floe_ptx::mbar_test_wait(&empty[st], (us / ns) & 1u)) return false;
            }
          return true;
        };
        while (k_early < nsC && (K + k_early) % nsC < c_lim &&
               !floe_ptx::mbar_test_wait(&listbar, P)) {
          const uint32_t f = kEarlyRecords ? ld_acquire_s(&lf[k_early]) : 0u;
          if ((f & kValid) && stages_free((K + k_early) % nsC)) {
            const uint32_t r = k_early, s2 = (f >> kSlotShift) & 0x7fu, c = f & 0xffffffu;
            issueC(K + r, rec_s[s2] + (size_t)c * 2 * DH, lv[r] * w_s[s2], l2_stream);
            ++k_early;
          } else {
            __nanosleep(32);
          }
        }
      }
      // ---- phase C: own records, the CTA-pair plan
      mbar_spin(&listbar, P, 12u << 28);
      const uint32_t n_own = n_list;
      const uint32_t Pf = min(n_own, nsC);
      auto own_item = [&](uint32_t k) {
        const uint32_t f = lf[k], s2 = (f >> kSlotShift) & 0x7fu, c = f & 0xffffffu;
        issueC(K + k, rec_s[s2] + (size_t)c * 2 * DH, lv[k] * w_s[s2], l2_stream);
      };
      mark(18);
      if (a.paired) {
        n_pub = n_own;
        floe_ptx::mbar_arrive_remote(floe_ptx::mapa(&peerbar, (b ^ 1u) & 1u));
      }
      for (uint32_t k = k_early; k < Pf; ++k) own_item(k);
      uint32_t own = n_own, take = 0, pfirst = 0;
      if (a.paired) {
        const uint32_t peer = b ^ 1u;
        floe_ptx::mbar_wait_cluster(&peerbar, P, 17u << 28);
        const uint32_t n_p = floe_ptx::ld_cluster_u32(floe_ptx::mapa(&n_pub, peer & 1u));
        const uint32_t T = n_own + n_p;
        const uint32_t t_me = (b & 1u) ? T / 2 : (T + 1) / 2, t_p = T - t_me;
        own = max(Pf, min(n_own, t_me));
        const uint32_t own_p = max(min(n_p, nsC), min(n_p, t_p));
        take = t_me > own ? min(t_me - own, n_p - own_p) : 0u;
        pfirst = own_p;
      }
      n_total = own + take;
      floe_ptx::mbar_arrive(&totbar);
      for (uint32_t k = Pf; k < own; ++k) own_item(k);
      if (a.paired) {
        const uint32_t pr = (b ^ 1u) & 1u;
        for (uint32_t k = 0; k < take; ++k) {
          const uint32_t f = floe_ptx::ld_cluster_u32(floe_ptx::mapa(&lf[pfirst + k], pr));
          const float v = __uint_as_float(floe_ptx::ld_cluster_u32(floe_ptx::mapa(&lv[pfirst + k], pr)));
          const uint32_t s2 = (f >> kSlotShift) & 0x7fu, c = f & 0xffffffu;
          issueC(K + own + k, rec_s[s2] + (size_t)c * 2 * DH, v * w_s[s2], l2_stream);
        }
        floe_ptx::mbar_arrive_remote(floe_ptx::mapa(&donebar, pr));
      }
      K += own + take;
      mark(19);
      if (l + 1 == a.n_layers) break;
      // ---- the next layer's chunk: by this CTA's finishing position
      mbar_spin(&tickbar, P, 19u << 28);
      const uint32_t tau = tau_s;
      chunk = tau < NCH ? tau : 0xffffffffu;
      floe_ptx::mbar_wait(&parbar, P, 20u << 28);  // ld_s of layer l + 1
      mark_prev(20);
      if (chunk != 0xffffffffu) {
        chunk_begin(l + 1, chunk);
        mark_prev(21);
        mbar_spin(&lpass, P, 21u << 28);  // every CTA finished layer l
        mark_prev(22);
        asm volatile("fence.proxy.async.global;" ::: "memory");
        floe_ptx::mbar_arrive_expect_tx(&hbar, 4u * DH);
        floe_ptx::bulk_g2s(hs, layer_in<DH>(a, l + 1), 4u * DH, &hbar);
        mark_prev(27);
      } else {
        // no chunk: thread 0 arrived right after the ticket; every phase of
        // lpass is waited on (no arrival on an unobserved phase)
        mbar_spin(&lpass, P, 21u << 28);
      }
    }
    return;
  }

  if (router_warp) {
    // =================== router warp ===================
    pdl_wait();
    auto sum_partials = [&](const float *part, uint32_t n) {  // lane e returns logit e
      float lg = -__int_as_float(0x7f800000);
      for (uint32_t e0 = 0; e0 < E; e0 += 8) {
        float sv[8];
#pragma unroll
        for (int ee = 0; ee < 8; ++ee) {
          const uint32_t e = e0 + ee;
          float pv[kMaxGrid / 32];
#pragma unroll
          for (int j = 0; j < kMaxGrid / 32; ++j) {
            const uint32_t bb = lane + 32 * j;
            pv[j] = (e < E && bb < n) ? __ldcg(&part[e * kMaxGrid + bb]) : 0.0f;
          }
          float s = 0.0f;
#pragma unroll
          for (int j = 0; j < kMaxGrid / 32; ++j) s += pv[j];
          sv[ee] = s;
        }
#pragma unroll
        for (int ee = 0; ee < 8; ++ee) {
          float s = sv[ee];
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == e0 + ee) lg = s;
        }
      }
      return lg;
    };
    uint32_t owned = 0;  // chunk-owning layers so far (hbar / rbar parity)
    for (l = 0; l < a.n_layers; ++l) {
      const uint32_t P = l & 1u;
      const ExpertDesc *tab = table_s[P];
      // ---- this CTA's predicted partial (router_pred * h over its chunk's
      // rows), published with a count of G per layer; the router warp does it
      // so that no consumer warp waits on the fence and the atomic
      if (l > 0) floe_ptx::mbar_wait(&tickbar, (l - 1) & 1u, 23u << 28);
      const uint32_t tau = l == 0 ? b : tau_s;
      unsigned long long target = 0;
      if (tau < NCH) {
        floe_ptx::mbar_wait(&hbar, owned & 1u, 3u << 28);
        floe_ptx::mbar_wait(&rbar, owned & 1u, 9u << 28);
        ++owned;
        if (lane < E) {
          float s = 0.0f;
          for (uint32_t r = 0; r < (uint32_t)kChunkRows; ++r)
            s = fmaf(rsl[1][lane][r], hs[tau * kChunkRows + r], s);
          a.pred_partial[lane * kMaxGrid + tau] = s;
        }
        __syncwarp();
      }
      if (lane == 0) {
        const unsigned long long old = atom_add_release(a.pcnt);
        target = (old / G + 1) * G;
        poll_until(a.pcnt, target, "prediction", l);
      }
      __syncwarp();
      {
        float plg = sum_partials(a.pred_partial, NCH);
        if (a.debug & 8u) plg = -plg;
        const uint32_t ptaken = warp_topk(lane < E ? plg : -__int_as_float(0x7f800000), lane, E, a.top_k);
        if (lane == 0) {  // the thread that arrives writes them (producer reads after predbar)
          uint32_t i = 0;
          for (uint32_t m = ptaken; m; m &= m - 1, ++i) {
            const uint32_t e = __ffs(m) - 1;
            ptiles_s[i] = reinterpret_cast<const uint8_t *>(tab[e].tiles);
            pthr_s[i] = tab[e].threshold;
          }
          ptaken_s = ptaken;
          mark(26);
          floe_ptx::mbar_arrive(&predbar);
        }
      }
      floe_ptx::mbar_wait(&bar1, P, 10u << 28);
      if (lane == 0) mark(24);
      const float lg = sum_partials(a.partial, NCH);
      const uint32_t taken = warp_topk(lane < E ? lg : -__int_as_float(0x7f800000), lane, E, a.top_k);
      const bool mine = (taken >> lane) & 1u;
      float mx = mine ? lg : -__int_as_float(0x7f800000);
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      const float ex = mine ? expf(lg - mx) : 0.0f;
      float sum = 0.0f;
      for (uint32_t m = taken; m; m &= m - 1) sum += __shfl_sync(0xffffffffu, ex, __ffs(m) - 1);
      if (mine) {
        const uint32_t i = __popc(taken & ((1u << lane) - 1));
        w_s[i] = ex / sum;
        rec_s[i] = tab[lane].records;
        rhost_s[i] = tab[lane].host_records;
        etiles_s[i] = reinterpret_cast<const uint8_t *>(tab[lane].tiles);
        ethr_s[i] = tab[lane].threshold;
      }
      __syncwarp();
      if (lane == 0) {
        spec_ok = taken == ptaken_s ? 1u : 0u;
        mark(25);
        floe_ptx::mbar_arrive(&routebar);
      }
      // ---- the next layer's descriptors into the other buffer
      if (l + 1 < a.n_layers) {
        const uint32_t Q = (l + 1) & 1u;
        if (lane == 0) ld_s[Q] = a.layers[l + 1];
        if (lane < E) table_s[Q][lane] = a.layers[l + 1].table[lane];
        __syncwarp();
        if (lane == 0) floe_ptx::mbar_arrive(&parbar);
      }
    }
    return;
  }

  // =================== consumer warps (threads 0..511) ===================
  pdl_wait();
  const bool setup_warp = warp >= kConsumerWarps / 2;
  const uint32_t ts = t - kConsumers / 2;
  const bool act = setup_warp && ts < SPANS * 4;
  const uint32_t span = ts >> 2, tig = ts & 3;
  float xv[16];
  auto setup1 = [&]() {
    const float4 *x4 = reinterpret_cast<const float4 *>(hs + (act ? 64 * span + 16 * tig : 0));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 f = x4[i];
      xv[4 * i] = f.x;
      xv[4 * i + 1] = f.y;
      xv[4 * i + 2] = f.z;
      xv[4 * i + 3] = f.w;
    }
    float mx = 0.0f;
    bool fin = true;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      mx = fmaxf(mx, fabsf(xv[i]));
      fin = fin && isfinite(xv[i]);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const bool wfin = __all_sync(0xffffffffu, fin);
    if (lane == 0) redmax[warp] = wfin ? mx : -1.0f;
  };
  auto x_scale = [&](bool &fin_all, float &S, float &invS) {
    fin_all = true;
    float mx = 0.0f;
#pragma unroll
    for (int w = kConsumerWarps / 2; w < kConsumerWarps; ++w) {
      fin_all = fin_all && redmax[w] >= 0.0f;
      mx = fmaxf(mx, redmax[w]);
    }
    int ex = 0;
    frexpf(mx, &ex);
    const bool scaled = mx > 0.0f && fin_all;
    S = scaled ? __int_as_float((127 + 22 - ex) << 23) : 1.0f;
    invS = scaled ? __int_as_float((127 - 22 + ex) << 23) : 1.0f;
  };
  auto setup2 = [&]() {
    bool fin_all;
    float S, invS;
    x_scale(fin_all, S, invS);
    {  // x again from shared memory (not kept live across the barrier: registers)
      const float4 *x4 = reinterpret_cast<const float4 *>(hs + (act ? 64 * span + 16 * tig : 0));
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 f = x4[i];
        xv[4 * i] = f.x;
        xv[4 * i + 1] = f.y;
        xv[4 * i + 2] = f.z;
        xv[4 * i + 3] = f.w;
      }
    }
    if (act && fin_all) {
      int X[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) X[i] = __float2int_rn(xv[i] * S);
      const uint32_t p = span >> 1, sodd = span & 1;
      uint4 *xt = reinterpret_cast<uint4 *>(xtab) + (p * 2 + sodd) * 32;
      uint32_t lw[3][2][2];
#pragma unroll
      for (int q = 0; q < 3; ++q)
#pragma unroll
        for (int m = 0; m < 2; ++m)
#pragma unroll
          for (int j = 0; j < 2; ++j) lw[q][m][j] = 0;
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const int v = X[i];
        const int l0 = ((v + 128) & 255) - 128;
        const int r1 = (v - l0) >> 8;
        const int l1 = ((r1 + 128) & 255) - 128;
        const int l2 = (r1 - l1) >> 8;
        const int bb = i >> 2, m = (i >> 1) & 1, j = i & 1;
        lw[0][m][j] |= (uint32_t)(l0 & 255) << (8 * bb);
        lw[1][m][j] |= (uint32_t)(l1 & 255) << (8 * bb);
        lw[2][m][j] |= (uint32_t)(l2 & 255) << (8 * bb);
      }
#pragma unroll
      for (int n = 0; n < 8; ++n) {
        const int lim = n == 0 || n == 2 ? 0 : (n == 1 || n == 3 ? 1 : 2);
        const bool c1 = n == 0 || n == 1 || n == 4, c4 = n == 2 || n == 3 || n == 6;
        xt[4 * n + tig] = make_uint4(c1 ? lw[lim][0][0] : 0u, c4 ? lw[lim][0][1] : 0u,
                                     c1 ? lw[lim][1][0] : 0u, c4 ? lw[lim][1][1] : 0u);
      }
    }
    float s16 = 0.0f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s16 += xv[i];
    s16 += __shfl_xor_sync(0xffffffffu, s16, 1);
    s16 += __shfl_xor_sync(0xffffffffu, s16, 2);
    if (act && tig == 0) xs[span] = s16;
  };

  constexpr int EPT2 = DH / 256;
  using Vec = typename std::conditional<EPT2 == 16, uint4, uint2>::type;
  const uint32_t grp = warp / 8, gw = warp % 8, gt = t % 256;
  // transposed warp reduction of NV values: lanes (32/NV) r hold value r's warp sum
  auto warp_reduce_t = [&](float *v, auto nv_tag) {
    constexpr int NV = decltype(nv_tag)::value;
#pragma unroll
    for (int sft = 16, cnt = NV / 2; cnt >= 1; sft >>= 1, cnt >>= 1) {
      const bool upper = (lane & sft) != 0;
#pragma unroll
      for (int r = 0; r < cnt; ++r) {
        const float send = upper ? v[r] : v[r + cnt];
        const float keep = upper ? v[r + cnt] : v[r];
        v[r] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
      }
    }
#pragma unroll
    for (int sft = 32 / NV / 2; sft >= 1; sft >>= 1) v[0] += __shfl_xor_sync(0xffffffffu, v[0], sft);
  };
  uint32_t U = 0, K = 0, batch = 0;
  uint32_t chunk = b < NCH ? b : 0xffffffffu;
  uint32_t owned = 0;  // chunk-owning layers so far: hbar / rbar complete once per such layer

  for (l = 0; l < a.n_layers; ++l) {
    const uint32_t P = l & 1u;
    float *yl = layer_out<DH>(a, l);
    if (t == 0) mark(0);
    // ============================ phase A ============================
    if (chunk != 0xffffffffu) {
      const uint32_t r0 = chunk * kChunkRows;
      // warp 0 waits for h, the router slices and the prefetched items, one
      // lane per barrier (an mbarrier wait costs ~0.1 us of latency: in
      // parallel, not in sequence), then hands them to every consumer warp
      constexpr uint32_t PRE = (uint32_t)kChunkItems < nsC ? (uint32_t)kChunkItems : nsC;
      if (warp == 0 && lane < 2 + PRE) {
        uint64_t *bar;
        uint32_t par;
        if (lane < 2) {
          bar = lane == 0 ? &hbar : &rbar;
          par = owned & 1u;
        } else {
          const uint32_t k = K + lane - 2;
          bar = &fullC[k % nsC];
          par = (k / nsC) & 1u;
        }
        mbar_spin(bar, par, (3u << 28) | lane);  // all lanes at once
      }
      cbar();
      if (kRacecheck) {
        floe_ptx::mbar_wait(&hbar, owned & 1u, 3u << 28);
        floe_ptx::mbar_wait(&rbar, owned & 1u, 3u << 28);
        for (uint32_t j = 0; j < PRE; ++j)
          floe_ptx::mbar_wait(&fullC[(K + j) % nsC], ((K + j) / nsC) & 1u, 3u << 28);
      }
      ++owned;
      mark(7);
      // u rows: group g takes items g, g + 2, ...; thread gt owns elements
      // [EPT2 gt, EPT2 gt + EPT2) of both rows of an item
      float2 h2[EPT2 / 2];
      {
        const float4 *ha = reinterpret_cast<const float4 *>(hs + EPT2 * gt);
#pragma unroll
        for (int i = 0; i < EPT2 / 4; ++i) {
          const float4 q = ha[i];
          h2[2 * i] = make_float2(q.x, q.y);
          h2[2 * i + 1] = make_float2(q.z, q.w);
        }
      }
      uint32_t k = K + grp;
      uint32_t stg = k % nsC, ph = (k / nsC) & 1u;
      for (uint32_t i0 = 0; i0 < (uint32_t)kChunkItems / 2; i0 += 2, ++batch) {
        // one thread of the group waits for both items (the other warps do
        // no mbarrier operation: each costs ~0.1 us of latency), the group
        // barrier hands them over, and after the reduction barrier the same
        // thread releases both stages for the group
        float dv[4];
        const uint32_t stg0 = stg, ph0 = ph;
        const uint32_t stg1 = stg0 + 2 >= nsC ? stg0 + 2 - nsC : stg0 + 2;
        const uint32_t ph1 = stg0 + 2 >= nsC ? ph0 ^ 1u : ph0;
        if (grp + 2 * i0 + 2 >= PRE) {  // an item past the prefetched ones
          if (gw == 0 && lane < 2) mbar_spin(&fullC[lane ? stg1 : stg0], lane ? ph1 : ph0, (4u << 28) | lane);
          gbar(grp);
          if (kRacecheck) {
            floe_ptx::mbar_wait(&fullC[stg0], ph0, 4u << 28);
            floe_ptx::mbar_wait(&fullC[stg1], ph1, 4u << 28);
          }
        }
#pragma unroll
        for (int r = 0; r < 2; ++r) {
          const Vec *rec = reinterpret_cast<const Vec *>(ring + stg * REC_B);
          const Vec g0 = rec[2 * gt], g1 = rec[2 * gt + 1];
          const Vec d0 = rec[512 + 2 * gt], d1 = rec[512 + 2 * gt + 1];
          const __half2 *p0 = reinterpret_cast<const __half2 *>(&g0);
          const __half2 *p1 = reinterpret_cast<const __half2 *>(&g1);
          const __half2 *q0 = reinterpret_cast<const __half2 *>(&d0);
          const __half2 *q1 = reinterpret_cast<const __half2 *>(&d1);
          float2 sa = make_float2(0.0f, 0.0f), sb = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int jj = 0; jj < EPT2 / 4; ++jj) {
            sa = __ffma2_rn(__half22float2(p0[jj]), h2[jj], sa);
            sa = __ffma2_rn(__half22float2(p1[jj]), h2[EPT2 / 4 + jj], sa);
            sb = __ffma2_rn(__half22float2(q0[jj]), h2[jj], sb);
            sb = __ffma2_rn(__half22float2(q1[jj]), h2[EPT2 / 4 + jj], sb);
          }
          dv[2 * r] = sa.x + sa.y;
          dv[2 * r + 1] = sb.x + sb.y;
          stg += 2;
          if (stg >= nsC) {
            stg -= nsC;
            ph ^= 1u;
          }
        }
        warp_reduce_t(dv, std::integral_constant<int, 4>{});
        if ((lane & 7) == 0) red[grp][batch & 1][gw][lane >> 3] = dv[0];
        gbar(grp);
        if (gw == 0 && lane == 0) {  // every warp of the group has read both items
          floe_ptx::mbar_arrive_cnt(&emptyC[stg0], 8);
          floe_ptx::mbar_arrive_cnt(&emptyC[stg1], 8);
        }
        float s = red[grp][batch & 1][lane & 7][lane >> 3];
        s += __shfl_xor_sync(0xffffffffu, s, 4);
        s += __shfl_xor_sync(0xffffffffu, s, 2);
        s += __shfl_xor_sync(0xffffffffu, s, 1);
        if (gw == 0 && (lane & 7) == 0) {
          // value v = lane / 8: item grp + 2 (i0 + v / 2), row v % 2
          const uint32_t v = lane >> 3;
          const uint32_t row = 2u * chunk_item(chunk, grp + 2u * (i0 + (v >> 1))) + (v & 1u);
          u_s[row] = hs[r0 + row] + 1.0f * s;  // drift_scale 1 (model.cpp:151-152)
        }
      }
      K += kChunkItems;
      cbar();
      if (t == 0) {
        mark(14);
        if (a.phase_ns && l == a.trace_layer) {
          uint32_t smid;
          asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
          a.phase_ns[b * kTraceSlots + 52] = smid;
        }
      }
      if (warp == 0) {
        if (lane < E) {  // partial logits of the chunk, rows in order
          float s = 0.0f;
          for (uint32_t r = 0; r < (uint32_t)kChunkRows; ++r) s = fmaf(rsl[0][lane][r], u_s[r], s);
          a.partial[lane * kMaxGrid + chunk] = s;
        }
        a.u[r0 + lane] = u_s[lane];
        yl[r0 + lane] = u_s[lane];
      }
    }
    if (t == 0) mark(1);
    cbar();
    if (t == 0) {
      grid_barrier(a.bar, G);  // u, y = u and the partials of every chunk
      mark(2);
      floe_ptx::mbar_arrive(&bar1);
    }
    cbar();

    // ---- K1 setup
    floe_ptx::mbar_wait(&ubar, P, 16u << 28);
    if (t == 0) mark(34);
    if (setup_warp) setup1();
    cbar();
    if (setup_warp) setup2();
    cbar();
    if (t == 0) mark(3);
    float mult, zx;
    bool all_finite;
    {
      float S, invS;
      x_scale(all_finite, S, invS);
      const uint32_t mytig = lane & 3;
      mult = mytig == 0 ? invS : (mytig == 1 ? 0.25f * invS : (mytig == 2 ? 65536.0f * invS : 16384.0f * invS));
      zx = mytig == 0 ? 1.0f : 0.0f;
    }

    // ============================ phase B: K1 ============================
    auto k1_pass = [&](uint32_t u0, const float *thr_tab) {
      const uint32_t quad = warp / kQ, sub = warp % kQ;
      uint32_t n = 0;
      for (uint32_t j = 0; j < nB; ++j) {
        const uint32_t u = u0 + j;
        if ((u % 8) / 2 != quad) continue;
        const TileRef tr = tile_ref2(tile_lo + j, a.top_k, a.di);
        wait_full(u);
        float2 v2 = all_finite ? k1_tile<DH>(stage(u), xtab, xs, mult, zx, lane, sub)
                               : k1_tile_f32<DH>(stage(u), hs, lane, sub);
        __syncwarp();
        if (lane == 0) floe_ptx::mbar_arrive_cnt(&empty[u % ns], kConsumerWarps / kQ);
        if (sub != 0 && (lane & 3) == 0) xch[quad][n & 1][sub - 1][lane >> 2] = v2;
        qbar(quad);
        const uint32_t nb = n++;
        if (sub != 0) continue;
#pragma unroll
        for (int q = 0; q < kQ - 1; ++q) {
          const float2 o2 = xch[quad][nb & 1][q][lane >> 2];
          v2.x += o2.x;
          v2.y += o2.y;
        }
        const uint32_t g = lane >> 2;
        const bool q0 = (lane & 3) == 0;
        const float thr = thr_tab[tr.slot];
        const bool va = q0 && g < tr.nc, vb = q0 && g + 8 < tr.nc;
        const bool ka = va && !(fabsf(v2.x) < thr), kb = vb && !(fabsf(v2.y) < thr);
        const uint32_t ba = __ballot_sync(0xffffffffu, ka), bbal = __ballot_sync(0xffffffffu, kb);
        const uint32_t na = __popc(ba), cnt = na + __popc(bbal);
        if (cnt == 0) continue;
        uint32_t base = 0;
        if (lane == 0) {
          base = atomicAdd(&n_list, cnt);
          atomicAdd(&slot_cnt[tr.slot], cnt);
        }
        base = __shfl_sync(0xffffffffu, base, 0);
        const uint32_t lt = (1u << lane) - 1;
        if (ka) {
          const uint32_t pos = base + __popc(ba & lt);
          lv[pos] = v2.x;
          st_release_s(&lf[pos], kValid | (tr.slot << kSlotShift) | (tr.t * kTileCh + g));
        }
        if (kb) {
          const uint32_t pos = base + na + __popc(bbal & lt);
          lv[pos] = v2.y;
          st_release_s(&lf[pos], kValid | (tr.slot << kSlotShift) | (tr.t * kTileCh + g + 8));
        }
      }
    };
    k1_pass(U, pthr_s);
    U += nB;
    cbar();
    floe_ptx::mbar_wait(&routebar, P, 11u << 28);
    if (!spec_ok) {
      for (uint32_t i = t; i < list_cap; i += kConsumers) lf[i] = 0u;
      if (t < (uint32_t)floe_k::kMaxSlots) slot_cnt[t] = 0u;
      cbar();
      if (t == 0) n_list = 0u;
      cbar();
      k1_pass(U, ethr_s);
      U += nB;
      cbar();
    }
    const uint32_t n_items = n_list;
    if (t == 0) {
      mark(4);
      if (a.phase_ns && l == a.trace_layer) a.phase_ns[b * kTraceSlots + 9] = n_items;
      floe_ptx::mbar_arrive(&listbar);
      if (a.stats) {
        if (b == 0) atomicAdd(&a.stats[0], 1ull);
        atomicAdd(&a.stats[1], (unsigned long long)n_items);
      }
    }
    if (a.place_acc && t < a.top_k && slot_cnt[t])
      atomicAdd(&a.place_acc[rhost_s[t] ? 1 : 0], (unsigned long long)slot_cnt[t]);

    // ============================ phase C: K2 ============================
    float2 x2[EPT2 / 2], y2[EPT2 / 2];
    {
      const float4 *xa = reinterpret_cast<const float4 *>(hs + EPT2 * gt);
#pragma unroll
      for (int i = 0; i < EPT2 / 4; ++i) {
        const float4 q = xa[i];
        x2[2 * i] = make_float2(q.x, q.y);
        x2[2 * i + 1] = make_float2(q.z, q.w);
      }
#pragma unroll
      for (int i = 0; i < EPT2 / 2; ++i) y2[i] = make_float2(0.0f, 0.0f);
    }
    uint32_t stg = (K + grp) % nsC, ph = ((K + grp) / nsC) & 1u;
    uint32_t processed = 0;
    const uint32_t P0 = min(n_items, nsC);
    uint32_t total = a.paired ? 0xffffffffu : n_items;
    for (uint32_t i0 = 0;; i0 += kR, ++batch) {
      if (grp + 2 * (i0 + kR - 1) >= P0 && total == 0xffffffffu) {
        floe_ptx::mbar_wait(&totbar, P, 13u << 28);
        total = n_total;
      }
      const uint32_t lim = total == 0xffffffffu ? P0 : total;
      const uint32_t n_mine = lim > grp ? (lim - grp + 1) / 2 : 0u;
      if (i0 >= n_mine) break;
      Vec dv[kR][2];
      float gp[kR], sc[kR];
      bool proc[kR];
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        gp[r] = 0.0f;
        sc[r] = 0.0f;
        dv[r][0] = dv[r][1] = Vec{};
        proc[r] = i0 + r < n_mine;
        if (proc[r]) {
          floe_ptx::mbar_wait(&fullC[stg], ph, (4u << 28) | (grp + 2 * (i0 + r)));
          if (i0 + r == 0 && grp == 0 && t == 0) mark(5);
          sc[r] = stage_scale[stg];
          const Vec *rec = reinterpret_cast<const Vec *>(ring + stg * REC_B);
          const Vec g0 = rec[2 * gt];
          const Vec g1 = rec[2 * gt + 1];
          dv[r][0] = rec[512 + 2 * gt];
          dv[r][1] = rec[512 + 2 * gt + 1];
          __syncwarp();
          if (lane == 0) mbar_arrive1(&emptyC[stg]);
          const __half2 *h0 = reinterpret_cast<const __half2 *>(&g0);
          const __half2 *h1 = reinterpret_cast<const __half2 *>(&g1);
          float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int jj = 0; jj < EPT2 / 4; ++jj) {
            acc = __ffma2_rn(__half22float2(h0[jj]), x2[jj], acc);
            acc = __ffma2_rn(__half22float2(h1[jj]), x2[EPT2 / 4 + jj], acc);
          }
          gp[r] = acc.x + acc.y;
          stg += 2;
          if (stg >= nsC) {
            stg -= nsC;
            ph ^= 1u;
          }
        }
      }
      warp_reduce_t(gp, std::integral_constant<int, kR>{});
      if ((lane & (32 / kR - 1)) == 0) red[grp][batch & 1][gw][lane / (32 / kR)] = gp[0];
      gbar(grp);
      float g = red[grp][batch & 1][lane % 8][min(lane / 8, (uint32_t)kR - 1)];
      g += __shfl_xor_sync(0xffffffffu, g, 4);
      g += __shfl_xor_sync(0xffffffffu, g, 2);
      g += __shfl_xor_sync(0xffffffffu, g, 1);
      float scl = sc[0];
      bool pl = proc[0];
#pragma unroll
      for (int r = 1; r < kR; ++r)
        if (lane / 8 == (uint32_t)r) {
          scl = sc[r];
          pl = proc[r];
        }
      const float myaco = pl ? floe_k::silu_ref(g) * scl : 0.0f;
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        const float aco = __shfl_sync(0xffffffffu, myaco, 8 * r);
        if (!proc[r]) continue;
        ++processed;
        const float2 a2 = make_float2(aco, aco);
        const __half2 *e0 = reinterpret_cast<const __half2 *>(&dv[r][0]);
        const __half2 *e1 = reinterpret_cast<const __half2 *>(&dv[r][1]);
#pragma unroll
        for (int jj = 0; jj < EPT2 / 4; ++jj) {
          y2[jj] = __ffma2_rn(a2, __half22float2(e0[jj]), y2[jj]);
          y2[EPT2 / 4 + jj] = __ffma2_rn(a2, __half22float2(e1[jj]), y2[EPT2 / 4 + jj]);
        }
      }
    }
    if (total == 0xffffffffu) {  // paired, every item was in the first ring fill
      floe_ptx::mbar_wait(&totbar, P, 13u << 28);
      total = n_total;
    }
    K += total;
    if (processed > 0) {
      float *yo = yl + EPT2 * gt;
#pragma unroll
      for (int i = 0; i < EPT2 / 4; ++i)
        floe_k::red_add_v4(yo + 4 * i, y2[2 * i].x, y2[2 * i].y, y2[2 * i + 1].x, y2[2 * i + 1].y);
    }
    if (t == 0) {
      mark(6);
      if (a.paired) floe_ptx::mbar_wait_cluster(&donebar, P, 18u << 28);
    }
    cbar();
    // ---- end of layer: reset the list, take a finishing ticket
    for (uint32_t i = t; i < list_cap; i += kConsumers) lf[i] = 0u;
    if (t < (uint32_t)floe_k::kMaxSlots) slot_cnt[t] = 0u;
    if (l + 1 == a.n_layers) break;
    if (t == 0) {
      n_list = 0u;
      const unsigned long long old = atom_add_release(a.lbar);  // after this CTA's y adds
      const uint32_t tau = (uint32_t)(old % G);
      tau_s = tau;
      mark_prev(29);
      if (a.phase_ns && l + 1 == a.trace_layer) a.phase_ns[b * kTraceSlots + 28] = tau;
      floe_ptx::mbar_arrive(&tickbar);
      if (tau < NCH) {  // a chunk owner needs h: wait for every CTA
        if (tau != G - 1) poll_until(a.lbar, (old / G + 1) * G, "layer barrier", tau);
      }
      mark_prev(30);
      floe_ptx::mbar_arrive(&lpass);
    }
    cbar();
    chunk = tau_s < NCH ? tau_s : 0xffffffffu;
  }
}

}  // namespace floe_v3
