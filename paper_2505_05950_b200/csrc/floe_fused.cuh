// floe_fused.cuh -- ONE persistent sm_100a kernel per decode step.
//
// A kernel launch on B200 carries several microseconds of fixed ramp cost
// (profiles/r01_membench_cold_footprint.txt: an empty 148-CTA grid takes
// ~3.5 us cold; a 34 MB stream ~10 us), comparable to the whole roofline time
// of an expert-token (~10 us).  So the hot path runs as a single cooperative
// grid, one CTA per SM, that walks the reference's block_forward in phases
// separated by grid barriers (model.cpp:145-169):
//
//   A  (layer mode)  u = h + mixing.h; y = u; per-CTA partial router logits
//      --- grid barrier ---
//      every CTA sums the partials in the same fixed order and routes
//      (route, model.cpp:83-93): identical top-k/softmax in all CTAs
//   B  K1: v = qgemv_channels(up_e, u) for each selected expert over this
//      CTA's channel range, |v| >= t, kept channels appended to the CTA's
//      segment (quant.cpp:122-136, model.cpp:135)
//      --- grid barrier ---
//   C  K2: kept entries of all experts split evenly over CTAs; per entry
//      silu(gate_c . u) * v_c * w_e * down_c accumulated in registers and
//      reduced into y once (model.cpp:136-140, 162-166)
//
// All weight traffic is 1-D bulk copies (cp.async.bulk) through ONE shared
// memory ring that persists across phases and is re-carved per phase (16 KB
// stages for mixing rows and gate|down records, K1-tile stages for phase B);
// thread 0 refills a stage after the block barrier that retires it.
#pragma once

#include "floe_fast.cuh"

namespace floe_k {

struct FusedArgs {
  // phase A (layer mode only)
  const void *mixing;  // [dh][dh] f16 or f32
  const float *h;      // [dh]
  const float *router; // [E][dh]
  uint32_t n_experts, top_k;
  int has_mixing;
  float *partial;  // [grid][32]
  float *u_trace;
  uint32_t *sel_trace;
  float *w_trace;
  uint32_t *sel_out;  // [slots] routing result for later consumers
  float *w_out;
  // shared
  float *u;  // [dh] expert input (written in phase A in layer mode)
  float *y;  // [dh] output
  uint32_t dh, di, group_size, slots;
  const ExpertDesc *table;
  int use_threshold;
  float threshold;
  float *v_out;       // nullable [slots][di]
  uint8_t *mask_out;  // nullable [slots][di]
  uint32_t *kept_idx; // [slots][di]
  float *kept_v;      // [slots][di]
  uint32_t *seg_count;  // [slots][grid]
  unsigned long long *bar;  // grid barrier counter (monotonic, never reset)
  uint32_t *n_kept_out;
  uint32_t *kept_out;
  unsigned long long *stats;
  uint32_t ring_bytes;           // shared-memory ring size
  unsigned long long *phase_ns;  // nullable [grid][8]: %globaltimer at phase marks
  uint32_t debug;                // diagnostics: bit0 skip K1 math, bit1 skip K2 math
};

__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kTraceSlots = 64;  // per CTA: 0..7 phase marks, 8.. record arrivals

__device__ __forceinline__ void mark(const FusedArgs &a, int k) {
  if (a.phase_ns && threadIdx.x == 0 && k < kTraceSlots)
    a.phase_ns[blockIdx.x * kTraceSlots + k] = global_ns();
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

// Grid-wide barrier on a monotonic 64-bit counter (co-resident grid).
__device__ __forceinline__ void grid_sync(unsigned long long *bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned long long g = gridDim.x;
    const unsigned long long old = atomicAdd(bar, 1ull);
    const unsigned long long target = (old / g + 1) * g;
    const unsigned long long t0 = global_ns();
    for (uint32_t it = 1; ld_acquire_u64(bar) < target; ++it) {
      __nanosleep(20);
      if ((it & 1023u) == 0 && global_ns() - t0 > floe_ptx::kWatchdogNs)
        floe_ptx::watchdog_fire("grid barrier", (uint32_t)(target / g), (uint32_t)(old % g));
    }
    __threadfence();
  }
  __syncthreads();
}

constexpr uint32_t kFusedMaxStages = 24;
constexpr uint32_t kFusedRingBytes = 168 * 1024;
constexpr int kMaxGridPerWarp = 8;  // grid <= 256 CTAs

// Ring of bulk-copy stages in dynamic shared memory.  The kFusedMaxStages
// mbarriers are initialised ONCE per launch; each phase re-carves the ring
// with its own stage size and continues every barrier's phase sequence:
// `par` bit s is the parity of barrier s's completed phases when the current
// carving started, so use u waits for parity (u / ns + par_s) & 1.
struct Ring {
  uint8_t *base;
  uint64_t *full;
  uint32_t stage_bytes, ns, tag, par;  // tag: phase id for the watchdog
  __device__ uint8_t *stage(uint32_t u) const { return base + (u % ns) * stage_bytes; }
  __device__ uint64_t *bar(uint32_t u) const { return &full[u % ns]; }
  __device__ void wait(uint32_t u) const {
    floe_ptx::mbar_wait(bar(u), ((u / ns) + (par >> (u % ns))) & 1u, tag | u);
  }
  __device__ void issue(uint32_t u, const void *src, uint32_t bytes) const {
    floe_ptx::mbar_arrive_expect_tx(bar(u), bytes);
    floe_ptx::bulk_g2s(stage(u), src, bytes, bar(u));
  }
};

__device__ __forceinline__ uint32_t ring_ns(uint32_t stage_bytes, uint32_t ring_bytes) {
  return min(kFusedMaxStages, ring_bytes / stage_bytes);
}

// First carving: initialise the barriers.
__device__ __forceinline__ Ring ring_init(uint8_t *base, uint64_t *full, uint32_t stage_bytes,
                                          uint32_t ring_bytes, uint32_t tag) {
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < kFusedMaxStages; ++s) floe_ptx::mbar_init(&full[s], 1);
    floe_ptx::fence_barrier_init();
  }
  __syncthreads();
  return Ring{base, full, stage_bytes, ring_ns(stage_bytes, ring_bytes), tag, 0u};
}

// Re-carve after the previous carving's `used` stage uses were all issued and
// waited (block-uniform count): no barrier re-initialisation.
__device__ __forceinline__ Ring ring_next(const Ring &prev, uint32_t used, uint32_t stage_bytes,
                                          uint32_t ring_bytes, uint32_t tag) {
  uint32_t par = prev.par;
  for (uint32_t s = 0; s < prev.ns && s < used; ++s)
    par ^= (((used - 1 - s) / prev.ns + 1) & 1u) << s;
  __syncthreads();  // previous stages fully read before they are refilled
  return Ring{prev.base, prev.full, stage_bytes, ring_ns(stage_bytes, ring_bytes), tag, par};
}

// ---------------------------------------------------------------------------
template <typename T, int SPANS, int GPT>
__global__ void __launch_bounds__(256, 1) floe_fused(const FusedArgs a) {
  constexpr int TPB = 256;
  constexpr int NW = TPB / 32;
  constexpr int CH = kK1Ch;
  constexpr int CS = TPB / SPANS;
  constexpr int CPT = CH / CS;
  constexpr int WPP = 4 / GPT;
  constexpr uint32_t DH = SPANS * 64;
  constexpr uint32_t ROW = DH / 4;
  constexpr uint32_t REC = 4 * DH;  // gate|down record bytes
  constexpr int R = 4;              // K2 records per batch
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[kFusedMaxStages];
  __shared__ uint64_t hbar;
  __shared__ float u_s[kMaxRowsPerCta];
  __shared__ float rs[32 * kMaxRowsPerCta];
  __shared__ float logits[32];
  __shared__ uint32_t sel_s[kMaxSlots];
  __shared__ float w_s[kMaxSlots];
  __shared__ const __half *rec_s[kMaxSlots];
  __shared__ float thr_s[kMaxSlots];
  __shared__ ExpertDesc table_s[32];
  __shared__ float red_max[NW];
  __shared__ __align__(16) uint32_t limb_s[SPANS][4][12];  // read as uint4
  __shared__ float xsum_s[SPANS][4];
  __shared__ float wsum[2][NW][CPT];
  __shared__ float red[NW][R];
  __shared__ float aco_s[2][R];
  __shared__ const __half *ent_rec[kK2Chunk];
  __shared__ float ent_scale[kK2Chunk];
  __shared__ uint32_t own_cnt_s[kMaxSlots];
  __shared__ uint32_t plan_s[4];  // T, own_b, d_b, D_b

  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t G = gridDim.x, b = blockIdx.x;
  float *hs = reinterpret_cast<float *>(smem + a.ring_bytes);  // [dh] (layer mode)
  mark(a, 0);

  if (t == 0) {
    floe_ptx::mbar_init(&hbar, 1);
    floe_ptx::fence_barrier_init();
  }
  // expert descriptors of the whole layer, fetched once (hidden behind phase A)
  const uint32_t n_table = a.has_mixing ? a.n_experts : a.slots;
  if (t < n_table) table_s[t] = a.table[t];
  Ring ring = ring_init(smem, full, REC, a.ring_bytes, 1u << 24);
  uint32_t ring_used = 0;  // stage uses of the current carving

  // =========================== phase A: mixing ===========================
  if (a.has_mixing) {
    const uint32_t row_bytes = DH * (uint32_t)sizeof(T);
    const uint32_t rps = REC / row_bytes;  // rows per stage (2 for f16, 1 for f32)
    const uint32_t r_lo = seg_begin(DH, b, G), r_hi = seg_begin(DH, b + 1, G);
    const uint32_t n_items = (r_hi - r_lo + rps - 1) / rps;
    ring_used = n_items;
    const T *m = static_cast<const T *>(a.mixing);
    const uint32_t per_round = min(NW / rps, ring.ns / 2);  // stages per block barrier
    auto issue_rows = [&](uint32_t i) {
      const uint32_t r0 = r_lo + i * rps, nr = min(rps, r_hi - r0);
      ring.issue(i, m + (size_t)r0 * DH, nr * row_bytes);
    };
    if (t == 0) {
      floe_ptx::mbar_arrive_expect_tx(&hbar, 4u * DH);
      floe_ptx::bulk_g2s(hs, a.h, 4u * DH, &hbar);
      for (uint32_t i = 0; i < n_items && i < ring.ns; ++i) issue_rows(i);
    }
    for (uint32_t i = t; i < a.n_experts * kMaxRowsPerCta; i += TPB) {
      const uint32_t e = i / kMaxRowsPerCta, lr = i % kMaxRowsPerCta;
      if (r_lo + lr < r_hi) rs[i] = a.router[(size_t)e * DH + r_lo + lr];
    }
    floe_ptx::mbar_wait(&hbar, 0);
    constexpr uint32_t EPL = 16 / sizeof(T);
    for (uint32_t i0 = 0; i0 < n_items; i0 += per_round) {
      const uint32_t item = i0 + warp / rps, sub = warp % rps;
      const uint32_t row = r_lo + item * rps + sub;
      if (warp / rps < per_round && item < n_items && row < r_hi) {
        ring.wait(item);
        const T *rowp = reinterpret_cast<const T *>(ring.stage(item)) + (size_t)sub * DH;
        float acc0 = 0.0f, acc1 = 0.0f;
#pragma unroll 4
        for (uint32_t k = lane * EPL; k < DH; k += 32 * EPL) {
          const uint4 qv = *reinterpret_cast<const uint4 *>(rowp + k);
          const float4 h0 = *reinterpret_cast<const float4 *>(hs + k);
          if constexpr (sizeof(T) == 2) {
            const float4 h1 = *reinterpret_cast<const float4 *>(hs + k + 4);
            const __half2 *hh = reinterpret_cast<const __half2 *>(&qv);
            const float2 f0 = __half22float2(hh[0]), f1 = __half22float2(hh[1]);
            const float2 f2 = __half22float2(hh[2]), f3 = __half22float2(hh[3]);
            acc0 = fmaf(f0.x, h0.x, acc0);
            acc1 = fmaf(f0.y, h0.y, acc1);
            acc0 = fmaf(f1.x, h0.z, acc0);
            acc1 = fmaf(f1.y, h0.w, acc1);
            acc0 = fmaf(f2.x, h1.x, acc0);
            acc1 = fmaf(f2.y, h1.y, acc1);
            acc0 = fmaf(f3.x, h1.z, acc0);
            acc1 = fmaf(f3.y, h1.w, acc1);
          } else {
            acc0 = fmaf(__uint_as_float(qv.x), h0.x, acc0);
            acc1 = fmaf(__uint_as_float(qv.y), h0.y, acc1);
            acc0 = fmaf(__uint_as_float(qv.z), h0.z, acc0);
            acc1 = fmaf(__uint_as_float(qv.w), h0.w, acc1);
          }
        }
        float acc = acc0 + acc1;
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
        const float uu = hs[row] + 1.0f * acc;  // drift_scale = 1 (model.cpp:151-152)
        if (lane == 0) {
          a.u[row] = uu;
          a.y[row] = uu;
          if (a.u_trace) a.u_trace[row] = uu;
          if (row - r_lo < kMaxRowsPerCta) u_s[row - r_lo] = uu;
        }
      }
      __syncthreads();  // the round's stages are consumed
      if (t == 0)
        for (uint32_t k = 0; k < per_round; ++k) {
          const uint32_t nxt = i0 + k + ring.ns;
          if (i0 + k < n_items && nxt < n_items) issue_rows(nxt);
        }
    }
    // this CTA's share of router.u (fixed order: ascending rows)
    if (warp == 0 && lane < a.n_experts) {
      float s = 0.0f;
      for (uint32_t r = r_lo; r < r_hi; ++r) {
        const uint32_t lr = r - r_lo;
        const float w = lr < kMaxRowsPerCta ? rs[lane * kMaxRowsPerCta + lr]
                                            : a.router[(size_t)lane * DH + r];
        const float uu = lr < kMaxRowsPerCta ? u_s[lr] : a.u[r];
        s = fmaf(w, uu, s);
      }
      a.partial[b * 32 + lane] = s;
    }
    mark(a, 1);
    grid_sync(a.bar);
    // route (model.cpp:83-93): every CTA sums the partials in the same order
    for (uint32_t e = warp; e < a.n_experts; e += NW) {
      float pv[kMaxGridPerWarp];  // all loads in flight at once
#pragma unroll
      for (int j = 0; j < kMaxGridPerWarp; ++j) {
        const uint32_t bb = lane + 32 * j;
        pv[j] = bb < G ? __ldcg(&a.partial[bb * 32 + e]) : 0.0f;
      }
      float s = 0.0f;
#pragma unroll
      for (int j = 0; j < kMaxGridPerWarp; ++j) s += pv[j];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) logits[e] = s;
    }
    __syncthreads();
    if (t == 0) {
      uint32_t sel[32];
      float wv[32];
      route_finish(logits, a.n_experts, a.top_k, sel, wv,
                   b == 0 ? a.sel_trace : nullptr, b == 0 ? a.w_trace : nullptr);
      for (uint32_t s = 0; s < a.slots; ++s) {
        sel_s[s] = sel[s];
        w_s[s] = wv[s];
        if (b == 0 && a.sel_out) {
          a.sel_out[s] = sel[s];
          a.w_out[s] = wv[s];
        }
      }
    }
  } else {
    if (t < a.slots) {
      sel_s[t] = t;
      w_s[t] = 1.0f;
    }
    if (b == 0)
      for (uint32_t i = t; i < DH; i += TPB) a.y[i] = 0.0f;  // before barrier 2
  }
  __syncthreads();
  if (t < a.slots) {
    const ExpertDesc &d = table_s[sel_s[t]];
    rec_s[t] = d.records;
    thr_s[t] = a.use_threshold ? a.threshold : d.threshold;
  }

  mark(a, 2);
  // =========================== phase B: K1 ================================
  {
    const uint32_t span = t % SPANS, q = t / SPANS;
    const uint32_t c_lo = seg_begin(a.di, b, G), c_hi = seg_begin(a.di, b + 1, G);
    const uint32_t n_sub = (c_hi - c_lo + CH - 1) / CH;
    const uint32_t n_items = n_sub * a.slots;
    if (n_sub == 0 && t < a.slots) {  // di < grid: an empty segment still publishes its count
      a.seg_count[t * G + b] = 0;
      own_cnt_s[t] = 0;
    }
    const uint32_t gpc = DH / a.group_size;
    const uint32_t code_sz = round_up128(CH * ROW);
    ring = ring_next(ring, ring_used, k1_stage_bytes(DH, gpc), a.ring_bytes, 2u << 24);
    ring_used = n_items;
    auto issue_tile = [&](uint32_t i) {  // item i = (slot, sub-tile)
      const uint32_t s = i / n_sub, k = i % n_sub;
      const uint32_t c0 = c_lo + k * CH, nc = min((uint32_t)CH, c_hi - c0);
      const ExpertDesc &d = table_s[sel_s[s]];
      floe_ptx::mbar_arrive_expect_tx(ring.bar(i), nc * (ROW + gpc * 4u));
      floe_ptx::bulk_g2s(ring.stage(i), d.codes + (size_t)c0 * ROW, nc * ROW, ring.bar(i));
      floe_ptx::bulk_g2s(ring.stage(i) + code_sz, d.meta + (size_t)c0 * gpc, nc * gpc * 4u,
                         ring.bar(i));
    };
    if (t == 0)
      for (uint32_t i = 0; i < n_items && i < ring.ns; ++i) issue_tile(i);

    // x limbs (word q of this span), shared by the CS threads of the span
    const float *xg = a.u;
    float xw[16];
    {
      const float4 *x4 = reinterpret_cast<const float4 *>(xg + 64 * span + 16 * (q & 3));
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const float4 f = __ldcg(x4 + i);
        xw[4 * i] = f.x;
        xw[4 * i + 1] = f.y;
        xw[4 * i + 2] = f.z;
        xw[4 * i + 3] = f.w;
      }
    }
    float mx = 0.0f;
    bool finite = true;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      mx = fmaxf(mx, fabsf(xw[i]));
      finite = finite && isfinite(xw[i]);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const bool warp_finite = __all_sync(0xffffffffu, finite);
    if (lane == 0) red_max[warp] = warp_finite ? mx : -1.0f;
    __syncthreads();
    bool all_finite = true;
    mx = 0.0f;
#pragma unroll
    for (int w = 0; w < NW; ++w) {
      all_finite = all_finite && red_max[w] >= 0.0f;
      mx = fmaxf(mx, red_max[w]);
    }
    int ex = 0;
    frexpf(mx, &ex);
    const bool scaled = mx > 0.0f && all_finite;
    const float S = scaled ? __int_as_float((127 + 22 - ex) << 23) : 1.0f;
    const float invS = scaled ? __int_as_float((127 - 22 + ex) << 23) : 1.0f;
    if (q < 4) {
      float s16 = 0.0f;
#pragma unroll
      for (int mm = 0; mm < 4; ++mm) {
        uint32_t l0 = 0, l1 = 0, l2 = 0;
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) {
          const int X = all_finite ? __float2int_rn(xw[mm + 4 * bb] * S) : 0;
          const int X0 = ((X + 128) & 255) - 128;
          const int Rr = (X - X0) >> 8;
          const int X1 = ((Rr + 128) & 255) - 128;
          const int X2 = (Rr - X1) >> 8;
          l0 |= (uint32_t)(X0 & 255) << (8 * bb);
          l1 |= (uint32_t)(X1 & 255) << (8 * bb);
          l2 |= (uint32_t)(X2 & 255) << (8 * bb);
        }
        limb_s[span][q][mm] = l0;
        limb_s[span][q][4 + mm] = l1;
        limb_s[span][q][8 + mm] = l2;
      }
#pragma unroll
      for (int i = 0; i < 16; ++i) s16 += xw[i];
      xsum_s[span][q] = s16;
    }
    __syncthreads();
    uint32_t lw[4][12];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
      for (int k = 0; k < 12; k += 4) {
        const uint4 v4 = *reinterpret_cast<const uint4 *>(&limb_s[span][i][k]);
        lw[i][k] = v4.x;
        lw[i][k + 1] = v4.y;
        lw[i][k + 2] = v4.z;
        lw[i][k + 3] = v4.w;
      }
    float xpart[GPT];
#pragma unroll
    for (int p = 0; p < GPT; ++p) {
      xpart[p] = 0.0f;
#pragma unroll
      for (int i = p * WPP; i < (p + 1) * WPP; ++i) xpart[p] += xsum_s[span][i];
    }
    const uint32_t g0 = (64u * span) / a.group_size;

    uint32_t running = 0;  // warp 0: kept so far in the current slot's segment
    for (uint32_t i = 0; i < n_items; ++i) {
      const uint32_t s = i / n_sub, k = i % n_sub;
      if (k == 0) running = 0;
      ring.wait(i);
      const uint8_t *st = ring.stage(i);
      const uint32_t c0 = c_lo + k * CH;
      const uint32_t nc = min((uint32_t)CH, c_hi - c0);
      float part[CPT];
      if (a.debug & 1u) {
#pragma unroll
        for (int r = 0; r < CPT; ++r) part[r] = 0.0f;
      } else if (all_finite) {
        // channels past nc read stale stage bytes: their partials are never used
#pragma unroll
        for (int r = 0; r < CPT; ++r) {
          const uint32_t j = q + CS * r;
          const uint4 w4 = *reinterpret_cast<const uint4 *>(st + j * ROW + 16 * span);
          const uint32_t *meta = reinterpret_cast<const uint32_t *>(st + code_sz) + j * gpc + g0;
          const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
          float acc = 0.0f;
#pragma unroll
          for (int p = 0; p < GPT; ++p) {
            int a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
            for (int ii = p * WPP; ii < (p + 1) * WPP; ++ii) {
#pragma unroll
              for (int mm = 0; mm < 4; ++mm) {
                const int cb = (int)((wv[ii] >> (2 * mm)) & 0x03030303u);
                a0 = __dp4a(cb, (int)lw[ii][mm], a0);
                a1 = __dp4a(cb, (int)lw[ii][4 + mm], a1);
                a2 = __dp4a(cb, (int)lw[ii][8 + mm], a2);
              }
            }
            const int Tt = a2 * 65536 + a1 * 256 + a0;
            const uint32_t mz = meta[p];
            const float sc = __half2float(__ushort_as_half((uint16_t)(mz & 0xffffu)));
            const float zr = __half2float(__ushort_as_half((uint16_t)(mz >> 16)));
            acc = fmaf(sc * invS, (float)Tt, fmaf(zr, xpart[p], acc));
          }
          part[r] = acc;
        }
      } else {
#pragma unroll
        for (int r = 0; r < CPT; ++r) {
          const uint32_t j = q + CS * r;
          const uint4 w4 = *reinterpret_cast<const uint4 *>(st + j * ROW + 16 * span);
          const uint32_t *meta = reinterpret_cast<const uint32_t *>(st + code_sz) + j * gpc + g0;
          const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
          part[r] = j < nc ? k1_span_f32(wv, meta, a.group_size, xg + 64 * span) : 0.0f;
        }
      }
#pragma unroll
      for (int sft = 16, cnt = CPT / 2; cnt >= 1; sft >>= 1, cnt >>= 1) {
        const bool upper = (lane & sft) != 0;
#pragma unroll
        for (int r = 0; r < cnt; ++r) {
          const float send = upper ? part[r] : part[r + cnt];
          const float keep = upper ? part[r + cnt] : part[r];
          part[r] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
        }
      }
#pragma unroll
      for (int sft = 32 / CPT / 2; sft >= 1; sft >>= 1)
        part[0] += __shfl_xor_sync(0xffffffffu, part[0], sft);
      if ((lane & (32 / CPT - 1)) == 0) wsum[i & 1][warp][lane / (32 / CPT)] = part[0];
      __syncthreads();  // wsum[i&1] complete; stage retired
      if (t == 0 && i + ring.ns < n_items) issue_tile(i + ring.ns);
      if (warp == 0) {
        const uint32_t j = lane;
        float v = 0.0f;
        if (j < (uint32_t)CH) {
          const uint32_t qq = j % CS, rr = j / CS;
#pragma unroll
          for (int w = 0; w < SPANS / 32; ++w) v += wsum[i & 1][qq * (SPANS / 32) + w][rr];
        }
        const uint32_t c = c0 + j;
        const bool valid = j < nc;
        // model.cpp:135: `if (fabs(v) < t) continue;` -> ties and NaN are kept
        const bool keep = valid && !(fabsf(v) < thr_s[s]);
        const size_t off = (size_t)s * a.di + c;
        if (valid) {
          if (a.v_out) a.v_out[off] = v;
          if (a.mask_out) a.mask_out[off] = keep ? 1 : 0;
        }
        const uint32_t bal = __ballot_sync(0xffffffffu, keep);
        if (keep) {
          const size_t o = (size_t)s * a.di + c_lo + running + __popc(bal & ((1u << lane) - 1));
          a.kept_idx[o] = c;
          a.kept_v[o] = v;
        }
        running += __popc(bal);
        if (k + 1 == n_sub && lane == 0) {
          a.seg_count[s * G + b] = running;
          own_cnt_s[s] = running;
        }
      }
    }
  }

  // =========================== phase C: K2 ================================
  // Own-first balanced assignment.  Target per CTA t_b = T*(b+1)/G - T*b/G
  // kept entries; CTA b keeps own_b = min(n_b, t_b, kK2Chunk) of its OWN
  // entries (so their records can be prefetched BEFORE the barrier) and
  // fills the deficit t_b - own_b from the pool of every CTA's surplus, in a
  // fixed global order.  Stage uses: [0, E0) own items (prefetched first P,
  // processed iff < own_b), then pool items in chunks.
  {
    constexpr int TPB2 = DH / 16;  // threads owning 16 elements each
    const bool active = t < (uint32_t)TPB2;  // dh = 2048 uses half the CTA
    __syncthreads();  // own_cnt_s complete, last K1 stage retired
    ring = ring_next(ring, ring_used, REC, a.ring_bytes, 3u << 24);
    uint32_t n_own = 0;
    for (uint32_t s = 0; s < a.slots; ++s) n_own += own_cnt_s[s];
    const uint32_t c_lo = seg_begin(a.di, b, G);
    const uint32_t n_res = min(n_own, kK2Chunk);
    // own entry j -> (slot, position in the slot's segment)
    auto own_entry = [&](uint32_t j, uint32_t &s_out, size_t &o_out) {
      uint32_t s = 0;
      while (s + 1 < a.slots && j >= own_cnt_s[s]) {
        j -= own_cnt_s[s];
        ++s;
      }
      s_out = s;
      o_out = (size_t)s * a.di + c_lo + j;
    };
    for (uint32_t j = t; j < n_res; j += TPB) {
      uint32_t s;
      size_t o;
      own_entry(j, s, o);
      const uint32_t c = __ldcg(&a.kept_idx[o]);
      ent_rec[j] = rec_s[s] + (size_t)c * 2 * DH;
      ent_scale[j] = __ldcg(&a.kept_v[o]) * w_s[s];
    }
    __syncthreads();
    const uint32_t P = min(n_res, ring.ns);  // speculative prefetch, before the barrier
    if (t == 0)
      for (uint32_t k = 0; k < P; ++k) ring.issue(k, ent_rec[k], REC);
    float2 x2[8], y2[8];
    {
      const uint32_t tt = active ? t : 0;
      const float4 *xa = reinterpret_cast<const float4 *>(a.u + 8 * tt);
      const float4 *xb = reinterpret_cast<const float4 *>(a.u + 8 * (tt + TPB2));
      const float4 q0 = __ldcg(xa), q1 = __ldcg(xa + 1), q2 = __ldcg(xb), q3 = __ldcg(xb + 1);
      x2[0] = make_float2(q0.x, q0.y);
      x2[1] = make_float2(q0.z, q0.w);
      x2[2] = make_float2(q1.x, q1.y);
      x2[3] = make_float2(q1.z, q1.w);
      x2[4] = make_float2(q2.x, q2.y);
      x2[5] = make_float2(q2.z, q2.w);
      x2[6] = make_float2(q3.x, q3.y);
      x2[7] = make_float2(q3.z, q3.w);
#pragma unroll
      for (int i = 0; i < 8; ++i) y2[i] = make_float2(0.0f, 0.0f);
    }
    mark(a, 3);
    grid_sync(a.bar);
    mark(a, 4);

    // ---- the plan: per-CTA totals n_bb, targets, surplus/deficit prefixes
    uint32_t *S = reinterpret_cast<uint32_t *>(smem + a.ring_bytes +
                                               (a.has_mixing ? 4u * DH : 0u));  // [G+1]
    uint32_t *D = S + (G + 1);                                                  // [G+1]
    uint32_t *NB = D + (G + 1);                                                 // [G]
    uint32_t *SU = NB + G;                                                      // [G]
    for (uint32_t bb = t; bb < G; bb += TPB) {
      uint32_t n = 0;
      for (uint32_t s = 0; s < a.slots; ++s) n += __ldcg(&a.seg_count[s * G + bb]);
      NB[bb] = n;
    }
    __syncthreads();
    seg_prefix(NB, G, S);  // S[bb] = sum_{<bb} n  (reused below)
    const uint32_t T = S[G];
    auto plan = [&](uint32_t bb, uint32_t &own, uint32_t &sur, uint32_t &def) {
      const uint32_t tb = (uint32_t)(((uint64_t)T * (bb + 1)) / G - ((uint64_t)T * bb) / G);
      const uint32_t n = NB[bb];
      own = min(min(n, tb), kK2Chunk);
      sur = n - own;
      def = tb - own;
    };
    __syncthreads();
    for (uint32_t bb = t; bb < G; bb += TPB) {
      uint32_t own, sur, def;
      plan(bb, own, sur, def);
      D[bb] = def;  // deficits (prefix-summed below)
      SU[bb] = sur;
    }
    __syncthreads();
    // prefix of deficits into D (in place via S as scratch is not possible):
    seg_prefix(D, G, S);  // S = deficit prefix
    __syncthreads();
    for (uint32_t bb = t; bb <= G; bb += TPB) D[bb] = S[bb];
    __syncthreads();
    seg_prefix(SU, G, S);  // S = surplus prefix
    if (t == 0) {
      uint32_t own, sur, def;
      plan(b, own, sur, def);
      plan_s[0] = T;
      plan_s[1] = own;
      plan_s[2] = def;
      plan_s[3] = D[b];
    }
    __syncthreads();
    const uint32_t own_b = plan_s[1], d_b = plan_s[2], D_b = plan_s[3];
    if (b == 0) {
      if (t == 0 && a.stats) {
        atomicAdd(&a.stats[0], 1ull);
        atomicAdd(&a.stats[1], (unsigned long long)T);
      }
      if (warp < a.slots && a.n_kept_out) {
        uint32_t n = 0;
        for (uint32_t bb = lane; bb < G; bb += 32) n += __ldcg(&a.seg_count[warp * G + bb]);
#pragma unroll
        for (int o = 16; o >= 1; o >>= 1) n += __shfl_xor_sync(0xffffffffu, n, o);
        if (lane == 0) a.n_kept_out[warp] = n;
      }
    }
    if (a.kept_out && warp < a.slots) {
      // own segment's ids -> ascending per-slot position (prefix over lower CTAs)
      uint32_t base = 0;
      for (uint32_t bb = lane; bb < b; bb += 32) base += __ldcg(&a.seg_count[warp * G + bb]);
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) base += __shfl_xor_sync(0xffffffffu, base, o);
      const uint32_t cnt = own_cnt_s[warp];
      for (uint32_t j = lane; j < cnt; j += 32)
        a.kept_out[(size_t)warp * a.di + base + j] =
            __ldcg(&a.kept_idx[(size_t)warp * a.di + c_lo + j]);
    }

    // ---- consume a run of n items at stage uses [ub, ub+n) from ent[eb..]
    uint32_t batch = 0;
    auto run_items = [&](uint32_t ub, uint32_t n, uint32_t eb, uint32_t proc_end,
                         uint32_t pre_issued) {
      if (t == 0)
        for (uint32_t k = pre_issued; k < n && k < ring.ns; ++k)
          ring.issue(ub + k, ent_rec[eb + k], REC);
      for (uint32_t q0 = 0; q0 < n; q0 += R, ++batch) {
        uint4 dv[R][2];
        float gp[R];
#pragma unroll
        for (int r = 0; r < R; ++r) {
          gp[r] = 0.0f;
          dv[r][0] = dv[r][1] = make_uint4(0, 0, 0, 0);
          const uint32_t k = q0 + r;
          if (k < n) {
            const uint32_t u_idx = ub + k;
            ring.wait(u_idx);
            if (u_idx < (uint32_t)(kTraceSlots - 8)) mark(a, 8 + (int)u_idx);
            if (active && k < proc_end && !(a.debug & 2u)) {
              const uint4 *rec = reinterpret_cast<const uint4 *>(ring.stage(u_idx));
              const uint4 g0 = rec[t], g1 = rec[t + TPB2];
              dv[r][0] = rec[2 * TPB2 + t];
              dv[r][1] = rec[3 * TPB2 + t];
              const __half2 *h0 = reinterpret_cast<const __half2 *>(&g0);
              const __half2 *h1 = reinterpret_cast<const __half2 *>(&g1);
              float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
              for (int j = 0; j < 4; ++j) {
                acc = __ffma2_rn(__half22float2(h0[j]), x2[j], acc);
                acc = __ffma2_rn(__half22float2(h1[j]), x2[4 + j], acc);
              }
              gp[r] = acc.x + acc.y;
            }
          }
        }
        // transposed warp reduction of R values: lanes 8r hold record r's warp sum
#pragma unroll
        for (int sft = 16, cnt = R / 2; cnt >= 1; sft >>= 1, cnt >>= 1) {
          const bool upper = (lane & sft) != 0;
#pragma unroll
          for (int r = 0; r < cnt; ++r) {
            const float send = upper ? gp[r] : gp[r + cnt];
            const float keep = upper ? gp[r + cnt] : gp[r];
            gp[r] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
          }
        }
#pragma unroll
        for (int sft = 32 / R / 2; sft >= 1; sft >>= 1)
          gp[0] += __shfl_xor_sync(0xffffffffu, gp[0], sft);
        if ((lane & (32 / R - 1)) == 0) red[warp][lane / (32 / R)] = gp[0];
        __syncthreads();  // red complete; the batch's stages are read
        if (t == 0)
          for (int r = 0; r < R; ++r) {
            const uint32_t nq = q0 + r + ring.ns;
            if (q0 + r < n && nq < n) ring.issue(ub + nq, ent_rec[eb + nq], REC);
          }
        // warp r finishes record r once: block sum, silu, scale
        if (warp < (uint32_t)R && q0 + warp < n && q0 + warp < proc_end) {
          float g = lane < (uint32_t)NW ? red[lane][warp] : 0.0f;
#pragma unroll
          for (int o = 4; o >= 1; o >>= 1) g += __shfl_xor_sync(0xffffffffu, g, o);
          if (lane == 0) aco_s[batch & 1][warp] = silu_ref(g) * ent_scale[eb + q0 + warp];
        }
        __syncthreads();  // aco_s visible
#pragma unroll
        for (int r = 0; r < R; ++r) {
          const uint32_t k = q0 + r;
          if (k >= n || k >= proc_end) break;
          const float aco = aco_s[batch & 1][r];
          const float2 a2 = make_float2(aco, aco);
          const __half2 *e0 = reinterpret_cast<const __half2 *>(&dv[r][0]);
          const __half2 *e1 = reinterpret_cast<const __half2 *>(&dv[r][1]);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            y2[j] = __ffma2_rn(a2, __half22float2(e0[j]), y2[j]);
            y2[4 + j] = __ffma2_rn(a2, __half22float2(e1[j]), y2[4 + j]);
          }
        }
      }
    };
    // own items: [0, E0), processed iff < own_b (prefetched surplus is drained)
    const uint32_t E0 = max(P, own_b);
    run_items(0, E0, 0, own_b, P);
    // pool items in chunks of kK2Chunk
    uint32_t ub = E0;
    for (uint32_t q = 0; q < d_b; q += kK2Chunk) {
      const uint32_t n = min(kK2Chunk, d_b - q);
      __syncthreads();  // ent_* free
      for (uint32_t k = t; k < n; k += TPB) {
        const uint32_t pi = D_b + q + k;        // pool index
        const uint32_t bb = seg_find(S, G, pi);  // source CTA
        uint32_t own_src, sur_src, def_src;
        plan(bb, own_src, sur_src, def_src);
        uint32_t j = own_src + (pi - S[bb]);  // entry in bb's own list
        uint32_t s = 0;
        for (; s + 1 < a.slots; ++s) {
          const uint32_t cs = __ldcg(&a.seg_count[s * G + bb]);
          if (j < cs) break;
          j -= cs;
        }
        const size_t o = (size_t)s * a.di + seg_begin(a.di, bb, G) + j;
        const uint32_t c = __ldcg(&a.kept_idx[o]);
        ent_rec[k] = rec_s[s] + (size_t)c * 2 * DH;
        ent_scale[k] = __ldcg(&a.kept_v[o]) * w_s[s];
      }
      __syncthreads();
      run_items(ub, n, 0, n, 0);
      ub += n;
    }
    mark(a, 5);
    if (own_b + d_b > 0 && active) {
      float *ya = a.y + 8 * t, *yb = a.y + 8 * (t + TPB2);
      red_add_v4(ya, y2[0].x, y2[0].y, y2[1].x, y2[1].y);
      red_add_v4(ya + 4, y2[2].x, y2[2].y, y2[3].x, y2[3].y);
      red_add_v4(yb, y2[4].x, y2[4].y, y2[5].x, y2[5].y);
      red_add_v4(yb + 4, y2[6].x, y2[6].y, y2[7].x, y2[7].y);
    }
  }
}

}  // namespace floe_k
