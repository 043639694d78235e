// floe_kernels.cuh -- sm_100a kernels of the FloE compressed-expert FFN path.
//
// Reference algorithm (paths relative to /root/reference/proj/):
//   expert_forward_sparse(const CompressedExpert&, const Vec&)  core/src/model.cpp:128-142
//     v = qgemv_channels(up_q, x)                               core/src/quant.cpp:122-136
//     keep c iff !(|v[c]| < t)                                  core/src/model.cpp:135
//     y += silu(gate_c . x) * v[c] * down_c  (kept c only)      core/src/model.cpp:136-140
//
// Kernels (the INT2 fast path lives in floe_v2.cuh; these serve every other
// shape: any bits, any group size, any d_hidden)
//   K1g k1_generic         dequant GEMV + |v|>=t epilogue + compaction
//   K2g k2_generic         channel-sparse gate dot + SwiGLU + down accumulation
//   dequant_up             bit-exact f32 dequantisation (debug / parity)
//   mixing_gemv, route_topk, predict_experts_k   layer glue (model.cpp:83-93,145-169)
//
// HBM layout of one generic-path expert:
//   codes    u8 [di][dh*bits/8]  unchanged reference packing (LE in byte)
//   scales   u16[di][dh/g]       f16 bits, unchanged
//   zeros    u16[di][dh/g]       f16 bits, unchanged
//   records  f16[di][2][dh]      gate row c | down row c  (pack_compact wire format)
// Fast-path experts replace codes/scales/zeros by the tile-fragment layout.
#pragma once

#include <cuda_fp16.h>
#include <cstdint>

namespace floe_k {

constexpr int kMaxSlots = 8;

// Device-side descriptor of one resident expert.
struct ExpertDesc {
  const uint8_t *codes;    // generic path: reference packing (null on the fast path)
  const uint16_t *scales;  // generic path
  const uint16_t *zeros;   // generic path
  const __half *records;   // [di][2*dh]
  const uint32_t *tiles;   // fast path: tile-fragment up projection (floe_v2.cuh)
  float threshold;
  uint32_t host_records;   // records read in place from pinned host memory (over PCIe)
  uint32_t pad_[2];
};

// Kept-channel lists ("segments").  K1 runs on a (G1, slots) grid; CTA b of
// slot s owns the contiguous channel range [di*b/G1, di*(b+1)/G1) and writes
// its kept channels, ascending, to kept_idx/kept_v[s*di + di*b/G1 + j] for
// j < seg_count[s*G1 + b].  No atomics: every call overwrites every count.
// K2 prefix-scans seg_count, so the global entry order is (slot, channel)
// ascending -- deterministic, like the reference's ascending channel loop.
struct K1Args {
  const ExpertDesc *table;  // expert descriptors
  const uint32_t *sel;      // nullable: slot j uses table[sel[j]] (else table[j])
  const float *x;           // f32[dh]
  uint32_t dh, di, bits, group_size;
  int use_threshold;        // 1: use `threshold` instead of the expert's
  float threshold;
  float *v_out;             // nullable, [slots][di]
  uint8_t *mask_out;        // nullable, [slots][di]
  uint32_t *kept_idx;       // [slots][di]  (workspace)
  float *kept_v;            // [slots][di]  (workspace)
  uint32_t *seg_count;      // [slots][G1]
  float *y_zero;            // nullable: zeroed by CTA 0 (K2 accumulates into it)
};

struct K2Args {
  const ExpertDesc *table;
  const uint32_t *sel;       // nullable
  const float *weights;      // nullable: per-slot combine weight (routing softmax)
  const float *x;            // f32[dh]
  uint32_t dh, di, slots, g1;
  const uint32_t *kept_idx;  // [slots][di]
  const float *kept_v;       // [slots][di]
  const uint32_t *seg_count;  // [slots][g1]
  float *y;                  // f32[dh], accumulated with fp32 reductions
  uint32_t *n_kept_out;      // nullable [slots]
  uint32_t *kept_out;        // nullable [slots][di]: kept ids, ascending per slot
  unsigned long long *stats;  // nullable [2]: calls, kept channels (running totals)
};

__device__ __forceinline__ float h2f(uint16_t h) {
  return __half2float(__ushort_as_half(h));
}

__device__ __forceinline__ uint4 ldg_stream_u128(const void *p) {
  uint4 v;
  asm("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
      : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
      : "l"(p));
  return v;
}

__device__ __forceinline__ void red_add_v4(float *p, float a, float b, float c,
                                           float d) {
  asm volatile("red.global.add.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(a),
               "f"(b), "f"(c), "f"(d)
               : "memory");
}

// silu(z) = z / (1 + e^-z)  (core/src/la.cpp:31), IEEE division and expf.
__device__ __forceinline__ float silu_ref(float z) { return z / (1.0f + expf(-z)); }

// Reference get_code (core/src/quant.cpp:35-41) over a byte array.
__device__ __forceinline__ uint32_t get_code(const uint8_t *codes, uint32_t bits,
                                             uint64_t i) {
  uint64_t bit = i * bits;
  uint64_t idx = bit >> 3;
  uint32_t off = (uint32_t)(bit & 7);
  uint32_t v = (uint32_t)codes[idx] >> off;
  if (off + bits > 8) v |= (uint32_t)codes[idx + 1] << (8 - off);
  return v & ((1u << bits) - 1);
}

__device__ __forceinline__ uint32_t seg_begin(uint32_t di, uint32_t b, uint32_t g1) {
  return (uint32_t)(((uint64_t)di * b) / g1);
}

// K1 epilogue, called by one full warp; lane handles channel c (if valid).
// Appends kept channels to the CTA's segment in ascending order; `running`
// (warp-uniform) is the segment's count so far.
__device__ __forceinline__ void seg_emit(const K1Args &a, uint32_t slot, uint32_t seg_base,
                                         uint32_t c, bool valid, float v, float thr,
                                         uint32_t &running) {
  const uint32_t lane = threadIdx.x & 31;
  // model.cpp:135: `if (fabs(v) < t) continue;` -> ties and NaN are kept.
  const bool keep = valid && !(fabsf(v) < thr);
  const size_t off = (size_t)slot * a.di + c;
  if (valid) {
    if (a.v_out) a.v_out[off] = v;
    if (a.mask_out) a.mask_out[off] = keep ? 1 : 0;
  }
  const uint32_t bal = __ballot_sync(0xffffffffu, keep);
  if (keep) {
    const size_t o = (size_t)slot * a.di + seg_base + running + __popc(bal & ((1u << lane) - 1));
    a.kept_idx[o] = c;
    a.kept_v[o] = v;
  }
  running += __popc(bal);
}

// ---------------------------------------------------------------------------
// K1 generic: any bits in {1,2,3,4,8}, any group size dividing n, any dh.
// One warp per channel; per element the reference's own dequantize_at
// expression (quant.cpp:104-109): float(code)*scale + zero.
__global__ void __launch_bounds__(256) k1_generic(const K1Args a) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const uint32_t slot = blockIdx.y;
  const uint32_t e = a.sel ? a.sel[slot] : slot;
  const ExpertDesc d = a.table[e];
  const float thr = a.use_threshold ? a.threshold : d.threshold;
  if (a.y_zero && blockIdx.x == 0 && slot == 0)
    for (uint32_t i = threadIdx.x; i < a.dh; i += blockDim.x) a.y_zero[i] = 0.0f;
  const uint32_t c0 = seg_begin(a.di, blockIdx.x, gridDim.x);
  const uint32_t c1 = seg_begin(a.di, blockIdx.x + 1, gridDim.x);
  __shared__ float vbuf[32];
  uint32_t running = 0;
  for (uint32_t cb = c0; cb < c1; cb += 32) {
    for (uint32_t j = warp; j < 32; j += 8) {  // 4 channels per warp
      const uint32_t c = cb + j;
      float acc = 0.0f;
      if (c < c1) {
        const uint64_t base = (uint64_t)c * a.dh;
        for (uint32_t k = lane; k < a.dh; k += 32) {
          const uint64_t i = base + k;
          const uint64_t g = i / a.group_size;
          const float w = fmaf((float)get_code(d.codes, a.bits, i), h2f(d.scales[g]),
                               h2f(d.zeros[g]));
          acc = fmaf(w, a.x[k], acc);
        }
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) vbuf[j] = acc;
    }
    __syncthreads();
    if (warp == 0) {
      const uint32_t c = cb + lane;
      seg_emit(a, slot, c0 - 0, c, c < c1, vbuf[lane], thr, running);
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) a.seg_count[slot * gridDim.x + blockIdx.x] = running;
}

// ---------------------------------------------------------------------------
// Segment prefix: prefix[i] = sum_{j<i} seg_count[j] for i in [0, n], in
// shared memory, computed by the whole CTA (blockDim multiple of 32, <=1024).
__device__ inline void seg_prefix(const uint32_t *counts, uint32_t n, uint32_t *prefix) {
  __shared__ uint32_t warp_tot[32];
  const uint32_t t = threadIdx.x, nt = blockDim.x;
  const uint32_t per = (n + nt - 1) / nt;
  const uint32_t lo = min(n, t * per), hi = min(n, lo + per);
  uint32_t s = 0;
  for (uint32_t i = lo; i < hi; ++i) s += counts[i];
  // inclusive warp scan
  uint32_t inc = s;
  const uint32_t lane = t & 31, warp = t >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= (uint32_t)o) inc += y;
  }
  if (lane == 31) warp_tot[warp] = inc;
  __syncthreads();
  if (warp == 0) {
    const uint32_t nw = nt / 32;
    uint32_t wv = lane < nw ? warp_tot[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, wv, o);
      if (lane >= (uint32_t)o) wv += y;
    }
    if (lane < nw) warp_tot[lane] = wv;  // inclusive warp totals
  }
  __syncthreads();
  uint32_t run = inc - s + (warp ? warp_tot[warp - 1] : 0);  // exclusive start of chunk
  for (uint32_t i = lo; i < hi; ++i) {
    prefix[i] = run;
    run += counts[i];
  }
  if (t == nt - 1) prefix[n] = run;
  __syncthreads();
}

// Entry p (0 <= p < prefix[n]) -> segment index (largest i with prefix[i] <= p).
__device__ __forceinline__ uint32_t seg_find(const uint32_t *prefix, uint32_t n, uint32_t p) {
  uint32_t lo = 0, hi = n;  // invariant: prefix[lo] <= p < prefix[hi]
  while (hi - lo > 1) {
    const uint32_t mid = (lo + hi) >> 1;
    if (prefix[mid] <= p) lo = mid;
    else hi = mid;
  }
  return lo;
}

struct KeptEntry {
  uint32_t slot, c, slot_pos;
  float v;
};

__device__ __forceinline__ KeptEntry kept_entry(const K2Args &a, const uint32_t *prefix,
                                                uint32_t p) {
  const uint32_t nseg = a.slots * a.g1;
  const uint32_t idx = seg_find(prefix, nseg, p);
  const uint32_t slot = idx / a.g1, b = idx % a.g1;
  const size_t o = (size_t)slot * a.di + seg_begin(a.di, b, a.g1) + (p - prefix[idx]);
  KeptEntry k;
  k.slot = slot;
  k.c = a.kept_idx[o];
  k.v = a.kept_v[o];
  k.slot_pos = p - prefix[slot * a.g1];
  return k;
}

__device__ __forceinline__ float slot_weight(const K2Args &a, uint32_t slot) {
  return a.weights ? a.weights[slot] : 1.0f;
}

// Per-call bookkeeping by CTA 0 of K2 (or of k1_finalize).
__device__ __forceinline__ void k2_publish(const K2Args &a, const uint32_t *prefix) {
  if (blockIdx.x != 0) return;
  if (threadIdx.x < a.slots && a.n_kept_out)
    a.n_kept_out[threadIdx.x] =
        prefix[(threadIdx.x + 1) * a.g1] - prefix[threadIdx.x * a.g1];
  if (threadIdx.x == 0 && a.stats) {
    atomicAdd(&a.stats[0], 1ull);
    atomicAdd(&a.stats[1], (unsigned long long)prefix[a.slots * a.g1]);
  }
}

// ---------------------------------------------------------------------------
// K2 generic: one CTA per kept entry (grid-stride), fp32 atomics into y.
__global__ void __launch_bounds__(128) k2_generic(const K2Args a) {
  extern __shared__ uint32_t prefix[];
  const uint32_t nseg = a.slots * a.g1;
  seg_prefix(a.seg_count, nseg, prefix);
  k2_publish(a, prefix);
  const uint32_t total = prefix[nseg];
  __shared__ float red[4];
  for (uint32_t p = blockIdx.x; p < total; p += gridDim.x) {
    const KeptEntry k = kept_entry(a, prefix, p);
    if (a.kept_out && threadIdx.x == 0) a.kept_out[(size_t)k.slot * a.di + k.slot_pos] = k.c;
    if (!a.y) continue;
    const uint32_t e = a.sel ? a.sel[k.slot] : k.slot;
    const __half *rec = a.table[e].records + (size_t)k.c * 2 * a.dh;
    float acc = 0.0f;
    for (uint32_t i = threadIdx.x; i < a.dh; i += blockDim.x)
      acc = fmaf(__half2float(rec[i]), a.x[i], acc);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
    __syncthreads();
    const float g = red[0] + red[1] + red[2] + red[3];
    __syncthreads();
    const float aco = silu_ref(g) * k.v * slot_weight(a, k.slot);
    for (uint32_t i = threadIdx.x; i < a.dh; i += blockDim.x)
      atomicAdd(&a.y[i], aco * __half2float(rec[a.dh + i]));
  }
}

// ---------------------------------------------------------------------------
// dequantize (quant.cpp:104-120): out[i] = float(code)*scale + zero.  The
// product is exact (<= 8+11 significant bits), so one fmaf rounds exactly
// like the reference's mul-then-add: bit-exact.
__global__ void dequant_up(const ExpertDesc *table, uint64_t n, uint32_t bits,
                           uint32_t group_size, float *out) {
  const ExpertDesc d = table[0];
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t g = i / group_size;
    out[i] = fmaf((float)get_code(d.codes, bits, i), h2f(d.scales[g]), h2f(d.zeros[g]));
  }
}

// f32 -> f16 records with IEEE RNE (== floe::f32_to_f16 for finite values).
__global__ void pack_records(const float *gate, const float *down, uint32_t dh,
                             uint64_t di, __half *records) {
  const uint64_t n = (uint64_t)dh * di;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t c = i / dh, k = i % dh;
    records[c * 2 * dh + k] = __float2half_rn(gate[i]);
    records[c * 2 * dh + dh + k] = __float2half_rn(down[i]);
  }
}

// Device metadata layout for the K1 fast path: one u32 per group holding the
// f16 scale (low half) and f16 zero (high half) -> one 4-byte load per group.
__global__ void interleave_meta(const uint16_t *scales, const uint16_t *zeros, uint64_t n,
                                uint32_t *meta) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    meta[i] = (uint32_t)scales[i] | ((uint32_t)zeros[i] << 16);
}

__global__ void f32_to_f16_rn(const float *in, uint64_t n, __half *out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = __float2half_rn(in[i]);
}

// ---------------------------------------------------------------------------
// Layer glue (block_forward, model.cpp:145-169).
//
// u = h + mixing.h ; y = u ; logits = router.u ; top_k ; softmax -- one launch.
// Warp per row of the mixing matrix with the whole row's loads in flight; each
// CTA also reduces its rows' share of router.u into partial logits, and the
// last CTA (done counter, reset in-kernel) sums them in a fixed order and
// routes.  Deterministic: no float atomics.
struct MixArgs {
  const void *m;
  const float *h;
  uint32_t dh;
  const float *router;  // [E][dh]
  uint32_t E, k;
  float *u, *y_init, *u_trace;
  float *partial;  // [gridDim.x][E]
  uint32_t *done;
  uint32_t *sel;
  float *weights;
  uint32_t *sel_trace;
  float *w_trace;
};

// Total order for top_k: larger value first, ties (incl. -0 == +0) to the
// lower index, as la.cpp:52-55.  The reference's comparator is not a strict
// weak order once a NaN is present; here a NaN ranks below every number
// (-inf included), so every lane and thread agrees on an in-range selection
// for any input.  Key = (class|ordered value) << 8 | (255 - index); 0 never
// occurs for a real candidate.
__device__ __forceinline__ unsigned long long topk_key(float v, uint32_t i) {
  uint32_t hi;
  if (isnan(v)) {
    hi = 0u;
  } else {
    const uint32_t u = __float_as_uint(v == 0.0f ? 0.0f : v);
    hi = 1u + ((u >> 31) ? ~u : (u | 0x80000000u));  // -inf -> 0x00800000
  }
  return ((unsigned long long)hi << 8) | (255u - i);
}
__device__ __forceinline__ uint32_t topk_index(unsigned long long key) {
  return 255u - (uint32_t)(key & 255u);
}
__device__ inline void topk_small(const float *v, uint32_t n, uint32_t k, uint32_t *out);

// route (model.cpp:83-93) after the logits: top_k, softmax over the selected
// logits (la.cpp:37-46), outputs.  One thread.
__device__ inline void route_finish(const float *logits, uint32_t E, uint32_t k, uint32_t *sel,
                                    float *weights, uint32_t *sel_trace, float *w_trace) {
  uint32_t sidx[32];
  topk_small(logits, E, k, sidx);
  float wv[32];
  for (uint32_t i = 0; i < k; ++i) wv[i] = logits[sidx[i]];
  float mx = wv[0];
  for (uint32_t i = 1; i < k; ++i)
    if (mx < wv[i]) mx = wv[i];
  float sum = 0.0f;
  for (uint32_t i = 0; i < k; ++i) {
    wv[i] = expf(wv[i] - mx);
    sum += wv[i];
  }
  for (uint32_t i = 0; i < k; ++i) wv[i] /= sum;
  for (uint32_t i = 0; i < k; ++i) {
    sel[i] = sidx[i];
    weights[i] = wv[i];
    if (sel_trace) sel_trace[i] = sidx[i];
    if (w_trace) w_trace[i] = wv[i];
  }
}

template <typename T>
__global__ void __launch_bounds__(256) mixing_route(const MixArgs a) {
  extern __shared__ float hs[];
  __shared__ float pl[8][32];
  __shared__ bool last;
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t i = threadIdx.x; i < a.dh; i += blockDim.x) hs[i] = a.h[i];
  __syncthreads();
  const uint32_t row = blockIdx.x * 8 + warp;
  float uu = 0.0f;
  if (row < a.dh) {
    const T *mr = static_cast<const T *>(a.m) + (size_t)row * a.dh;
    constexpr uint32_t EPL = 16 / sizeof(T);  // elements per 128-bit load
    constexpr int U = 16;                     // loads in flight per lane
    float acc = 0.0f;
    for (uint32_t k0 = 0; k0 < a.dh; k0 += 32 * EPL * U) {
      uint4 q[U];
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const uint32_t k = k0 + (lane + 32 * j) * EPL;
        q[j] = k < a.dh ? ldg_stream_u128(mr + k) : make_uint4(0, 0, 0, 0);
      }
#pragma unroll
      for (int j = 0; j < U; ++j) {
        const uint32_t k = k0 + (lane + 32 * j) * EPL;
        if (k >= a.dh) break;
        if constexpr (sizeof(T) == 2) {
          const __half2 *hh = reinterpret_cast<const __half2 *>(&q[j]);
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(hh[i]);
            acc = fmaf(f.x, hs[k + 2 * i], acc);
            acc = fmaf(f.y, hs[k + 2 * i + 1], acc);
          }
        } else {
          acc = fmaf(__uint_as_float(q[j].x), hs[k], acc);
          acc = fmaf(__uint_as_float(q[j].y), hs[k + 1], acc);
          acc = fmaf(__uint_as_float(q[j].z), hs[k + 2], acc);
          acc = fmaf(__uint_as_float(q[j].w), hs[k + 3], acc);
        }
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    uu = hs[row] + 1.0f * acc;  // drift_scale = 1 (model.cpp:151-152)
    if (lane == 0) {
      a.u[row] = uu;
      a.y_init[row] = uu;
      if (a.u_trace) a.u_trace[row] = uu;
    }
  }
  // this CTA's rows' contribution to router.u
  if (lane < a.E) pl[warp][lane] = row < a.dh ? a.router[(size_t)lane * a.dh + row] * uu : 0.0f;
  __syncthreads();
  if (threadIdx.x < a.E) {
    float s = 0.0f;
#pragma unroll
    for (int w = 0; w < 8; ++w) s += pl[w][threadIdx.x];
    a.partial[blockIdx.x * a.E + threadIdx.x] = s;
  }
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(a.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ float logits[32];
  for (uint32_t e = warp; e < a.E; e += 8) {
    float s = 0.0f;
    for (uint32_t b = lane; b < gridDim.x; b += 32) s += __ldcg(&a.partial[b * a.E + e]);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (lane == 0) logits[e] = s;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *a.done = 0;
    route_finish(logits, a.E, a.k, a.sel, a.weights, a.sel_trace, a.w_trace);
  }
}

// top_k (la.cpp:48-61) over a short vector held by one thread.
__device__ inline void topk_small(const float *v, uint32_t n, uint32_t k,
                                  uint32_t *out) {
  uint32_t taken = 0;  // n <= 32
  for (uint32_t r = 0; r < k; ++r) {
    unsigned long long best = 0;
    for (uint32_t i = 0; i < n; ++i)
      if (!(taken & (1u << i))) best = max(best, topk_key(v[i], i));
    const uint32_t bi = topk_index(best);
    taken |= 1u << bi;
    out[r] = bi;
  }
  for (uint32_t i = 1; i < k; ++i)
    for (uint32_t j = i; j > 0 && out[j - 1] > out[j]; --j) {
      const uint32_t tmp = out[j];
      out[j] = out[j - 1];
      out[j - 1] = tmp;
    }
}

// logits = W u (+ b); top_k; optional softmax over the selected logits
// (route, model.cpp:83-93; predict_experts, predictor.cpp:164-177).
// One CTA, one warp per row.  E <= 32.
__global__ void __launch_bounds__(256) route_topk(const float *__restrict__ w,
                                                  const float *__restrict__ b,
                                                  const float *__restrict__ u,
                                                  uint32_t E, uint32_t dh,
                                                  uint32_t k, int softmax,
                                                  uint32_t *sel, float *weights,
                                                  uint32_t *sel_trace,
                                                  float *w_trace) {
  __shared__ float logits[32];
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (uint32_t r = warp; r < E; r += blockDim.x / 32) {
    float acc = 0.0f;
    for (uint32_t i = lane; i < dh; i += 32) acc = fmaf(w[(size_t)r * dh + i], u[i], acc);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    if (lane == 0) logits[r] = b ? acc + b[r] : acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t s[32];
    topk_small(logits, E, k, s);
    float wv[32];
    for (uint32_t i = 0; i < k; ++i) wv[i] = logits[s[i]];
    if (softmax) {  // softmax_inplace (la.cpp:37-46)
      float mx = wv[0];
      for (uint32_t i = 1; i < k; ++i)
        if (mx < wv[i]) mx = wv[i];
      float sum = 0.0f;
      for (uint32_t i = 0; i < k; ++i) {
        wv[i] = expf(wv[i] - mx);
        sum += wv[i];
      }
      for (uint32_t i = 0; i < k; ++i) wv[i] /= sum;
    }
    for (uint32_t i = 0; i < k; ++i) {
      sel[i] = s[i];
      if (weights) weights[i] = wv[i];
      if (sel_trace) sel_trace[i] = s[i];
      if (w_trace) w_trace[i] = wv[i];
    }
  }
}

// router_pred = router + router * mixing ([E][dh], E <= 32), the fused
// kernel's routing predictor.  Thread j owns column j; setup only.
template <typename MT>
__global__ void router_pred(const float *__restrict__ router, const MT *__restrict__ mixing,
                            uint32_t E, uint32_t dh, float *__restrict__ out) {
  const uint32_t j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= dh) return;
  // f64 accumulation, 8 experts per pass (registers)
  for (uint32_t e0 = 0; e0 < E; e0 += 8) {
    double acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) acc[e] = 0.0;
    for (uint32_t i = 0; i < dh; ++i) {
      const double m = static_cast<double>(static_cast<float>(mixing[(size_t)i * dh + j]));
#pragma unroll
      for (int e = 0; e < 8; ++e)
        if (e0 + e < E) acc[e] = fma((double)router[(size_t)(e0 + e) * dh + i], m, acc[e]);
    }
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (e0 + e < E)
        out[(size_t)(e0 + e) * dh + j] = (float)((double)router[(size_t)(e0 + e) * dh + j] + acc[e]);
  }
}

}  // namespace floe_k
