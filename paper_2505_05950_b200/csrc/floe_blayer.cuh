// floe_blayer.cuh -- the MoE block for a batch of tokens (SURVEY configs 4
// and 5): block_forward (core/src/model.cpp:145-169) for B tokens at once.
//   u = h + mixing h            mix_batched   (one warp per mixing row, all tokens)
//   logits = router u; route    route_batched (one warp per token: top_k with ties
//                                              to the lower index, softmax, la.cpp:37-61)
//   tokens grouped by expert    dispatch      (device counting, no host sort)
//   experts                     floe_gpu_expert_forward_batched per expert
//   y = u + sum_j w_j out_j     combine       (ascending expert order)
#pragma once

#include <cuda_fp16.h>

#include <cstdint>

#include "floe_kernels.cuh"

namespace floe_bl {

constexpr uint32_t kMixTok = 64;  // tokens per mixing pass (registers per lane)

// u[t][r] = h[t][r] + sum_k M[r][k] h[t][k] for T <= kMixTok tokens: one warp
// per row r streams the row once; every lane keeps T partial dots; h comes
// from shared memory in 256-element chunks (T x 1 KB).
template <typename MT>
__global__ void __launch_bounds__(256) mix_batched(const MT *__restrict__ M, uint32_t dh,
                                                   const float *__restrict__ h, uint32_t T,
                                                   float *__restrict__ u) {
  extern __shared__ float hs[];  // [T][256]
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t r = blockIdx.x * 8 + warp;
  float acc[kMixTok];
#pragma unroll
  for (uint32_t t = 0; t < kMixTok; ++t) acc[t] = 0.0f;
  for (uint32_t k0 = 0; k0 < dh; k0 += 256) {
    __syncthreads();
    for (uint32_t i = threadIdx.x; i < T * 256; i += blockDim.x) {
      const uint32_t t = i / 256, k = i % 256;
      hs[i] = k0 + k < dh ? h[(size_t)t * dh + k0 + k] : 0.0f;
    }
    __syncthreads();
    if (r >= dh) continue;
    float w[8];
    const uint32_t kk = k0 + 8 * lane;
    if (kk + 8 <= dh) {  // one 16-B (f16) or two 16-B (f32) loads per lane
      if constexpr (sizeof(MT) == 2) {
        const uint4 q = *reinterpret_cast<const uint4 *>(M + (size_t)r * dh + kk);
        const __half2 *p2 = reinterpret_cast<const __half2 *>(&q);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const float2 f = __half22float2(p2[i]);
          w[2 * i] = f.x;
          w[2 * i + 1] = f.y;
        }
      } else {
        const float4 a = *reinterpret_cast<const float4 *>(M + (size_t)r * dh + kk);
        const float4 b = *reinterpret_cast<const float4 *>(M + (size_t)r * dh + kk + 4);
        w[0] = a.x; w[1] = a.y; w[2] = a.z; w[3] = a.w;
        w[4] = b.x; w[5] = b.y; w[6] = b.z; w[7] = b.w;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        w[i] = kk + i < dh ? static_cast<float>(M[(size_t)r * dh + kk + i]) : 0.0f;
    }
#pragma unroll
    for (uint32_t t = 0; t < kMixTok; ++t) {
      if (t < T) {
        const float4 a = *reinterpret_cast<const float4 *>(hs + t * 256 + 8 * lane);
        const float4 b = *reinterpret_cast<const float4 *>(hs + t * 256 + 8 * lane + 4);
        float s = acc[t];
        s = fmaf(w[0], a.x, s);
        s = fmaf(w[1], a.y, s);
        s = fmaf(w[2], a.z, s);
        s = fmaf(w[3], a.w, s);
        s = fmaf(w[4], b.x, s);
        s = fmaf(w[5], b.y, s);
        s = fmaf(w[6], b.z, s);
        s = fmaf(w[7], b.w, s);
        acc[t] = s;
      }
    }
  }
  if (r >= dh) return;
#pragma unroll
  for (uint32_t t = 0; t < kMixTok; ++t) {
    if (t < T) {
      float s = acc[t];
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (lane == 0) u[(size_t)t * dh + r] = h[(size_t)t * dh + r] + s;  // drift_scale 1
    }
  }
}

// logits[t][e] = router_e . u_t (one warp per (token, expert)), then per token
// (one warp): top_k (la.cpp:48-61; ties to the lower index, NaN-safe order)
// and softmax over the selected logits (la.cpp:37-46).
__global__ void __launch_bounds__(256) router_logits(const float *__restrict__ router, uint32_t E,
                                                     uint32_t dh, const float *__restrict__ u,
                                                     uint32_t T, float *__restrict__ logits) {
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (gw >= T * E) return;
  const uint32_t t = gw / E, e = gw % E;
  const float *a = router + (size_t)e * dh, *x = u + (size_t)t * dh;
  float s = 0.0f;
  for (uint32_t k = lane; k < dh; k += 32) s = fmaf(a[k], x[k], s);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) logits[(size_t)t * E + e] = s;
}

__global__ void __launch_bounds__(256) route_batched(const float *__restrict__ logits, uint32_t T,
                                                     uint32_t E, uint32_t K,
                                                     uint32_t *__restrict__ sel,
                                                     float *__restrict__ w,
                                                     uint32_t *__restrict__ counts,
                                                     uint32_t *__restrict__ lists) {
  const uint32_t t = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (t >= T) return;
  const float lg = lane < E ? logits[(size_t)t * E + lane] : -__int_as_float(0x7f800000);
  const unsigned long long mykey = floe_k::topk_key(lg, lane);
  uint32_t taken = 0;
  for (uint32_t r = 0; r < K; ++r) {
    const bool cand = lane < E && !((taken >> lane) & 1u);
    unsigned long long bk = cand ? mykey : 0ull;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) bk = max(bk, __shfl_xor_sync(0xffffffffu, bk, o));
    taken |= 1u << floe_k::topk_index(bk);
  }
  const bool mine = (taken >> lane) & 1u;
  float mx = mine ? lg : -__int_as_float(0x7f800000);
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const float ex = mine ? expf(lg - mx) : 0.0f;
  float sum = 0.0f;
  for (uint32_t m = taken; m; m &= m - 1) sum += __shfl_sync(0xffffffffu, ex, __ffs(m) - 1);
  if (mine) {
    const uint32_t j = __popc(taken & ((1u << lane) - 1));  // ascending expert order
    sel[(size_t)t * K + j] = lane;
    w[(size_t)t * K + j] = ex / sum;
    const uint32_t pos = atomicAdd(&counts[lane], 1u);
    lists[(size_t)lane * T + pos] = t * K + j;  // (token, slot) pair id
  }
}

// X[i] = u[pair_i / K] for the expert's pairs (contiguous rows for the
// batched expert forward); the inverse scatter copies the expert's outputs
// back to their pair slots.
__global__ void gather_rows(const float *__restrict__ u, const uint32_t *__restrict__ pairs,
                            uint32_t n, uint32_t K, uint32_t dh, float *__restrict__ X) {
  const uint32_t i = blockIdx.y;
  if (i >= n) return;
  const float4 *src = reinterpret_cast<const float4 *>(u + (size_t)(pairs[i] / K) * dh);
  float4 *dst = reinterpret_cast<float4 *>(X + (size_t)i * dh);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < dh / 4; k += gridDim.x * blockDim.x)
    dst[k] = src[k];
}
__global__ void scatter_rows(const float *__restrict__ Y, const uint32_t *__restrict__ pairs,
                             uint32_t n, uint32_t dh, float *__restrict__ out) {
  const uint32_t i = blockIdx.y;
  if (i >= n) return;
  const float4 *src = reinterpret_cast<const float4 *>(Y + (size_t)i * dh);
  float4 *dst = reinterpret_cast<float4 *>(out + (size_t)pairs[i] * dh);
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < dh / 4; k += gridDim.x * blockDim.x)
    dst[k] = src[k];
}

// y[t] = u[t] + sum_j w[t][j] * out[t*K + j], ascending expert order
// (model.cpp:160-166 with drift_scale 1).
__global__ void combine(const float *__restrict__ u, const float *__restrict__ out,
                        const float *__restrict__ w, uint32_t K, uint32_t dh,
                        float *__restrict__ y) {
  const uint32_t t = blockIdx.y;
  for (uint32_t k = blockIdx.x * blockDim.x + threadIdx.x; k < dh; k += gridDim.x * blockDim.x) {
    float acc = u[(size_t)t * dh + k];
    for (uint32_t j = 0; j < K; ++j)
      acc += w[(size_t)t * K + j] * out[((size_t)t * K + j) * dh + k];
    y[(size_t)t * dh + k] = acc;
  }
}

}  // namespace floe_bl
