// floe_calib.cuh -- threshold calibration on the device: the reference's
// collect_stats / calibrate_model (core/src/model.cpp:242-330) and
// SampleReservoir / calibrate (core/src/sparsify.cpp:42-64,128-142), bit for
// bit.
//
// collect_stats runs the DENSE float model (f32 gate/up/down) over calibration
// tokens and records |up_c . u| of every channel of every routed expert in a
// per-(layer, expert) reservoir; calibrate takes the ceil(k N)-th smallest
// sample.  Bit-exactness with the reference needs its exact arithmetic:
//   * every dot product is a strictly ascending f32 sum of rounded products,
//     acc = acc + a*b with no FMA contraction (la.cpp:10-29, built for x86-64
//     without FMA) -> __fmul_rn / __fadd_rn, one thread per sum;
//   * silu and softmax use expf (la.cpp:31,37-46): glibc's expf is correctly
//     rounded, reproduced as (float)exp((double)x);
//   * the reservoir is Rng(seed ^ 0x5eedca11, layer*E + expert) with
//     below(n) = next_u64() % n (rng.cpp:26-63); draw d of a stream is
//     mix64(state0 + d*gamma), so every add past the cap is decided in
//     parallel and the last value landing on a slot wins.
// This is model preparation, not the decode path: correctness over speed,
// but the weight reads are coalesced (32x32 transposed tiles) so a Mixtral
// layer calibrates in milliseconds per token.
#pragma once

#include <cstdint>

#include "floe_gen.cuh"

namespace floe_cal {

__device__ __forceinline__ float fmul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float fadd(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ float exp_cr(float x) { return (float)exp((double)x); }
__device__ __forceinline__ float silu_cr(float x) {
  return __fdiv_rn(x, fadd(1.0f, exp_cr(-x)));
}

// y[t][r] = sum_c A[r][c] * x[t][c], ascending c (gemv, la.cpp:10-17); one
// warp per 32 rows of A and one token, A read in coalesced 32x32 tiles.
// out[t][r] = base ? base[t][r] + scale * acc : acc  (u = h + drift * mixed).
__global__ void __launch_bounds__(256) gemv_seq(const float *__restrict__ A, uint32_t rows,
                                                uint32_t cols, const float *__restrict__ x,
                                                const float *__restrict__ base, float scale,
                                                float *__restrict__ out) {
  __shared__ float tile[8][32][33];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t t = blockIdx.y;
  const uint32_t r0 = (blockIdx.x * 8 + warp) * 32;
  if (r0 >= rows) return;
  const float *xt = x + (size_t)t * cols;
  float acc = 0.0f;
  for (uint32_t c0 = 0; c0 < cols; c0 += 32) {
#pragma unroll 4
    for (uint32_t r = 0; r < 32; ++r)
      tile[warp][r][lane] =
          (r0 + r < rows && c0 + lane < cols) ? A[(size_t)(r0 + r) * cols + c0 + lane] : 0.0f;
    __syncwarp();
    const float xv = c0 + lane < cols ? xt[c0 + lane] : 0.0f;
    const uint32_t n = min(32u, cols - c0);
    for (uint32_t c = 0; c < n; ++c)
      acc = fadd(acc, fmul(tile[warp][lane][c], __shfl_sync(0xffffffffu, xv, c)));
    __syncwarp();
  }
  const uint32_t r = r0 + lane;
  if (r < rows) {
    float *o = out + (size_t)t * rows + r;
    *o = base ? fadd(base[(size_t)t * rows + r], fmul(scale, acc)) : acc;
  }
}

// route (model.cpp:83-93) of every token from its logits [T][E]: top_k with
// ties to the lower index, ascending output (la.cpp:48-61), softmax over the
// selected logits (la.cpp:37-46).  One thread per token.
__global__ void route_tokens(const float *__restrict__ logits, uint32_t T, uint32_t E,
                             uint32_t K, uint32_t *__restrict__ sel, float *__restrict__ w) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= T) return;
  const float *lg = logits + (size_t)t * E;
  uint32_t taken = 0;  // E <= 32
  for (uint32_t r = 0; r < K; ++r) {
    int best = -1;
    for (uint32_t i = 0; i < E; ++i) {
      if ((taken >> i) & 1u) continue;
      // better(a, b): v[a] > v[b], ties to the lower index (a NaN never wins)
      if (best < 0 || lg[i] > lg[best]) best = (int)i;
    }
    taken |= 1u << best;
  }
  float v[32];
  uint32_t n = 0;
  for (uint32_t i = 0; i < E; ++i)
    if ((taken >> i) & 1u) {
      sel[(size_t)t * K + n] = i;
      v[n++] = lg[i];
    }
  float mx = v[0];
  for (uint32_t i = 1; i < n; ++i) mx = fmaxf(mx, v[i]);
  float sum = 0.0f;
  for (uint32_t i = 0; i < n; ++i) {
    v[i] = exp_cr(v[i] - mx);
    sum = fadd(sum, v[i]);
  }
  for (uint32_t i = 0; i < n; ++i) w[(size_t)t * K + i] = __fdiv_rn(v[i], sum);
}

// For the (token, expert) pairs `pairs` [P] (token index, slot j, expert e,
// position of the token among expert e's tokens in this batch): v_c =
// up_c . u_t, g_c = silu(gate_c . u_t), a_c = g_c * v_c for every channel c;
// |v_c| -> vals[e][pos][c], a_c -> acoef[pair][c].  One warp per 32
// channels, weights read in coalesced transposed tiles.
struct Pair {
  uint32_t t, j, e, pos;
};
__global__ void __launch_bounds__(128) up_gate_seq(const float *const *__restrict__ up,
                                                   const float *const *__restrict__ gate,
                                                   const float *__restrict__ u, uint32_t dh,
                                                   uint32_t di, const Pair *__restrict__ pairs,
                                                   float *const *__restrict__ vals,
                                                   float *__restrict__ acoef) {
  __shared__ float tu[4][32][33], tg[4][32][33];
  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Pair pr = pairs[blockIdx.y];
  const uint32_t c0 = (blockIdx.x * 4 + warp) * 32;
  if (c0 >= di) return;
  const float *U = up[pr.e], *Gt = gate[pr.e];
  const float *ut = u + (size_t)pr.t * dh;
  float av = 0.0f, ag = 0.0f;
  for (uint32_t k0 = 0; k0 < dh; k0 += 32) {
#pragma unroll 4
    for (uint32_t r = 0; r < 32; ++r) {
      const bool ok = c0 + r < di && k0 + lane < dh;
      tu[warp][r][lane] = ok ? U[(size_t)(c0 + r) * dh + k0 + lane] : 0.0f;
      tg[warp][r][lane] = ok ? Gt[(size_t)(c0 + r) * dh + k0 + lane] : 0.0f;
    }
    __syncwarp();
    const float xv = k0 + lane < dh ? ut[k0 + lane] : 0.0f;
    const uint32_t n = min(32u, dh - k0);
    for (uint32_t k = 0; k < n; ++k) {
      const float xk = __shfl_sync(0xffffffffu, xv, k);
      av = fadd(av, fmul(tu[warp][lane][k], xk));
      ag = fadd(ag, fmul(tg[warp][lane][k], xk));
    }
    __syncwarp();
  }
  const uint32_t c = c0 + lane;
  if (c < di) {
    vals[pr.e][(size_t)pr.pos * di + c] = fabsf(av);
    acoef[(size_t)blockIdx.y * di + c] = fmul(silu_cr(ag), av);  // float a = g * vi
  }
}

// out_pair[k] = sum_c a_c * down_c[k], ascending c (model.cpp:283-284);
// thread per output element k, coalesced over k.
__global__ void down_seq(const float *const *__restrict__ down, const Pair *__restrict__ pairs,
                         const float *__restrict__ acoef, uint32_t dh, uint32_t di,
                         float *__restrict__ out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= dh) return;
  const Pair pr = pairs[blockIdx.y];
  const float *D = down[pr.e];
  const float *ac = acoef + (size_t)blockIdx.y * di;
  float acc = 0.0f;
  for (uint32_t c = 0; c < di; ++c) acc = fadd(acc, fmul(ac[c], D[(size_t)c * dh + k]));
  out[(size_t)blockIdx.y * dh + k] = acc;
}

// y_t = u_t + sum_j (drift * w_tj) * out_tj in slot order (model.cpp:286-290).
__global__ void combine_seq(const float *__restrict__ u, const float *__restrict__ out,
                            const float *__restrict__ w, const int32_t *__restrict__ pair_of,
                            uint32_t T, uint32_t K, uint32_t dh, float drift,
                            float *__restrict__ y) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x, t = blockIdx.y;
  if (k >= dh) return;
  float acc = u[(size_t)t * dh + k];
  for (uint32_t j = 0; j < K; ++j) {
    const int32_t p = pair_of[t * K + j];
    acc = fadd(acc, fmul(fmul(drift, w[t * K + j]), out[(size_t)p * dh + k]));
  }
  y[(size_t)t * dh + k] = acc;
}

// ---- reservoir (SampleReservoir::add, sparsify.cpp:56-64)
struct ResState {
  unsigned long long seen;   // values added so far
  unsigned long long state0, gamma;  // Rng(seed ^ 0x5eedca11, stream)
};

// value i of this batch has global index g = seen + i: g < cap -> slot g;
// otherwise draw d = g - cap + 1 decides slot j = mix64(state0 + d gamma) %
// (g + 1) (kept if j < cap).  The last value of the batch landing on a slot
// wins: owner[j] = 1 + max i.
__global__ void reservoir_claim(const ResState *__restrict__ st, uint64_t cap,
                                uint64_t n, uint32_t *__restrict__ owner) {
  const uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const unsigned long long g = st->seen + i;
  unsigned long long j;
  if (g < cap) {
    j = g;
  } else {
    const unsigned long long d = g - cap + 1;
    j = floe_gen::mix64(st->state0 + d * st->gamma) % (g + 1);
    if (j >= cap) return;
  }
  atomicMax(&owner[j], (uint32_t)i + 1u);  // 0 = no value of this batch
}
__global__ void reservoir_apply(uint64_t cap, const float *__restrict__ vals,
                                const uint32_t *__restrict__ owner, float *__restrict__ samples) {
  const uint64_t j = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  if (j < cap && owner[j] != 0u) samples[j] = vals[owner[j] - 1u];
}
__global__ void reservoir_init(ResState *st, uint64_t seed, uint64_t stream0, uint32_t n) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const floe_gen::StreamState s = floe_gen::stream_init(seed, stream0 + i);
  st[i].seen = 0;
  st[i].state0 = s.state0;
  st[i].gamma = s.gamma;
}
// threshold of reservoir i from its sorted samples: sorted[rank - 1],
// rank = clamp(ceil(k * n), 1, n) (calibrate_threshold, sparsify.cpp:42-54)
__global__ void reservoir_pick(const ResState *__restrict__ st, const float *__restrict__ sorted,
                               uint64_t cap, uint32_t n_res, double k, float *__restrict__ out) {
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n_res) return;
  const uint64_t n = st[i].seen < cap ? st[i].seen : cap;
  if (k == 0.0) {
    out[i] = 0.0f;
    return;
  }
  if (n == 0) {
    out[i] = __int_as_float(0x7fc00000);
    return;
  }
  uint64_t rank = (uint64_t)ceil(k * (double)n);
  if (rank == 0) rank = 1;
  if (rank > n) rank = n;
  out[i] = sorted[(uint64_t)i * cap + rank - 1];
}
__global__ void reservoir_advance(ResState *st, uint64_t n) { st->seen += n; }

}  // namespace floe_cal
