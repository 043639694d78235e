// floe_prefill.cuh -- the expert FFN for many tokens at once (config 5 prefill,
// large config-4 batches): expert_forward_sparse (core/src/model.cpp:128-142)
// for n tokens as three dense f16 tensor-core GEMMs with f32 accumulation.
// With ~1000 tokens per expert every channel is kept by some token, so the
// gate/down products are dense; the per-token mask is applied to the
// coefficients (a = 0 for a dropped channel), which gives the reference's sum
// over kept channels.
//
// Precision: every operand is scaled per token row by a power of two (no f16
// overflow or subnormals at any token magnitude).  The up projection decides
// the masks, so it is computed to ~22 bits with f16 hi + lo splits:
//   v = x . W      = [x_hi | x_hi | x_lo] . [W_hi | W_lo | W_hi]   (K = 3 dh)
// the gate and down products use the f16-rounded activations / coefficients
// against the f16 records (relative error ~1e-4 of g and y, against the 1e-2
// tolerance; the records themselves are f16):
//   g = x_hi . gate,   y = a_hi . down
// W = float(code) * scale + zero (quant.cpp:104-109) is dequantized from the
// tile layout per call (the compressed expert stays the source of truth).
#pragma once

#include "floe_v2.cuh"

namespace floe_pf {

// W -> Wb [di][3 dh] f16 = [W_hi | W_lo | W_hi], from the tile layout.
template <int DH>
__global__ void wcat_tiled(const uint32_t *tiles, uint32_t di, __half *wb) {
  constexpr uint32_t TB = floe_v2::tile_bytes(DH) / 4;
  const uint64_t n = (uint64_t)di * DH / 2;  // element pairs
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = (uint32_t)(2 * i / DH), kk = (uint32_t)(2 * i % DH);
    const uint32_t t = c / floe_v2::kTileCh, row = c % floe_v2::kTileCh, span = kk / 64, e = kk % 64;
    const uint32_t p = span / 2, kidx = (span & 1) * 2 + (row >= 8);
    const uint32_t lane = 4 * (row & 7) + e / 16;
    const uint32_t *tile = tiles + (uint64_t)t * TB;
    const uint32_t w = tile[(p * 32 + lane) * 4 + kidx];
    const uint32_t m = tile[DH + (p * 8 + (row & 7)) * 4 + kidx];
    const float sc = floe_k::h2f((uint16_t)(m & 0xffffu)), zr = floe_k::h2f((uint16_t)(m >> 16));
    const float w0 = fmaf((float)((w >> (2 * (e % 16))) & 3u), sc, zr);
    const float w1 = fmaf((float)((w >> (2 * (e % 16 + 1))) & 3u), sc, zr);
    const __half h0 = __float2half_rn(w0), h1 = __float2half_rn(w1);
    const __half l0 = __float2half_rn(w0 - __half2float(h0)), l1 = __float2half_rn(w1 - __half2float(h1));
    __half2 *row3 = reinterpret_cast<__half2 *>(wb + (uint64_t)c * 3 * DH + kk);
    row3[0] = __halves2half2(h0, h1);
    row3[DH / 2] = __halves2half2(l0, l1);
    row3[DH] = __halves2half2(h0, h1);
  }
}

// Per-row power-of-two scale: s = 2^-e with max|row| < 2^e (1 for an all-zero
// or non-finite row), so the scaled row's magnitudes are in [0.5, 1).
__device__ __forceinline__ float pow2_inv_scale(float mx) {
  if (!(mx > 0.0f) || !isfinite(mx)) return 1.0f;
  int e = 0;
  frexpf(mx, &e);
  return ldexpf(1.0f, -e);
}

// x [n][dh] f32 -> xa [n][3 dh] = [hi | hi | lo] of x * s_row, inv[row] = 1 / s_row.
__global__ void xcat(const float *x, uint32_t dh, __half *xa, float *inv) {
  const uint32_t r = blockIdx.x;
  const float *xr = x + (size_t)r * dh;
  __shared__ float red[32];
  float mx = 0.0f;
  for (uint32_t k = threadIdx.x; k < dh; k += blockDim.x) mx = fmaxf(mx, fabsf(xr[k]));
  for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float m = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0f;
    for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  const float s = pow2_inv_scale(red[0]);
  if (threadIdx.x == 0) inv[r] = 1.0f / s;
  __half *xo = xa + (size_t)r * 3 * dh;
  for (uint32_t k = threadIdx.x; k < dh; k += blockDim.x) {
    const float v = xr[k] * s;  // exact (power of two)
    const __half hi = __float2half_rn(v);
    xo[k] = hi;
    xo[dh + k] = hi;
    xo[2 * dh + k] = __float2half_rn(v - __half2float(hi));
  }
}

// a = silu(g) * v where !(|v| < t) (model.cpp:135-137, la.cpp:31), else 0;
// g (and v unless v_true) are the scaled GEMM outputs (times inv[row] for the
// true values);
// ah [n][di] = f16(a * s_a[row]), ainv[row] = 1 / s_a.  One block per token
// row: the row maximum first (exact power-of-two scale).
__global__ void coeffs(const float *v, const float *g, const float *inv, uint32_t di, float t,
                       __half *acat, float *ainv, int v_true) {
  const uint32_t r = blockIdx.x;
  const float ig = inv[r], iv = v_true ? 1.0f : ig;  // v from the exact batched K1: unscaled
  const float *vr = v + (size_t)r * di, *gr = g + (size_t)r * di;
  __shared__ float red[32];
  float mx = 0.0f;
  for (uint32_t c = threadIdx.x; c < di; c += blockDim.x) {
    const float vv = vr[c] * iv;
    const float a = !(fabsf(vv) < t) ? floe_k::silu_ref(gr[c] * ig) * vv : 0.0f;
    mx = fmaxf(mx, fabsf(a));
  }
  for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float m = threadIdx.x < blockDim.x / 32 ? red[threadIdx.x] : 0.0f;
    for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  const float s = pow2_inv_scale(red[0]);
  if (threadIdx.x == 0) ainv[r] = 1.0f / s;
  __half *ao = acat + (size_t)r * di;
  for (uint32_t c = threadIdx.x; c < di; c += blockDim.x) {
    const float vv = vr[c] * iv;
    ao[c] = __float2half_rn((!(fabsf(vv) < t) ? floe_k::silu_ref(gr[c] * ig) * vv : 0.0f) * s);
  }
}

// coeffs for di <= KM * 1024 with 1024 threads per row: each thread keeps its
// KM coefficients in registers between the row maximum and the f16 write (one
// read of v and g, KM independent loads in flight per thread; the 256-thread
// two-pass version took 67 us per 16-token call under ncu).  Same arithmetic,
// so the same bits as coeffs.
template <int KM>
__global__ void __launch_bounds__(1024) coeffs_reg(const float *v, const float *g, const float *inv,
                                                   uint32_t di, float t, __half *acat, float *ainv,
                                                   int v_true) {
  const uint32_t r = blockIdx.x;
  const float ig = inv[r], iv = v_true ? 1.0f : ig;
  const float *vr = v + (size_t)r * di, *gr = g + (size_t)r * di;
  __shared__ float red[32];
  float a[KM], mx = 0.0f;
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    const uint32_t c = threadIdx.x + 1024u * k;
    float av = 0.0f;
    if (c < di) {
      const float vv = vr[c] * iv;
      av = !(fabsf(vv) < t) ? floe_k::silu_ref(gr[c] * ig) * vv : 0.0f;
    }
    a[k] = av;
    mx = fmaxf(mx, fabsf(av));
  }
  for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x / 32] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    float m = red[threadIdx.x];
    for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  const float s = pow2_inv_scale(red[0]);
  if (threadIdx.x == 0) ainv[r] = 1.0f / s;
  __half *ao = acat + (size_t)r * di;
#pragma unroll
  for (int k = 0; k < KM; ++k) {
    const uint32_t c = threadIdx.x + 1024u * k;
    if (c < di) ao[c] = __float2half_rn(a[k] * s);
  }
}

// u = h + mh * inv[row] (the block input, model.cpp:150-152: drift scale 1).
__global__ void residual(const float *h, const float *mh, const float *inv, uint32_t dh, float *u) {
  const uint32_t r = blockIdx.x;
  const float s = inv[r];
  for (uint32_t k = threadIdx.x; k < dh; k += blockDim.x)
    u[(size_t)r * dh + k] = h[(size_t)r * dh + k] + mh[(size_t)r * dh + k] * s;
}

// y[row] *= ainv[row] (the coefficients' scale), in place.
__global__ void unscale_rows(float *y, uint32_t dh, const float *ainv) {
  const uint32_t r = blockIdx.x;
  const float s = ainv[r];
  for (uint32_t k = threadIdx.x; k < dh; k += blockDim.x) y[(size_t)r * dh + k] *= s;
}

}  // namespace floe_pf
