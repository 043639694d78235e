// floe_fast.cuh -- specialised sm_100a kernels for the Mixtral-shaped path
// (INT2 codes, d_hidden = 16*TPB).  Both kernels stream their weights with
// 1-D bulk copies (cp.async.bulk, the TMA engine) into an NS-deep shared
// memory ring tracked by mbarriers, so every SM keeps NS-1 tiles in flight
// without spending registers on loads.
//
// Reference (paths relative to /root/reference/proj/):
//   K1 = qgemv_channels + threshold    core/src/quant.cpp:122-136, core/src/model.cpp:135
//   K2 = gate dot + silu + down        core/src/model.cpp:136-140, core/src/la.cpp:25-31
#pragma once

#include "floe_kernels.cuh"
#include "floe_ptx.cuh"

namespace floe_k {

constexpr int kK1Ch = 16;  // channels per K1 tile

__host__ __device__ constexpr uint32_t round_up128(uint32_t x) { return (x + 127u) & ~127u; }

// Shared-memory bytes of one K1 stage for a given d_hidden / groups-per-channel.
__host__ __device__ constexpr uint32_t k1_stage_bytes(uint32_t tpb, uint32_t gpc) {
  return round_up128(kK1Ch * tpb * 4u) + 2u * round_up128(kK1Ch * gpc * 2u);
}

// Exact INT2 dot product of one code word with 16 pre-scaled inputs.
// c*4^i is formed exactly as (2^23 + c*4^i) - 2^23 from one LOP3 and one
// packed FADD2; the packed FFMA2 accumulates even/odd lanes of x.
__device__ __forceinline__ float dot16_int2(uint32_t w, const float2 (&xs)[8]) {
  const uint32_t magic = 0x4B000000u;
  const uint32_t w2 = w >> 22;
  const float2 off = make_float2(-8388608.0f, -8388608.0f);
  float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
  for (int p = 0; p < 8; ++p) {
    const int i0 = 2 * p, i1 = 2 * p + 1;
    const uint32_t s0 = i0 < 11 ? w : w2, s1 = i1 < 11 ? w : w2;
    const int h0 = i0 < 11 ? 2 * i0 : 2 * (i0 - 11);
    const int h1 = i1 < 11 ? 2 * i1 : 2 * (i1 - 11);
    float2 f;
    f.x = __uint_as_float(floe_ptx::and_or(s0, 3u << h0, magic));
    f.y = __uint_as_float(floe_ptx::and_or(s1, 3u << h1, magic));
    f = __fadd2_rn(f, off);
    acc = __ffma2_rn(f, xs[p], acc);
  }
  return acc.x + acc.y;
}

// ---------------------------------------------------------------------------
// K1: v[c] = sum_k deq(up[c,k]) x[k]; keep |v|>=t; compact kept channels.
//
// Tiles of 16 channels are claimed dynamically (one atomic per tile, issued
// NS-1 tiles ahead) and bulk-copied: codes 16*dh/4 B, scales and zeros
// 16*dh/g*2 B each.  Thread t owns x[16t, 16t+16) (one code word per
// channel, all in group 16t/g) -- x stays in registers pre-scaled by 4^-i,
// and the group-affine dequant is folded out of the inner loop:
//   sum_k (c_k s + z) x_k  =  s * sum_k c_k x_k  +  z * sum_k x_k .
template <int TPB, int NS>
__global__ void __launch_bounds__(TPB, 2) k1_int2(const K1Args a) {
  constexpr int NW = TPB / 32;
  constexpr int CH = kK1Ch;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[NS];
  __shared__ uint32_t stage_tile[NS];
  __shared__ float wsum[NW][CH];

  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t slot = blockIdx.y;
  const uint32_t e = a.sel ? a.sel[slot] : slot;
  const ExpertDesc d = a.table[e];
  const float thr = a.use_threshold ? a.threshold : d.threshold;
  const uint32_t gpc = a.dh / a.group_size;
  const uint32_t code_sz = round_up128(CH * TPB * 4u);
  const uint32_t meta_sz = round_up128(CH * gpc * 2u);
  const uint32_t stage_sz = code_sz + 2 * meta_sz;
  const uint32_t n_tiles = (a.di + CH - 1) / CH;

  auto issue = [&](uint32_t s) {  // thread 0 only
    const uint32_t tile = atomicAdd(&a.tile_ctr[slot], 1u);
    stage_tile[s] = tile;
    if (tile < n_tiles) {
      const uint32_t c0 = tile * CH;
      const uint32_t nc = min((uint32_t)CH, a.di - c0);
      const uint32_t cb = nc * TPB * 4u, mb = nc * gpc * 2u;
      uint8_t *st = smem + s * stage_sz;
      floe_ptx::mbar_arrive_expect_tx(&full[s], cb + 2 * mb);
      floe_ptx::bulk_g2s(st, d.codes + (size_t)c0 * TPB * 4u, cb, &full[s]);
      floe_ptx::bulk_g2s(st + code_sz, d.scales + (size_t)c0 * gpc, mb, &full[s]);
      floe_ptx::bulk_g2s(st + code_sz + meta_sz, d.zeros + (size_t)c0 * gpc, mb, &full[s]);
    }
  };

  if (t == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) floe_ptx::mbar_init(&full[s], 1);
    floe_ptx::fence_barrier_init();
#pragma unroll
    for (int s = 0; s < NS; ++s) issue(s);
  }
  if (a.y_zero && blockIdx.x == 0 && slot == 0)
    for (uint32_t i = t; i < a.dh; i += TPB) a.y_zero[i] = 0.0f;

  float2 xs[8];
  float xsum = 0.0f;
  {
    const float4 *x4 = reinterpret_cast<const float4 *>(a.x) + 4 * t;
    float xr[16];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float4 f = x4[q];
      xr[4 * q] = f.x;
      xr[4 * q + 1] = f.y;
      xr[4 * q + 2] = f.z;
      xr[4 * q + 3] = f.w;
    }
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      xsum += xr[i];
      const int sh = i < 11 ? 2 * i : 2 * (i - 11);
      xr[i] *= __int_as_float((127 - sh) << 23);  // * 4^-i, exact
    }
#pragma unroll
    for (int p = 0; p < 8; ++p) xs[p] = make_float2(xr[2 * p], xr[2 * p + 1]);
  }
  const uint32_t gcol = (16u * t) / a.group_size;
  __syncthreads();

  uint32_t phase = 0;  // bit s = parity of stage s
  for (uint32_t s = 0;; s = (s + 1 == NS) ? 0 : s + 1) {
    const uint32_t tile = stage_tile[s];
    if (tile >= n_tiles) break;
    floe_ptx::mbar_wait(&full[s], (phase >> s) & 1u);
    phase ^= 1u << s;
    const uint8_t *st = smem + s * stage_sz;
    const uint32_t *cw = reinterpret_cast<const uint32_t *>(st);
    const uint16_t *sc = reinterpret_cast<const uint16_t *>(st + code_sz);
    const uint16_t *zr = reinterpret_cast<const uint16_t *>(st + code_sz + meta_sz);
    const uint32_t c0 = tile * CH;
    float part[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      const uint32_t w = cw[j * TPB + t];
      const float sj = h2f(sc[j * gpc + gcol]);
      const float zj = h2f(zr[j * gpc + gcol]);
      part[j] = fmaf(sj, dot16_int2(w, xs), zj * xsum);  // channels past di read 0-padded garbage; masked below
    }
    // transposed butterfly over 16 channels, then fold the two half-warps:
    // lane l (and l^16) ends with the warp sum of channel l&15.
#pragma unroll
    for (int sft = 8; sft >= 1; sft >>= 1) {
      const bool upper = (lane & sft) != 0;
#pragma unroll
      for (int j = 0; j < sft; ++j) {
        const float send = upper ? part[j] : part[j + sft];
        const float keep = upper ? part[j + sft] : part[j];
        part[j] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
      }
    }
    part[0] += __shfl_xor_sync(0xffffffffu, part[0], 16);
    if (lane < CH) wsum[warp][lane] = part[0];
    __syncthreads();  // wsum complete; stage s fully consumed
    if (t == 0) issue(s);
    if (warp == 0) {
      float v = 0.0f;
#pragma unroll
      for (int w = 0; w < NW; ++w) v += wsum[w][lane & (CH - 1)];
      const uint32_t c = c0 + lane;
      k1_emit(a, slot, c, lane < CH && c < a.di, v, thr);
    }
    __syncthreads();  // stage_tile[s] / wsum reuse
  }
  k1_finish(a, gridDim.y);
}

// ---------------------------------------------------------------------------
// K2: y += sum_{kept c} silu(gate_c . x) * v[c] * w_slot * down_c.
//
// Kept entries of all slots are split evenly over CTAs (balance is exact
// regardless of where channels were kept).  Each entry's 4*dh-byte record
// (gate row | down row, f16) arrives with ONE bulk copy.  Thread t owns
// 16-byte chunks t and t+TPB of each half-record (elements [8t, 8t+8) and
// [8(t+TPB), ...)), so shared-memory reads are conflict-free 128-bit loads.
template <int TPB, int NS>
__global__ void __launch_bounds__(TPB, 1) k2_gate_down(const K2Args a) {
  constexpr int NW = TPB / 32;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[NS];
  __shared__ float stage_scale[NS];  // v[c] * routing weight of the entry
  __shared__ float red[2][NW];

  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t rec_bytes = 4u * a.dh;  // == 64 * TPB
  uint32_t total = 0;
  for (uint32_t s = 0; s < a.slots; ++s) total += a.count_final[s];
  const uint32_t begin = (uint32_t)(((uint64_t)total * blockIdx.x) / gridDim.x);
  const uint32_t end = (uint32_t)(((uint64_t)total * (blockIdx.x + 1)) / gridDim.x);
  const uint32_t n = end - begin;

  auto issue = [&](uint32_t i) {  // thread 0 only: entry begin+i -> stage i%NS
    const uint32_t s = i % NS;
    const KeptEntry k = kept_entry(a, begin + i);
    const uint32_t e = a.sel ? a.sel[k.slot] : k.slot;
    stage_scale[s] = k.v * slot_weight(a, k.slot);
    floe_ptx::mbar_arrive_expect_tx(&full[s], rec_bytes);
    floe_ptx::bulk_g2s(smem + s * rec_bytes, a.table[e].records + (size_t)k.c * 2 * a.dh,
                       rec_bytes, &full[s]);
  };
  if (t == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) floe_ptx::mbar_init(&full[s], 1);
    floe_ptx::fence_barrier_init();
    for (uint32_t i = 0; i < n && i < (uint32_t)NS; ++i) issue(i);
  }

  float2 x2[8], y2[8];
  {
    const float4 *xa = reinterpret_cast<const float4 *>(a.x + 8 * t);
    const float4 *xb = reinterpret_cast<const float4 *>(a.x + 8 * (t + TPB));
    const float4 q0 = xa[0], q1 = xa[1], q2 = xb[0], q3 = xb[1];
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
  __syncthreads();

  for (uint32_t i = 0; i < n; ++i) {
    const uint32_t s = i % NS;
    floe_ptx::mbar_wait(&full[s], (i / NS) & 1u);
    const uint4 *rec = reinterpret_cast<const uint4 *>(smem + s * rec_bytes);
    const uint4 g0 = rec[t], g1 = rec[t + TPB];
    const uint4 d0 = rec[2 * TPB + t], d1 = rec[3 * TPB + t];
    const float sc = stage_scale[s];
    float2 acc = make_float2(0.0f, 0.0f);
    {
      const __half2 *h0 = reinterpret_cast<const __half2 *>(&g0);
      const __half2 *h1 = reinterpret_cast<const __half2 *>(&g1);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        acc = __ffma2_rn(__half22float2(h0[q]), x2[q], acc);
        acc = __ffma2_rn(__half22float2(h1[q]), x2[4 + q], acc);
      }
    }
    float gp = acc.x + acc.y;
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) gp += __shfl_xor_sync(0xffffffffu, gp, o);
    if (lane == 0) red[i & 1][warp] = gp;
    __syncthreads();  // red complete; stage s fully read
    if (t == 0 && i + NS < n) issue(i + NS);
    float g = 0.0f;
#pragma unroll
    for (int w = 0; w < NW; ++w) g += red[i & 1][w];
    const float aco = silu_ref(g) * sc;
    const float2 a2 = make_float2(aco, aco);
    const __half2 *e0 = reinterpret_cast<const __half2 *>(&d0);
    const __half2 *e1 = reinterpret_cast<const __half2 *>(&d1);
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      y2[q] = __ffma2_rn(a2, __half22float2(e0[q]), y2[q]);
      y2[4 + q] = __ffma2_rn(a2, __half22float2(e1[q]), y2[4 + q]);
    }
  }
  if (n > 0) {
    float *ya = a.y + 8 * t, *yb = a.y + 8 * (t + TPB);
    red_add_v4(ya, y2[0].x, y2[0].y, y2[1].x, y2[1].y);
    red_add_v4(ya + 4, y2[2].x, y2[2].y, y2[3].x, y2[3].y);
    red_add_v4(yb, y2[4].x, y2[4].y, y2[5].x, y2[5].y);
    red_add_v4(yb + 4, y2[6].x, y2[6].y, y2[7].x, y2[7].y);
  }
}

}  // namespace floe_k
