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
// CTA b owns channels [di*b/G1, di*(b+1)/G1) (contiguous, balanced to one
// channel) and walks them in sub-tiles of 16 channels, each bulk-copied:
// codes 16*dh/4 B, scales and zeros 16*dh/g*2 B.  NS sub-tiles are in flight
// and nothing on the issue path waits on global memory.  Thread t owns
// x[16t, 16t+16) (one code word per channel, all in group 16t/g): x stays in
// registers pre-scaled by 4^-i and the group-affine dequant is folded out of
// the inner loop:  sum_k (c_k s + z) x_k = s * sum_k c_k x_k + z * sum_k x_k.
template <int TPB, int NS>
__global__ void __launch_bounds__(TPB, 2) k1_int2(const K1Args a) {
  constexpr int NW = TPB / 32;
  constexpr int CH = kK1Ch;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[NS];
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
  const uint32_t c_lo = seg_begin(a.di, blockIdx.x, gridDim.x);
  const uint32_t c_hi = seg_begin(a.di, blockIdx.x + 1, gridDim.x);
  const uint32_t n_sub = (c_hi - c_lo + CH - 1) / CH;

  auto issue = [&](uint32_t i) {  // thread 0 only: sub-tile i -> stage i % NS
    const uint32_t s = i % NS;
    const uint32_t c0 = c_lo + i * CH;
    const uint32_t nc = min((uint32_t)CH, c_hi - c0);
    const uint32_t cb = nc * TPB * 4u, mb = nc * gpc * 2u;
    uint8_t *st = smem + s * stage_sz;
    floe_ptx::mbar_arrive_expect_tx(&full[s], cb + 2 * mb);
    floe_ptx::bulk_g2s(st, d.codes + (size_t)c0 * TPB * 4u, cb, &full[s]);
    floe_ptx::bulk_g2s(st + code_sz, d.scales + (size_t)c0 * gpc, mb, &full[s]);
    floe_ptx::bulk_g2s(st + code_sz + meta_sz, d.zeros + (size_t)c0 * gpc, mb, &full[s]);
  };

  if (t == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) floe_ptx::mbar_init(&full[s], 1);
    floe_ptx::fence_barrier_init();
    for (uint32_t i = 0; i < n_sub && i < (uint32_t)NS; ++i) issue(i);
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
  uint32_t running = 0;
  __syncthreads();

  for (uint32_t i = 0; i < n_sub; ++i) {
    const uint32_t s = i % NS;
    floe_ptx::mbar_wait(&full[s], (i / NS) & 1u);
    const uint8_t *st = smem + s * stage_sz;
    const uint32_t *cw = reinterpret_cast<const uint32_t *>(st);
    const uint16_t *sc = reinterpret_cast<const uint16_t *>(st + code_sz);
    const uint16_t *zr = reinterpret_cast<const uint16_t *>(st + code_sz + meta_sz);
    const uint32_t c0 = c_lo + i * CH;
    const uint32_t nc = min((uint32_t)CH, c_hi - c0);
    float part[CH];
#pragma unroll
    for (int j = 0; j < CH; ++j) {
      part[j] = 0.0f;
      if ((uint32_t)j < nc) {  // CTA-uniform
        const uint32_t w = cw[j * TPB + t];
        const float sj = h2f(sc[j * gpc + gcol]);
        const float zj = h2f(zr[j * gpc + gcol]);
        part[j] = fmaf(sj, dot16_int2(w, xs), zj * xsum);
      }
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
    if (t == 0 && i + NS < n_sub) issue(i + NS);
    if (warp == 0) {
      float v = 0.0f;
#pragma unroll
      for (int w = 0; w < NW; ++w) v += wsum[w][lane & (CH - 1)];
      seg_emit(a, slot, c_lo, c0 + lane, lane < nc, v, thr, running);
    }
    __syncthreads();  // wsum reuse
  }
  if (t == 0) a.seg_count[slot * gridDim.x + blockIdx.x] = running;
}

// ---------------------------------------------------------------------------
// K2: y += sum_{kept c} silu(gate_c . x) * v[c] * w_slot * down_c.
//
// Kept entries of all slots are split evenly over CTAs (exact balance however
// the channels fell).  The CTA first resolves its entries' (record address,
// v * routing weight) into shared memory with all threads in parallel, so the
// issuing thread never waits on global memory; then each entry's 4*dh-byte
// record (gate row | down row, f16) arrives with ONE bulk copy into an
// NS-deep ring.  Thread t owns 16-byte chunks t and t+TPB of each half-record
// (elements [8t, 8t+8) and [8(t+TPB), ...)): conflict-free 128-bit smem reads.
constexpr uint32_t kK2Chunk = 256;  // entries resolved per preload round

template <int TPB, int NS>
__global__ void __launch_bounds__(TPB, 1) k2_gate_down(const K2Args a) {
  constexpr int NW = TPB / 32;
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[NS];
  __shared__ float red[2][NW];
  __shared__ const __half *ent_rec[kK2Chunk];
  __shared__ float ent_scale[kK2Chunk];

  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t rec_bytes = 4u * a.dh;  // == 64 * TPB
  const uint32_t nseg = a.slots * a.g1;
  uint32_t *prefix = reinterpret_cast<uint32_t *>(smem + NS * rec_bytes);
  seg_prefix(a.seg_count, nseg, prefix);
  k2_publish(a, prefix);
  const uint32_t total = prefix[nseg];
  const uint32_t begin = (uint32_t)(((uint64_t)total * blockIdx.x) / gridDim.x);
  const uint32_t end = (uint32_t)(((uint64_t)total * (blockIdx.x + 1)) / gridDim.x);

  if (t == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) floe_ptx::mbar_init(&full[s], 1);
    floe_ptx::fence_barrier_init();
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

  uint32_t it = 0;  // global iteration count (ring position / parity)
  for (uint32_t cb = begin; cb < end; cb += kK2Chunk) {
    const uint32_t n = min(kK2Chunk, end - cb);
    __syncthreads();  // previous chunk's ent_* fully consumed
    for (uint32_t q = t; q < n; q += TPB) {
      const KeptEntry k = kept_entry(a, prefix, cb + q);
      const uint32_t e = a.sel ? a.sel[k.slot] : k.slot;
      ent_rec[q] = a.table[e].records + (size_t)k.c * 2 * a.dh;
      ent_scale[q] = k.v * slot_weight(a, k.slot);
      if (a.kept_out) a.kept_out[(size_t)k.slot * a.di + k.slot_pos] = k.c;
    }
    __syncthreads();
    if (t == 0)
      for (uint32_t q = 0; q < n && q < (uint32_t)NS; ++q) {
        const uint32_t s = (it + q) % NS;
        floe_ptx::mbar_arrive_expect_tx(&full[s], rec_bytes);
        floe_ptx::bulk_g2s(smem + s * rec_bytes, ent_rec[q], rec_bytes, &full[s]);
      }
    for (uint32_t q = 0; q < n; ++q, ++it) {
      const uint32_t s = it % NS;
      floe_ptx::mbar_wait(&full[s], (it / NS) & 1u);
      const uint4 *rec = reinterpret_cast<const uint4 *>(smem + s * rec_bytes);
      const uint4 g0 = rec[t], g1 = rec[t + TPB];
      const uint4 d0 = rec[2 * TPB + t], d1 = rec[3 * TPB + t];
      float2 acc = make_float2(0.0f, 0.0f);
      {
        const __half2 *h0 = reinterpret_cast<const __half2 *>(&g0);
        const __half2 *h1 = reinterpret_cast<const __half2 *>(&g1);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc = __ffma2_rn(__half22float2(h0[j]), x2[j], acc);
          acc = __ffma2_rn(__half22float2(h1[j]), x2[4 + j], acc);
        }
      }
      float gp = acc.x + acc.y;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) gp += __shfl_xor_sync(0xffffffffu, gp, o);
      if (lane == 0) red[it & 1][warp] = gp;
      __syncthreads();  // red complete; stage s fully read
      if (t == 0 && q + NS < n) {
        floe_ptx::mbar_arrive_expect_tx(&full[s], rec_bytes);
        floe_ptx::bulk_g2s(smem + s * rec_bytes, ent_rec[q + NS], rec_bytes, &full[s]);
      }
      float g = 0.0f;
#pragma unroll
      for (int w = 0; w < NW; ++w) g += red[it & 1][w];
      const float aco = silu_ref(g) * ent_scale[q];
      const float2 a2 = make_float2(aco, aco);
      const __half2 *e0 = reinterpret_cast<const __half2 *>(&d0);
      const __half2 *e1 = reinterpret_cast<const __half2 *>(&d1);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        y2[j] = __ffma2_rn(a2, __half22float2(e0[j]), y2[j]);
        y2[4 + j] = __ffma2_rn(a2, __half22float2(e1[j]), y2[4 + j]);
      }
    }
  }
  if (end > begin) {
    float *ya = a.y + 8 * t, *yb = a.y + 8 * (t + TPB);
    red_add_v4(ya, y2[0].x, y2[0].y, y2[1].x, y2[1].y);
    red_add_v4(ya + 4, y2[2].x, y2[2].y, y2[3].x, y2[3].y);
    red_add_v4(yb, y2[4].x, y2[4].y, y2[5].x, y2[5].y);
    red_add_v4(yb + 4, y2[6].x, y2[6].y, y2[7].x, y2[7].y);
  }
}

}  // namespace floe_k
