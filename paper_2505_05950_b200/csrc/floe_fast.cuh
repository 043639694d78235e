// floe_fast.cuh -- specialised sm_100a kernels for the Mixtral-shaped path
// (INT2 codes, d_hidden in {2048, 4096}).  All three stream their weights with
// 1-D bulk copies (cp.async.bulk, the TMA engine) into an NS-deep shared
// memory ring tracked by mbarriers, so each SM keeps up to ~190 KB in flight
// without spending registers on loads, and nothing on an issue path waits on
// a dependent global load.
//
// Reference (paths relative to /root/reference/proj/):
//   K1 = qgemv_channels + threshold     core/src/quant.cpp:122-136, core/src/model.cpp:135
//   K2 = gate dot + silu + down         core/src/model.cpp:136-140, core/src/la.cpp:25-31
//   mixing_route = block_forward head   core/src/model.cpp:150-154, 83-93
#pragma once

#include "floe_kernels.cuh"
#include "floe_ptx.cuh"

namespace floe_k {

constexpr int kK1Ch = 16;  // channels per K1 sub-tile

__host__ __device__ constexpr uint32_t round_up128(uint32_t x) { return (x + 127u) & ~127u; }

// Shared-memory bytes of one K1 stage: codes (16 ch x dh/4 B) + interleaved
// scale|zero metadata (16 ch x dh/g x 4 B).
__host__ __device__ constexpr uint32_t k1_stage_bytes(uint32_t dh, uint32_t gpc) {
  return round_up128(kK1Ch * dh / 4u) + round_up128(kK1Ch * gpc * 4u);
}

// f32 fallback for one channel's 64-element span when x holds inf/NaN (the
// fixed-point limbs cannot represent them): the reference's own expression
// float(code)*scale + zero, accumulated in element order.
__device__ __noinline__ float k1_span_f32(const uint32_t *w, const uint32_t *meta, uint32_t g,
                                          const float *xg) {
  float acc = 0.0f;
  for (int i = 0; i < 64; ++i) {
    const uint32_t mz = meta[g >= 64 ? 0 : (uint32_t)i / g];
    const float sc = __half2float(__ushort_as_half((uint16_t)(mz & 0xffffu)));
    const float zr = __half2float(__ushort_as_half((uint16_t)(mz >> 16)));
    const uint32_t code = (w[i / 16] >> (2 * (i % 16))) & 3u;
    acc = fmaf(fmaf((float)code, sc, zr), xg[i], acc);
  }
  return acc;
}

// ---------------------------------------------------------------------------
// K1: v[c] = sum_k deq(up[c,k]) x[k]; keep |v| >= t; compact kept channels.
//
// Integer formulation (exact products, 24-bit input precision):
//   x is scaled once per launch by S = 2^(22-E) (max|x| < 2^E) and rounded to
//   a 23-bit integer X, split into three signed 8-bit limbs.  Per group g of a
//   channel, sum_k c_k X_k is accumulated EXACTLY in int32 with IDP4A (four
//   2-bit codes x four limb bytes per instruction), and
//       v[c] = sum_g  s_g * (sum_k c_k X_k) / S  +  z_g * sum_k x_k ,
//   i.e. the group-affine dequant c*s+z of dequantize_at (quant.cpp:104-109)
//   folded out of the inner loop.  About 1.3 instructions per weight.
//
// Work split: CTA b owns channels [di*b/G1, di*(b+1)/G1) (balanced to one
// channel), walked in sub-tiles of 16 channels, each ONE bulk copy of codes
// plus one of interleaved metadata, NS sub-tiles in flight.  Thread t owns the
// 64-element span (t % SPANS) of dh for every channel (x limbs stay in 48
// registers) and channels q, q+CS, ... of each sub-tile (q = t / SPANS).  The
// CS threads sharing a span split the limb preparation (one code word each)
// and exchange it through shared memory.
template <int SPANS, int GPT, int NS>
__global__ void __launch_bounds__(256, 2) k1_int2(const K1Args a) {
  constexpr int TPB = 256;
  constexpr int NW = TPB / 32;
  constexpr int CH = kK1Ch;
  constexpr int CS = TPB / SPANS;  // channel slots per CTA (threads per span)
  constexpr int CPT = CH / CS;     // channels per thread per sub-tile
  constexpr int WPP = 4 / GPT;     // code words per group part
  static_assert(SPANS == 64 || SPANS == 32, "dh must be 4096 or 2048");
  constexpr uint32_t DH = SPANS * 64;
  constexpr uint32_t ROW = DH / 4;  // code bytes per channel
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[NS];
  __shared__ float wsum[NW][CPT];
  __shared__ float red_max[NW];
  __shared__ __align__(16) uint32_t limb_s[SPANS][4][12];  // [span][word][limb*4 + m], read as uint4
  __shared__ float xsum_s[SPANS][4];

  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t span = t % SPANS, q = t / SPANS;
  const uint32_t slot = blockIdx.y;
  const uint32_t c_lo = seg_begin(a.di, blockIdx.x, gridDim.x);
  const uint32_t c_hi = seg_begin(a.di, blockIdx.x + 1, gridDim.x);
  const uint32_t n_sub = (c_hi - c_lo + CH - 1) / CH;
  const uint32_t gpc = DH / a.group_size;
  const uint32_t code_sz = round_up128(CH * ROW);
  const uint32_t stage_sz = code_sz + round_up128(CH * gpc * 4u);

  const uint32_t e = a.sel ? a.sel[slot] : slot;
  const ExpertDesc d = a.table[e];
  const float thr = a.use_threshold ? a.threshold : d.threshold;

  if (t == 0) {
#pragma unroll
    for (int s = 0; s < NS; ++s) floe_ptx::mbar_init(&full[s], 1);
    floe_ptx::fence_barrier_init();
    for (uint32_t i = 0; i < n_sub && i < (uint32_t)NS; ++i) {
      const uint32_t c0 = c_lo + i * CH, nc = min((uint32_t)CH, c_hi - c0);
      floe_ptx::mbar_arrive_expect_tx(&full[i], nc * (ROW + gpc * 4u));
      floe_ptx::bulk_g2s(smem + i * stage_sz, d.codes + (size_t)c0 * ROW, nc * ROW, &full[i]);
      floe_ptx::bulk_g2s(smem + i * stage_sz + code_sz, d.meta + (size_t)c0 * gpc, nc * gpc * 4u,
                         &full[i]);
    }
  }
  if (a.y_zero && blockIdx.x == 0 && slot == 0)
    for (uint32_t i = t; i < a.dh; i += TPB) a.y_zero[i] = 0.0f;

  // ---- x: word q of this span (16 elements) -> block max|x| -> limbs ----
  const bool word_owner = q < 4;
  float xw[16];
  {
    const float4 *x4 = reinterpret_cast<const float4 *>(a.x + 64 * span + 16 * (q & 3));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 f = x4[i];
      xw[4 * i] = f.x;
      xw[4 * i + 1] = f.y;
      xw[4 * i + 2] = f.z;
      xw[4 * i + 3] = f.w;
    }
  }
  float m = 0.0f;
  bool finite = true;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    m = fmaxf(m, fabsf(xw[i]));
    finite = finite && isfinite(xw[i]);
  }
#pragma unroll
  for (int o = 16; o >= 1; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
  const bool warp_finite = __all_sync(0xffffffffu, finite);
  if (lane == 0) red_max[warp] = warp_finite ? m : -1.0f;
  __syncthreads();
  bool all_finite = true;
  m = 0.0f;
#pragma unroll
  for (int w = 0; w < NW; ++w) {
    all_finite = all_finite && red_max[w] >= 0.0f;
    m = fmaxf(m, red_max[w]);
  }
  int ex = 0;
  frexpf(m, &ex);  // m < 2^ex
  const float S = (m > 0.0f && all_finite) ? __int_as_float((127 + 22 - ex) << 23) : 1.0f;
  const float invS = (m > 0.0f && all_finite) ? __int_as_float((127 - 22 + ex) << 23) : 1.0f;
  if (word_owner) {
    // limb l of elements mm + 4b (b = 0..3) in byte b: the byte order of
    // (w >> 2mm) & 0x03030303 on this code word.
    float s16 = 0.0f;
#pragma unroll
    for (int mm = 0; mm < 4; ++mm) {
      uint32_t l0 = 0, l1 = 0, l2 = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const float xf = xw[mm + 4 * b];
        const int X = all_finite ? __float2int_rn(xf * S) : 0;
        const int X0 = ((X + 128) & 255) - 128;
        const int R = (X - X0) >> 8;
        const int X1 = ((R + 128) & 255) - 128;
        const int X2 = (R - X1) >> 8;
        l0 |= (uint32_t)(X0 & 255) << (8 * b);
        l1 |= (uint32_t)(X1 & 255) << (8 * b);
        l2 |= (uint32_t)(X2 & 255) << (8 * b);
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
  const uint32_t g0 = (64u * span) / a.group_size;  // first group of this span

  uint32_t running = 0;
  for (uint32_t it = 0; it < n_sub; ++it) {
    const uint32_t s = it % NS;
    floe_ptx::mbar_wait(&full[s], (it / NS) & 1u);
    const uint8_t *st = smem + s * stage_sz;
    const uint32_t c0 = c_lo + it * CH;
    const uint32_t nc = min((uint32_t)CH, c_hi - c0);
    float part[CPT];
#pragma unroll
    for (int r = 0; r < CPT; ++r) {
      const uint32_t j = q + CS * r;
      float acc = 0.0f;
      if (j < nc) {
        const uint4 w4 = *reinterpret_cast<const uint4 *>(st + j * ROW + 16 * span);
        const uint32_t *meta = reinterpret_cast<const uint32_t *>(st + code_sz) + j * gpc + g0;
        if (all_finite) {
          const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
          for (int p = 0; p < GPT; ++p) {
            int a0 = 0, a1 = 0, a2 = 0;
#pragma unroll
            for (int i = p * WPP; i < (p + 1) * WPP; ++i) {
#pragma unroll
              for (int mm = 0; mm < 4; ++mm) {
                const int cb = (int)((wv[i] >> (2 * mm)) & 0x03030303u);
                a0 = __dp4a(cb, (int)lw[i][mm], a0);
                a1 = __dp4a(cb, (int)lw[i][4 + mm], a1);
                a2 = __dp4a(cb, (int)lw[i][8 + mm], a2);
              }
            }
            const int T = a2 * 65536 + a1 * 256 + a0;
            const uint32_t mz = meta[p];
            const float sc = __half2float(__ushort_as_half((uint16_t)(mz & 0xffffu)));
            const float zr = __half2float(__ushort_as_half((uint16_t)(mz >> 16)));
            acc = fmaf(sc * invS, (float)T, fmaf(zr, xpart[p], acc));
          }
        } else {
          const uint32_t wv[4] = {w4.x, w4.y, w4.z, w4.w};
          acc = k1_span_f32(wv, meta, a.group_size, a.x + 64 * span);
        }
      }
      part[r] = acc;
    }
    // transposed butterfly: CPT values -> lane holds channel r(lane) summed
    // over the lanes of its warp; lanes with (lane & (32/CPT - 1)) == 0 write.
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
    if ((lane & (32 / CPT - 1)) == 0) wsum[warp][lane / (32 / CPT)] = part[0];
    __syncthreads();  // wsum complete; stage s fully consumed
    if (t == 0 && it + NS < n_sub) {
      const uint32_t c1 = c_lo + (it + NS) * CH, n1 = min((uint32_t)CH, c_hi - c1);
      floe_ptx::mbar_arrive_expect_tx(&full[s], n1 * (ROW + gpc * 4u));
      floe_ptx::bulk_g2s(smem + s * stage_sz, d.codes + (size_t)c1 * ROW, n1 * ROW, &full[s]);
      floe_ptx::bulk_g2s(smem + s * stage_sz + code_sz, d.meta + (size_t)c1 * gpc,
                         n1 * gpc * 4u, &full[s]);
    }
    if (warp == 0) {
      // channel j = q + CS*r is reduced by warps q*SPANS/32 .. +SPANS/32-1
      const uint32_t j = lane;
      float v = 0.0f;
      if (j < (uint32_t)CH) {
        const uint32_t qq = j % CS, rr = j / CS;
#pragma unroll
        for (int w = 0; w < SPANS / 32; ++w) v += wsum[qq * (SPANS / 32) + w][rr];
      }
      seg_emit(a, slot, c_lo, c0 + j, j < nc, v, thr, running);
    }
    __syncthreads();  // wsum reuse
  }
  if (t == 0) a.seg_count[slot * gridDim.x + blockIdx.x] = running;
}

// ---------------------------------------------------------------------------
// K2: y += sum_{kept c} silu(gate_c . x) * v[c] * w_slot * down_c.
//
// One CTA per SM.  Kept entries of all slots are split evenly over CTAs
// (exact balance however the channels fell).  The per-slot record base
// (sel -> table -> records) and routing weight are resolved once per CTA in
// parallel with the segment scan; then all entries' (record address, v * w)
// are resolved in one parallel round, so the issuing thread never waits on
// global memory.  Each entry's 4*dh-byte record (gate row | down row, f16)
// is ONE bulk copy into an NS-deep ring (NS*16 KB in flight per SM), and R
// records are consumed per block barrier (R independent dot chains, one
// transposed warp reduction).  Thread t owns 16-byte chunks t and t+TPB of
// each half-record (elements [8t, 8t+8) and [8(t+TPB), ...)): conflict-free
// 128-bit smem reads, y kept in registers.
constexpr uint32_t kK2Chunk = 512;  // entries resolved per preload round (multiple of R)

template <int TPB, int NS, int R>
__global__ void __launch_bounds__(TPB, 1) k2_gate_down(const K2Args a) {
  constexpr int NW = TPB / 32;
  static_assert(NS % R == 0 && (R == 1 || R == 2 || R == 4), "ring holds whole batches");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[NS];
  __shared__ float red[2][NW][R];
  __shared__ const __half *ent_rec[kK2Chunk];
  __shared__ float ent_scale[kK2Chunk];
  __shared__ const __half *slot_rec[kMaxSlots];
  __shared__ float slot_w[kMaxSlots];

  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t rec_bytes = 4u * a.dh;  // == 64 * TPB
  const uint32_t nseg = a.slots * a.g1;
  if (t < a.slots) {
    const uint32_t e = a.sel ? a.sel[t] : t;
    slot_rec[t] = a.table[e].records;
    slot_w[t] = slot_weight(a, t);
  }
  uint32_t *prefix = reinterpret_cast<uint32_t *>(smem + NS * rec_bytes);
  seg_prefix(a.seg_count, nseg, prefix);  // contains __syncthreads
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

  uint32_t it = 0;  // entries consumed so far (ring position)
  uint32_t batch = 0;
  for (uint32_t cb = begin; cb < end; cb += kK2Chunk) {
    const uint32_t n = min(kK2Chunk, end - cb);
    __syncthreads();  // previous chunk's ent_* consumed; slot_* visible
    for (uint32_t qq = t; qq < n; qq += TPB) {
      const uint32_t p = cb + qq;
      const uint32_t idx = seg_find(prefix, nseg, p);
      const uint32_t slot = idx / a.g1, b = idx % a.g1;
      const size_t o = (size_t)slot * a.di + seg_begin(a.di, b, a.g1) + (p - prefix[idx]);
      const uint32_t c = a.kept_idx[o];
      ent_rec[qq] = slot_rec[slot] + (size_t)c * 2 * a.dh;
      ent_scale[qq] = a.kept_v[o] * slot_w[slot];
      if (a.kept_out) a.kept_out[(size_t)slot * a.di + (p - prefix[slot * a.g1])] = c;
    }
    __syncthreads();
    // `it` counts stage uses in order across chunks (every chunk but the
    // last holds a whole number of batches), so stage = use % NS and the
    // mbarrier parity = (use / NS) & 1 stay consistent.
    if (t == 0)
      for (uint32_t k = 0; k < n && k < (uint32_t)NS; ++k) {
        const uint32_t s = (it + k) % NS;
        floe_ptx::mbar_arrive_expect_tx(&full[s], rec_bytes);
        floe_ptx::bulk_g2s(smem + s * rec_bytes, ent_rec[k], rec_bytes, &full[s]);
      }
    for (uint32_t q0 = 0; q0 < n; q0 += R, ++batch) {
      uint4 gv[R][2], dv[R][2];
      float gp[R];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const uint32_t qq = q0 + r;
        gp[r] = 0.0f;
        if (qq < n) {
          const uint32_t s = (it + r) % NS;
          floe_ptx::mbar_wait(&full[s], ((it + r) / NS) & 1u);
          const uint4 *rec = reinterpret_cast<const uint4 *>(smem + s * rec_bytes);
          gv[r][0] = rec[t];
          gv[r][1] = rec[t + TPB];
          dv[r][0] = rec[2 * TPB + t];
          dv[r][1] = rec[3 * TPB + t];
          const __half2 *h0 = reinterpret_cast<const __half2 *>(&gv[r][0]);
          const __half2 *h1 = reinterpret_cast<const __half2 *>(&gv[r][1]);
          float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            acc = __ffma2_rn(__half22float2(h0[j]), x2[j], acc);
            acc = __ffma2_rn(__half22float2(h1[j]), x2[4 + j], acc);
          }
          gp[r] = acc.x + acc.y;
        } else {
          dv[r][0] = dv[r][1] = make_uint4(0, 0, 0, 0);
        }
      }
      // transposed warp reduction of R values
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
      if ((lane & (32 / R - 1)) == 0) red[batch & 1][warp][lane / (32 / R)] = gp[0];
      __syncthreads();  // red complete; the batch's stages fully read
      if (t == 0)
        for (int r = 0; r < R; ++r) {
          const uint32_t nq = q0 + r + NS;
          if (nq < n) {
            const uint32_t s = (it + r) % NS;
            floe_ptx::mbar_arrive_expect_tx(&full[s], rec_bytes);
            floe_ptx::bulk_g2s(smem + s * rec_bytes, ent_rec[nq], rec_bytes, &full[s]);
          }
        }
#pragma unroll
      for (int r = 0; r < R; ++r) {
        if (q0 + r >= n) break;
        float g = 0.0f;
#pragma unroll
        for (int w = 0; w < NW; ++w) g += red[batch & 1][w][r];
        const float aco = silu_ref(g) * ent_scale[q0 + r];
        const float2 a2 = make_float2(aco, aco);
        const __half2 *e0 = reinterpret_cast<const __half2 *>(&dv[r][0]);
        const __half2 *e1 = reinterpret_cast<const __half2 *>(&dv[r][1]);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          y2[j] = __ffma2_rn(a2, __half22float2(e0[j]), y2[j]);
          y2[4 + j] = __ffma2_rn(a2, __half22float2(e1[j]), y2[4 + j]);
        }
      }
      it += R;
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

// ---------------------------------------------------------------------------
// Block head: u = h + mixing.h; y = u; logits = router.u; top-k; softmax.
//
// One CTA per SM; CTA b owns rows [dh*b/G, dh*(b+1)/G), streamed in chunks
// of RPC <= 8 rows (one row per warp) by bulk copy through an NS-deep ring;
// h is bulk-copied once.  Each warp finishes its own row (u, y, and the
// row's contribution to the router logits) -- one block barrier per chunk,
// only to release the stage.  The last CTA (done counter, reset in-kernel)
// sums the per-CTA partial logits in a fixed order and routes.
// Deterministic: no float atomics.
constexpr uint32_t kMaxRowsPerCta = 48;
constexpr uint32_t kMixChunkBytes = 96 * 1024;  // bytes of rows per stage (cap)

__host__ __device__ inline uint32_t mix_rows_per_chunk(uint32_t row_bytes) {
  uint32_t r = kMixChunkBytes / row_bytes;
  return r > 8 ? 8 : (r < 1 ? 1 : r);
}

template <typename T, int NS>
__global__ void __launch_bounds__(256, 1) mixing_route_bulk(const MixArgs a) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[NS + 1];  // [NS] = h
  __shared__ float plw[8][32];       // per-warp partial logits
  __shared__ float logits[32];
  __shared__ float rs[32 * kMaxRowsPerCta];  // router[e][this CTA's rows]
  __shared__ bool last;
  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t row_bytes = a.dh * (uint32_t)sizeof(T);
  const uint32_t rpc = mix_rows_per_chunk(row_bytes);
  const uint32_t r_lo = seg_begin(a.dh, blockIdx.x, gridDim.x);
  const uint32_t r_hi = seg_begin(a.dh, blockIdx.x + 1, gridDim.x);
  const uint32_t n_chunks = (r_hi - r_lo + rpc - 1) / rpc;
  const uint32_t stage_sz = round_up128(rpc * row_bytes);
  float *hs = reinterpret_cast<float *>(smem + NS * stage_sz);
  const T *m = static_cast<const T *>(a.m);

  if (t == 0) {
#pragma unroll
    for (int s = 0; s <= NS; ++s) floe_ptx::mbar_init(&full[s], 1);
    floe_ptx::fence_barrier_init();
    floe_ptx::mbar_arrive_expect_tx(&full[NS], 4u * a.dh);
    floe_ptx::bulk_g2s(hs, a.h, 4u * a.dh, &full[NS]);
    for (uint32_t i = 0; i < n_chunks && i < (uint32_t)NS; ++i) {
      const uint32_t r0 = r_lo + i * rpc, nr = min(rpc, r_hi - r0);
      floe_ptx::mbar_arrive_expect_tx(&full[i], nr * row_bytes);
      floe_ptx::bulk_g2s(smem + i * stage_sz, m + (size_t)r0 * a.dh, nr * row_bytes, &full[i]);
    }
  }
  // router slice for this CTA's rows, fetched while the bulk copies fly
  for (uint32_t i = t; i < a.E * kMaxRowsPerCta; i += 256) {
    const uint32_t e = i / kMaxRowsPerCta, lr = i % kMaxRowsPerCta;
    if (r_lo + lr < r_hi) rs[i] = a.router[(size_t)e * a.dh + r_lo + lr];
  }
  __syncthreads();
  floe_ptx::mbar_wait(&full[NS], 0);

  constexpr uint32_t EPL = 16 / sizeof(T);  // elements per 128-bit smem load
  float pl = 0.0f;                          // lane e < E: this warp's partial logit e
  for (uint32_t ci = 0; ci < n_chunks; ++ci) {
    const uint32_t s = ci % NS;
    const uint32_t r0 = r_lo + ci * rpc, nr = min(rpc, r_hi - r0);
    if (warp < nr) {
      floe_ptx::mbar_wait(&full[s], (ci / NS) & 1u);
      const T *rowp = reinterpret_cast<const T *>(smem + s * stage_sz) + (size_t)warp * a.dh;
      float acc0 = 0.0f, acc1 = 0.0f;
      for (uint32_t k = lane * EPL; k < a.dh; k += 32 * EPL) {
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
      const uint32_t row = r0 + warp;
      const float uu = hs[row] + 1.0f * acc;  // drift_scale = 1 (model.cpp:151-152)
      if (lane == 0) {
        a.u[row] = uu;
        a.y_init[row] = uu;
        if (a.u_trace) a.u_trace[row] = uu;
      }
      if (lane < a.E) {
        const uint32_t lr = row - r_lo;
        const float w = lr < kMaxRowsPerCta ? rs[lane * kMaxRowsPerCta + lr]
                                            : a.router[(size_t)lane * a.dh + row];
        pl = fmaf(w, uu, pl);
      }
    }
    __syncthreads();  // stage s consumed by every warp
    if (t == 0 && ci + NS < n_chunks) {
      const uint32_t r1 = r_lo + (ci + NS) * rpc, n1 = min(rpc, r_hi - r1);
      floe_ptx::mbar_arrive_expect_tx(&full[s], n1 * row_bytes);
      floe_ptx::bulk_g2s(smem + s * stage_sz, m + (size_t)r1 * a.dh, n1 * row_bytes, &full[s]);
    }
  }
  plw[warp][lane] = pl;
  __syncthreads();
  if (t < a.E) {
    float sacc = 0.0f;
#pragma unroll
    for (int w = 0; w < 8; ++w) sacc += plw[w][t];
    a.partial[blockIdx.x * a.E + t] = sacc;
  }
  __threadfence();
  __syncthreads();
  if (t == 0) last = atomicAdd(a.done, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  for (uint32_t e = warp; e < a.E; e += 8) {
    float sacc = 0.0f;
    for (uint32_t b = lane; b < gridDim.x; b += 32) sacc += __ldcg(&a.partial[b * a.E + e]);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
    if (lane == 0) logits[e] = sacc;
  }
  __syncthreads();
  if (t == 0) {
    *a.done = 0;
    route_finish(logits, a.E, a.k, a.sel, a.weights, a.sel_trace, a.w_trace);
  }
}

}  // namespace floe_k
