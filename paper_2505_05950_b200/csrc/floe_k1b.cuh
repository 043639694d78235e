// floe_k1b.cuh -- batched up projection for small batches (config 4: a routed
// expert sees ~4 of 16 decode tokens): qgemv_channels (core/src/quant.cpp:
// 122-136) for up to 8 tokens per pass, straight from the tile-fragment layout
// (floe_v2.cuh) with exact integer IMMA, every SM busy.
//
// Same arithmetic as floe_tc::k1_batched and the batch-1 K1 of the fused
// kernel: x_t scaled by S_t = 2^(22-e_t) to X = L0 + 256 L1 + 65536 L2
// (signed 8-bit limbs); per 64-element span the exact integer sums
// sum code * L_l on mma.sync m16n8k32 s8 (A = 16 channels x 32 codes, B = 32
// positions x 8 tokens of ONE limb), recombined exactly in s32, then
//   acc1 += scale * float(isum),  acc2 += zero * sum_span x,
//   v = invS * acc1 + acc2.
//
// Why not tcgen05 here: at <= 8 tokens the product is tiny (N = 24 limb
// columns) and the kernel is bound by moving the 2-bit codes.  The tcgen05
// path must expand every code to a byte in shared memory for the A operand
// (8 KB of stores and a proxy fence per span of 128 channels); IMMA takes the
// A fragments straight from the tile layout in registers (one LDS.128 per two
// spans, shift+mask per code word), so the codes cross shared memory once, as
// bulk copies.  floe_tc::k1_batched stays the path for more tokens.
//
// Work split: the grid is one CTA per SM over contiguous tile ranges; a tile
// (16 channels, 5 DH bytes) is cut into 8 items along K (DH/1024 span pairs
// each); CTA b takes the contiguous item range [NI b / G, NI (b+1) / G) of all
// NI = 8 tiles items (balanced to one item: whole tiles per CTA left 8 CTAs
// with 7 tiles and 140 with 6).  A tile's items arrive by one bulk copy (two
// for a tile cut by the CTA boundary) into a 4-slot ring (small copies are
// expensive: per-item 2.5 KB copies ran at 0.9 TB/s), go round-robin to 16
// consumer warps (balanced per SM sub-partition), and a channel's item
// partials are added in fixed order at the end.  A tile cut between two CTAs
// gets both halves by atomicAdd onto zeros (limbs() zeroes those channels):
// 0 + a + b == 0 + b + a, so the result is deterministic.
#pragma once

#include "floe_v2.cuh"

namespace floe_k1b {

constexpr int kTok = 8;                      // tokens per pass (the IMMA N)
constexpr int kWarps = 16;                   // consumer warps
constexpr int kThreads = 32 * (kWarps + 1);  // + producer warp
constexpr int kSlots = 4;                    // tile ring
constexpr int kItems = 8;                    // items per tile (K eighths)
constexpr int kMaxTokens = 64;               // passes of kTok tokens up to here
constexpr int kDefaultMax = 16;              // the library's default switch to floe_tc (FLOE_K1_IMMA_MAX)

// x limbs: [span][limb][lane] uint4 (B fragments of both IMMAs of the span)
__host__ __device__ constexpr uint32_t xt_bytes(uint32_t dh) { return (dh / 64u) * 3u * 512u; }
__host__ __device__ constexpr uint32_t xs_bytes(uint32_t dh) { return (dh / 64u) * kTok * 4u; }

// local tiles of one CTA: its items span at most ceil(NI / G) / 8 + 2 tiles
__host__ __device__ inline uint32_t tiles_per_cta(uint32_t di, uint32_t G) {
  const uint64_t NI = (uint64_t)((di + 15u) / 16u) * kItems;
  return (uint32_t)(((NI + G - 1) / G + kItems - 1) / kItems) + 1u;
}

struct Smem {
  uint32_t xt, xs, ring, part, total;
};
__host__ __device__ inline Smem smem_layout(uint32_t dh, uint32_t tiles_per_cta) {
  Smem L;
  uint32_t o = 0;
  L.xt = o;   o += xt_bytes(dh);
  L.xs = o;   o += xs_bytes(dh);
  L.ring = o; o += kSlots * floe_v2::tile_bytes(dh);
  L.part = o; o += tiles_per_cta * kItems * 16u * kTok * 4u;
  L.total = o;
  return L;
}

// Limb tables of one pass (tokens x[0..B), B <= 8; columns past B are zero).
// Per token first S = 2^(22-e) (max|x| < 2^e) and 1/S (NaN for a non-finite
// token), as floe_tc::token_scale computes them; every block computes them
// (B * dh floats from L2) so that one launch prepares the pass.
// Word m, byte b of xt[span][l][lane = 4n + tig] is limb l of
// x_n[64 span + 16 tig + 4 b + m]: the k order in which the A fragments come
// out of a code word (code 16 tig + 4 b + m sits in bits 8b + 2m).  xs[span][n]
// = the span's f32 sum (the zero term), reduced as in floe_tc::token_limbs.
// Also zeroes v[0..B) on the channels of tiles that k1's grid of G CTAs cuts.
template <int DH>
__global__ void __launch_bounds__(256) limbs(const float *__restrict__ x, uint32_t B,
                                             float *__restrict__ invS, uint8_t *__restrict__ xt,
                                             float *__restrict__ xs, float *__restrict__ v,
                                             uint32_t di, uint32_t G) {
  const uint32_t span = blockIdx.x;
  floe_v2::pdl_launch_dependents();  // k1 starts streaming its tiles meanwhile
  __shared__ float S_s[kTok];
  {
    const uint64_t NI = (uint64_t)((di + 15u) / 16u) * kItems;
    for (uint32_t cta = 1u + blockIdx.x; cta < G; cta += gridDim.x) {
      const uint64_t ilo = NI * cta / G;
      if (ilo % kItems == 0) continue;
      const uint32_t c0 = (uint32_t)(ilo / kItems) * 16u;
      for (uint32_t i = threadIdx.x; i < 16u * B; i += blockDim.x)
        if (c0 + i % 16u < di) v[(size_t)(i / 16u) * di + c0 + i % 16u] = 0.0f;
    }
  }
  const uint32_t n = threadIdx.x >> 5, ln = threadIdx.x & 31u;  // one warp per token
  if (n < B) {
    const float4 *x4 = reinterpret_cast<const float4 *>(x + (size_t)n * DH);
    float mx = 0.0f;
    int nf = 0;
#pragma unroll 16
    for (uint32_t k = ln; k < DH / 4u; k += 32u) {
      const float4 q = x4[k];
      mx = fmaxf(fmaxf(mx, fmaxf(fabsf(q.x), fabsf(q.y))), fmaxf(fabsf(q.z), fabsf(q.w)));
      nf |= !isfinite(q.x) | !isfinite(q.y) | !isfinite(q.z) | !isfinite(q.w);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      nf |= __shfl_xor_sync(0xffffffffu, nf, o);
    }
    if (ln == 0) {
      int ex = 0;
      frexpf(mx, &ex);  // mx < 2^ex
      const bool scaled = mx > 0.0f;
      S_s[n] = scaled ? __int_as_float((127 + 22 - ex) << 23) : 1.0f;
      if (span == 0)
        invS[n] = nf ? __int_as_float(0x7fc00000) : (scaled ? __int_as_float((127 - 22 + ex) << 23) : 1.0f);
    }
  }
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kTok * 64u; i += blockDim.x) {
    const uint32_t tn = i / 64u, e = i % 64u;
    int X = 0;
    if (tn < B) {
      const float xv = x[(size_t)tn * DH + 64u * span + e];
      X = isfinite(xv) ? __float2int_rn(xv * S_s[tn]) : 0;
    }
    const int l0 = ((X + 128) & 255) - 128;
    const int r1 = (X - l0) >> 8;
    const int l1 = ((r1 + 128) & 255) - 128;
    const int l2 = (r1 - l1) >> 8;
    const uint32_t tig = e >> 4, b = (e >> 2) & 3u, m = e & 3u;
    const uint32_t off = (4u * tn + tig) * 16u + 4u * m + b;
    uint8_t *o = xt + (size_t)span * 3u * 512u;
    o[off] = (uint8_t)(l0 & 255);
    o[512u + off] = (uint8_t)(l1 & 255);
    o[1024u + off] = (uint8_t)(l2 & 255);
  }
  if (n < (uint32_t)kTok) {
    float sum = 0.0f;
    if (n < B) {
      const float2 v2 = *reinterpret_cast<const float2 *>(x + (size_t)n * DH + 64u * span + 2u * ln);
      sum = v2.x + v2.y;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (ln == 0) xs[span * kTok + n] = sum;
  }
}

// test_wait spin: mbarrier.try_wait lowers to a suspend (NANOSLEEP.SYNCS of up
// to 20 us) that wakes late when the phase completes (ncu: 20 us per call)
__device__ __forceinline__ void spin(uint64_t *bar, uint32_t parity, uint32_t tag) {
  if (floe_ptx::mbar_test_wait(bar, parity)) return;
  const unsigned long long t0 = floe_ptx::now_ns();
  for (uint32_t it = 1;; ++it) {
    if (floe_ptx::mbar_test_wait(bar, parity)) return;
    if ((it & 1023u) == 0 && floe_ptx::now_ns() - t0 > floe_ptx::kWatchdogNs)
      floe_ptx::watchdog_fire("mbarrier", tag, parity);
  }
}

struct Args {
  const uint32_t *tiles;  // the expert's tile-fragment layout
  uint32_t di, B;         // B <= 8 tokens in this pass
  const uint8_t *xt;      // limbs() output
  const float *xs;
  const float *invS;      // [B] 1/S_t (NaN for a non-finite token)
  float *v;               // [B][di]
  unsigned long long *trace;  // nullable [G][8] %globaltimer marks (diagnostics, FLOE_K1B_TRACE)
};
__device__ __forceinline__ void mark(const Args &a, int k) {
  if (a.trace) a.trace[blockIdx.x * 8u + (uint32_t)k] = floe_ptx::now_ns();
}

template <int DH>
__global__ void __launch_bounds__(kThreads, 1) k1(const Args a) {
  constexpr uint32_t PQ = DH / 1024u;  // span pairs per item
  constexpr uint32_t TB = floe_v2::tile_bytes(DH);
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kSlots], empty[kSlots], xbar;
  const uint32_t t = threadIdx.x, warp = t >> 5, lane = t & 31u;
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const uint64_t NI = (uint64_t)((a.di + 15u) / 16u) * kItems;
  const uint32_t ilo = (uint32_t)(NI * b / G), ihi = (uint32_t)(NI * (b + 1) / G);
  const uint32_t items = ihi - ilo, tlo = ilo / kItems;
  const uint32_t ntl = items ? (ihi - 1u) / kItems - tlo + 1u : 0u;
  const Smem L = smem_layout(DH, tiles_per_cta(a.di, G));
  // items [q0, q1) of local tile j belong to this CTA
  auto qlo = [&](uint32_t j) { return j == 0 ? ilo - tlo * kItems : 0u; };
  auto qhi = [&](uint32_t j) { return min((uint32_t)kItems, ihi - (tlo + j) * kItems); };
  if (t == 0) {
    for (int s = 0; s < kSlots; ++s) {
      floe_ptx::mbar_init(&full[s], 1);
      floe_ptx::mbar_init(&empty[s], kItems);  // one arrival per item
    }
    floe_ptx::mbar_init(&xbar, 1);
    floe_ptx::fence_barrier_init();
  }
  __syncthreads();
  if (t == 0) mark(a, 0);

  if (warp == kWarps) {
    // ============================== producer ==============================
    if (lane == 0) {
      // (launched with programmatic stream serialization after limbs(): the
      // first tiles stream before griddepcontrol.wait, the limb tables after)
      auto issue_tile = [&](uint32_t j) {
        const uint32_t s = j % kSlots;
        const uint8_t *src = reinterpret_cast<const uint8_t *>(a.tiles) + (size_t)(tlo + j) * TB;
        uint8_t *dst = smem + L.ring + s * TB;
        const uint32_t q0 = qlo(j), q1 = qhi(j);
        if (q0 == 0 && q1 == (uint32_t)kItems) {
          floe_ptx::mbar_arrive_expect_tx(&full[s], TB);
          floe_ptx::bulk_g2s(dst, src, TB, &full[s]);
        } else {  // codes and meta of items [q0, q1)
          floe_ptx::mbar_arrive_expect_tx(&full[s], (q1 - q0) * PQ * 640u);
          floe_ptx::bulk_g2s(dst + q0 * PQ * 512u, src + q0 * PQ * 512u, (q1 - q0) * PQ * 512u, &full[s]);
          floe_ptx::bulk_g2s(dst + 4u * DH + q0 * PQ * 128u, src + 4u * DH + q0 * PQ * 128u,
                             (q1 - q0) * PQ * 128u, &full[s]);
        }
      };
      const uint32_t first = min(ntl, (uint32_t)kSlots);
      for (uint32_t j = 0; j < first; ++j) issue_tile(j);
      floe_v2::pdl_wait();  // limbs() done: its tables, invS and the zeroed v
      floe_ptx::mbar_arrive_expect_tx(&xbar, xt_bytes(DH) + xs_bytes(DH));
      floe_ptx::bulk_g2s(smem + L.xt, a.xt, xt_bytes(DH), &xbar);
      floe_ptx::bulk_g2s(smem + L.xs, a.xs, xs_bytes(DH), &xbar);
      for (uint32_t j = first; j < ntl; ++j) {
        spin(&empty[j % kSlots], ((j / kSlots) - 1u) & 1u, (1u << 28) | j);
        issue_tile(j);
      }
    }
    return;
  }

  // ============================== consumers ===============================
  const uint32_t g = lane >> 2, tig = lane & 3u;
  const uint4 *xt4 = reinterpret_cast<const uint4 *>(smem + L.xt);
  const float *xs_s = reinterpret_cast<const float *>(smem + L.xs);
  float *part = reinterpret_cast<float *>(smem + L.part);
  floe_v2::pdl_wait();
  const float inv0 = 2u * tig < a.B ? a.invS[2u * tig] : 0.0f;
  const float inv1 = 2u * tig + 1u < a.B ? a.invS[2u * tig + 1u] : 0.0f;
  spin(&xbar, 0, 2u << 28);
  if (t == 0) mark(a, 1);
  constexpr uint32_t M = 0x03030303u;
  for (uint32_t k = warp; k < items; k += kWarps) {
    const uint32_t i = ilo + k, j = i / kItems - tlo, s = j % kSlots, q = i % kItems;
    spin(&full[s], (j / kSlots) & 1u, (3u << 28) | k);
    const uint8_t *st = smem + L.ring + s * TB;
    const uint4 *cw = reinterpret_cast<const uint4 *>(st + q * PQ * 512u) + lane;         // [pair][lane]
    const uint4 *mw = reinterpret_cast<const uint4 *>(st + 4u * DH + q * PQ * 128u) + g;  // [pair][g]
    // (row g, token 2tig), (g, 2tig+1), (g+8, 2tig), (g+8, 2tig+1)
    float acc1[4] = {0.0f, 0.0f, 0.0f, 0.0f}, acc2[4] = {0.0f, 0.0f, 0.0f, 0.0f};
    auto span_step = [&](uint32_t wa, uint32_t wb, uint32_t mg, uint32_t mg8, uint32_t sp) {
      const uint32_t a0 = wa & M, a1 = wb & M, a2 = (wa >> 2) & M, a3 = (wb >> 2) & M;
      const uint32_t a4 = (wa >> 4) & M, a5 = (wb >> 4) & M, a6 = (wa >> 6) & M, a7 = (wb >> 6) & M;
      int c[3][4];
#pragma unroll
      for (int l = 0; l < 3; ++l) {
        const uint4 xf = xt4[(sp * 3u + (uint32_t)l) * 32u + lane];
        c[l][0] = c[l][1] = c[l][2] = c[l][3] = 0;
        floe_v2::imma16832(c[l], a0, a1, a2, a3, xf.x, xf.y);
        floe_v2::imma16832(c[l], a4, a5, a6, a7, xf.z, xf.w);
      }
      const float sg = floe_k::h2f((uint16_t)(mg & 0xffffu)), sg8 = floe_k::h2f((uint16_t)(mg8 & 0xffffu));
      const float zg = floe_k::h2f((uint16_t)(mg >> 16)), zg8 = floe_k::h2f((uint16_t)(mg8 >> 16));
      const float2 xv = *reinterpret_cast<const float2 *>(xs_s + sp * kTok + 2u * tig);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int isum = c[0][j] + 256 * c[1][j] + 65536 * c[2][j];  // exact
        acc1[j] = fmaf(j < 2 ? sg : sg8, (float)isum, acc1[j]);
        acc2[j] = fmaf(j < 2 ? zg : zg8, (j & 1) ? xv.y : xv.x, acc2[j]);
      }
    };
#pragma unroll 2
    for (uint32_t p = 0; p < PQ; ++p) {
      const uint4 c4 = cw[p * 32u], m4 = mw[p * 8u];
      const uint32_t sp = 2u * (q * PQ + p);
      span_step(c4.x, c4.y, m4.x, m4.y, sp);
      span_step(c4.z, c4.w, m4.z, m4.w, sp + 1u);
    }
    __syncwarp();
    if (lane == 0) {  // this item's part of the tile is done (the first item of a cut tile
                      // also arrives for the items that belong to the other CTA)
      const uint32_t n = qhi(j) - qlo(j);
      floe_ptx::mbar_arrive_cnt(&empty[s], q == qlo(j) ? 1u + kItems - n : 1u);
    }
    if (t == 0 && k == 0) mark(a, 2);
    float *pp = part + (j * kItems + q) * 16u * kTok;  // [tile][item][row][token]
    pp[g * kTok + 2u * tig] = fmaf(inv0, acc1[0], acc2[0]);
    pp[g * kTok + 2u * tig + 1u] = fmaf(inv1, acc1[1], acc2[1]);
    pp[(g + 8u) * kTok + 2u * tig] = fmaf(inv0, acc1[2], acc2[2]);
    pp[(g + 8u) * kTok + 2u * tig + 1u] = fmaf(inv1, acc1[3], acc2[3]);
  }
  if (lane == 0) mark(a, 3 + (warp == kWarps - 1 ? 1 : 0));
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kWarps) : "memory");
  if (t == 0) mark(a, 5);
  // v[token][channel]: the item partials in fixed order; consecutive threads
  // take consecutive channels of one token (coalesced rows of v)
  const uint32_t nch = ntl * 16u;
  for (uint32_t o = t; o < nch * a.B; o += 32u * kWarps) {
    const uint32_t tok = o / nch, cl = o % nch, j = cl / 16u, row = cl % 16u;
    const uint32_t c = tlo * 16u + cl, q0 = qlo(j), q1 = qhi(j);
    const float *pp = part + j * kItems * 16u * kTok + row * kTok + tok;
    float sum = pp[q0 * 16u * kTok];
    for (uint32_t q = q0 + 1u; q < q1; ++q) sum += pp[q * 16u * kTok];
    if (c < a.di) {
      float *dst = a.v + (size_t)tok * a.di + c;
      if (q1 - q0 == (uint32_t)kItems) *dst = sum;
      else atomicAdd(dst, sum);  // a cut tile: the other CTA adds its part too
    }
  }
}

}  // namespace floe_k1b
