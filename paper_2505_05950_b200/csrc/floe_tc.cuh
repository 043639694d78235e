// floe_tc.cuh -- batched up projection on the 5th-generation tensor cores.
//
// qgemv_channels (core/src/quant.cpp:122-136) for B tokens at once, the up
// projection of batched decode:
//   v[t][c] = sum_g scale[c,g] * sum_{k in g} code[c,k] x_t[k] + zero[c,g] * sum_{k in g} x_t[k]
// (the reference's dequantize_at = code*scale + zero, quant.cpp:104-109, with
// the per-group factors pulled out of the inner sum).
//
// Exactness.  x_t is scaled by S_t = 2^(22-e_t) (max|x_t| < 2^e_t) and rounded
// to a 23-bit integer X = L0 + 256 L1 + 65536 L2 with signed 8-bit limbs.  The
// group sums sum code*L_l are computed EXACTLY by tcgen05.mma kind::i8 (u8
// codes x s8 limbs -> s32 in TMEM), recombined exactly in s32
// (|sum| <= 64*3*2^23 < 2^31), and only the epilogue rounds: one cvt and one
// FMA per group, then an FMA for the zero term (the same arithmetic as the
// batch-1 fused kernel's IMMA K1).
//
// Operands (SWIZZLE_NONE, K-major canonical layout: 8-row x 16-byte core
// matrices, LBO = 128 B between core matrices along K, SBO = 512 B between
// 8-row groups; validated by tools/umma_i8_test.cu):
//   A = codes of 128 channels x 64 elements (one group), unpacked from the
//       expert's tile-fragment layout (floe_v2.cuh) to one byte per code: the
//       16 codes of a 32-bit code word w go out as (w >> 2m) & 0x03030303,
//       m = 0..3, so K position 4m + b of a 16-byte chunk holds element
//       16*chunk + 4b + m -- a fixed permutation of K that B follows too;
//   B = limbs, row n = l * Bp + t (limb l of token t, Bp = B rounded up to 16).
// One CTA per 128-channel block; a 3-stage ring of span pairs (codes, meta,
// limbs) arrives by bulk copies; thread 0 issues copies and MMAs; all 128
// threads unpack, and drain TMEM (thread = channel row) once per batch of
// spans that fills the 512 TMEM columns.
#pragma once

#include <cuda_fp16.h>
#include <cstdint>

#include "floe_ptx.cuh"

namespace floe_tc {

constexpr int kThreads = 128;
constexpr int kRows = 128;      // channels per CTA (MMA M)
constexpr int kStages = 3;      // ring of span pairs
constexpr int kMaxTokens = 64;

__host__ __device__ constexpr uint32_t padded_tokens(uint32_t B) { return (B + 15u) / 16u * 16u; }
// columns of one span's accumulator (3 limbs x Bp tokens)
__host__ __device__ constexpr uint32_t span_cols(uint32_t B) { return 3u * padded_tokens(B); }
// bytes of one span's B operand (limb table)
__host__ __device__ constexpr uint32_t xl_span_bytes(uint32_t B) { return span_cols(B) * 64u; }

__device__ __forceinline__ uint32_t kmaj_off(uint32_t row, uint32_t k) {
  return (row & 7u) * 16u + (k & 15u) + (k >> 4) * 128u + (row >> 3) * 512u;
}

// ------------------------------------------------------------- token prep
// Per token: S_t, 1/S_t (0 if x_t is not finite) -- one CTA per token.
__global__ void __launch_bounds__(256) token_scale(const float *__restrict__ x, uint32_t dh,
                                                   float *__restrict__ invS_out,
                                                   float *__restrict__ S_out) {
  const uint32_t t = blockIdx.x;
  __shared__ float red[8];
  __shared__ int bad[8];
  float mx = 0.0f;
  int nf = 0;
  for (uint32_t k = threadIdx.x; k < dh; k += blockDim.x) {
    const float v = x[(size_t)t * dh + k];
    mx = fmaxf(mx, fabsf(v));
    nf |= !isfinite(v);
  }
  for (int o = 16; o >= 1; o >>= 1) {
    mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    nf |= __shfl_xor_sync(0xffffffffu, nf, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = mx;
    bad[threadIdx.x >> 5] = nf;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    float m = 0.0f;
    int b = 0;
    for (int w = 0; w < 8; ++w) {
      m = fmaxf(m, red[w]);
      b |= bad[w];
    }
    int ex = 0;
    frexpf(m, &ex);  // m < 2^ex
    const bool scaled = m > 0.0f;
    S_out[t] = scaled ? __int_as_float((127 + 22 - ex) << 23) : 1.0f;
    // a non-finite token cannot be limb-encoded: its v comes out NaN
    invS_out[t] = b ? __int_as_float(0x7fc00000) : (scaled ? __int_as_float((127 - 22 + ex) << 23) : 1.0f);
  }
}

// Limb tables xl[span][n][64 B] in the B-operand layout and span sums
// xs[span][Bp].  Grid: spans; block: 256.
__global__ void __launch_bounds__(256) token_limbs(const float *__restrict__ x, uint32_t dh,
                                                   uint32_t B, const float *__restrict__ S,
                                                   uint8_t *__restrict__ xl,
                                                   float *__restrict__ xs) {
  const uint32_t span = blockIdx.x, Bp = padded_tokens(B), N = 3u * Bp;
  uint8_t *out = xl + (size_t)span * N * 64u;
  // one thread per (token, element of the span)
  for (uint32_t i = threadIdx.x; i < Bp * 64u; i += blockDim.x) {
    const uint32_t t = i / 64u, e = i % 64u;
    int X = 0;
    if (t < B) {
      const float v = x[(size_t)t * dh + 64u * span + e];
      X = isfinite(v) ? __float2int_rn(v * S[t]) : 0;
    }
    const int l0 = ((X + 128) & 255) - 128;
    const int r1 = (X - l0) >> 8;
    const int l1 = ((r1 + 128) & 255) - 128;
    const int l2 = (r1 - l1) >> 8;
    // element e = 16*chunk + 4b + m sits at K position 16*chunk + 4m + b
    const uint32_t chunk = e >> 4, b = (e >> 2) & 3u, m = e & 3u;
    const uint32_t kp = 16u * chunk + 4u * m + b;
    out[kmaj_off(0u * Bp + t, kp)] = (uint8_t)(l0 & 255);
    out[kmaj_off(1u * Bp + t, kp)] = (uint8_t)(l1 & 255);
    out[kmaj_off(2u * Bp + t, kp)] = (uint8_t)(l2 & 255);
  }
  // span sums in f32, ascending (the zero term: zero * sum_k x_k)
  for (uint32_t t = threadIdx.x; t < Bp; t += blockDim.x) {
    float s = 0.0f;
    if (t < B)
      for (uint32_t e = 0; e < 64u; ++e) s += x[(size_t)t * dh + 64u * span + e];
    xs[(size_t)span * Bp + t] = s;
  }
}

// ------------------------------------------------------------- main kernel
struct BatchedArgs {
  const uint32_t *tiles;  // expert tile-fragment layout (floe_v2::tile_up)
  uint32_t dh, di, B;
  const uint8_t *xl;      // [spans][N][64]
  const float *xs;        // [spans][Bp]
  const float *invS;      // [Bp]
  float *v;               // [B][di]
};

struct BatchedSmem {
  uint32_t stage_bytes, codes, meta, xlb, a, meta_batch, xs, vacc, total;
};
__host__ __device__ inline BatchedSmem batched_smem(uint32_t dh, uint32_t B) {
  BatchedSmem L;
  const uint32_t Bp = padded_tokens(B), N = 3u * Bp;
  const uint32_t SB = (512u / N) & ~1u;  // spans per TMEM batch (even)
  // per stage: codes 8 tiles x 512 B, meta 8 x 128 B, limbs 2 spans, A 2 x 8 KB
  L.codes = 0;
  L.meta = 4096;
  L.xlb = 4096 + 1024;
  L.a = (L.xlb + 2u * N * 64u + 1023u) & ~1023u;
  L.stage_bytes = L.a + 2u * 8192u;
  uint32_t o = kStages * L.stage_bytes;
  L.meta_batch = o;  o += SB * kRows * 4u;
  L.xs = o;          o += (dh / 64u) * Bp * 4u;
  L.vacc = o;        o += Bp * kRows * 4u;
  L.total = o;
  (void)dh;
  return L;
}

template <int DH>
__global__ void __launch_bounds__(kThreads, 1) k1_batched(const BatchedArgs a) {
  constexpr uint32_t SPANS = DH / 64, PAIRS = DH / 128;
  constexpr uint32_t TILE_W = 5u * DH / 4u;  // u32 per tile
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[kStages], mdone[kStages];
  __shared__ uint32_t tmem_base;
  __shared__ float invS_s[kMaxTokens];
  const uint32_t t = threadIdx.x, warp = t >> 5, lane = t & 31;
  const uint32_t B = a.B, Bp = padded_tokens(B), N = 3u * Bp;
  const uint32_t SB = (512u / N) & ~1u;
  const BatchedSmem L = batched_smem(DH, B);
  const uint32_t blk = blockIdx.x, tiles_total = (a.di + 15u) / 16u;
  const uint32_t tile0 = blk * 8u;
  auto stage_ptr = [&](uint32_t s) { return smem + s * L.stage_bytes; };
  uint32_t *meta_batch = reinterpret_cast<uint32_t *>(smem + L.meta_batch);
  float *xs_s = reinterpret_cast<float *>(smem + L.xs);
  float *vacc = reinterpret_cast<float *>(smem + L.vacc);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        floe_ptx::smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    for (int s = 0; s < kStages; ++s) {
      floe_ptx::mbar_init(&full[s], 1);
      floe_ptx::mbar_init(&mdone[s], 1);
    }
    floe_ptx::fence_barrier_init();
  }
  for (uint32_t i = t; i < Bp; i += kThreads) invS_s[i] = i < B ? a.invS[i] : 0.0f;
  for (uint32_t i = t; i < SPANS * Bp; i += kThreads) xs_s[i] = a.xs[i];
  for (uint32_t i = t; i < Bp * kRows; i += kThreads) vacc[i] = 0.0f;
  // tiles past the expert's end: their codes are zero in the whole ring
  const uint32_t ntiles = tile0 < tiles_total ? min(8u, tiles_total - tile0) : 0u;
  if (ntiles < 8u)
    for (uint32_t s = 0; s < kStages; ++s)
      for (uint32_t i = t; i < 5120u / 4u; i += kThreads)
        reinterpret_cast<uint32_t *>(stage_ptr(s))[i] = 0u;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;

  // producer: pair p -> stage p % kStages
  auto issue = [&](uint32_t p) {
    const uint32_t s = p % kStages;
    uint8_t *st = stage_ptr(s);
    const uint32_t xlb = 2u * N * 64u;
    floe_ptx::mbar_arrive_expect_tx(&full[s], ntiles * (512u + 128u) + xlb);
    for (uint32_t j = 0; j < ntiles; ++j) {
      const uint32_t *tile = a.tiles + (size_t)(tile0 + j) * TILE_W;
      floe_ptx::bulk_g2s(st + L.codes + 512u * j, tile + p * 128u, 512u, &full[s]);
      floe_ptx::bulk_g2s(st + L.meta + 128u * j, tile + DH + p * 32u, 128u, &full[s]);
    }
    floe_ptx::bulk_g2s(st + L.xlb, a.xl + (size_t)(2u * p) * N * 64u, xlb, &full[s]);
  };
  if (t == 0)
    for (uint32_t p = 0; p < min((uint32_t)kStages, PAIRS); ++p) issue(p);

  // instruction descriptor: D s32, A u8, B s8, K-major both, N, M = 128
  const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((N >> 3) << 17) | ((uint32_t)(kRows >> 4) << 24);
  auto desc = [](uint32_t saddr) -> uint64_t {
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)(128u >> 4) << 16) |
           ((uint64_t)(512u >> 4) << 32) | ((uint64_t)1 << 46);
  };

  const uint32_t row = t;  // TMEM lane / channel row of this thread in the epilogue
  uint32_t batch_begin = 0;  // first span of the current TMEM batch
  for (uint32_t p = 0; p < PAIRS; ++p) {
    const uint32_t s = p % kStages;
    uint8_t *st = stage_ptr(s);
    floe_ptx::mbar_wait(&full[s], (p / kStages) & 1u, (7u << 28) | p);
    // unpack: 8 tiles x 32 lanes x 4 words -> A (2 spans x 128 rows x 64 B)
    {
      const uint32_t *cw = reinterpret_cast<const uint32_t *>(st + L.codes);
      uint8_t *A = st + L.a;
#pragma unroll 2
      for (uint32_t i = t; i < 8u * 128u; i += kThreads) {
        const uint32_t j = i >> 7, q = i & 127u;          // tile, word in the pair
        const uint32_t k = q & 3u, ln = q >> 2;           // word slot, lane
        const uint32_t r = 16u * j + (ln >> 2) + 8u * (k & 1u), sp = k >> 1, chunk = ln & 3u;
        const uint32_t w = cw[i];
        const uint4 o = make_uint4(w & 0x03030303u, (w >> 2) & 0x03030303u,
                                   (w >> 4) & 0x03030303u, (w >> 6) & 0x03030303u);
        *reinterpret_cast<uint4 *>(A + sp * 8192u + kmaj_off(r, 16u * chunk)) = o;
      }
      // meta of the two spans -> this TMEM batch's table [span][row]
      const uint32_t *mw = reinterpret_cast<const uint32_t *>(st + L.meta);
      for (uint32_t i = t; i < 8u * 32u; i += kThreads) {
        const uint32_t j = i >> 5, q = i & 31u, k = q & 3u, g = q >> 2;
        const uint32_t r = 16u * j + g + 8u * (k & 1u), sp = k >> 1;
        meta_batch[(2u * p + sp - batch_begin) * kRows + r] = mw[i];
      }
    }
    asm volatile("fence.proxy.async.shared::cta;");  // generic writes -> tensor-core reads
    __syncthreads();
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (uint32_t sp = 0; sp < 2; ++sp) {
        const uint32_t col = (2u * p + sp - batch_begin) * N;
        const uint32_t a0 = floe_ptx::smem_u32(st + L.a + sp * 8192u);
        const uint32_t b0 = floe_ptx::smem_u32(st + L.xlb + sp * N * 64u);
        for (uint32_t kh = 0; kh < 2; ++kh) {  // K = 64: two K=32 instructions
          const uint64_t da = desc(a0 + kh * 256u), db = desc(b0 + kh * 256u);
          const uint32_t acc = kh;
          asm volatile(
              "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, q;\n\t}" ::"r"(tmem + col),
              "l"(da), "l"(db), "r"(idesc), "r"(acc));
        }
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          floe_ptx::smem_u32(&mdone[s])));
      // refill this stage once its MMAs have read it
      if (p + kStages < PAIRS) {
        floe_ptx::mbar_wait(&mdone[s], (p / kStages) & 1u, (8u << 28) | p);
        issue(p + kStages);
      }
    }
    const uint32_t span_end = 2u * p + 2u;
    if (span_end - batch_begin == SB || p + 1 == PAIRS) {
      // drain TMEM: wait for this pair's MMAs (commit covers all earlier ones)
      if (!(t == 0 && p + kStages < PAIRS))  // (thread 0 waited above)
        floe_ptx::mbar_wait(&mdone[s], (p / kStages) & 1u, (9u << 28) | p);
      asm volatile("tcgen05.fence::after_thread_sync;");
      for (uint32_t sp = batch_begin; sp < span_end; ++sp) {
        const uint32_t mv = meta_batch[(sp - batch_begin) * kRows + row];
        const float scale = __half2float(__ushort_as_half((unsigned short)(mv & 0xffffu)));
        const float zero = __half2float(__ushort_as_half((unsigned short)(mv >> 16)));
        const uint32_t col0 = (sp - batch_begin) * N;
        for (uint32_t tc = 0; tc < Bp; tc += 16u) {
          uint32_t c[3][16];
#pragma unroll
          for (int l = 0; l < 3; ++l) {
            const uint32_t addr = tmem + ((warp * 32u) << 16) + col0 + (uint32_t)l * Bp + tc;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(c[l][0]), "=r"(c[l][1]), "=r"(c[l][2]), "=r"(c[l][3]), "=r"(c[l][4]),
                  "=r"(c[l][5]), "=r"(c[l][6]), "=r"(c[l][7]), "=r"(c[l][8]), "=r"(c[l][9]),
                  "=r"(c[l][10]), "=r"(c[l][11]), "=r"(c[l][12]), "=r"(c[l][13]), "=r"(c[l][14]),
                  "=r"(c[l][15])
                : "r"(addr));
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const uint32_t tok = tc + (uint32_t)i;
            const int isum = (int)c[0][i] + 256 * (int)c[1][i] + 65536 * (int)c[2][i];  // exact
            float &acc = vacc[tok * kRows + row];
            acc = fmaf(scale * invS_s[tok], (float)isum, fmaf(zero, xs_s[sp * Bp + tok], acc));
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;");
      __syncthreads();  // TMEM may be overwritten by the next batch's MMAs
      batch_begin = span_end;
    }
  }
  // v[t][c] for the block's channels
  const uint32_t c = blk * kRows + row;
  if (c < a.di)
    for (uint32_t tok = 0; tok < B; ++tok) a.v[(size_t)tok * a.di + c] = vacc[tok * kRows + row];
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

}  // namespace floe_tc
