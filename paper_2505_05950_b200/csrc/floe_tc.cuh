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
// One CTA per 128-channel block.  A copy warp streams span pairs by bulk
// copies (a ring of 4-pair codes+meta stages, 2-4 operand stages of limbs), an
// MMA warp issues the MMAs, and 16 consumer warps unpack codes into the A
// operand and drain TMEM (thread = channel row, 16 tokens) once per batch of
// spans that fills the 512 TMEM columns.
#pragma once

#include <cuda_fp16.h>
#include <cstdint>

#include "floe_kernels.cuh"
#include "floe_ptx.cuh"

namespace floe_tc {

constexpr int kRows = 128;      // channels per CTA (MMA M)
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
  const float4 *x4 = reinterpret_cast<const float4 *>(x + (size_t)t * dh);
  for (uint32_t k = threadIdx.x; k < dh / 4u; k += blockDim.x) {
    const float4 v = x4[k];
    mx = fmaxf(fmaxf(mx, fmaxf(fabsf(v.x), fabsf(v.y))), fmaxf(fabsf(v.z), fabsf(v.w)));
    nf |= !isfinite(v.x) | !isfinite(v.y) | !isfinite(v.z) | !isfinite(v.w);
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
  // span sums in f32 (the zero term: zero * sum_k x_k): one warp per token,
  // two elements per lane, butterfly reduction
  for (uint32_t t = threadIdx.x >> 5; t < Bp; t += blockDim.x >> 5) {
    const uint32_t ln = threadIdx.x & 31u;
    float s = 0.0f;
    if (t < B) {
      const float2 v2 = *reinterpret_cast<const float2 *>(x + (size_t)t * dh + 64u * span + 2u * ln);
      s = v2.x + v2.y;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (ln == 0) xs[(size_t)span * Bp + t] = s;
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
  unsigned long long *trace;  // nullable [blocks][32] %globaltimer marks (diagnostics)
};
__device__ __forceinline__ void tmark(const BatchedArgs &a, int k) {
  if (a.trace) {
    unsigned long long g;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g));
    a.trace[blockIdx.x * 32u + (uint32_t)k] = g;
  }
}

// Roles: warps 0..15 consume (unpack, epilogue), warp 16 lane 0 issues the
// MMAs, warp 17 lane 0 issues the bulk copies (so neither waits on the other).  Epilogue: warp w reads TMEM lane
// quadrant w % 4 (its 32 channel rows) for token chunk w / 4 (16 tokens).
constexpr int kConsumerWarps = 16;
constexpr int kBThreads = 32 * (kConsumerWarps + 2);  // + MMA warp + copy warp
constexpr int kPS = 4;   // packed ring stages
constexpr int kPPS = 4;  // span pairs per packed stage: per tile one 2 KB codes + one 512 B meta copy

// Span pairs are handled in groups of ppg (2 while the 4 spans' accumulators
// fit TMEM twice over, else 1): one unpack/arrive, one limb copy, one MMA
// batch and one commit per group.
struct BatchedSmem {
  uint32_t ppg, sb, nos, pstage, ostage, p, o, meta_batch, xs, total;
};
__host__ __device__ inline BatchedSmem batched_smem(uint32_t dh, uint32_t B) {
  BatchedSmem L;
  const uint32_t Bp = padded_tokens(B), N = 3u * Bp;
  L.ppg = N <= 96u ? 2u : 1u;
  L.sb = (512u / N) / (2u * L.ppg) * (2u * L.ppg);  // spans per TMEM batch (whole groups)
  const uint32_t SB = L.sb;
  L.nos = N <= 48u ? 3u : 2u;  // operand stages (A + limbs of a group)
  L.pstage = kPPS * 5120u;
  L.ostage = (L.ppg * 16384u + L.ppg * 2u * N * 64u + 1023u) & ~1023u;
  uint32_t o = 0;
  L.o = o;            o += L.nos * L.ostage;  // 1024-aligned operand stages first
  L.p = o;            o += kPS * L.pstage;
  L.meta_batch = o;   o += SB * 128u * 4u;
  L.xs = o;           o += (dh / 64u) * Bp * 4u;
  L.total = o;
  return L;
}

template <int DH>
__global__ void __launch_bounds__(kBThreads, 1) k1_batched(const BatchedArgs a) {
  constexpr uint32_t PAIRS = DH / 128;
  constexpr uint32_t TILE_W = 5u * DH / 4u;  // u32 per tile
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t pfull[kPS], pempty[kPS];
  __shared__ __align__(8) uint64_t xfull[3], aready[3], mdone[3], tfree;
  __shared__ uint32_t tmem_base;
  __shared__ float invS_s[kMaxTokens];
  const uint32_t t = threadIdx.x, warp = t >> 5, lane = t & 31;
  if (t == 0) tmark(a, 0);
  const uint32_t B = a.B, Bp = padded_tokens(B), N = 3u * Bp;
  const BatchedSmem L = batched_smem(DH, B);
  const uint32_t SB = L.sb, PPG = L.ppg, NG = PAIRS / PPG;
  const uint32_t NOS = L.nos;
  const uint32_t blk = blockIdx.x, tiles_total = (a.di + 15u) / 16u, tile0 = blk * 8u;
  const uint32_t ntiles = tile0 < tiles_total ? min(8u, tiles_total - tile0) : 0u;
  auto pst = [&](uint32_t s) { return smem + L.p + s * L.pstage; };
  auto ost = [&](uint32_t o) { return smem + L.o + o * L.ostage; };
  uint32_t *meta_batch = reinterpret_cast<uint32_t *>(smem + L.meta_batch);
  float *xs_s = reinterpret_cast<float *>(smem + L.xs);

  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
        floe_ptx::smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    for (int s = 0; s < kPS; ++s) {
      floe_ptx::mbar_init(&pfull[s], 1);
      floe_ptx::mbar_init(&pempty[s], kConsumerWarps);
    }
    for (int o = 0; o < 3; ++o) {
      floe_ptx::mbar_init(&xfull[o], 1);
      floe_ptx::mbar_init(&aready[o], kConsumerWarps);
      floe_ptx::mbar_init(&mdone[o], 1);
    }
    floe_ptx::mbar_init(&tfree, kConsumerWarps);
    floe_ptx::fence_barrier_init();
  }
  for (uint32_t i = t; i < Bp; i += kBThreads) invS_s[i] = i < B ? a.invS[i] : 0.0f;
  for (uint32_t i = t; i < (DH / 64u) * Bp; i += kBThreads) xs_s[i] = a.xs[i];
  if (ntiles < 8u)  // tiles past the expert's end: zero codes/meta in the whole ring
    for (uint32_t i = t; i < kPS * L.pstage / 4u; i += kBThreads)
      reinterpret_cast<uint32_t *>(smem + L.p)[i] = 0u;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  if (t == 0) tmark(a, 1);

  // packed stage q = span pairs kPPS*q ..: per tile the codes (kPPS x 512 B)
  // and meta (kPPS x 128 B) of those pairs are contiguous in the tile
  auto issue_packed = [&](uint32_t q) {
    const uint32_t s = q % kPS, p0 = q * kPPS;
    uint8_t *st = pst(s);
    floe_ptx::mbar_arrive_expect_tx(&pfull[s], ntiles * kPPS * (512u + 128u));
    for (uint32_t j = 0; j < ntiles; ++j) {
      const uint32_t *tile = a.tiles + (size_t)(tile0 + j) * TILE_W;
      floe_ptx::bulk_g2s(st + kPPS * 512u * j, tile + p0 * 128u, kPPS * 512u, &pfull[s]);
      floe_ptx::bulk_g2s(st + kPPS * 4096u + kPPS * 128u * j, tile + DH + p0 * 32u, kPPS * 128u,
                         &pfull[s]);
    }
  };
  auto issue_xl = [&](uint32_t g) {  // limbs of group g's 2*PPG spans (contiguous)
    const uint32_t o = g % NOS, bytes = PPG * 2u * N * 64u;
    floe_ptx::mbar_arrive_expect_tx(&xfull[o], bytes);
    floe_ptx::bulk_g2s(ost(o) + PPG * 16384u, a.xl + (size_t)(2u * PPG * g) * N * 64u, bytes,
                       &xfull[o]);
  };
  constexpr uint32_t QS = PAIRS / kPPS;  // packed stages in all

  if (warp == kConsumerWarps + 1) {
    // ============================= copy warp =============================
    if (lane == 0) {
      for (uint32_t q = 0; q < min((uint32_t)kPS, QS); ++q) issue_packed(q);
      for (uint32_t g = 0; g < min(NOS, NG); ++g) issue_xl(g);
      for (uint32_t g = 0; g < NG; ++g) {
        const uint32_t plast = PPG * g + PPG - 1u;
        if (plast % kPPS == kPPS - 1 && plast / kPPS + kPS < QS) {  // stage fully unpacked
          const uint32_t q = plast / kPPS;
          floe_ptx::mbar_wait(&pempty[q % kPS], (q / kPS) & 1u, (13u << 28) | g);
          issue_packed(q + kPS);
        }
        if (g + NOS < NG) {  // group g's MMAs done: its operand stage takes group g + NOS
          floe_ptx::mbar_wait(&mdone[g % NOS], (g / NOS) & 1u, (14u << 28) | g);
          issue_xl(g + NOS);
        }
      }
    }
    __syncwarp();
  } else if (warp == kConsumerWarps) {
    // ============================= MMA warp ==============================
    if (lane == 0) {
      const uint32_t idesc = (2u << 4) | (0u << 7) | (1u << 10) | ((N >> 3) << 17) |
                             ((uint32_t)(128 >> 4) << 24);
      auto desc = [](uint32_t saddr) -> uint64_t {
        return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)(128u >> 4) << 16) |
               ((uint64_t)(512u >> 4) << 32) | ((uint64_t)1 << 46);
      };
      uint32_t batch = 0, batch_begin = 0;
      for (uint32_t g = 0; g < NG; ++g) {
        const uint32_t o = g % NOS, s0 = 2u * PPG * g;  // first span of the group
        if (s0 == batch_begin + SB) {  // a new TMEM batch: wait for the epilogue
          floe_ptx::mbar_wait(&tfree, batch & 1u, (10u << 28) | g);
          ++batch;
          batch_begin = s0;
        }
        if (g == 4) tmark(a, 22);
        floe_ptx::mbar_wait(&aready[o], (g / NOS) & 1u, (11u << 28) | g);
        if (g == 0) tmark(a, 2);
        if (g == 4) tmark(a, 23);
        floe_ptx::mbar_wait(&xfull[o], (g / NOS) & 1u, (12u << 28) | g);
        if (g == 0) tmark(a, 3);
        if (g == 4) tmark(a, 24);
        asm volatile("tcgen05.fence::after_thread_sync;");
        for (uint32_t sg = 0; sg < 2u * PPG; ++sg) {  // span within the group
          const uint32_t col = (s0 + sg - batch_begin) * N;
          const uint32_t a0 = floe_ptx::smem_u32(ost(o) + sg * 8192u);
          const uint32_t b0 = floe_ptx::smem_u32(ost(o) + PPG * 16384u + sg * N * 64u);
          for (uint32_t kh = 0; kh < 2; ++kh) {
            const uint64_t da = desc(a0 + kh * 256u), db = desc(b0 + kh * 256u);
            asm volatile(
                "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, q;\n\t}" ::"r"(tmem + col),
                "l"(da), "l"(db), "r"(idesc), "r"(kh));
          }
        }
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
            floe_ptx::smem_u32(&mdone[o])));
        if (g == 4) tmark(a, 25);
      }
    }
    __syncwarp();
  } else {
    // ============================ consumers =============================
    // epilogue role: TMEM lane quadrant, token chunk of 16, and (when there
    // are fewer than 4 token chunks) which of the batch's spans, so that all
    // 16 warps drain TMEM for any batch size
    const uint32_t nchunk = Bp / 16u, spg = 4u / nchunk;  // span groups per chunk
    const uint32_t quad = warp & 3u, wg = warp >> 2;
    const uint32_t tchunk = wg % nchunk, sphase = wg / nchunk;
    const uint32_t row = 32u * quad + lane;
    const bool ep = sphase < spg;
    float acc1[16], acc2[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) acc1[i] = acc2[i] = 0.0f;
    uint32_t batch = 0, batch_begin = 0;
    for (uint32_t g = 0; g < NG; ++g) {
      const uint32_t p0 = PPG * g, q = p0 / kPPS, s = q % kPS, o = g % NOS;
      if (t == 0 && g == 4) tmark(a, 19);
      floe_ptx::mbar_wait(&pfull[s], (q / kPS) & 1u, (15u << 28) | g);  // (a group lies in one stage)
      if (t == 0 && g == 4) tmark(a, 27);
      if (g >= NOS)  // A[o] free: MMAs of group g - NOS done
        floe_ptx::mbar_wait(&mdone[o], ((g / NOS) - 1u) & 1u, (16u << 28) | g);
      if (t == 0 && g == 4) tmark(a, 28);
      {
        uint8_t *A = ost(o);
        if (t < PPG * 256u) {  // thread = (pair of the group, tile j, lane ln): 4 code words
          const uint32_t pg = t >> 8, j = (t >> 5) & 7u, ln = t & 31u, g8 = ln >> 2, chunk = ln & 3u;
          const uint32_t pp = (p0 + pg) % kPPS;
          const uint32_t *cw = reinterpret_cast<const uint32_t *>(pst(s) + pp * 512u);
          const uint4 w4 = *reinterpret_cast<const uint4 *>(cw + j * (kPPS * 128u) + 4u * ln);
          const uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
#pragma unroll
          for (uint32_t k = 0; k < 4; ++k) {  // slot k: row g8 + 8(k&1), span k>>1
            const uint32_t w = ws[k], r = 16u * j + g8 + 8u * (k & 1u);
            const uint4 ov = make_uint4(w & 0x03030303u, (w >> 2) & 0x03030303u,
                                        (w >> 4) & 0x03030303u, (w >> 6) & 0x03030303u);
            *reinterpret_cast<uint4 *>(A + pg * 16384u + (k >> 1) * 8192u + kmaj_off(r, 16u * chunk)) = ov;
          }
        }
        for (uint32_t i = t; i < PPG * 256u; i += 32u * kConsumerWarps) {  // meta -> batch table
          const uint32_t pg = i >> 8, tm = i & 255u;
          const uint32_t pp = (p0 + pg) % kPPS;
          const uint32_t *mw = reinterpret_cast<const uint32_t *>(pst(s) + kPPS * 4096u + pp * 128u);
          const uint32_t j = tm >> 5, mq = tm & 31u, k = mq & 3u, g8 = mq >> 2;
          const uint32_t r = 16u * j + g8 + 8u * (k & 1u), sp = k >> 1;
          meta_batch[(2u * (p0 + pg) + sp - batch_begin) * 128u + r] = mw[j * (kPPS * 32u) + mq];
        }
      }
      asm volatile("fence.proxy.async.shared::cta;");  // generic writes -> tensor-core reads
      __syncwarp();
      if (lane == 0) {
        if ((p0 + PPG - 1u) % kPPS == kPPS - 1) floe_ptx::mbar_arrive(&pempty[s]);
        floe_ptx::mbar_arrive(&aready[o]);
      }
      if (t == 0 && g == 4) tmark(a, 29);
      const uint32_t span_end = 2u * PPG * (g + 1u);
      if (span_end - batch_begin == SB || g + 1 == NG) {
        // all MMAs of the batch are done when group g's commit fires
        if (t == 0 && batch < 12) tmark(a, 4 + 2 * (int)batch);
        floe_ptx::mbar_wait(&mdone[o], (g / NOS) & 1u, (17u << 28) | g);
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps));  // meta_batch complete
        asm volatile("tcgen05.fence::after_thread_sync;");
        if (ep) {
          for (uint32_t sp = batch_begin + sphase; sp < span_end; sp += spg) {
            const uint32_t mv = meta_batch[(sp - batch_begin) * 128u + row];
            const float scale = __half2float(__ushort_as_half((unsigned short)(mv & 0xffffu)));
            const float zero = __half2float(__ushort_as_half((unsigned short)(mv >> 16)));
            const uint32_t col0 = (sp - batch_begin) * N + 16u * tchunk;
            uint32_t c[3][16];
#pragma unroll
            for (int l = 0; l < 3; ++l) {
              const uint32_t addr = tmem + ((32u * quad) << 16) + col0 + (uint32_t)l * Bp;
              asm volatile(
                  "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                  : "=r"(c[l][0]), "=r"(c[l][1]), "=r"(c[l][2]), "=r"(c[l][3]), "=r"(c[l][4]),
                    "=r"(c[l][5]), "=r"(c[l][6]), "=r"(c[l][7]), "=r"(c[l][8]), "=r"(c[l][9]),
                    "=r"(c[l][10]), "=r"(c[l][11]), "=r"(c[l][12]), "=r"(c[l][13]), "=r"(c[l][14]),
                    "=r"(c[l][15])
                  : "r"(addr));
            }
            asm volatile("tcgen05.wait::ld.sync.aligned;");
            const float4 *xsv = reinterpret_cast<const float4 *>(xs_s + sp * Bp + 16u * tchunk);
#pragma unroll
            for (int i4 = 0; i4 < 4; ++i4) {
              const float4 z = xsv[i4];
              const float zz[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
              for (int u = 0; u < 4; ++u) {
                const int i = 4 * i4 + u;
                const int isum = (int)c[0][i] + 256 * (int)c[1][i] + 65536 * (int)c[2][i];  // exact
                acc1[i] = fmaf(scale, (float)isum, acc1[i]);
                acc2[i] = fmaf(zero, zz[u], acc2[i]);
              }
            }
          }
        }
        asm volatile("tcgen05.fence::before_thread_sync;");
        __syncwarp();
        if (t == 0 && batch < 12) tmark(a, 5 + 2 * (int)batch);
        if (lane == 0) floe_ptx::mbar_arrive(&tfree);  // TMEM and meta_batch reusable
        asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps));  // meta_batch reuse
        ++batch;
        batch_begin = span_end;
      }
    }
    // combine the span groups' partials (through the packed ring, free now),
    // then v = invS * sum_g scale*isum + sum_g zero*xs (invS a power of two)
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps));
    float *red = reinterpret_cast<float *>(smem + L.p);  // [wg][row][32]
    if (ep && sphase > 0)
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        red[(wg * 128u + row) * 32u + i] = acc1[i];
        red[(wg * 128u + row) * 32u + 16 + i] = acc2[i];
      }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kConsumerWarps));
    const uint32_t c = blk * 128u + row;
    if (ep && sphase == 0) {
      for (uint32_t ph = 1; ph < spg; ++ph) {
        const uint32_t og = ph * nchunk + tchunk;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          acc1[i] += red[(og * 128u + row) * 32u + i];
          acc2[i] += red[(og * 128u + row) * 32u + 16 + i];
        }
      }
      if (c < a.di)
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const uint32_t tok = 16u * tchunk + (uint32_t)i;
          if (tok < B) a.v[(size_t)tok * a.di + c] = fmaf(invS_s[tok], acc1[i], acc2[i]);
        }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (t == 0) tmark(a, 30);
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
}

// ------------------------------------------------------- batched gate/down
// expert_forward_sparse (model.cpp:128-142) for B tokens after the batched up
// projection: token t keeps channel c iff !(|v[t][c]| < t_e) (model.cpp:135:
// ties and NaN kept); the union of kept channels is read once.
//   union_masks: per channel a token bitmask; kept channels appended to a list
//   coeffs:      A[u][t] = silu(gate_c . x_t) * v[t][c] for the tokens keeping c
//                (la.cpp:25-31), one warp per union channel, x from L2
//   down_accum:  y[t][j] = sum_u A[u][t] * down_c[j], CTAs over (1024-column
//                chunk, union-row chunk), partial sums added into y

__global__ void __launch_bounds__(256) union_masks(const float *__restrict__ v, uint32_t B,
                                                   uint32_t di, float thr,
                                                   uint32_t *__restrict__ count,
                                                   uint32_t *__restrict__ uc,
                                                   unsigned long long *__restrict__ um) {
  const uint32_t c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= di) return;
  unsigned long long m = 0;
  for (uint32_t t = 0; t < B; ++t)
    if (!(fabsf(v[(size_t)t * di + c]) < thr)) m |= 1ull << t;
  if (m) {
    const uint32_t i = atomicAdd(count, 1u);
    uc[i] = c;
    um[i] = m;
  }
}

template <int DH>
__global__ void __launch_bounds__(256) coeffs(const __half *__restrict__ records,
                                              const float *__restrict__ x, const float *__restrict__ v,
                                              uint32_t B, uint32_t di,
                                              const uint32_t *__restrict__ count,
                                              const uint32_t *__restrict__ uc,
                                              const unsigned long long *__restrict__ um,
                                              float *__restrict__ A /* [n][B] */,
                                              uint32_t *__restrict__ amax) {
  // one warp per union channel, one pass: the gate row stays in registers and
  // each keeping token's x streams from L2 (x is B x 16 KB, shared by all SMs)
  const uint32_t n = *count, lane = threadIdx.x & 31u, warp = threadIdx.x >> 5;
  for (uint32_t u = blockIdx.x * 8u + warp; u < n; u += gridDim.x * 8u) {
    const uint32_t c = uc[u];
    const unsigned long long m = um[u];
    const uint4 *g4 = reinterpret_cast<const uint4 *>(records + (size_t)c * 2 * DH);
    uint4 gr[DH / 256];
#pragma unroll
    for (int i = 0; i < DH / 256; ++i) gr[i] = __ldg(g4 + lane + 32 * i);
    for (uint32_t t = lane; t < B; t += 32u)
      if (!((m >> t) & 1ull)) A[(size_t)u * B + t] = 0.0f;
    for (unsigned long long mm = m; mm; mm &= mm - 1) {
      const uint32_t tt = (uint32_t)__ffsll((long long)mm) - 1u;
      const float4 *xt = reinterpret_cast<const float4 *>(x + (size_t)tt * DH);
      float acc = 0.0f;
#pragma unroll
      for (int i = 0; i < DH / 256; ++i) {
        const __half2 *h2 = reinterpret_cast<const __half2 *>(&gr[i]);
        const float4 xa = __ldg(xt + 2 * (lane + 32 * i));
        const float4 xb = __ldg(xt + 2 * (lane + 32 * i) + 1);
        float2 f;
        f = __half22float2(h2[0]); acc = fmaf(f.x, xa.x, acc); acc = fmaf(f.y, xa.y, acc);
        f = __half22float2(h2[1]); acc = fmaf(f.x, xa.z, acc); acc = fmaf(f.y, xa.w, acc);
        f = __half22float2(h2[2]); acc = fmaf(f.x, xb.x, acc); acc = fmaf(f.y, xb.y, acc);
        f = __half22float2(h2[3]); acc = fmaf(f.x, xb.z, acc); acc = fmaf(f.y, xb.w, acc);
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      if (lane == 0) {
        const float z = acc;
        const float av = z / (1.0f + expf(-z)) * v[(size_t)tt * di + c];  // silu(g) * v
        A[(size_t)u * B + tt] = av;
        if (amax) atomicMax(&amax[tt], __float_as_uint(fabsf(av)));
      }
    }
  }
}

// ------------------------------------- fused union gate/down (<= 4 tokens)
// expert_forward_sparse's phase C (model.cpp:136-140, la.cpp:25-31) over the
// union of kept channels for up to 4 tokens in ONE pass over the records, the
// decode kernel's way: one CTA per SM takes a contiguous range of union rows,
// a producer warp streams each row's gate|down record (16 KB, one bulk copy)
// through an 8-stage ring, and 16 consumer warps each own a 1/16 column slice
// of x (registers) and of y (register accumulators).  Per batch of kUR records:
// per-warp gate partials -> shared memory -> fixed-order sum, silu(g) * v (0
// for a token that drops the channel) -> every warp adds a * down into its y
// slice.  y gets one red.add per element per CTA at the end.  (coeffs +
// down_accum read the records with per-thread loads and stayed latency-bound
// at ~0.3 of HBM.)
constexpr int kUTok = 4;                  // tokens
constexpr int kUWarps = 16;               // consumer warps
constexpr int kUThreads = 32 * (kUWarps + 1);
constexpr int kUStages = 8;
constexpr int kUR = 8;                    // records per barrier batch (default)
constexpr uint32_t kUMaxRows = 256;       // union rows per CTA (host checks n <= G * kUMaxRows)

// PL consecutive f16 values (PL = 4: one 8-B load, PL % 8 == 0: 16-B loads)
template <uint32_t PL>
__device__ __forceinline__ void load_half_row(const __half *p, float (&f)[PL]) {
  if constexpr (PL % 8 == 0) {
#pragma unroll
    for (uint32_t e = 0; e < PL; e += 8) {
      const uint4 q = *reinterpret_cast<const uint4 *>(p + e);
      const __half2 *h2 = reinterpret_cast<const __half2 *>(&q);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float2 v2 = __half22float2(h2[j]);
        f[e + 2 * j] = v2.x;
        f[e + 2 * j + 1] = v2.y;
      }
    }
  } else {
    static_assert(PL == 4, "union_ffn: 4 or a multiple of 8 elements per lane");
    const uint2 q = *reinterpret_cast<const uint2 *>(p);
    const float2 a = __half22float2(*reinterpret_cast<const __half2 *>(&q.x));
    const float2 b = __half22float2(*reinterpret_cast<const __half2 *>(&q.y));
    f[0] = a.x; f[1] = a.y; f[2] = b.x; f[3] = b.y;
  }
}

template <int DH, int UR = kUR>
__global__ void __launch_bounds__(kUThreads, 1) union_ffn(const __half *__restrict__ records,
                                                         const float *__restrict__ x,
                                                         const float *__restrict__ v, uint32_t B,
                                                         uint32_t di,
                                                         const uint32_t *__restrict__ count,
                                                         const uint32_t *__restrict__ uc,
                                                         const unsigned long long *__restrict__ um,
                                                         float *__restrict__ y) {
  constexpr uint32_t PL = DH / (32u * kUWarps);  // elements per lane (8 at dh 4096)
  constexpr uint32_t RB = 4u * DH;               // record bytes (gate | down, f16)
  extern __shared__ __align__(128) uint8_t ring[];  // [kUStages][RB]
  __shared__ __align__(8) uint64_t full[kUStages], empty[kUStages];
  __shared__ uint32_t rows_s[kUMaxRows];
  __shared__ float va_s[kUMaxRows][kUTok];   // v of the token, or 0 if it drops the row
  static_assert(UR * kUTok <= 32, "union_ffn: one lane of warp 0 per (record, token)");
  __shared__ float part[UR][kUTok][kUWarps];
  __shared__ float acoef[UR][kUTok];
  const uint32_t t = threadIdx.x, warp = t >> 5, lane = t & 31u;
  const uint32_t G = gridDim.x, b = blockIdx.x, n = *count;
  const uint32_t r0 = (uint32_t)((uint64_t)n * b / G), r1 = (uint32_t)((uint64_t)n * (b + 1) / G);
  const uint32_t nr = min(r1 - r0, kUMaxRows);
  if (t == 0) {
    for (int s = 0; s < kUStages; ++s) {
      floe_ptx::mbar_init(&full[s], 1);
      floe_ptx::mbar_init(&empty[s], kUWarps);
    }
    floe_ptx::fence_barrier_init();
  }
  for (uint32_t i = t; i < nr; i += blockDim.x) rows_s[i] = uc[r0 + i];
  __syncthreads();
  auto spin = [](uint64_t *bar, uint32_t parity) {
    while (!floe_ptx::mbar_test_wait(bar, parity)) {
    }
  };
  if (warp == kUWarps) {
    // ============================== producer ==============================
    if (lane == 0)
      for (uint32_t i = 0; i < nr; ++i) {
        const uint32_t s = i % kUStages;
        if (i >= (uint32_t)kUStages) spin(&empty[s], ((i / kUStages) - 1u) & 1u);
        floe_ptx::mbar_arrive_expect_tx(&full[s], RB);
        floe_ptx::bulk_g2s(ring + s * RB, records + (size_t)rows_s[i] * 2u * DH, RB, &full[s]);
      }
    return;
  }
  // ============================== consumers ===============================
  for (uint32_t i = t; i < nr * kUTok; i += 32u * kUWarps) {
    const uint32_t r = i / kUTok, tk = i % kUTok;
    const bool keep = tk < B && ((um[r0 + r] >> tk) & 1ull);
    va_s[r][tk] = keep ? v[(size_t)tk * di + rows_s[r]] : 0.0f;
  }
  const uint32_t k0 = warp * (DH / kUWarps) + lane * PL;  // this lane's columns
  float xr[kUTok][PL], ya[kUTok][PL];
#pragma unroll
  for (int tk = 0; tk < kUTok; ++tk)
#pragma unroll
    for (uint32_t e = 0; e < PL; e += 4) {
      const float4 q = (uint32_t)tk < B ? *reinterpret_cast<const float4 *>(x + (size_t)tk * DH + k0 + e)
                                        : make_float4(0.0f, 0.0f, 0.0f, 0.0f);
      xr[tk][e] = q.x; xr[tk][e + 1] = q.y; xr[tk][e + 2] = q.z; xr[tk][e + 3] = q.w;
      ya[tk][e] = ya[tk][e + 1] = ya[tk][e + 2] = ya[tk][e + 3] = 0.0f;
    }
  asm volatile("bar.sync 1, %0;" ::"n"(32 * kUWarps) : "memory");  // va_s complete
  for (uint32_t i0 = 0; i0 < nr; i0 += UR) {
    const uint32_t nb = min((uint32_t)UR, nr - i0);
    // gate partials of this warp's column slice
    for (uint32_t rr = 0; rr < nb; ++rr) {
      const uint32_t i = i0 + rr, s = i % kUStages;
      spin(&full[s], (i / kUStages) & 1u);
      float gf[PL], p[kUTok];
      load_half_row<PL>(reinterpret_cast<const __half *>(ring + s * RB) + k0, gf);
#pragma unroll
      for (int tk = 0; tk < kUTok; ++tk) {
        p[tk] = 0.0f;
#pragma unroll
        for (uint32_t e = 0; e < PL; ++e) p[tk] = fmaf(gf[e], xr[tk][e], p[tk]);
      }
      // transposed butterfly: the 4 token sums in 6 shuffles (not 20); lane
      // 8 tk ends with token tk's sum
      static_assert(kUTok == 4, "union_ffn: the butterfly reduces 4 token sums");
      const bool hi16 = (lane & 16u) != 0, hi8 = (lane & 8u) != 0;
      const float r0 = __shfl_xor_sync(0xffffffffu, hi16 ? p[0] : p[2], 16);
      const float r1 = __shfl_xor_sync(0xffffffffu, hi16 ? p[1] : p[3], 16);
      const float k0s = (hi16 ? p[2] : p[0]) + r0, k1s = (hi16 ? p[3] : p[1]) + r1;
      float q = (hi8 ? k1s : k0s) + __shfl_xor_sync(0xffffffffu, hi8 ? k0s : k1s, 8);
#pragma unroll
      for (int o = 4; o >= 1; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
      if ((lane & 7u) == 0) part[rr][lane >> 3][warp] = q;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kUWarps) : "memory");
    if (warp == 0 && lane < nb * kUTok) {  // a = silu(g) * v, fixed-order sum of the slices
      const uint32_t rr = lane / kUTok, tk = lane % kUTok;
      float gs = 0.0f;
#pragma unroll
      for (int w = 0; w < kUWarps; ++w) gs += part[rr][tk][w];
      const float va = va_s[i0 + rr][tk];
      acoef[rr][tk] = va != 0.0f ? floe_k::silu_ref(gs) * va : 0.0f;
    }
    asm volatile("bar.sync 1, %0;" ::"n"(32 * kUWarps) : "memory");
    for (uint32_t rr = 0; rr < nb; ++rr) {
      const uint32_t i = i0 + rr, s = i % kUStages;
      float a[kUTok], df[PL];
#pragma unroll
      for (int tk = 0; tk < kUTok; ++tk) a[tk] = acoef[rr][tk];
      load_half_row<PL>(reinterpret_cast<const __half *>(ring + s * RB) + DH + k0, df);
#pragma unroll
      for (uint32_t e = 0; e < PL; ++e)
#pragma unroll
        for (int tk = 0; tk < kUTok; ++tk) ya[tk][e] = fmaf(a[tk], df[e], ya[tk][e]);
      __syncwarp();
      if (lane == 0) floe_ptx::mbar_arrive(&empty[s]);
    }
  }
  if (nr > 0)
#pragma unroll
    for (int tk = 0; tk < kUTok; ++tk)
      if ((uint32_t)tk < B)
#pragma unroll
        for (uint32_t e = 0; e < PL; e += 4)
          floe_k::red_add_v4(y + (size_t)tk * DH + k0 + e, ya[tk][e], ya[tk][e + 1], ya[tk][e + 2],
                             ya[tk][e + 3]);
}

// ---------------------------------------------- gate GEMM on tcgen05 (f16)
// G[u][t] = gate_{c_u} . x_t for 128 union channels per CTA as one tensor-core
// GEMM: A = the channels' f16 gate rows (gathered with cp.async, K-major
// SWIZZLE_NONE, LBO 128 B / SBO 1024 B), B = x split into f16 hi + lo (x =
// hi + lo to ~22 bits, rows 2t and 2t+1), D f32 in TMEM; g = D[2t] + D[2t+1].
// 64-element K chunks through a 4-stage ring; then A[u][t] = silu(g) * v.
constexpr int kGemmStages = 4;

__host__ __device__ constexpr uint32_t gemm_n(uint32_t B) { return 2u * ((B + 7u) / 8u * 8u); }

__device__ __forceinline__ uint32_t kmaj_off128(uint32_t row, uint32_t kbyte) {
  return (row & 7u) * 16u + (kbyte & 15u) + (kbyte >> 4) * 128u + (row >> 3) * 1024u;
}

// Power-of-two scale that puts max|a| in [64, 128): the f16 hi + lo split of
// a*scale then keeps ~22 significant bits without f16 underflow or overflow
// whatever the token's magnitude (1 when amax is 0 or not finite).  amax_bits
// = float bits of a non-negative max (uint order == float order).
__device__ __forceinline__ float hilo_scale(uint32_t amax_bits) {
  if (amax_bits == 0u || amax_bits >= 0x7f800000u) return 1.0f;
  const int e = (int)((amax_bits >> 23) & 255u) - 127;  // amax < 2^(e+1)
  const int se = max(-100, min(100, 6 - e));
  return __int_as_float((127 + se) << 23);
}

// Per token: the hi/lo scale of x (xsc[t], inv_xsc[t]); clears amax[t] (the
// per-token max|A| the gate stage accumulates for the down GEMM's A scale).
__global__ void __launch_bounds__(256) hilo_token_scale(const float *__restrict__ x, uint32_t dh,
                                                        float *__restrict__ xsc,
                                                        float *__restrict__ inv_xsc,
                                                        uint32_t *__restrict__ amax) {
  const uint32_t t = blockIdx.x;
  __shared__ uint32_t red[8];
  uint32_t mx = 0;
  const float4 *x4 = reinterpret_cast<const float4 *>(x + (size_t)t * dh);
  for (uint32_t k = threadIdx.x; k < dh / 4u; k += blockDim.x) {
    const float4 v = x4[k];
    mx = max(mx, max(max(__float_as_uint(fabsf(v.x)), __float_as_uint(fabsf(v.y))),
                     max(__float_as_uint(fabsf(v.z)), __float_as_uint(fabsf(v.w)))));
  }
  mx = __reduce_max_sync(0xffffffffu, mx);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = max(mx, red[w]);
    const float sc = hilo_scale(max(mx, red[0]));
    xsc[t] = sc;
    inv_xsc[t] = 1.0f / sc;
    amax[t] = 0u;
  }
}

// x -> hi/lo table [chunk][N rows][128 B] in the B-operand layout, x_t scaled
// by xsc[t] (undone in the gate epilogue).  Grid: chunks.
__global__ void __launch_bounds__(256) x_hilo(const float *__restrict__ x, uint32_t dh, uint32_t B,
                                              const float *__restrict__ xsc,
                                              uint8_t *__restrict__ xh) {
  const uint32_t ch = blockIdx.x, N = gemm_n(B);
  uint8_t *out = xh + (size_t)ch * N * 128u;
  for (uint32_t i = threadIdx.x; i < (N / 2u) * 64u; i += blockDim.x) {
    const uint32_t t = i / 64u, e = i % 64u;
    __half hi = __float2half_rn(0.0f), lo = hi;
    if (t < B) {
      const float xv = x[(size_t)t * dh + 64u * ch + e] * xsc[t];
      hi = __float2half_rn(xv);
      lo = __float2half_rn(xv - __half2float(hi));
    }
    *reinterpret_cast<__half *>(out + kmaj_off128(2u * t, 2u * e)) = hi;
    *reinterpret_cast<__half *>(out + kmaj_off128(2u * t + 1u, 2u * e)) = lo;
  }
}

__device__ __forceinline__ void cp_async16(void *dst, const void *src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(floe_ptx::smem_u32(dst)), "l"(src)
               : "memory");
}

template <int DH>
__global__ void __launch_bounds__(128, 1) gate_gemm(const __half *__restrict__ records,
                                                    const uint8_t *__restrict__ xh,
                                                    const float *__restrict__ v, uint32_t B,
                                                    uint32_t di, const uint32_t *__restrict__ count,
                                                    const uint32_t *__restrict__ uc,
                                                    const unsigned long long *__restrict__ um,
                                                    float *__restrict__ A /* [n][B] */,
                                                    float *__restrict__ G /* split K: [n][B] */,
                                                    const float *__restrict__ inv_xsc,
                                                    uint32_t *__restrict__ amax) {
  // K (d_hidden) split over gridDim.y CTAs: each adds its partial dot into G,
  // gate_finish applies silu * v; with one part the epilogue does it directly
  constexpr uint32_t CHUNKS = DH / 64u;
  const uint32_t c_lo = CHUNKS * blockIdx.y / gridDim.y, c_hi = CHUNKS * (blockIdx.y + 1) / gridDim.y;
  const uint32_t NCH = c_hi - c_lo;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t mdone[kGemmStages];
  __shared__ uint32_t tmem_base;
  __shared__ uint32_t ucs[128];
  __shared__ uint32_t amax_s[kMaxTokens];
  const uint32_t n = *count, u0 = blockIdx.x * 128u;
  if (u0 >= n) return;
  const uint32_t t = threadIdx.x, warp = t >> 5, lane = t & 31u;
  const uint32_t N = gemm_n(B), nr = min(128u, n - u0);
  const uint32_t stageA = 16384u, stage = stageA + N * 128u;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;" ::"r"(
        floe_ptx::smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    for (int s = 0; s < kGemmStages; ++s) floe_ptx::mbar_init(&mdone[s], 1);
    floe_ptx::fence_barrier_init();
  }
  ucs[t] = t < nr ? uc[u0 + t] : uc[u0];  // rows past the union repeat a valid channel
  if (t < kMaxTokens) amax_s[t] = 0u;
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  // chunk loads: A = 128 rows x 128 B (8 x 16 B per row), B = N rows x 128 B
  auto load = [&](uint32_t j) {  // local chunk j = global chunk c_lo + j
    const uint32_t c = c_lo + j;
    uint8_t *st = smem + (j % kGemmStages) * stage;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const uint32_t idx = t + 128u * (uint32_t)i, row = idx >> 3, kb = (idx & 7u) * 16u;
      const uint8_t *src = reinterpret_cast<const uint8_t *>(records + (size_t)ucs[row] * 2 * DH) +
                           128u * c + kb;
      cp_async16(st + kmaj_off128(row, kb), src);
    }
    const uint8_t *xs = xh + (size_t)c * N * 128u;
    for (uint32_t i = t; i < N * 8u; i += 128u) cp_async16(st + stageA + 16u * i, xs + 16u * i);
  };
  const uint32_t idesc = (1u << 4) | (0u << 7) | (0u << 10) | ((N >> 3) << 17) | ((128u >> 4) << 24);
  auto desc = [](uint32_t saddr) -> uint64_t {
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)(128u >> 4) << 16) |
           ((uint64_t)(1024u >> 4) << 32) | ((uint64_t)1 << 46);
  };
  for (uint32_t c = 0; c < kGemmStages - 1; ++c) {
    if (c < NCH) load(c);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (uint32_t c = 0; c < NCH; ++c) {
    // stage of chunk c + 3 was last read by the MMAs of chunk c - 1
    if (c >= 1 && c + kGemmStages - 1 < NCH)
      floe_ptx::mbar_wait(&mdone[(c - 1) % kGemmStages], ((c - 1) / kGemmStages) & 1u, c);
    if (c + kGemmStages - 1 < NCH) load(c + kGemmStages - 1);
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(kGemmStages - 1) : "memory");  // chunk c landed
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = floe_ptx::smem_u32(smem + (c % kGemmStages) * stage);
      const uint32_t b0 = a0 + stageA;
#pragma unroll
      for (uint32_t kk = 0; kk < 4; ++kk) {  // K = 16 halves (32 B) per instruction
        const uint32_t acc = (c > 0 || kk > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n\t}" ::"r"(tmem),
            "l"(desc(a0 + kk * 256u)), "l"(desc(b0 + kk * 256u)), "r"(idesc), "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          floe_ptx::smem_u32(&mdone[c % kGemmStages])));
    }
  }
  floe_ptx::mbar_wait(&mdone[(NCH - 1) % kGemmStages], ((NCH - 1) / kGemmStages) & 1u, 999u);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: thread = union row; columns (2t, 2t+1) = x_t hi, lo
  const uint32_t u = u0 + t;
  const unsigned long long m = t < nr ? um[u] : 0ull;
  const uint32_t c_ch = ucs[t];
  for (uint32_t c0 = 0; c0 < N; c0 += 16u) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15])
        : "r"(tmem + ((warp * 32u) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    if (t < nr)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const uint32_t tok = c0 / 2u + (uint32_t)i;
        if (tok < B) {
          const float z = (__uint_as_float(r[2 * i]) + __uint_as_float(r[2 * i + 1])) * inv_xsc[tok];
          if (gridDim.y > 1) {
            atomicAdd(G + (size_t)u * B + tok, z);
          } else {
            const float av =
                ((m >> tok) & 1ull) ? z / (1.0f + expf(-z)) * v[(size_t)tok * di + c_ch] : 0.0f;
            A[(size_t)u * B + tok] = av;
            atomicMax(&amax_s[tok], __float_as_uint(fabsf(av)));
          }
        }
      }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (gridDim.y == 1 && t < B && amax_s[t]) atomicMax(&amax[t], amax_s[t]);
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;" ::"r"(tmem));
  (void)lane;
}

// A[u][t] = silu(G[u][t]) * v[t][c_u] for the tokens keeping c_u, else 0.
__global__ void __launch_bounds__(256) gate_finish(const float *__restrict__ G,
                                                   const float *__restrict__ v, uint32_t B,
                                                   uint32_t di, const uint32_t *__restrict__ count,
                                                   const uint32_t *__restrict__ uc,
                                                   const unsigned long long *__restrict__ um,
                                                   float *__restrict__ A,
                                                   uint32_t *__restrict__ amax) {
  __shared__ uint32_t amax_s[kMaxTokens];
  if (threadIdx.x < kMaxTokens) amax_s[threadIdx.x] = 0u;
  __syncthreads();
  const uint32_t n = *count;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n * B; i += gridDim.x * blockDim.x) {
    const uint32_t u = i / B, tok = i % B;
    const float z = G[i];
    const float av = ((um[u] >> tok) & 1ull) ? z / (1.0f + expf(-z)) * v[(size_t)tok * di + uc[u]] : 0.0f;
    A[i] = av;
    atomicMax(&amax_s[tok], __float_as_uint(fabsf(av)));
  }
  __syncthreads();
  if (threadIdx.x < B && amax_s[threadIdx.x]) atomicMax(&amax[threadIdx.x], amax_s[threadIdx.x]);
}

// ---------------------------------------------- down GEMM on tcgen05 (f16)
// Y[t][m] = sum_u A[u][t] * down_{c_u}[m] for a 256-wide slice of m and a range
// of kDownKRange union channels per CTA: M = 2 rows per token (the f32
// coefficient split into f16 hi + lo, zero rows past 2B), N = 256 (d_hidden
// slice), K = channels.  A (K-major) is built from the coefficients; B is the
// gathered f16 down rows, N-contiguous per channel = the MN-major operand
// (validated by tools/umma_f16_mn_test.cu: core matrices 8 k x 16 B of n,
// n-adjacent 128 B apart; descriptor LBO = k-core stride, SBO = 128 B).
// Partial sums of the channel range are added into y.
constexpr uint32_t kDownKRange = 256;   // union channels per CTA
constexpr uint32_t kDownKChunk = 64;    // channels per pipeline stage
constexpr int kDownStages = 2;

template <int DH>
__global__ void __launch_bounds__(128, 1) down_gemm(const __half *__restrict__ records,
                                                    uint32_t B, const uint32_t *__restrict__ count,
                                                    const uint32_t *__restrict__ uc,
                                                    const float *__restrict__ A, float *__restrict__ y,
                                                    const uint32_t *__restrict__ amax) {
  constexpr uint32_t NS = 256;  // d_hidden columns per CTA
  constexpr uint32_t SA = 128u * kDownKChunk * 2u;   // 16 KB: 128 rows x 64 k f16
  constexpr uint32_t SBB = kDownKChunk * NS * 2u;    // 32 KB: 64 k x 256 n f16
  constexpr uint32_t ST = SA + SBB;
  extern __shared__ __align__(1024) uint8_t smem[];
  __shared__ __align__(8) uint64_t mdone[kDownStages];
  __shared__ uint32_t tmem_base;
  __shared__ float asc[kMaxTokens], inv_asc[kMaxTokens];
  const uint32_t n = *count, k0 = blockIdx.y * kDownKRange;
  if (k0 >= n) return;
  if (threadIdx.x < B) {  // per-token power-of-two scale of the coefficients
    const float sc = hilo_scale(amax[threadIdx.x]);
    asc[threadIdx.x] = sc;
    inv_asc[threadIdx.x] = 1.0f / sc;
  }
  const uint32_t m0 = blockIdx.x * NS, t = threadIdx.x, warp = t >> 5, lane = t & 31u;
  const uint32_t nk = min(kDownKRange, n - k0), nch = (nk + kDownKChunk - 1) / kDownKChunk;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(
        floe_ptx::smem_u32(&tmem_base)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (t == 0) {
    for (int s2 = 0; s2 < kDownStages; ++s2) floe_ptx::mbar_init(&mdone[s2], 1);
    floe_ptx::fence_barrier_init();
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  // zero the A rows past 2B in every stage once (never written afterwards)
  for (uint32_t s2 = 0; s2 < (uint32_t)kDownStages; ++s2)
    for (uint32_t i = t; i < (128u - 2u * B) * kDownKChunk; i += 128u) {
      const uint32_t row = 2u * B + i / kDownKChunk, kk = i % kDownKChunk;
      *reinterpret_cast<__half *>(smem + s2 * ST + kmaj_off128(row, 2u * kk)) = __float2half_rn(0.0f);
    }
  __syncthreads();
  const uint32_t tmem = tmem_base;
  // stage c: B = down rows (cp.async gather), A = coefficient hi/lo rows
  auto load = [&](uint32_t c) {
    uint8_t *st = smem + (c % kDownStages) * ST;
    const uint32_t kc0 = k0 + c * kDownKChunk;
    // B: 64 channels x 32 pieces of 16 B (8 n each)
    for (uint32_t i = t; i < kDownKChunk * 32u; i += 128u) {
      const uint32_t kk = i >> 5, piece = i & 31u;
      uint8_t *dst = st + SA + (kk & 7u) * 16u + piece * 128u + (kk >> 3) * (NS / 8u * 128u);
      if (kc0 + kk < k0 + nk) {
        const uint8_t *src = reinterpret_cast<const uint8_t *>(records + (size_t)uc[kc0 + kk] * 2 * DH +
                                                               DH + m0) + 16u * piece;
        cp_async16(dst, src);
      } else {
        *reinterpret_cast<uint4 *>(dst) = make_uint4(0u, 0u, 0u, 0u);
      }
    }
    // A: rows 2t (hi), 2t+1 (lo) for t < B (rows past 2B stay zero from the
    // start); coefficients read token-contiguous
    for (uint32_t i = t; i < kDownKChunk * B; i += 128u) {
      const uint32_t kk = i / B, tok = i % B;
      const float a = kc0 + kk < k0 + nk ? A[(size_t)kc0 * B + i] * asc[tok] : 0.0f;
      const __half hi = __float2half_rn(a), lo = __float2half_rn(a - __half2float(hi));
      *reinterpret_cast<__half *>(st + kmaj_off128(2u * tok, 2u * kk)) = hi;
      *reinterpret_cast<__half *>(st + kmaj_off128(2u * tok + 1u, 2u * kk)) = lo;
    }
  };
  const uint32_t idesc = (1u << 4) | (1u << 16) | ((NS >> 3) << 17) | ((128u >> 4) << 24);
  auto descA = [](uint32_t saddr) -> uint64_t {
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)(128u >> 4) << 16) |
           ((uint64_t)(1024u >> 4) << 32) | ((uint64_t)1 << 46);
  };
  auto descB = [](uint32_t saddr) -> uint64_t {
    return (uint64_t)((saddr >> 4) & 0x3fffu) | ((uint64_t)((NS / 8u * 128u) >> 4) << 16) |
           ((uint64_t)(128u >> 4) << 32) | ((uint64_t)1 << 46);
  };
  for (uint32_t c = 0; c < kDownStages - 1; ++c) {  // (empty groups keep the count uniform)
    if (c < nch) load(c);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (uint32_t c = 0; c < nch; ++c) {
    if (c + kDownStages - 1 < nch) {
      if (c >= 1)  // stage of chunk c + 2 was last read by the MMAs of chunk c - 1
        floe_ptx::mbar_wait(&mdone[(c - 1) % kDownStages], ((c - 1) / kDownStages) & 1u, c);
      load(c + kDownStages - 1);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(kDownStages - 1) : "memory");
    asm volatile("fence.proxy.async.shared::cta;");
    __syncthreads();
    if (t == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;");
      const uint32_t a0 = floe_ptx::smem_u32(smem + (c % kDownStages) * ST), b0 = a0 + SA;
#pragma unroll
      for (uint32_t kk = 0; kk < kDownKChunk / 16u; ++kk) {
        const uint32_t acc = (c > 0 || kk > 0) ? 1u : 0u;
        asm volatile(
            "{\n\t.reg .pred q;\n\tsetp.ne.b32 q, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, q;\n\t}" ::"r"(tmem),
            "l"(descA(a0 + kk * 256u)), "l"(descB(b0 + kk * 2u * (NS / 8u * 128u))), "r"(idesc),
            "r"(acc));
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          floe_ptx::smem_u32(&mdone[c % kDownStages])));
    }
  }
  floe_ptx::mbar_wait(&mdone[(nch - 1) % kDownStages], ((nch - 1) / kDownStages) & 1u, 998u);
  asm volatile("tcgen05.fence::after_thread_sync;");
  // epilogue: TMEM lane = row 2t + h; the hi and lo rows are adjacent lanes
  const uint32_t row = warp * 32u + lane, tok = row >> 1;
  if (warp * 16u < B) {  // this warp holds tokens 16 warp .. 16 warp + 15
    for (uint32_t c0 = 0; c0 < NS; c0 += 16u) {
      uint32_t r[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
            "=r"(r[14]), "=r"(r[15])
          : "r"(tmem + ((warp * 32u) << 16) + c0));
      asm volatile("tcgen05.wait::ld.sync.aligned;");
      float f[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float mine = __uint_as_float(r[i]);
        f[i] = (mine + __shfl_xor_sync(0xffffffffu, mine, 1)) * inv_asc[min(tok, B - 1)];  // hi + lo
      }
      if (!(row & 1u) && tok < B)
#pragma unroll
        for (int i = 0; i < 16; i += 4)
          floe_k::red_add_v4(y + (size_t)tok * DH + m0 + c0 + i, f[i], f[i + 1], f[i + 2], f[i + 3]);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem));
}

// Grid (DH / 1024 column chunks) x (row chunks): each CTA reads 2 KB of each of
// its union rows' down halves (a warp: 256 contiguous bytes), thread = 4
// columns x 16 tokens in registers, token groups of 16 in turn; partial sums
// are added into y (zeroed by the caller) with vector reductions.
constexpr uint32_t kDownRowCap = 128;  // union rows per CTA (staged in shared memory)

template <int DH>
__global__ void __launch_bounds__(256) down_accum(const __half *__restrict__ records,
                                                  uint32_t B, const uint32_t *__restrict__ count,
                                                  const uint32_t *__restrict__ uc,
                                                  const float *__restrict__ A, float *__restrict__ y) {
  const uint32_t n = *count;
  const uint32_t r0 = (uint32_t)(((uint64_t)n * blockIdx.y) / gridDim.y);
  const uint32_t r1 = (uint32_t)(((uint64_t)n * (blockIdx.y + 1)) / gridDim.y);
  const uint32_t col = blockIdx.x * 1024u + 4u * threadIdx.x;
  // the chunk's channel ids and coefficients (row stride padded to 4 tokens)
  // in shared memory: record loads do not wait on them, coefficients are
  // broadcast 16-byte reads
  __shared__ uint32_t ucs[kDownRowCap];
  extern __shared__ __align__(16) float As[];  // [r1 - r0][B4]
  const uint32_t B4 = (B + 3u) & ~3u;
  const uint32_t nr = r1 - r0;  // <= kDownRowCap (host sizes the grid for it)
  for (uint32_t i = threadIdx.x; i < nr; i += blockDim.x) ucs[i] = uc[r0 + i];
  for (uint32_t i = threadIdx.x; i < nr * B4; i += blockDim.x) {
    const uint32_t r = i / B4, t = i % B4;
    As[i] = t < B ? A[(size_t)(r0 + r) * B + t] : 0.0f;
  }
  __syncthreads();
  for (uint32_t tg = 0; tg < B4; tg += 16u) {
    const uint32_t nq = min(4u, (B4 - tg) / 4u);  // token quads in this group
    float2 acc[16][2];
#pragma unroll
    for (int t = 0; t < 16; ++t) acc[t][0] = acc[t][1] = make_float2(0.0f, 0.0f);
    auto row = [&](uint32_t r, uint2 d) {
      const float2 d01 = __half22float2(*reinterpret_cast<const __half2 *>(&d.x));
      const float2 d23 = __half22float2(*reinterpret_cast<const __half2 *>(&d.y));
      const float4 *aq = reinterpret_cast<const float4 *>(As + (size_t)r * B4 + tg);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if ((uint32_t)q < nq) {
          const float4 a4 = aq[q];
          const float av[4] = {a4.x, a4.y, a4.z, a4.w};
#pragma unroll
          for (int k = 0; k < 4; ++k) {
            const float2 a2 = make_float2(av[k], av[k]);
            acc[4 * q + k][0] = __ffma2_rn(a2, d01, acc[4 * q + k][0]);
            acc[4 * q + k][1] = __ffma2_rn(a2, d23, acc[4 * q + k][1]);
          }
        }
      }
    };
    uint32_t r = 0;
    for (; r + 8u <= nr; r += 8u) {  // eight rows' loads in flight
      uint2 d[8];
#pragma unroll
      for (int k = 0; k < 8; ++k)
        d[k] = __ldg(reinterpret_cast<const uint2 *>(records + (size_t)ucs[r + k] * 2 * DH + DH + col));
#pragma unroll
      for (int k = 0; k < 8; ++k) row(r + k, d[k]);
    }
    for (; r < nr; ++r)
      row(r, __ldg(reinterpret_cast<const uint2 *>(records + (size_t)ucs[r] * 2 * DH + DH + col)));
    if (nr > 0)
#pragma unroll
      for (int t = 0; t < 16; ++t)
        if (tg + (uint32_t)t < B)
          floe_k::red_add_v4(y + (size_t)(tg + t) * DH + col, acc[t][0].x, acc[t][0].y,
                             acc[t][1].x, acc[t][1].y);
  }
}

}  // namespace floe_tc
