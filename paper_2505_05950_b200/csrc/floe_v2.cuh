// floe_v2.cuh -- the sm_100a fast path: ONE warp-specialised persistent
// kernel per decode step over a tile-fragment HBM layout of the INT2 up
// projection, with the up-projection GEMV on the tensor cores (exact integer
// IMMA).
//
// Reference (paths relative to /root/reference/proj/):
//   block_forward / route        core/src/model.cpp:145-169, 83-93   (phase A)
//   qgemv_channels + threshold   core/src/quant.cpp:122-136, model.cpp:135 (phase B)
//   gate dot + silu + down       core/src/model.cpp:136-140, la.cpp:25-31 (phase C)
//
// ---------------------------------------------------------------------------
// Up projection as an exact integer tensor-core product.
//
//   v[c] = sum_s  scale[c,s] * sum_{k in span s} code[c,k] * x[k]  +  zero[c,s] * sum_{k in s} x[k]
//
// (the group-affine dequant code*scale+zero of dequantize_at, quant.cpp:104-109,
// folded out of the inner sum; s runs over 64-element spans, each inside one
// quantisation group because g % 64 == 0).  x is scaled once per call by
// S = 2^(22-E) (max|x| < 2^E) to a 23-bit integer X = X0 + 256 X1 + 65536 X2
// with signed 8-bit limbs, and sum code*X is computed EXACTLY with
// mma.sync m16n8k32 s8.s8.s32 (IMMA): A = 16 channels x 32 codes (0..3 as s8),
// B = 32 x-positions x 8 columns, columns 0..2 = the three limbs.  One IMMA
// covers 512 weights; two cover a 64-element span of 16 channels.  The limb
// columns land in lanes tig=0 (limbs 0,1) and tig=1 (limb 2) of each quad, so
// each lane scales its own columns (mult = 1/S or 65536/S) and a final quad
// reduction sums them -- no shuffles in the inner loop.
//
// Tile-fragment HBM layout of one expert's up projection (built at upload by
// tile_up; bit-exact dequant from it is checked by dequant_tiled):
//   tile t = channels [16t, 16t+16) (zero-padded past d_intermediate), 5*DH bytes:
//   codes [pair p < DH/128][lane < 32][4 x u32]    = 4*DH bytes
//         lane = 4*g + tig; the 4 words are word `tig` (codes 16tig..16tig+15)
//         of (row g, span 2p), (row g+8, span 2p), (row g, span 2p+1), (row g+8, span 2p+1)
//   meta  [pair p][g < 8][4 x u32]                 = DH bytes
//         scale16 | zero16 << 16 of the group of the same four (row, span)
// so every lane reads its IMMA A-fragments with one conflict-free LDS.128 per
// two spans.  Extracting 2-bit codes to s8: (w >> 2m) & 0x03030303 gives bytes
// = codes 16tig + 4b + m, which fixes the logical k order; the B table (x limbs)
// is built in the same order once per call.
#pragma once

#include <type_traits>

#include "floe_kernels.cuh"
#include "floe_ptx.cuh"

namespace floe_v2 {

using floe_k::ExpertDesc;
using floe_k::h2f;

constexpr int kTileCh = 16;
constexpr int kConsumerWarps = 16;
constexpr int kConsumers = 32 * kConsumerWarps;   // 512
constexpr int kThreads = kConsumers + 64;         // + 1 producer warp + 1 router warp
constexpr int kPairs = kConsumerWarps / 2;        // stage owners in phases A/B: warps p, p+8
constexpr int kMaxStages = 24;  // ring stages: a multiple of kPairs (see phase B)
constexpr int kMaxGrid = 256;                     // plan scans: one value per consumer
#ifndef FLOE_KR
#define FLOE_KR 2
#endif
constexpr int kR = FLOE_KR;                             // phase-C records per consumer barrier
constexpr int kMaxRowsPerCta = 28;                // phase-A router slice in smem (dh/148 rows)

__host__ __device__ constexpr uint32_t tile_bytes(uint32_t dh) { return 5u * dh; }
__host__ __device__ constexpr uint32_t xtab_bytes(uint32_t dh) { return (dh / 128u) * 2u * 32u * 16u; }
__host__ __device__ inline uint32_t tiles_per_expert(uint32_t di) { return (di + kTileCh - 1) / kTileCh; }

// ------------------------------------------------------------ layout kernels
// Reference codes/scales/zeros (device) -> tile-fragment layout.
__global__ void tile_up(const uint8_t *codes, const uint16_t *scales, const uint16_t *zeros,
                        uint32_t dh, uint32_t di, uint32_t gsize, uint32_t *out) {
  const uint32_t tb = tile_bytes(dh) / 4;  // u32 per tile
  const uint32_t code_w = dh;              // u32 of codes per tile (4*dh bytes)
  const uint64_t n = (uint64_t)tiles_per_expert(di) * tb;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(i / tb), q = (uint32_t)(i % tb);
    uint32_t row, span, word;
    const bool is_code = q < code_w;
    if (is_code) {
      const uint32_t k = q & 3, lane = (q >> 2) & 31, p = q >> 7;
      row = (lane >> 2) + 8 * (k & 1);
      span = 2 * p + (k >> 1);
      word = lane & 3;
    } else {
      const uint32_t m = q - code_w;
      const uint32_t k = m & 3, g = (m >> 2) & 7, p = m >> 5;
      row = g + 8 * (k & 1);
      span = 2 * p + (k >> 1);
      word = 0;
    }
    const uint32_t c = t * kTileCh + row;
    uint32_t val = 0;
    if (c < di) {
      const uint64_t e0 = (uint64_t)c * dh + 64u * span;  // first element of the span
      if (is_code) {
        val = *reinterpret_cast<const uint32_t *>(codes + e0 / 4 + 4u * word);
      } else {
        const uint64_t grp = e0 / gsize;
        val = (uint32_t)scales[grp] | ((uint32_t)zeros[grp] << 16);
      }
    }
    out[i] = val;
  }
}

// Inverse of tile_up: the tile layout -> the reference packing (codes,
// scales, zeros; quant.hpp:20-31).  Groups of g > 64 elements appear in
// several spans with the same scale|zero, written identically.
__global__ void untile_up(const uint32_t *tiles, uint32_t dh, uint32_t di, uint32_t gsize,
                          uint8_t *codes, uint16_t *scales, uint16_t *zeros) {
  const uint32_t tb = tile_bytes(dh) / 4;
  const uint32_t code_w = dh;
  const uint64_t n = (uint64_t)tiles_per_expert(di) * tb;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t t = (uint32_t)(i / tb), q = (uint32_t)(i % tb);
    uint32_t row, span, word;
    const bool is_code = q < code_w;
    if (is_code) {
      const uint32_t k = q & 3, lane = (q >> 2) & 31, p = q >> 7;
      row = (lane >> 2) + 8 * (k & 1);
      span = 2 * p + (k >> 1);
      word = lane & 3;
    } else {
      const uint32_t m = q - code_w;
      const uint32_t k = m & 3, g = (m >> 2) & 7, p = m >> 5;
      row = g + 8 * (k & 1);
      span = 2 * p + (k >> 1);
      word = 0;
    }
    const uint32_t c = t * kTileCh + row;
    if (c >= di) continue;
    const uint64_t e0 = (uint64_t)c * dh + 64u * span;
    const uint32_t val = tiles[i];
    if (is_code) {
      *reinterpret_cast<uint32_t *>(codes + e0 / 4 + 4u * word) = val;
    } else {
      const uint64_t grp = e0 / gsize;
      scales[grp] = (uint16_t)(val & 0xffffu);
      zeros[grp] = (uint16_t)(val >> 16);
    }
  }
}

// dequantize (quant.cpp:104-120) from the tile layout: bit-exact (one fmaf of
// an exact product, like the reference's mul-then-add).
__global__ void dequant_tiled(const uint32_t *tiles, uint32_t dh, uint32_t di, float *out) {
  const uint64_t n = (uint64_t)dh * di;
  const uint32_t tb = tile_bytes(dh) / 4;
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint32_t c = (uint32_t)(i / dh), kk = (uint32_t)(i % dh);
    const uint32_t t = c / kTileCh, row = c % kTileCh, span = kk / 64, e = kk % 64;
    const uint32_t p = span / 2, kidx = (span & 1) * 2 + (row >= 8);
    const uint32_t lane = 4 * (row & 7) + e / 16;
    const uint32_t *tile = tiles + (uint64_t)t * tb;
    const uint32_t w = tile[(p * 32 + lane) * 4 + kidx];
    const uint32_t m = tile[dh + (p * 8 + (row & 7)) * 4 + kidx];
    const uint32_t code = (w >> (2 * (e % 16))) & 3u;
    out[i] = fmaf((float)code, h2f((uint16_t)(m & 0xffffu)), h2f((uint16_t)(m >> 16)));
  }
}

// --------------------------------------------------------------- K1 tile math
__device__ __forceinline__ void imma16832(int (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                          uint32_t a3, uint32_t b0, uint32_t b1) {
  asm("mma.sync.aligned.m16n8k32.row.col.s32.s8.s8.s32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+r"(c[0]), "+r"(c[1]), "+r"(c[2]), "+r"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// One 64-element span of 16 channels: wa/wb = this lane's code word of rows
// g / g+8, xb = the lane's B fragments (column groupID) for the span's two
// IMMAs, mg/mg8 = scale|zero of rows g / g+8.
//
// Code extraction in two classes, without per-class shifts: bits 0-1 of each
// byte (`& 0x03030303`, class x1: codes 4b+0 / 4b+2) and bits 2-3 left in
// place (`& 0x0C0C0C0C`, class x4: 4 * codes 4b+1 / 4b+3), one shift by 4
// for the second IMMA -- 5 ops per code word instead of 7.  The classes sit
// in the k-halves of each IMMA; the B columns separate them (columns 0,1,4
// carry limbs 0,1,2 of the class-x1 elements and are zero on class-x4 rows,
// columns 2,3,6 the converse), so lane tig of a quad holds one class and
// limb pair and scales it by its own constant `mult` (1, 1/4, 65536, 16384
// times 1/S).
__device__ __forceinline__ void span_step(float2 &acc, uint32_t wa, uint32_t wb, uint4 xb,
                                          uint32_t mg, uint32_t mg8, float zxs, float mult) {
  constexpr uint32_t M1 = 0x03030303u, M4 = 0x0C0C0C0Cu;
  int c[4] = {0, 0, 0, 0};
  imma16832(c, wa & M1, wb & M1, wa & M4, wb & M4, xb.x, xb.y);
  const uint32_t wa4 = wa >> 4, wb4 = wb >> 4;
  imma16832(c, wa4 & M1, wb4 & M1, wa4 & M4, wb4 & M4, xb.z, xb.w);
  // exact in f32: |c0 + 256 c1| < 2^24 for every class/limb pair
  const float2 t2 = make_float2((float)(c[0] + 256 * c[1]), (float)(c[2] + 256 * c[3]));
  const float2 s2 = __fmul2_rn(make_float2(h2f((uint16_t)(mg & 0xffffu)), h2f((uint16_t)(mg8 & 0xffffu))),
                               make_float2(mult, mult));
  const float2 z2 = make_float2(h2f((uint16_t)(mg >> 16)), h2f((uint16_t)(mg8 >> 16)));
  acc = __ffma2_rn(s2, t2, __ffma2_rn(z2, make_float2(zxs, zxs), acc));
}

// v of rows (g, g+8) over span quarter `qtr` (16 spans) of one tile in stage
// memory; all four lanes of a quad return the same pair.
constexpr int kQ = 4;  // warps per K1 tile (span quarters)
template <int DH>
__device__ __forceinline__ float2 k1_tile(const uint8_t *stage, const uint8_t *xtab,
                                          const float *xs, float mult, float zx, uint32_t lane,
                                          uint32_t qtr) {
  constexpr int PAIRS = DH / (128 * kQ);  // span pairs of this quarter of the tile
  const uint4 *cw = reinterpret_cast<const uint4 *>(stage + qtr * PAIRS * 32 * 16) + lane;
  const uint4 *mw = reinterpret_cast<const uint4 *>(stage + 4 * DH + qtr * PAIRS * 8 * 16) +
                    (lane >> 2);
  const uint4 *xw = reinterpret_cast<const uint4 *>(xtab + qtr * PAIRS * 64 * 16) + lane;
  xs += qtr * PAIRS * 2;
  float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll 4
  for (int p = 0; p < PAIRS; ++p) {
    const uint4 c4 = cw[p * 32];
    const uint4 m4 = mw[p * 8];
    const uint4 x0 = xw[p * 64], x1 = xw[p * 64 + 32];
    const float2 xsp = *reinterpret_cast<const float2 *>(xs + 2 * p);
    span_step(acc, c4.x, c4.y, x0, m4.x, m4.y, xsp.x * zx, mult);
    span_step(acc, c4.z, c4.w, x1, m4.z, m4.w, xsp.y * zx, mult);
  }
  acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
  acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
  acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 2);
  acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 2);
  return acc;
}

// Non-finite x (inf/NaN cannot be limb-encoded): the reference's own f32
// expression float(code)*scale + zero per element, so NaN/inf propagate exactly
// as in qgemv_channels.  xf = x in shared memory.
template <int DH>
__device__ __noinline__ float2 k1_tile_f32(const uint8_t *stage, const float *xf, uint32_t lane,
                                           uint32_t qtr) {
  const uint32_t *cw = reinterpret_cast<const uint32_t *>(stage);
  const uint32_t *mw = reinterpret_cast<const uint32_t *>(stage + 4 * DH);
  const uint32_t g = lane >> 2, tig = lane & 3;
  constexpr uint32_t SPQ = DH / 64 / kQ;  // spans per quarter
  float2 acc = make_float2(0.0f, 0.0f);
  for (uint32_t span = qtr * SPQ; span < (qtr + 1) * SPQ; ++span) {
    const uint32_t p = span / 2, hi = span & 1;
    for (uint32_t r = 0; r < 2; ++r) {
      const uint32_t kidx = hi * 2 + r;
      const uint32_t w = cw[(p * 32 + lane) * 4 + kidx];
      const uint32_t m = mw[(p * 8 + g) * 4 + kidx];
      const float sc = h2f((uint16_t)(m & 0xffffu)), zr = h2f((uint16_t)(m >> 16));
      float s = 0.0f;
      for (uint32_t q = 0; q < 16; ++q)
        s = fmaf(fmaf((float)((w >> (2 * q)) & 3u), sc, zr), xf[64 * span + 16 * tig + q], s);
      if (r == 0) acc.x += s;
      else acc.y += s;
    }
  }
  acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 1);
  acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 1);
  acc.x += __shfl_xor_sync(0xffffffffu, acc.x, 2);
  acc.y += __shfl_xor_sync(0xffffffffu, acc.y, 2);
  return acc;
}

// ----------------------------------------------------------------- utilities
// Named barriers.  __syncwarp() first: an inline-asm barrier is not a
// reconvergence point for the compiler, and a warp arriving diverged would be
// counted twice.
__device__ __forceinline__ void cbar() {  // consumers
  __syncwarp();
  asm volatile("barrier.sync 1, %0;" ::"n"(kConsumers) : "memory");
}
__device__ __forceinline__ void qbar(uint32_t quad) {  // the four warps of a K1 quad
  __syncwarp();
  asm volatile("barrier.sync %0, 128;" ::"r"(3 + quad) : "memory");
}
__device__ __forceinline__ void gbar(uint32_t grp) {  // phase C: one 8-warp record group
  __syncwarp();
  asm volatile("barrier.sync %0, 256;" ::"r"(11 + grp) : "memory");
}

__device__ __forceinline__ void mbar_arrive1(uint64_t *bar) { floe_ptx::mbar_arrive(bar); }

// Programmatic dependent launch: the next fused launch on the stream may start
// its prologue (barrier init, weight prefetch) while this grid drains; it
// waits for this grid's completion before touching anything this grid
// writes or reads (workspace, h/x, y).
__device__ __forceinline__ void pdl_launch_dependents() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

constexpr int kTraceSlots = 96;

// Grid barrier on a monotonic counter; called by consumer thread 0 only,
// between two consumer barriers.
__device__ __forceinline__ void grid_arrive_wait(unsigned long long *bar, uint32_t G) {
  __threadfence();
  const unsigned long long old = atomicAdd(bar, 1ull);
  const unsigned long long target = (old / G + 1) * G;
  const unsigned long long t0 = gtime();
  for (uint32_t it = 1;; ++it) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(bar) : "memory");
    if (v >= target) break;
    if ((it & 255u) == 0 && gtime() - t0 > floe_ptx::kWatchdogNs)
      floe_ptx::watchdog_fire("grid barrier", (uint32_t)(target / G), (uint32_t)(old % G));
  }
  __threadfence();
}



// Early record issue: the producer polls the kept list (release/acquire on
// shared-memory flag words) and streams records before K1 ends.
// compute-sanitizer's racecheck does not model release/acquire on shared
// memory and reports every such handoff as a hazard; the racecheck build
// (-DFLOE_RACECHECK) compiles the polling out, so the list is read only after
// the mbarrier that closes it, and racecheck checks everything else.
// The same build also makes every consumer thread observe the mbarriers that
// one thread waited on before a named-barrier handoff (racecheck only credits
// the thread that waited; floe_v3.cuh phase A).
#ifdef FLOE_RACECHECK
constexpr bool kRacecheck = true;
#else
constexpr bool kRacecheck = false;
#endif
constexpr bool kEarlyRecords = !kRacecheck;

// shared-memory flag words of the producer <-> consumer list protocol
__device__ __forceinline__ uint32_t ld_acquire_s(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.cta.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(floe_ptx::smem_u32(p))
               : "memory");
  return v;
}
__device__ __forceinline__ void st_release_s(uint32_t *p, uint32_t v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(floe_ptx::smem_u32(p)), "r"(v)
               : "memory");
}

// -------------------------------------------------------------- the kernel
//
// One persistent CTA per SM: 16 consumer warps, 1 producer warp (lane 0
// issues every bulk copy), 1 router warp (layer mode: exact routing).  All
// weight bytes flow through ONE ring of `ns` 20 KB stages, in one sequence of
// ring uses per CTA:
//   [mixing rows]  [K1 tiles of the predicted experts]  [own kept records]
// Layer mode:
//   * at kernel start the consumers compute PREDICTED logits router_pred * h
//     (router_pred = router + router * mixing, so router_pred * h ==
//     router * (h + mixing * h) up to f32 rounding) and the producer streams
//     the predicted experts' K1 tiles right behind the mixing rows: the ring is
//     full of K1 tiles when phase A ends;
//   * phase A (mixing GEMV, u, y = u, partial router logits), ONE grid barrier;
//   * the router warp computes the EXACT routing from the partial logits
//     (model.cpp:83-93) while the consumers run K1 on the predicted experts;
//     the prediction is checked before any record is issued, and a
//     misprediction re-runs K1 on the exact experts (tests force it);
//   * K1 epilogues append kept channels to the CTA's own list in shared memory
//     and the producer streams their gate|down records as they appear, so the
//     records flow in while the last K1 tiles are still being consumed;
//   * phase C: the CTA's own kept records, no second grid barrier.
// Expert mode: no phase A; K1 starts at once; y is zeroed by CTA 0 and the
// other CTAs check a per-call flag before their final y reduction.
struct FusedArgs {
  int has_mixing;  // layer mode (phase A) vs single-expert mode
  int k1_only;     // qgemv_channels / predict_mask: no phase C
  // phase A
  const void *mixing;  // [DH][DH] f16 or f32
  int mix_f16;
  const float *h;
  const float *router;       // [E][DH]
  const float *router_pred;  // [E][DH] router + router * mixing (layer mode)
  uint32_t n_experts, top_k;
  float *partial;  // [32][kMaxGrid] per-CTA partial router logits
  float *pred_partial;       // [32][kMaxGrid] per-CTA partial predicted logits
  unsigned long long *pcnt;  // monotonic count of published predicted partials
  float *u_trace;
  uint32_t *sel_trace;
  float *w_trace;
  uint32_t *sel_out;
  float *w_out;
  // expert input/outputs
  const float *x;  // expert mode input (layer mode: x = u)
  float *u;        // layer mode: block input u (written in phase A)
  float *y;        // output (nullable when k1_only)
  uint32_t di, slots;
  const ExpertDesc *table;  // layer: [E]; expert mode: [slots]
  int use_threshold;
  float threshold;
  float *v_out;          // nullable [slots][di]
  uint8_t *mask_out;     // nullable [slots][di]
  uint32_t *n_kept_out;  // nullable [slots]
  uint32_t *kept_out;    // nullable [slots][di], unordered
  uint32_t *kcount;      // [kMaxSlots] per-call kept counts (zero between calls)
  unsigned long long *tick;    // monotonic CTA ticket (last CTA publishes the counts)
  unsigned long long *bar;     // monotonic grid-barrier counter
  unsigned long long *y_flag;  // expert mode: [0] index + 1 of the last call whose y is
                               // zeroed, [1] monotonic CTA count (G per call)
  unsigned long long *stats;
  unsigned long long *place_acc;  // nullable [2]: kept records read from HBM / over PCIe
  unsigned long long *phase_ns;   // nullable [G][kTraceSlots]
  int paired;          // launched as clusters of 2: the CTA pair balances phase C over DSMEM
  const void *next_mixing;      // nullable: the next launch's mixing matrix (L2 prefetch)
  uint64_t next_mixing_bytes;
  unsigned long long *pf_tick;  // monotonic ticket: the order CTAs finish issuing records
  uint32_t ns;         // ring stages
  uint32_t max_tiles;  // per-CTA tile capacity of the shared-memory kept list
  uint32_t debug;      // test hook: bit 3 = invert the predicted logits (misprediction path)
  uint32_t early;      // mixing stages issued before griddepcontrol.wait
};

// Dynamic shared memory layout (bytes), host and device agree.
struct SmemLayout {
  uint32_t ring, uni, ubuf, xs, lf, lv, total;
};

__host__ __device__ inline SmemLayout smem_layout(uint32_t dh, uint32_t ns, uint32_t max_tiles,
                                                  uint32_t G) {
  (void)G;
  SmemLayout L;
  uint32_t o = 0;
  L.ring = o; o += ns * tile_bytes(dh);
  L.uni = o;  o += xtab_bytes(dh);  // K1 B fragments (x limbs)
  L.ubuf = o; o += 4u * dh;          // phase A: h; then x (u in layer mode), f32
  L.xs = o;   o += 4u * (dh / 64);
  L.lf = o;   o += 4u * kTileCh * max_tiles;  // kept list: flattened channel | kValid
  L.lv = o;   o += 4u * kTileCh * max_tiles;  //            v
  L.total = (o + 127u) & ~127u;
  return L;
}

constexpr uint32_t kValid = 0x80000000u;
#ifndef FLOE_EARLY_STAGES
#define FLOE_EARLY_STAGES 2
#endif
constexpr uint32_t kEarly = FLOE_EARLY_STAGES;  // mixing stages issued before griddepcontrol.wait

// Phase trace (diagnostics): %globaltimer at fixed points by consumer thread 0
// (marks 0..15), producer lane 0 (16..23) and router lane 0 (24..27).
__device__ __forceinline__ void mark(const FusedArgs &a, int k) {
  if (a.phase_ns && k < kTraceSlots) a.phase_ns[blockIdx.x * kTraceSlots + k] = gtime();
}

// Ring geometry, fixed per d_hidden so every ring index is a shift or a
// multiply by a constant (the producer is one thread: a runtime division on
// each issued copy costs ~100 cycles on its critical path).
__host__ __device__ constexpr uint32_t ring_stages(uint32_t dh) { return dh == 4096 ? 8u : 16u; }
__host__ __device__ constexpr uint32_t rec_stages(uint32_t dh) {
  return (ring_stages(dh) * tile_bytes(dh) + xtab_bytes(dh)) / (4u * dh);
}
constexpr uint32_t kSlotShift = 24;  // kept-list entry: kValid | slot << 24 | channel

// Tile i of the launch (tile-granular split of slots x tiles_per_expert over
// the grid, slots interleaved: every CTA gets the same channel range of each
// slot, so its kept-record count does not depend on which expert keeps more
// channels for this token): slot, tile within expert, channel count,
// flattened position.
struct TileRef {
  uint32_t slot, t, nc, f0;
};
__device__ __forceinline__ TileRef tile_ref(uint32_t i, uint32_t slots, uint32_t di) {
  TileRef r;
  r.slot = i % slots;
  r.t = i / slots;
  r.nc = min((uint32_t)kTileCh, di - r.t * kTileCh);
  r.f0 = r.slot * di + r.t * kTileCh;
  return r;
}

// tile_ref without runtime divisions for 1 or 2 slots (the expert call, top-2)
__device__ __forceinline__ TileRef tile_ref2(uint32_t i, uint32_t slots, uint32_t di) {
  if (slots > 2) return tile_ref(i, slots, di);
  TileRef r;
  r.slot = slots == 2 ? (i & 1u) : 0u;
  r.t = slots == 2 ? (i >> 1) : i;
  r.nc = min((uint32_t)kTileCh, di - r.t * kTileCh);
  r.f0 = r.slot * di + r.t * kTileCh;
  return r;
}

// top_k as k warp arg-max rounds over lanes < E holding one logit each
// (la.cpp:48-61; NaN-safe total order, floe_k::topk_key); returns the
// selection as a lane mask (ascending order = rank of the set bits).
__device__ __forceinline__ uint32_t warp_topk(float lg, uint32_t lane, uint32_t E, uint32_t K) {
  const unsigned long long mykey = floe_k::topk_key(lg, lane);
  uint32_t taken = 0;
#pragma unroll 1
  for (uint32_t r = 0; r < K; ++r) {
    const bool cand = lane < E && !((taken >> lane) & 1u);
    unsigned long long bk = cand ? mykey : 0ull;
#pragma unroll 1
    for (int o = 16; o >= 1; o >>= 1) bk = max(bk, __shfl_xor_sync(0xffffffffu, bk, o));
    taken |= 1u << floe_k::topk_index(bk);
  }
  return taken;
}

template <int DH>
__global__ void __launch_bounds__(kThreads, 1) fused(const FusedArgs a) {
  constexpr uint32_t TILE_B = tile_bytes(DH);
  constexpr uint32_t REC_B = 4 * DH;
  constexpr uint32_t SPANS = DH / 64;
  static_assert(DH == 4096 || DH == 2048, "d_hidden 4096 or 2048");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[kMaxStages], empty[kMaxStages];
  __shared__ float stage_scale[kMaxStages];
  __shared__ uint64_t hbar, predbar, bar1, routebar, lreset, listbar, pubbar, ubar;
  __shared__ uint64_t peerbar, donebar, totbar;  // CTA pair: partner's list final / reads done; item count
  __shared__ uint32_t n_pub, n_total;
  __shared__ unsigned long long pc_target, y_target;
  __shared__ ExpertDesc table_s[32];
  __shared__ float rs[32 * kMaxRowsPerCta];
  __shared__ float plw[kConsumerWarps][32];  // phase A partial logits per warp
  __shared__ float rps[32 * kMaxRowsPerCta];  // router_pred slice (predicted logits)
  // predicted selection (the K1 pass) and exact routing (the records)
  __shared__ uint32_t ptaken_s, spec_ok;
  __shared__ float pthr_s[floe_k::kMaxSlots];
  __shared__ const uint8_t *ptiles_s[floe_k::kMaxSlots];
  __shared__ float ethr_s[floe_k::kMaxSlots];
  __shared__ const uint8_t *etiles_s[floe_k::kMaxSlots];
  __shared__ float w_s[floe_k::kMaxSlots];
  __shared__ const __half *rec_s[floe_k::kMaxSlots];
  __shared__ uint32_t rhost_s[floe_k::kMaxSlots];
  __shared__ uint32_t slot_cnt[floe_k::kMaxSlots], kbase_s[floe_k::kMaxSlots],
      kpos_s[floe_k::kMaxSlots];
  __shared__ uint32_t n_list;
  __shared__ uint64_t fullC[kMaxStages], emptyC[kMaxStages];
  __shared__ float redmax[kConsumerWarps];
  __shared__ float2 xch[kConsumerWarps / kQ][2][kQ - 1][8];  // phase B: quarter partials
  __shared__ float red[2][2][8][kR];    // phase C: [group][batch parity][warp][record]

  const uint32_t t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const uint32_t G = gridDim.x, b = blockIdx.x;
  const bool producer = warp == kConsumerWarps;
  const bool router_warp = warp == kConsumerWarps + 1;
  constexpr uint32_t ns = ring_stages(DH);
  const SmemLayout L = smem_layout(DH, ns, a.max_tiles, G);
  uint8_t *ring = smem + L.ring;
  float *hs = reinterpret_cast<float *>(smem + L.ubuf);  // phase A: h; then x (u), f32
  uint8_t *xtab = smem + L.uni;
  float *xs = reinterpret_cast<float *>(smem + L.xs);
  uint32_t *lf = reinterpret_cast<uint32_t *>(smem + L.lf);
  float *lv = reinterpret_cast<float *>(smem + L.lv);
  const uint32_t list_cap = kTileCh * a.max_tiles;

  // Streamed weights (read once per call) go through L2 as evict-first, so the
  // ~165 MB per layer do not evict the kernel's code, the routing partials or
  // router_pred.
  const uint64_t l2_stream = floe_ptx::policy_evict_first();
  auto stage = [&](uint32_t u) { return ring + (u % ns) * TILE_B; };
  auto wait_full = [&](uint32_t u) {
    floe_ptx::mbar_wait(&full[u % ns], (u / ns) & 1u, (1u << 28) | u);
  };
  // producer side: stage use u may be (re)filled once use u - ns is released
  auto wait_empty = [&](uint32_t u) {
    if (u >= ns) floe_ptx::mbar_wait(&empty[u % ns], ((u / ns) + 1) & 1u, (2u << 28) | u);
  };
  auto issue = [&](uint32_t u, const void *src, uint32_t bytes) {
    floe_ptx::mbar_arrive_expect_tx(&full[u % ns], bytes);
    floe_ptx::bulk_g2s_hint(stage(u), src, bytes, &full[u % ns], l2_stream);
  };
  // Phase C re-carves the ring plus the x-table area (both free once every K1
  // tile is consumed) into 4*DH-byte record stages with their own barriers:
  // 12 records (192 KB) in flight at d_hidden 4096.
  constexpr uint32_t nsC = rec_stages(DH);
  static_assert(nsC <= (uint32_t)kMaxStages, "record ring");
  auto stageC = [&](uint32_t k) { return ring + (k % nsC) * REC_B; };
  auto issueC = [&](uint32_t k, const void *src, float scale) {
    if (k >= nsC) floe_ptx::mbar_wait(&emptyC[k % nsC], ((k / nsC) + 1) & 1u, (5u << 28) | k);
    stage_scale[k % nsC] = scale;
    floe_ptx::mbar_arrive_expect_tx(&fullC[k % nsC], REC_B);
    floe_ptx::bulk_g2s_hint(stageC(k), src, REC_B, &fullC[k % nsC], l2_stream);
  };

  if (t == 0) {
    mark(a, 0);
    for (uint32_t s = 0; s < ns; ++s) {
      floe_ptx::mbar_init(&full[s], 1);
      // released by all 16 consumer warps: count 8 from each warp of the
      // owning pair (phases A/B), 2 from each warp of the record group (C)
      floe_ptx::mbar_init(&empty[s], kConsumerWarps);
    }
    for (uint32_t s = 0; s < nsC; ++s) {
      floe_ptx::mbar_init(&fullC[s], 1);
      floe_ptx::mbar_init(&emptyC[s], 8);  // the 8 warps of the record's group
    }
    floe_ptx::mbar_init(&hbar, 1);
    floe_ptx::mbar_init(&predbar, 1);
    floe_ptx::mbar_init(&bar1, 1);
    floe_ptx::mbar_init(&routebar, 1);
    floe_ptx::mbar_init(&lreset, 1);
    floe_ptx::mbar_init(&listbar, 1);  // consumers: K1 done, own list final
    floe_ptx::mbar_init(&pubbar, 1);   // warp 0: predicted partial published
    floe_ptx::mbar_init(&ubar, 1);     // x (u) in shared memory
    floe_ptx::mbar_init(&peerbar, 1);  // remote arrive: the partner's kept list is final
    floe_ptx::mbar_init(&donebar, 1);  // remote arrive: the partner finished reading ours
    floe_ptx::mbar_init(&totbar, 1);   // producer: this CTA's phase-C item count
    floe_ptx::fence_barrier_init();
    spec_ok = 1u;
    n_list = 0u;
    pdl_launch_dependents();
  }
  const uint32_t n_table = a.has_mixing ? a.n_experts : a.slots;
  if (t < n_table) table_s[t] = a.table[t];
  if (t < (uint32_t)floe_k::kMaxSlots) {
    slot_cnt[t] = 0u;
    kpos_s[t] = 0u;
  }
  for (uint32_t i = t; i < list_cap; i += kThreads) lf[i] = 0u;
  __syncthreads();
  if (!a.has_mixing && t < a.slots) {  // expert mode: the slots are the experts
    const ExpertDesc &d = table_s[t];
    const float thr = a.use_threshold ? a.threshold : d.threshold;
    pthr_s[t] = ethr_s[t] = thr;
    ptiles_s[t] = etiles_s[t] = reinterpret_cast<const uint8_t *>(d.tiles);
    w_s[t] = 1.0f;
    rec_s[t] = d.records;
    rhost_s[t] = d.host_records;
  }
  if (a.paired) floe_ptx::cluster_sync_all();  // partner barriers initialised (remote arrivals)
  else __syncthreads();

  // ---- geometry
  const uint32_t tps = tiles_per_expert(a.di);
  const uint32_t NT = a.slots * tps;
  const uint32_t tile_lo = (uint32_t)(((uint64_t)NT * b) / G);
  const uint32_t nB = (uint32_t)(((uint64_t)NT * (b + 1)) / G) - tile_lo;
  const uint32_t rpi = a.mix_f16 ? 2u : 1u;  // mixing rows per stage
  const uint32_t r_lo = floe_k::seg_begin(DH, b, G), r_hi = floe_k::seg_begin(DH, b + 1, G);
  const uint32_t nA = a.has_mixing ? (r_hi - r_lo + rpi - 1) / rpi : 0u;
  const uint32_t uB = nA;  // first K1 ring use

  if (producer) {
    // =================== producer warp ===================
    // lane 0 issues every copy; the whole warp computes the phase-C plan
    uint32_t k_early = 0;  // own records issued before the end of K1
    if (lane == 0) {
      uint32_t u = 0;
      if (a.has_mixing) {
        const uint32_t row_bytes = DH * (a.mix_f16 ? 2u : 4u);
        const uint8_t *m = static_cast<const uint8_t *>(a.mixing);
        // mixing rows are read-only weights: the first kEarly stream in before
        // the previous grid has finished (PDL); h (the previous layer's output)
        // goes right after them so it is not queued behind the whole ring
        for (uint32_t i = 0; i < nA; ++i) {
          if (i == min(nA, a.early)) {
            pdl_wait();
            floe_ptx::mbar_arrive_expect_tx(&hbar, 4u * DH);
            floe_ptx::bulk_g2s(hs, a.h, 4u * DH, &hbar);
            // h lands ahead of the burst of mixing copies every CTA issues once
            // the previous grid completes (measured: h otherwise queues 3-5 us)
            floe_ptx::mbar_wait(&hbar, 0, 3u << 28);
          }
          const uint32_t r0 = r_lo + i * rpi, nr = min(rpi, r_hi - r0);
          wait_empty(u);
          issue(u++, m + (size_t)r0 * row_bytes, nr * row_bytes);
        }
        if (nA <= a.early) {
          pdl_wait();
          floe_ptx::mbar_arrive_expect_tx(&hbar, 4u * DH);
          floe_ptx::bulk_g2s(hs, a.h, 4u * DH, &hbar);
        }
        floe_ptx::mbar_wait(&predbar, 0, 6u << 28);  // predicted routing
        mark(a, 16);
      }
      // x into shared memory (layer mode: u, complete once the grid barrier
      // passed; the K1 tiles are issued after it, not during phase A: a
      // global read waits behind the SM's queued bulk copies, and the
      // barrier's polls are global reads), then the K1 tiles of the predicted
      // (layer) / given (expert) experts
      if (a.has_mixing) {
        floe_ptx::mbar_wait(&bar1, 0, 15u << 28);
        asm volatile("fence.proxy.async.global;" ::: "memory");  // u: generic-proxy writes
      } else {
        pdl_wait();
      }
      floe_ptx::mbar_arrive_expect_tx(&ubar, 4u * DH);
      floe_ptx::bulk_g2s(hs, a.has_mixing ? a.u : a.x, 4u * DH, &ubar);
      for (uint32_t j = 0; j < nB; ++j) {
        const TileRef tr = tile_ref2(tile_lo + j, a.slots, a.di);
        wait_empty(u);
        issue(u++, ptiles_s[tr.slot] + (size_t)tr.t * TILE_B, TILE_B);
      }
      mark(a, 17);
      if (a.has_mixing && !a.k1_only) {
        floe_ptx::mbar_wait(&routebar, 0, 7u << 28);
        if (!spec_ok)  // misprediction: the exact experts' tiles follow
          for (uint32_t j = 0; j < nB; ++j) {
            const TileRef tr = tile_ref2(tile_lo + j, a.slots, a.di);
            wait_empty(u);
            issue(u++, etiles_s[tr.slot] + (size_t)tr.t * TILE_B, TILE_B);
          }
      }
      // Early records: while the last K1 tiles are consumed, record stage r
      // is filled with kept record r as soon as the ring stages under it have
      // seen their last K1 use released and the K1 epilogues have appended
      // entry r, so phase C starts on landed data instead of a cold ring.
      // Record stages over the x table wait for the end of K1.
      if (!a.k1_only && spec_ok) {
        const uint32_t uEnd = u;
        const uint32_t r_max = min(nsC, ns * TILE_B / REC_B);
        auto stages_free = [&](uint32_t r) {  // ring stages under record stage r: last use released
          const uint32_t lo = r * REC_B, hi = lo + REC_B;
          for (uint32_t st = lo / TILE_B; st <= (hi - 1) / TILE_B; ++st)
            if (uEnd > st) {
              const uint32_t us = st + ((uEnd - 1 - st) / ns) * ns;
              if (!floe_ptx::mbar_test_wait(&empty[st], (us / ns) & 1u)) return false;
            }
          return true;
        };
        // never blocks past the end of K1: once the list is final the normal
        // path issues the rest (the whole ring is free by then)
        while (k_early < r_max && !floe_ptx::mbar_test_wait(&listbar, 0)) {
          const uint32_t f = kEarlyRecords ? ld_acquire_s(&lf[k_early]) : 0u;
          if ((f & kValid) && stages_free(k_early)) {
            const uint32_t r = k_early, s2 = (f >> kSlotShift) & 0x7fu, c = f & 0xffffffu;
            issueC(r, rec_s[s2] + (size_t)c * 2 * DH, lv[r] * w_s[s2]);
            ++k_early;
          } else {
            __nanosleep(32);
          }
        }
      }
    }
    if (a.k1_only) return;
    // ---- phase C: the record ring fills as soon as K1 is done (every tile
    // consumed, the list final)
    floe_ptx::mbar_wait(&listbar, 0, 12u << 28);
    const uint32_t n_own = n_list;
    const uint32_t P = min(n_own, nsC);  // the first ring fill: always this CTA's own
    auto own_item = [&](uint32_t k) {
      const uint32_t f = lf[k], s2 = (f >> kSlotShift) & 0x7fu, c = f & 0xffffffu;
      issueC(k, rec_s[s2] + (size_t)c * 2 * DH, lv[k] * w_s[s2]);
    };
    if (lane == 0) {
      mark(a, 18);
      if (a.paired) {  // publish the list to the partner CTA (release: the list writes
        n_pub = n_own;  // were acquired through listbar)
        floe_ptx::mbar_arrive_remote(floe_ptx::mapa(&peerbar, (b ^ 1u) & 1u));
      }
      for (uint32_t k = k_early; k < P; ++k) own_item(k);
      uint32_t own = n_own, take = 0, pfirst = 0;
      const uint32_t peer = b ^ 1u;
      if (a.paired) {
        // CTA pair plan over distributed shared memory (no global round trip:
        // a global read waits behind the SM's queued bulk copies): T = n_me +
        // n_peer, even CTA target ceil(T/2), odd floor(T/2); each keeps
        // max(min(n, nsC), min(n, target)) own records and the deficit CTA
        // takes the partner's surplus from the end of its list
        floe_ptx::mbar_wait_cluster(&peerbar, 0, 17u << 28);
        const uint32_t n_p = floe_ptx::ld_cluster_u32(floe_ptx::mapa(&n_pub, peer & 1u));
        const uint32_t T = n_own + n_p;
        const uint32_t t_me = (b & 1u) ? T / 2 : (T + 1) / 2, t_p = T - t_me;
        own = max(P, min(n_own, t_me));
        const uint32_t own_p = max(min(n_p, nsC), min(n_p, t_p));
        take = t_me > own ? min(t_me - own, n_p - own_p) : 0u;
        pfirst = own_p;
      }
      n_total = own + take;
      floe_ptx::mbar_arrive(&totbar);
      for (uint32_t k = P; k < own; ++k) own_item(k);
      if (a.paired) {
        const uint32_t pr = (b ^ 1u) & 1u;
        for (uint32_t k = 0; k < take; ++k) {
          const uint32_t f =
              floe_ptx::ld_cluster_u32(floe_ptx::mapa(&lf[pfirst + k], pr));
          const float v = __uint_as_float(floe_ptx::ld_cluster_u32(floe_ptx::mapa(&lv[pfirst + k], pr)));
          const uint32_t s2 = (f >> kSlotShift) & 0x7fu, c = f & 0xffffffu;
          issueC(own + k, rec_s[s2] + (size_t)c * 2 * DH, v * w_s[s2]);
        }
        floe_ptx::mbar_arrive_remote(floe_ptx::mapa(&donebar, pr));  // done reading its list
      }
      mark(a, 19);
      // The CTAs that finish early pull the NEXT layer's mixing matrix into L2
      // (evict-last) while the slow ones still stream their records: the next
      // launch's phase A, which waits for this grid, then reads it from L2.
      // Finish order decides the chunk: the first G/2 finishers cover it all.
      if (a.next_mixing) {
        const uint32_t ticket = (uint32_t)(atomicAdd(a.pf_tick, 1ull) % G);
        const uint32_t nchunk = max(1u, G / 2);
        if (ticket < nchunk) {
          const uint64_t per = (a.next_mixing_bytes / nchunk + 4095) & ~4095ull;
          const uint64_t lo = per * ticket;
          const uint64_t hi = lo + per < a.next_mixing_bytes ? lo + per : a.next_mixing_bytes;
          const uint64_t pol = floe_ptx::policy_evict_last();
          const uint8_t *base = static_cast<const uint8_t *>(a.next_mixing);
          for (uint64_t o = lo; o < hi; o += 65536)
            floe_ptx::bulk_prefetch_l2_hint(base + o, (uint32_t)(hi - o < 65536 ? hi - o : 65536),
                                            pol);
        }
      }
    }
    return;
  }

  if (router_warp) {
    // =================== router warp (layer mode) ===================
    if (!a.has_mixing) return;
    pdl_wait();
    // sum of the per-CTA partials of E logits, the same fixed order in every
    // CTA; all loads in flight at once; lane e returns logit e
    auto sum_partials = [&](const float *part) {
      float lg = -__int_as_float(0x7f800000);
      for (uint32_t e0 = 0; e0 < a.n_experts; e0 += 8) {
        float sv[8];
#pragma unroll
        for (int ee = 0; ee < 8; ++ee) {
          const uint32_t e = e0 + ee;
          float pv[kMaxGrid / 32];
#pragma unroll
          for (int j = 0; j < kMaxGrid / 32; ++j) {
            const uint32_t bb = lane + 32 * j;
            pv[j] = (e < a.n_experts && bb < G) ? __ldcg(&part[e * kMaxGrid + bb]) : 0.0f;
          }
          float s = 0.0f;
#pragma unroll
          for (int j = 0; j < kMaxGrid / 32; ++j) s += pv[j];
          sv[ee] = s;
        }
#pragma unroll
        for (int ee = 0; ee < 8; ++ee) {
          float s = sv[ee];
#pragma unroll
          for (int o = 16; o >= 1; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == e0 + ee) lg = s;
        }
      }
      return lg;
    };
    // ---- predicted routing: wait for every CTA's predicted partials
    floe_ptx::mbar_wait(&pubbar, 0, 14u << 28);
    if (lane == 0) {
      const unsigned long long target = pc_target, t0 = gtime();
      for (uint32_t it = 1;; ++it) {
        unsigned long long v;
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a.pcnt) : "memory");
        if (v >= target) break;
        if ((it & 255u) == 0 && gtime() - t0 > floe_ptx::kWatchdogNs)
          floe_ptx::watchdog_fire("prediction", (uint32_t)(target / G), 0u);
      }
    }
    __syncwarp();
    {
      float plg = sum_partials(a.pred_partial);
      if (a.debug & 8u) plg = -plg;  // test hook: force a misprediction
      const uint32_t ptaken = warp_topk(lane < a.n_experts ? plg : -__int_as_float(0x7f800000),
                                        lane, a.n_experts, a.top_k);
      if (lane == 0) {  // the thread that arrives writes them (producer reads after predbar)
        uint32_t i = 0;
        for (uint32_t m = ptaken; m; m &= m - 1, ++i) {
          const uint32_t e = __ffs(m) - 1;
          ptiles_s[i] = reinterpret_cast<const uint8_t *>(table_s[e].tiles);
          pthr_s[i] = a.use_threshold ? a.threshold : table_s[e].threshold;
        }
        ptaken_s = ptaken;
        mark(a, 26);
        floe_ptx::mbar_arrive(&predbar);
      }
    }
    floe_ptx::mbar_wait(&bar1, 0, 10u << 28);
    if (lane == 0) mark(a, 24);
    // route (model.cpp:83-93) on the exact logits router * u
    const float lg = sum_partials(a.partial);
    // top_k (la.cpp:48-61: ties to the lower index, output ascending); softmax
    // over the selected logits (la.cpp:37-46): mx, then the sum in ascending
    // expert order
    const uint32_t taken = warp_topk(lane < a.n_experts ? lg : -__int_as_float(0x7f800000), lane,
                                     a.n_experts, a.top_k);
    const bool mine = (taken >> lane) & 1u;
    float mx = mine ? lg : -__int_as_float(0x7f800000);
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const float ex = mine ? expf(lg - mx) : 0.0f;
    float sum = 0.0f;
    for (uint32_t m = taken; m; m &= m - 1) sum += __shfl_sync(0xffffffffu, ex, __ffs(m) - 1);
    if (mine) {
      const uint32_t i = __popc(taken & ((1u << lane) - 1));  // rank = ascending position
      const float w = ex / sum;
      const ExpertDesc &d = table_s[lane];
      w_s[i] = w;
      rec_s[i] = d.records;
      rhost_s[i] = d.host_records;
      etiles_s[i] = reinterpret_cast<const uint8_t *>(d.tiles);
      ethr_s[i] = a.use_threshold ? a.threshold : d.threshold;
      if (b == 0) {
        if (a.sel_out) {
          a.sel_out[i] = lane;
          a.w_out[i] = w;
        }
        if (a.sel_trace) a.sel_trace[i] = lane;
        if (a.w_trace) a.w_trace[i] = w;
      }
    }
    __syncwarp();
    if (lane == 0) {
      spec_ok = taken == ptaken_s ? 1u : 0u;
      mark(a, 25);
      floe_ptx::mbar_arrive(&routebar);
    }
    return;
  }

  // =================== consumer warps (threads 0..511) ===================
  const uint32_t nrows = r_hi - r_lo;
  const bool rs_ok = a.has_mixing && nrows <= (uint32_t)kMaxRowsPerCta;
  if (rs_ok)
    for (uint32_t i = t; i < a.n_experts * kMaxRowsPerCta; i += kConsumers) {
      const uint32_t e = i / kMaxRowsPerCta, lr = i % kMaxRowsPerCta;
      if (lr < nrows) {
        rs[i] = a.router[(size_t)e * DH + r_lo + lr];
        rps[i] = a.router_pred[(size_t)e * DH + r_lo + lr];
      }
    }
  if (rs_ok) cbar();  // warp 0 reads every consumer's router rows in phase A
  pdl_wait();  // from here on: workspace, inputs and outputs shared with the previous grid
  if (t == 0) mark(a, 11);
  if (!a.has_mixing && a.y && !a.k1_only) {
    // expert mode: CTA 0 zeroes y, the others check a flag before their final
    // reduction; the call index comes from a counter every CTA bumps once
    if (t == 0) y_target = atomicAdd(a.y_flag + 1, 1ull) / G + 1;
    if (b == 0) {
      for (uint32_t i = t; i < DH; i += kConsumers) a.y[i] = 0.0f;
      cbar();
      if (t == 0) {
        __threadfence();
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(a.y_flag), "l"(y_target)
                     : "memory");
      }
    }
  }

  // ---- K1 operand setup (warps 8..15): x -> max|x| -> limbs (IMMA B
  // fragments) + span sums
  const bool setup_warp = warp >= kConsumerWarps / 2;
  const uint32_t ts = t - kConsumers / 2;  // setup thread index (warps 8..15)
  const bool act = setup_warp && ts < SPANS * 4;
  const uint32_t span = ts >> 2, tig = ts & 3;
  float xv[16];
  auto setup1 = [&]() {  // x from shared memory, this warp's max|x| and finiteness
    const float4 *x4 = reinterpret_cast<const float4 *>(hs + (act ? 64 * span + 16 * tig : 0));
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float4 f = x4[i];
      xv[4 * i] = f.x;
      xv[4 * i + 1] = f.y;
      xv[4 * i + 2] = f.z;
      xv[4 * i + 3] = f.w;
    }
    float mx = 0.0f;
    bool fin = true;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      mx = fmaxf(mx, fabsf(xv[i]));
      fin = fin && isfinite(xv[i]);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    const bool wfin = __all_sync(0xffffffffu, fin);
    if (lane == 0) redmax[warp] = wfin ? mx : -1.0f;
  };
  // global max|x| over the setup warps -> scale S = 2^(22 - e), max|x| < 2^e
  auto x_scale = [&](bool &fin_all, float &S, float &invS) {
    fin_all = true;
    float mx = 0.0f;
#pragma unroll
    for (int w = kConsumerWarps / 2; w < kConsumerWarps; ++w) {
      fin_all = fin_all && redmax[w] >= 0.0f;
      mx = fmaxf(mx, redmax[w]);
    }
    int ex = 0;
    frexpf(mx, &ex);  // mx < 2^ex
    const bool scaled = mx > 0.0f && fin_all;
    S = scaled ? __int_as_float((127 + 22 - ex) << 23) : 1.0f;
    invS = scaled ? __int_as_float((127 - 22 + ex) << 23) : 1.0f;
  };
  auto setup2 = [&]() {  // limbs -> xtab (or the f32 copy), span sums -> xs
    bool fin_all;
    float S, invS;
    x_scale(fin_all, S, invS);
    if (act) {
      if (fin_all) {
        int X[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) X[i] = __float2int_rn(xv[i] * S);
        const uint32_t p = span >> 1, sodd = span & 1;
        uint4 *xt = reinterpret_cast<uint4 *>(xtab) + (p * 2 + sodd) * 32;
        // limb bytes of the 16 elements: lb[l][i] for element i
        uint32_t lw[3][2][2];  // [limb][m][j]: element 4b + 2m + j, byte b
#pragma unroll
        for (int l = 0; l < 3; ++l)
#pragma unroll
          for (int m = 0; m < 2; ++m)
#pragma unroll
            for (int j = 0; j < 2; ++j) lw[l][m][j] = 0;
#pragma unroll
        for (int i = 0; i < 16; ++i) {
          const int v = X[i];
          const int l0 = ((v + 128) & 255) - 128;
          const int r1 = (v - l0) >> 8;
          const int l1 = ((r1 + 128) & 255) - 128;
          const int l2 = (r1 - l1) >> 8;
          const int bb = i >> 2, m = (i >> 1) & 1, j = i & 1;
          lw[0][m][j] |= (uint32_t)(l0 & 255) << (8 * bb);
          lw[1][m][j] |= (uint32_t)(l1 & 255) << (8 * bb);
          lw[2][m][j] |= (uint32_t)(l2 & 255) << (8 * bb);
        }
        // column n -> (class, limb): 0 (x1,L0) 1 (x1,L1) 2 (x4,L0) 3 (x4,L1)
        // 4 (x1,L2) 6 (x4,L2); 5, 7 zero.  Class x1 rides in b0 (j = 0, the
        // even elements), class x4 in b1 (j = 1, the odd elements).
#pragma unroll
        for (int n = 0; n < 8; ++n) {
          const int lim = n == 0 || n == 2 ? 0 : (n == 1 || n == 3 ? 1 : 2);
          const bool c1 = n == 0 || n == 1 || n == 4, c4 = n == 2 || n == 3 || n == 6;
          xt[4 * n + tig] = make_uint4(c1 ? lw[lim][0][0] : 0u, c4 ? lw[lim][0][1] : 0u,
                                       c1 ? lw[lim][1][0] : 0u, c4 ? lw[lim][1][1] : 0u);
        }
      }  // (not finite: K1 reads x from shared memory in f32)
    }
    float s16 = 0.0f;
#pragma unroll
    for (int i = 0; i < 16; ++i) s16 += xv[i];
    s16 += __shfl_xor_sync(0xffffffffu, s16, 1);
    s16 += __shfl_xor_sync(0xffffffffu, s16, 2);
    if (act && tig == 0) xs[span] = s16;
  };

  // ============================ phase A: mixing ============================
  if (a.has_mixing) {
    floe_ptx::mbar_wait(&hbar, 0, 3u << 28);
    // predicted logits router_pred * h (router_pred = router + router *
    // mixing), distributed like the exact ones: this CTA's rows of h give
    // per-CTA partials, published with a counter; the router warp sums them
    // in the background while phase A streams
    if (warp == 0) {
      for (uint32_t e = lane; e < a.n_experts; e += 32) {
        float s = 0.0f;
        for (uint32_t lr = 0; lr < nrows; ++lr)
          s = fmaf(rs_ok ? rps[e * kMaxRowsPerCta + lr] : a.router_pred[(size_t)e * DH + r_lo + lr],
                   hs[r_lo + lr], s);
        a.pred_partial[e * kMaxGrid + b] = s;
      }
      __syncwarp();
      if (lane == 0) {
        __threadfence();
        const unsigned long long old = atomicAdd(a.pcnt, 1ull);
        pc_target = (old / G + 1) * G;  // this call's last publication
        mark(a, 7);
        floe_ptx::mbar_arrive(&pubbar);
      }
    }
    float pl = 0.0f;  // lane e < E: this warp's partial logit e
    const uint32_t pair = warp % kPairs, sub = warp / kPairs;
    // item i (stage use i) belongs to pair i % 8; warp `sub` of the pair takes
    // row `sub` of the item (f16: 2 rows per stage; f32: 1 row, sub 1 idles)
    for (uint32_t i = pair; i < nA; i += kPairs) {
      wait_full(i);
      if (i == 0 && t == 0) mark(a, 8);
      const uint32_t r0 = r_lo + i * rpi, nr = min(rpi, r_hi - r0);
      const bool mine = sub < nr;
      float acc0 = 0.0f, acc1 = 0.0f;
      if (mine && a.mix_f16) {
        const __half *row = reinterpret_cast<const __half *>(stage(i)) + sub * DH;
#pragma unroll 4
        for (uint32_t k = lane * 8; k < DH; k += 256) {
          const float4 h0 = *reinterpret_cast<const float4 *>(hs + k);
          const float4 h1 = *reinterpret_cast<const float4 *>(hs + k + 4);
          const uint4 q0 = *reinterpret_cast<const uint4 *>(row + k);
          const __half2 *p0 = reinterpret_cast<const __half2 *>(&q0);
          float2 f;
          f = __half22float2(p0[0]); acc0 = fmaf(f.x, h0.x, acc0); acc1 = fmaf(f.y, h0.y, acc1);
          f = __half22float2(p0[1]); acc0 = fmaf(f.x, h0.z, acc0); acc1 = fmaf(f.y, h0.w, acc1);
          f = __half22float2(p0[2]); acc0 = fmaf(f.x, h1.x, acc0); acc1 = fmaf(f.y, h1.y, acc1);
          f = __half22float2(p0[3]); acc0 = fmaf(f.x, h1.z, acc0); acc1 = fmaf(f.y, h1.w, acc1);
        }
      } else if (mine) {
        const float *row = reinterpret_cast<const float *>(stage(i));
#pragma unroll 4
        for (uint32_t k = lane * 4; k < DH; k += 128) {
          const float4 h0 = *reinterpret_cast<const float4 *>(hs + k);
          const float4 q0 = *reinterpret_cast<const float4 *>(row + k);
          acc0 = fmaf(q0.x, h0.x, acc0);
          acc1 = fmaf(q0.y, h0.y, acc1);
          acc0 = fmaf(q0.z, h0.z, acc0);
          acc1 = fmaf(q0.w, h0.w, acc1);
        }
      }
      float acc = acc0 + acc1;
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
      __syncwarp();
      if (lane == 0) floe_ptx::mbar_arrive_cnt(&empty[i % ns], kPairs);  // done with the stage
      if (mine) {
        const uint32_t row = r0 + sub;
        const float uu = hs[row] + 1.0f * acc;  // drift_scale 1 (model.cpp:151-152)
        if (lane == 0) {
          a.u[row] = uu;
          a.y[row] = uu;
          if (a.u_trace) a.u_trace[row] = uu;
        }
        if (lane < a.n_experts) {
          const float w = rs_ok ? rs[lane * kMaxRowsPerCta + (row - r_lo)]
                                : a.router[(size_t)lane * DH + row];
          pl = fmaf(w, uu, pl);
        }
      }
    }
    plw[warp][lane] = pl;
    cbar();
    if (t < a.n_experts) {
      float s = 0.0f;
#pragma unroll
      for (int w = 0; w < kConsumerWarps; ++w) s += plw[w][t];
      a.partial[t * kMaxGrid + b] = s;  // [expert][CTA]: coalesced reads by the router warp
    }
    if (t == 0) mark(a, 1);
    cbar();
    if (t == 0) {
      grid_arrive_wait(a.bar, G);  // u, y = u and the partials of every CTA
      mark(a, 2);
      floe_ptx::mbar_arrive(&bar1);
    }
    cbar();
  }

  // ---- K1 setup: x limbs, span sums, epilogue multipliers
  floe_ptx::mbar_wait(&ubar, 0, 16u << 28);
  if (setup_warp) setup1();
  cbar();
  if (setup_warp) setup2();
  cbar();
  if (t == 0) mark(a, 3);
  float mult, zx;
  bool all_finite;
  {
    float S, invS;
    x_scale(all_finite, S, invS);
    const uint32_t mytig = lane & 3;
    // column pair of this lane (see span_step): (c1L0,c1L1) (c4L0,c4L1) (c1L2,-) (c4L2,-)
    mult = mytig == 0 ? invS : (mytig == 1 ? 0.25f * invS : (mytig == 2 ? 65536.0f * invS : 16384.0f * invS));
    zx = mytig == 0 ? 1.0f : 0.0f;
  }

  // ============================ phase B: K1 ================================
  // Quads of 4 warps (one per SMSP) own 2 ring stages each and alternate
  // between them, so a quad computes one tile while its other stage refills:
  // tile j (ring use u0 + j) belongs to quad ((u0 + j) % 8) / 2.  With ns a
  // multiple of 8 every stage is consumed by ONE quad in phase B and every
  // phase-A use of it was consumed before the grid barrier, so a warp never
  // waits on a stage more than one fill ahead (mbarrier parity waits cannot
  // tell phase k from phase k+2).  Warp `sub` of the quad computes span
  // quarter `sub`; the partials go through xch (double-buffered by the quad's
  // tile parity) to warp 0 of the quad, which sums them in a fixed order,
  // thresholds and appends kept channels to the CTA's list.
  auto k1_pass = [&](uint32_t u0, const float *thr_tab) {
    const uint32_t quad = warp / kQ, sub = warp % kQ;
    uint32_t n = 0;  // tiles this quad has done
    for (uint32_t j = 0; j < nB; ++j) {
      const uint32_t u = u0 + j;
      if ((u % 8) / 2 != quad) continue;
      const TileRef tr = tile_ref2(tile_lo + j, a.slots, a.di);
      wait_full(u);
      float2 v2 = all_finite ? k1_tile<DH>(stage(u), xtab, xs, mult, zx, lane, sub)
                             : k1_tile_f32<DH>(stage(u), hs, lane, sub);
      __syncwarp();
      if (lane == 0) floe_ptx::mbar_arrive_cnt(&empty[u % ns], kConsumerWarps / kQ);
      if (sub != 0 && (lane & 3) == 0) xch[quad][n & 1][sub - 1][lane >> 2] = v2;
      qbar(quad);
      const uint32_t nb = n++;
      if (sub != 0) continue;
#pragma unroll
      for (int q = 0; q < kQ - 1; ++q) {
        const float2 o2 = xch[quad][nb & 1][q][lane >> 2];
        v2.x += o2.x;
        v2.y += o2.y;
      }
      const uint32_t g = lane >> 2;
      const bool q0 = (lane & 3) == 0;
      const float thr = thr_tab[tr.slot];
      // model.cpp:135: `if (fabs(v) < t) continue;` -> ties and NaN are kept
      const bool va = q0 && g < tr.nc, vb = q0 && g + 8 < tr.nc;
      const bool ka = va && !(fabsf(v2.x) < thr), kb = vb && !(fabsf(v2.y) < thr);
      const size_t o = (size_t)tr.f0;
      if (a.v_out) {
        if (va) a.v_out[o + g] = v2.x;
        if (vb) a.v_out[o + g + 8] = v2.y;
      }
      if (a.mask_out) {
        if (va) a.mask_out[o + g] = ka ? 1 : 0;
        if (vb) a.mask_out[o + g + 8] = kb ? 1 : 0;
      }
      const uint32_t ba = __ballot_sync(0xffffffffu, ka), bbal = __ballot_sync(0xffffffffu, kb);
      const uint32_t na = __popc(ba), cnt = na + __popc(bbal);
      if (cnt == 0) continue;
      uint32_t base = 0;
      if (lane == 0) {
        base = atomicAdd(&n_list, cnt);
        atomicAdd(&slot_cnt[tr.slot], cnt);
      }
      base = __shfl_sync(0xffffffffu, base, 0);
      const uint32_t lt = (1u << lane) - 1;
      if (ka) {
        const uint32_t pos = base + __popc(ba & lt);
        lv[pos] = v2.x;
        st_release_s(&lf[pos], kValid | (tr.slot << kSlotShift) | (tr.t * kTileCh + g));  // read early by the producer
      }
      if (kb) {
        const uint32_t pos = base + na + __popc(bbal & lt);
        lv[pos] = v2.y;
        st_release_s(&lf[pos], kValid | (tr.slot << kSlotShift) | (tr.t * kTileCh + g + 8));
      }
    }
  };
  k1_pass(uB, pthr_s);
  cbar();
  if (a.has_mixing) {
    floe_ptx::mbar_wait(&routebar, 0, 11u << 28);  // exact routing known
    if (!spec_ok) {
      // misprediction: drop the list, K1 again on the exact experts (their
      // tiles follow the predicted ones in the ring)
      for (uint32_t i = t; i < list_cap; i += kConsumers) lf[i] = 0u;
      if (t < (uint32_t)floe_k::kMaxSlots) slot_cnt[t] = 0u;
      cbar();
      if (t == 0) {
        n_list = 0u;
        floe_ptx::mbar_arrive(&lreset);
      }
      cbar();
      k1_pass(uB + nB, ethr_s);
      cbar();
    }
  }
  const uint32_t n_items = n_list;
  if (t == 0) {
    mark(a, 4);
    if (a.phase_ns) a.phase_ns[b * kTraceSlots + 9] = n_items;  // (a count, not a time)
    if (!a.k1_only) floe_ptx::mbar_arrive(&listbar);  // the producer streams the own records
  }

  // ---- per-call accounting (the calls / kept totals behind the byte
  // identity, HBM vs PCIe record counts, kept ids and counts)
  if (t == 0 && a.stats && !a.k1_only) {
    if (b == 0) atomicAdd(&a.stats[0], 1ull);
    atomicAdd(&a.stats[1], (unsigned long long)n_items);
  }
  if (a.place_acc && t < a.slots && slot_cnt[t])
    atomicAdd(&a.place_acc[rhost_s[t] ? 1 : 0], (unsigned long long)slot_cnt[t]);
  if (a.kept_out || a.n_kept_out) {
    if (t < a.slots) kbase_s[t] = slot_cnt[t] ? atomicAdd(&a.kcount[t], slot_cnt[t]) : 0u;
    cbar();
    if (a.kept_out)
      for (uint32_t i = t; i < n_items; i += kConsumers) {
        const uint32_t f = lf[i], s = (f >> kSlotShift) & 0x7fu;
        const uint32_t pos = kbase_s[s] + atomicAdd(&kpos_s[s], 1u);
        a.kept_out[(size_t)s * a.di + pos] = f & 0xffffffu;
      }
    cbar();
    if (t == 0) {
      __threadfence();
      const unsigned long long tk = atomicAdd(a.tick, 1ull);
      if (tk % G == G - 1) {  // the last CTA of this call: publish and reset
        __threadfence();
        for (uint32_t s = 0; s < a.slots; ++s) {
          const uint32_t nk = atomicExch(&a.kcount[s], 0u);
          if (a.n_kept_out) a.n_kept_out[s] = nk;
        }
      }
    }
  }
  if (a.k1_only) return;

  // ============================ phase C: K2 ================================
  // Ring items: the CTA's own kept records in list order (ring use uC + k).
  // Two groups of 8 warps take alternate records (group g: items g, g+2, ...)
  // so each record costs the bookkeeping of 8 warps, not 16; thread gt of a
  // group owns elements [EPT2 gt, EPT2 gt + EPT2) of both record halves.
  constexpr int EPT2 = DH / 256;  // 16 (d_hidden 4096) or 8
  using Vec = typename std::conditional<EPT2 == 16, uint4, uint2>::type;  // EPT2/2 halves
  const uint32_t grp = warp / 8, gw = warp % 8, gt = t % 256;
  float2 x2[EPT2 / 2], y2[EPT2 / 2];
  {
    const float4 *xa = reinterpret_cast<const float4 *>(hs + EPT2 * gt);
#pragma unroll
    for (int i = 0; i < EPT2 / 4; ++i) {
      const float4 q = xa[i];
      x2[2 * i] = make_float2(q.x, q.y);
      x2[2 * i + 1] = make_float2(q.z, q.w);
    }
#pragma unroll
    for (int i = 0; i < EPT2 / 2; ++i) y2[i] = make_float2(0.0f, 0.0f);
  }
  uint32_t stg = grp % nsC, ph = 0;  // ring position of item grp + 2i
  uint32_t batch = 0, processed = 0;
  // items k < P0 (the first ring fill, own records) always exist; past them
  // the count comes from the producer's pair plan
  const uint32_t P0 = min(n_items, nsC);
  uint32_t total = a.paired ? 0xffffffffu : n_items;
  for (uint32_t i0 = 0;; i0 += kR, ++batch) {
    if (grp + 2 * (i0 + kR - 1) >= P0 && total == 0xffffffffu) {
      floe_ptx::mbar_wait(&totbar, 0, 13u << 28);
      total = n_total;
    }
    const uint32_t lim = total == 0xffffffffu ? P0 : total;
    const uint32_t n_mine = lim > grp ? (lim - grp + 1) / 2 : 0u;
    if (i0 >= n_mine) break;
    Vec dv[kR][2];
    float gp[kR], sc[kR];
    bool proc[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      gp[r] = 0.0f;
      sc[r] = 0.0f;
      dv[r][0] = dv[r][1] = Vec{};
      proc[r] = i0 + r < n_mine;
      if (proc[r]) {
        floe_ptx::mbar_wait(&fullC[stg], ph, (4u << 28) | (grp + 2 * (i0 + r)));
        if (i0 + r == 0 && grp == 0 && t == 0) mark(a, 5);
        sc[r] = stage_scale[stg];
        const Vec *rec = reinterpret_cast<const Vec *>(stageC(stg));
        const Vec g0 = rec[2 * gt];
        const Vec g1 = rec[2 * gt + 1];
        dv[r][0] = rec[512 + 2 * gt];
        dv[r][1] = rec[512 + 2 * gt + 1];
        __syncwarp();
        if (lane == 0) mbar_arrive1(&emptyC[stg]);  // this warp's slice is in registers
        const __half2 *h0 = reinterpret_cast<const __half2 *>(&g0);
        const __half2 *h1 = reinterpret_cast<const __half2 *>(&g1);
        float2 acc = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int jj = 0; jj < EPT2 / 4; ++jj) {
          acc = __ffma2_rn(__half22float2(h0[jj]), x2[jj], acc);
          acc = __ffma2_rn(__half22float2(h1[jj]), x2[EPT2 / 4 + jj], acc);
        }
        gp[r] = acc.x + acc.y;
        stg += 2;
        if (stg >= nsC) {
          stg -= nsC;
          ph ^= 1u;
        }
      }
    }
    // transposed warp reduction of kR values: lanes 8r hold record r's warp sum
#pragma unroll
    for (int sft = 16, cnt = kR / 2; cnt >= 1; sft >>= 1, cnt >>= 1) {
      const bool upper = (lane & sft) != 0;
#pragma unroll
      for (int r = 0; r < cnt; ++r) {
        const float send = upper ? gp[r] : gp[r + cnt];
        const float keep = upper ? gp[r + cnt] : gp[r];
        gp[r] = keep + __shfl_xor_sync(0xffffffffu, send, sft);
      }
    }
#pragma unroll
    for (int sft = 32 / kR / 2; sft >= 1; sft >>= 1)
      gp[0] += __shfl_xor_sync(0xffffffffu, gp[0], sft);
    if ((lane & (32 / kR - 1)) == 0) red[grp][batch & 1][gw][lane / (32 / kR)] = gp[0];
    gbar(grp);  // the group's partials for this batch (double-buffered: one barrier)
    // lane l: record r = l / 8, warp partial l % 8 -> lanes 8r finish record r
    // (block sum in a fixed order, silu, scale) and broadcast its coefficient
    float g = red[grp][batch & 1][lane % 8][min(lane / 8, (uint32_t)kR - 1)];
    g += __shfl_xor_sync(0xffffffffu, g, 4);
    g += __shfl_xor_sync(0xffffffffu, g, 2);
    g += __shfl_xor_sync(0xffffffffu, g, 1);
    float scl = sc[0];
    bool pl = proc[0];
#pragma unroll
    for (int r = 1; r < kR; ++r)
      if (lane / 8 == (uint32_t)r) {
        scl = sc[r];
        pl = proc[r];
      }
    const float myaco = pl ? floe_k::silu_ref(g) * scl : 0.0f;
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      const float aco = __shfl_sync(0xffffffffu, myaco, 8 * r);
      if (!proc[r]) continue;
      ++processed;
      const float2 a2 = make_float2(aco, aco);
      const __half2 *e0 = reinterpret_cast<const __half2 *>(&dv[r][0]);
      const __half2 *e1 = reinterpret_cast<const __half2 *>(&dv[r][1]);
#pragma unroll
      for (int jj = 0; jj < EPT2 / 4; ++jj) {
        y2[jj] = __ffma2_rn(a2, __half22float2(e0[jj]), y2[jj]);
        y2[EPT2 / 4 + jj] = __ffma2_rn(a2, __half22float2(e1[jj]), y2[EPT2 / 4 + jj]);
      }
    }
  }
  if (t == 0) {
    mark(a, 6);
    // the partner may still read this CTA's kept list (distributed shared
    // memory lives as long as the CTA): wait until it is done
    if (a.paired && !a.k1_only) floe_ptx::mbar_wait_cluster(&donebar, 0, 18u << 28);
  }
  if (!a.has_mixing) {  // expert mode: y was zeroed by CTA 0 for this call
    if (t == 0) {
      const unsigned long long t0 = gtime();
      for (uint32_t it = 1;; ++it) {
        unsigned long long v;
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(a.y_flag) : "memory");
        if (v >= y_target) break;
        if ((it & 255u) == 0 && gtime() - t0 > floe_ptx::kWatchdogNs)
          floe_ptx::watchdog_fire("y flag", (uint32_t)y_target, 0u);
      }
    }
    cbar();
  }
  if (processed > 0) {
    float *yo = a.y + EPT2 * gt;
#pragma unroll
    for (int i = 0; i < EPT2 / 4; ++i)
      floe_k::red_add_v4(yo + 4 * i, y2[2 * i].x, y2[2 * i].y, y2[2 * i + 1].x, y2[2 * i + 1].y);
  }
}

}  // namespace floe_v2
