// floe_gen.cuh -- device-side model preparation: the reference's random
// streams and its group quantizer, so Mixtral-scale compressed models are
// built in HBM in seconds instead of minutes of host work.
//
//   SplitMix64 streams + Box-Muller   core/src/rng.cpp:12-64
//   gen_model fill_gaussian sharding  core/src/model.cpp:25-39
//   quantize                          core/src/quant.cpp:43-86
#pragma once

#include <cuda_fp16.h>
#include <cstdint>

namespace floe_gen {

__device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}

struct StreamState {
  uint64_t state0, gamma;
};

__device__ __forceinline__ StreamState stream_init(uint64_t seed, uint64_t stream) {
  StreamState s;
  s.gamma = mix64(stream * 2 + 1) | 1ULL;
  s.state0 = mix64(seed ^ mix64(stream + 0x632BE59BD9B4E019ULL));
  return s;
}

// Normals 2p and 2p+1 of a fresh stream: draws 2p+1 (uniform_pos) and 2p+2
// (uniform); cos first, sin as the spare.  SplitMix state after m draws is
// state0 + m*gamma, so each pair is independent.
__device__ __forceinline__ void normal_pair(const StreamState &s, uint64_t p, double &c,
                                            double &sn) {
  const uint64_t s1 = s.state0 + (2 * p + 1) * s.gamma;
  const uint64_t d1 = mix64(s1), d2 = mix64(s1 + s.gamma);
  const double u1 = ((double)(d1 >> 11) + 0.5) * 0x1.0p-53;
  const double u2 = (double)(d2 >> 11) * 0x1.0p-53;
  const double r = sqrt(-2.0 * log(u1));
  const double theta = 2.0 * 3.14159265358979323846 * u2;
  sincos(theta, &sn, &c);
  c *= r;
  sn *= r;
}

// out[i] = sigma * (float)normal.  sharded: 64 logical shards (gen_model).
__global__ void gen_normals(uint64_t seed, uint64_t stream, uint64_t n, float sigma,
                            int sharded, float *out) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  const uint64_t nthreads = (uint64_t)gridDim.x * blockDim.x;
  if (!sharded) {
    const StreamState s = stream_init(seed, stream);
    for (uint64_t p = tid; 2 * p < n; p += nthreads) {
      double c, sn;
      normal_pair(s, p, c, sn);
      out[2 * p] = sigma * (float)c;
      if (2 * p + 1 < n) out[2 * p + 1] = sigma * (float)sn;
    }
    return;
  }
  // shard s covers [n*s/64, n*(s+1)/64); pairs are local to the shard.
  for (uint64_t sh = 0; sh < 64; ++sh) {
    const uint64_t lo = n * sh / 64, hi = n * (sh + 1) / 64;
    const uint64_t len = hi - lo;
    const StreamState s = stream_init(seed, stream + sh);
    for (uint64_t p = tid; 2 * p < len; p += nthreads) {
      double c, sn;
      normal_pair(s, p, c, sn);
      out[lo + 2 * p] = sigma * (float)c;
      if (2 * p + 1 < len) out[lo + 2 * p + 1] = sigma * (float)sn;
    }
  }
}

// quantize (quant.cpp:59-84), one thread per group.  Metadata is rounded to
// f16 first (RNE; __float2half_rn == floe::f32_to_f16 on finite inputs),
// then codes are fit to the stored values with IEEE division and rintf
// (== std::nearbyint under the default rounding mode).
__global__ void quantize_groups(const float *x, uint64_t groups, uint32_t g, uint32_t bits,
                                uint8_t *codes, uint16_t *scales, uint16_t *zeros,
                                int aligned_words) {
  const float levels = (float)((1u << bits) - 1);
  for (uint64_t gi = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; gi < groups;
       gi += (uint64_t)gridDim.x * blockDim.x) {
    const float *src = x + gi * g;
    float lo = src[0], hi = src[0];
    for (uint32_t k = 1; k < g; ++k) {
      const float v = src[k];
      lo = (v < lo) ? v : lo;
      hi = (hi < v) ? v : hi;
    }
    const __half z16 = __float2half_rn(lo);
    __half s16 = __float2half_rn((hi - lo) / levels);
    if (!(__half2float(s16) > 0.0f)) s16 = __float2half_rn(1.0f);
    zeros[gi] = __half_as_ushort(z16);
    scales[gi] = __half_as_ushort(s16);
    const float zero = __half2float(z16), scale = __half2float(s16);
    if (aligned_words) {
      // the group's codes fill whole 32-bit words: build them locally
      uint32_t *wp = reinterpret_cast<uint32_t *>(codes + gi * g * bits / 8);
      const uint32_t per_word = 32 / bits;
      for (uint32_t w0 = 0; w0 < g; w0 += per_word) {
        uint32_t word = 0;
        for (uint32_t k = 0; k < per_word; ++k) {
          float t = rintf(__fdiv_rn(src[w0 + k] - zero, scale));
          t = t < 0.0f ? 0.0f : (levels < t ? levels : t);
          word |= (uint32_t)t << (k * bits);
        }
        wp[w0 / per_word] = word;
      }
    } else {
      for (uint32_t k = 0; k < g; ++k) {
        float t = rintf(__fdiv_rn(src[k] - zero, scale));
        t = t < 0.0f ? 0.0f : (levels < t ? levels : t);
        const uint32_t c = (uint32_t)t;
        const uint64_t bit = (gi * g + k) * bits;
        // put_code (quant.cpp:27-33) with 32-bit atomics on the containing word(s)
        const uint64_t byte = bit >> 3;
        const uint32_t off = (uint32_t)(bit & 7);
        const uint64_t wbyte = byte & ~uint64_t(3);
        const uint32_t sh = (uint32_t)(byte - wbyte) * 8 + off;
        const uint64_t v64 = (uint64_t)c << sh;
        atomicOr(reinterpret_cast<unsigned int *>(codes + wbyte), (unsigned int)v64);
        if (v64 >> 32) atomicOr(reinterpret_cast<unsigned int *>(codes + wbyte + 4),
                                (unsigned int)(v64 >> 32));
      }
    }
  }
}

}  // namespace floe_gen
