// ringbench.cu -- does the consumer-side synchronisation pattern of the
// record ring limit streaming?  148 CTAs (one per SM), one producer thread
// streams N 16 KB bulk copies from a private contiguous region into an NS-stage
// ring; consumers follow one of several patterns:
//   0: one warp waits full / arrives empty (count 1), nobody reads
//   1: 2 groups of 8 warps take alternate items; every warp of the group waits
//      full, reads its 1/256 slice (64 B per thread), arrives (count 8) --
//      the fused kernel's phase-C pattern
//   2: as 1, plus one named barrier per 2 items per group (the gate-dot reduction)
//   3: as 2, but only warp 0 of the group waits full; a named barrier hands
//      the item to the group; the group's reads end in a second named barrier,
//      then warp 0 arrives empty (count 1)
//   4: all 16 warps wait every item, read 1/512, arrive (count 16)
// Prints aggregate GB/s over the steady-state region.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/ringbench tools/ringbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "../paper_2505_05950_b200/csrc/floe_ptx.cuh"

constexpr uint32_t REC = 16384;
constexpr uint32_t NITEMS = 256;

__device__ __forceinline__ void gbar(uint32_t g) {
  __syncwarp();
  asm volatile("barrier.sync %0, 256;" ::"r"(11 + g) : "memory");
}

__global__ void __launch_bounds__(544, 1) ring(const uint8_t *src, uint32_t ns, int mode,
                                               unsigned long long *out, uint32_t *sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[16], empty[16];
  const uint32_t t = threadIdx.x, warp = t / 32, lane = t % 32, b = blockIdx.x;
  const uint8_t *base = src + (size_t)b * NITEMS * REC;
  const uint32_t ecount = mode == 0 || mode == 3 ? 1 : (mode == 4 ? 16 : 8);
  if (t == 0) {
    for (uint32_t s = 0; s < ns; ++s) {
      floe_ptx::mbar_init(&full[s], 1);
      floe_ptx::mbar_init(&empty[s], ecount);
    }
    floe_ptx::fence_barrier_init();
  }
  __syncthreads();
  const unsigned long long t0 = floe_ptx::now_ns();
  if (warp == 16) {
    if (lane == 0)
      for (uint32_t i = 0; i < NITEMS; ++i) {
        const uint32_t s = i % ns;
        if (i >= ns) floe_ptx::mbar_wait(&empty[s], ((i / ns) + 1) & 1u);
        floe_ptx::mbar_arrive_expect_tx(&full[s], REC);
        floe_ptx::bulk_g2s(smem + (size_t)s * REC, base + (size_t)i * REC, REC, &full[s]);
      }
  } else {
    uint32_t acc = 0;
    const uint32_t grp = warp / 8, gt = t % 256;
    if (mode == 0) {
      if (warp == 0)
        for (uint32_t i = 0; i < NITEMS; ++i) {
          floe_ptx::mbar_wait(&full[i % ns], (i / ns) & 1u);
          __syncwarp();
          if (lane == 0) floe_ptx::mbar_arrive(&empty[i % ns]);
        }
    } else if (mode == 4) {
      for (uint32_t i = 0; i < NITEMS; ++i) {
        floe_ptx::mbar_wait(&full[i % ns], (i / ns) & 1u);
        const uint2 *p = reinterpret_cast<const uint2 *>(smem + (size_t)(i % ns) * REC);
        const uint2 v = p[t];
        acc ^= v.x ^ v.y;
        const uint2 w = p[t + 512 + 512];
        acc ^= w.x;
        __syncwarp();
        if (lane == 0) floe_ptx::mbar_arrive(&empty[i % ns]);
      }
    } else {
      uint32_t batch = 0;
      for (uint32_t i = grp; i < NITEMS; i += 2) {
        const uint32_t s = i % ns, ph = (i / ns) & 1u;
        if (mode == 3) {
          if (warp % 8 == 0) floe_ptx::mbar_wait(&full[s], ph);
          gbar(grp);
        } else {
          floe_ptx::mbar_wait(&full[s], ph);
        }
        const uint4 *p = reinterpret_cast<const uint4 *>(smem + (size_t)s * REC);
        const uint4 a = p[2 * gt], c = p[2 * gt + 1], d = p[512 + 2 * gt], e = p[512 + 2 * gt + 1];
        acc ^= a.x ^ c.y ^ d.z ^ e.w;
        if (mode == 3) {
          gbar(grp);
          if (warp % 8 == 0 && lane == 0) floe_ptx::mbar_arrive(&empty[s]);
        } else {
          __syncwarp();
          if (lane == 0) floe_ptx::mbar_arrive(&empty[s]);
          if (mode == 2 && (++batch & 1) == 0) gbar(grp);
        }
      }
    }
    if (acc == 0x12345678u) *sink = acc;
  }
  __syncthreads();
  if (t == 0) {
    out[b * 2 + 0] = t0;
    out[b * 2 + 1] = floe_ptx::now_ns();
  }
}

int main() {
  const int G = 148;
  uint8_t *src;
  uint32_t *sink;
  unsigned long long *out;
  cudaMalloc(&src, (size_t)G * NITEMS * REC);
  cudaMemset(src, 1, (size_t)G * NITEMS * REC);
  cudaMalloc(&sink, 4);
  cudaMalloc(&out, 16 * G);
  for (uint32_t ns : {8u, 12u}) {
    cudaFuncSetAttribute(ring, cudaFuncAttributeMaxDynamicSharedMemorySize, ns * REC);
    for (int mode = 0; mode <= 4; ++mode) {
      double best = 0;
      for (int rep = 0; rep < 5; ++rep) {
        ring<<<G, 544, ns * REC>>>(src, ns, mode, out, sink);
        cudaDeviceSynchronize();
        unsigned long long o[2 * 148];
        cudaMemcpy(o, out, 16 * G, cudaMemcpyDeviceToHost);
        unsigned long long lo = ~0ull, hi = 0;
        for (int i = 0; i < G; ++i) {
          lo = o[2 * i] < lo ? o[2 * i] : lo;
          hi = o[2 * i + 1] > hi ? o[2 * i + 1] : hi;
        }
        const double gbs = (double)G * NITEMS * REC / (double)(hi - lo);
        best = gbs > best ? gbs : best;
      }
      printf("ns %2u mode %d: %7.1f GB/s (%5.1f per SM) %s\n", ns, mode, best, best / G,
             cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
