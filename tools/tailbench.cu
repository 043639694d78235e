// tailbench.cu -- phase-C shaped record streaming (16 KB bulk copies through
// an NS-stage ring, one producer thread, 256 consumers) with a per-CTA record
// count: how fast does a CTA stream (a) when every SM streams, (b) alone, and
// how long does a global load issued mid-stream take to return (it queues
// behind the SM's outstanding bulk copies)?
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/tailbench tools/tailbench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>
#include <algorithm>

#include "../paper_2505_05950_b200/csrc/floe_ptx.cuh"

constexpr uint32_t REC = 16384;

__global__ void __launch_bounds__(288, 1) stream_n(const uint8_t *src, const uint32_t *cnt,
                                                   uint32_t ns, unsigned long long *out,
                                                   const uint32_t *probe, uint32_t *sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[16], empty[16];
  const uint32_t b = blockIdx.x, n = cnt[b] & 0xffffu, dep = cnt[b] >> 16 ? cnt[b] >> 16 : ns;
  const uint8_t *base = src + (size_t)b * 64 * REC;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < ns; ++s) {
      floe_ptx::mbar_init(&full[s], 1);
      floe_ptx::mbar_init(&empty[s], 8);
    }
    floe_ptx::fence_barrier_init();
  }
  __syncthreads();
  unsigned long long t0 = floe_ptx::now_ns();
  if (threadIdx.x == 256) {  // producer
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t s = i % ns;
      if (i >= dep) floe_ptx::mbar_wait(&empty[(i - dep) % ns], ((i - dep) / ns) & 1u);
      if (i >= ns) floe_ptx::mbar_wait(&empty[s], ((i / ns) + 1) & 1u);
      floe_ptx::mbar_arrive_expect_tx(&full[s], REC);
      floe_ptx::bulk_g2s(smem + (size_t)s * REC, base + (size_t)(i % 64) * REC, REC, &full[s]);
    }
  } else if (threadIdx.x == 288 - 1) {  // probe: a global load issued after the ring filled
    if (n > ns) {
      floe_ptx::mbar_wait(&full[0], 0);
      const unsigned long long a = floe_ptx::now_ns();
      uint32_t v;
      asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(probe + b * 32) : "memory");
      unsigned long long c;
      asm volatile("add.u32 %1, %1, 1;\n\tmov.u64 %0, %%globaltimer;" : "=l"(c), "+r"(v));
      if (v == 0x7777u) sink[1] = v;
      out[b * 4 + 2] = c - a;
      const unsigned long long d = floe_ptx::now_ns();
      atomicAdd(sink + 2, 1u);
      __threadfence();
      out[b * 4 + 3] = floe_ptx::now_ns() - d;
    }
  } else if (threadIdx.x < 256) {
    uint32_t acc = 0;
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t s = i % ns;
      floe_ptx::mbar_wait(&full[s], (i / ns) & 1u);
      const uint4 *p = reinterpret_cast<const uint4 *>(smem + (size_t)s * REC);
      for (uint32_t k = threadIdx.x; k < REC / 16; k += 256) acc ^= p[k].x;
      __syncwarp();
      if ((threadIdx.x & 31) == 0) floe_ptx::mbar_arrive(&empty[s]);
    }
    if (acc == 0x12345678u) *sink = acc;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    out[b * 4 + 0] = t0;
    out[b * 4 + 1] = floe_ptx::now_ns();
  }
}

int main() {
  const int G = 148;
  uint8_t *src;
  uint32_t *cnt, *probe, *sink;
  unsigned long long *out;
  cudaMalloc(&src, (size_t)G * 64 * REC);
  cudaMemset(src, 1, (size_t)G * 64 * REC);
  cudaMalloc(&cnt, 4 * G);
  cudaMalloc(&probe, 4 * 32 * G);
  cudaMemset(probe, 0, 4 * 32 * G);
  cudaMalloc(&sink, 4);
  cudaMalloc(&out, 8 * 4 * G);
  uint8_t *flush;
  cudaMalloc(&flush, 512u << 20);
  for (uint32_t ns : {8u, 12u}) {
    cudaFuncSetAttribute(stream_n, cudaFuncAttributeMaxDynamicSharedMemorySize, ns * REC);
    if (ns != 12) continue;
    struct Sc { const char *name; int active; int n; int n0; int d; int d0; };
    for (Sc sc : {Sc{"all 40", G, 40, 40, 0, 0}, Sc{"all 40, cta0 60", G, 40, 60, 0, 0},
                  Sc{"all 40 d8, cta0 60 d12", G, 40, 60, 8, 12}, Sc{"all 40 d6, cta0 60 d12", G, 40, 60, 6, 12},
                  Sc{"all 40 d4, cta0 60 d12", G, 40, 60, 4, 12}, Sc{"all 40 d8", G, 40, 40, 8, 8},
                  Sc{"all 40 d6", G, 40, 40, 6, 6}}) {
      std::vector<uint32_t> h(G, 0);
      for (int i = 0; i < sc.active; ++i) h[i] = sc.n | (sc.d << 16);
      h[0] = sc.n0 | (sc.d0 << 16);
      cudaMemcpy(cnt, h.data(), 4 * G, cudaMemcpyHostToDevice);
      double sum_rate = 0, mx = 0, lat = 0, flat = 0;
      int nl = 0;
      for (int rep = 0; rep < 5; ++rep) {
        cudaMemset(flush, rep, 512u << 20);
        stream_n<<<G, 288, ns * REC>>>(src, cnt, ns, out, probe, sink);
        cudaDeviceSynchronize();
        std::vector<unsigned long long> o(4 * G);
        cudaMemcpy(o.data(), out, 8 * 4 * G, cudaMemcpyDeviceToHost);
        unsigned long long tmin = ~0ull, tmax = 0;
        for (int i = 0; i < G; ++i) if (h[i] & 0xffff) { tmin = std::min(tmin, o[4 * i]); tmax = std::max(tmax, o[4 * i + 1]); }
        const double us0 = (o[1] - o[0]) / 1e3;
        sum_rate += (h[0] & 0xffff) * (double)REC / (us0 * 1e3);
        mx += (tmax - tmin) / 1e3;
        for (int i = 0; i < G; ++i) if ((h[i] & 0xffff) > ns) { lat += o[4 * i + 2] / 1e3; flat += o[4 * i + 3] / 1e3; ++nl; }
      }
      printf("ns %2u %-18s cta0 %6.1f GB/s, all-done %7.2f us, mid-stream load %5.2f us, atomic+fence %5.2f us (%s)\n", ns,
             sc.name, sum_rate / 5, mx / 5, nl ? lat / nl : 0.0, nl ? flat / nl : 0.0, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
