// pubbench.cu -- how long does a relaxed global store by one SM take to be
// seen by polls of the other SMs while every SM streams 16 KB bulk copies
// (phase C)?  Each CTA publishes a tagged word after record `at`, then its
// poll thread waits until all G words carry the tag.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -o tools/pubbench tools/pubbench.cu
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#include "../paper_2505_05950_b200/csrc/floe_ptx.cuh"

constexpr uint32_t REC = 16384;

__device__ __forceinline__ uint32_t ldr(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__global__ void __launch_bounds__(320, 1) pub(const uint8_t *src, uint32_t n, uint32_t ns,
                                              uint32_t at, uint32_t tag, uint32_t mode,
                                              uint32_t *words, unsigned long long *out) {
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ uint64_t full[16], empty[16];
  __shared__ uint64_t atbar;
  const uint32_t b = blockIdx.x, G = gridDim.x;
  const uint8_t *base = src + (size_t)b * 64 * REC;
  if (threadIdx.x == 0) {
    for (uint32_t s = 0; s < ns; ++s) {
      floe_ptx::mbar_init(&full[s], 1);
      floe_ptx::mbar_init(&empty[s], 8);
    }
    floe_ptx::mbar_init(&atbar, 1);
    floe_ptx::fence_barrier_init();
  }
  __syncthreads();
  if (threadIdx.x == 256) {  // producer
    for (uint32_t i = 0; i < n; ++i) {
      const uint32_t s = i % ns;
      if (i >= ns) floe_ptx::mbar_wait(&empty[s], ((i / ns) + 1) & 1u);
      floe_ptx::mbar_arrive_expect_tx(&full[s], REC);
      floe_ptx::bulk_g2s(smem + (size_t)s * REC, base + (size_t)(i % 64) * REC, REC, &full[s]);
    }
  } else if (threadIdx.x >= 288) {  // poll warp
    const uint32_t lane = threadIdx.x & 31;
    floe_ptx::mbar_wait(&atbar, 0);
    const unsigned long long t0 = floe_ptx::now_ns();
    for (;;) {
      bool ok = true;
      if (mode == 0) {
        for (uint32_t j = lane; j < G; j += 32) ok = ok && ldr(words + j) == tag;
      } else {
        uint32_t w[8];
        for (int i = 0; i < 8; ++i) w[i] = 8 * lane + i < G ? ldr(words + 8 * lane + i) : tag;
        for (int i = 0; i < 8; ++i) ok = ok && w[i] == tag;
      }
      if (__all_sync(0xffffffffu, ok)) break;
    }
    if (lane == 0) {
      out[b * 4 + 1] = floe_ptx::now_ns();
      out[b * 4 + 2] = t0;
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
      if (i == at && threadIdx.x == 0) {
        asm volatile("st.relaxed.gpu.global.u32 [%0], %1;" ::"l"(words + b), "r"(tag) : "memory");
        out[b * 4 + 0] = floe_ptx::now_ns();
        floe_ptx::mbar_arrive(&atbar);
      }
    }
    if (acc == 0x12345678u) out[0] = acc;
  }
}

int main() {
  const int G = 148;
  uint8_t *src;
  uint32_t *words;
  unsigned long long *out;
  cudaMalloc(&src, (size_t)G * 64 * REC);
  cudaMemset(src, 1, (size_t)G * 64 * REC);
  cudaMalloc(&words, 4 * 256);
  cudaMemset(words, 0, 4 * 256);
  cudaMalloc(&out, 8 * 4 * G);
  uint32_t tag = 1;
  for (uint32_t ns : {4u, 8u, 12u})
    for (uint32_t mode : {0u, 1u}) {
      cudaFuncSetAttribute(pub, cudaFuncAttributeMaxDynamicSharedMemorySize, ns * REC);
      double lat = 0, own = 0;
      for (int rep = 0; rep < 5; ++rep) {
        ++tag;
        pub<<<G, 320, ns * REC>>>(src, 40, ns, 8, tag, mode, words, out);
        cudaDeviceSynchronize();
        std::vector<unsigned long long> o(4 * G);
        cudaMemcpy(o.data(), out, 8 * 4 * G, cudaMemcpyDeviceToHost);
        unsigned long long last = 0;
        for (int i = 0; i < G; ++i) last = std::max(last, o[4 * i]);
        double s = 0, s2 = 0;
        for (int i = 0; i < G; ++i) {
          s += (double)(o[4 * i + 1] - last) / 1e3;
          s2 += (double)(o[4 * i + 1] - o[4 * i + 2]) / 1e3;
        }
        lat += s / G;
        own += s2 / G;
      }
      printf("ns %2u poll mode %u: all seen %.2f us after the last publication (%.2f us after own)  %s\n",
             ns, mode, lat / 5, own / 5, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
