// instbench.cu -- per-SM throughput of the inner-loop instructions K1 can use:
// IDP.4A (dp4a), FFMA2 (fma.rn.f32x2), FFMA, LOP3, HFMA2 and the IMMA-free
// integer paths.  Each thread runs 8 independent chains; lanes/clk/SM printed.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/instbench tools/instbench.cu
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

constexpr int ITERS = 4096;

__global__ void k_dp4a(int *out, int seed) {
  int a[8], b = seed * 3 + threadIdx.x;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = i + threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __dp4a(b, a[i] ^ 0x01010101, a[i]);
  }
  int s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 0x7fffffff) out[0] = s;
}

__global__ void k_ffma2(float *out, float seed) {
  float2 a[8], b = make_float2(seed, seed * 0.5f);
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = make_float2(i, threadIdx.x);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __ffma2_rn(a[i], b, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i].x + a[i].y;
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_ffma(float *out, float seed) {
  float a[8], b = seed;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = i + threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1234.5f) out[0] = s;
}

__global__ void k_lop3(int *out, int seed) {
  uint32_t a[8], b = seed, c = seed * 7;
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = i + threadIdx.x;
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      uint32_t d;
      asm volatile("lop3.b32 %0, %1, %2, %3, 0xEA;" : "=r"(d) : "r"(a[i]), "r"(b), "r"(c));
      a[i] = d;
    }
  }
  uint32_t s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 0x7fffffff) out[0] = s;
}

__global__ void k_hfma2(float *out, float seed) {
  __half2 a[8], b = __floats2half2_rn(seed, seed);
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = __floats2half2_rn(i, threadIdx.x);
  for (int it = 0; it < ITERS; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __hfma2(a[i], b, b);
  }
  float s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += __low2float(a[i]);
  if (s == 1234.5f) out[0] = s;
}

int main() {
  int sm = 0;
  cudaDeviceGetAttribute(&sm, cudaDevAttrMultiProcessorCount, 0);
  int clk_khz = 0;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  void *buf;
  cudaMalloc(&buf, 64);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  auto run = [&](const char *name, auto launch, double ops_per_thread_iter) {
    for (int blocks_per_sm : {4, 8}) {
      const int grid = sm * blocks_per_sm, block = 256;
      launch(grid, block);
      cudaDeviceSynchronize();
      cudaEventRecord(a);
      launch(grid, block);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      const double lane_ops = (double)grid * block * ITERS * ops_per_thread_iter;
      const double per_sm_per_clk = lane_ops / sm / (ms * 1e-3) / (clk_khz * 1e3);
      printf("%-6s %d CTA/SM: %8.1f lane-ops/clk/SM (at %d MHz nominal) %s\n", name, blocks_per_sm,
             per_sm_per_clk, clk_khz / 1000, cudaGetErrorString(cudaGetLastError()));
    }
  };
  run("dp4a", [&](int g, int bl) { k_dp4a<<<g, bl>>>((int *)buf, 3); }, 8);
  run("ffma2", [&](int g, int bl) { k_ffma2<<<g, bl>>>((float *)buf, 0.999f); }, 8);
  run("ffma", [&](int g, int bl) { k_ffma<<<g, bl>>>((float *)buf, 0.999f); }, 8);
  run("lop3", [&](int g, int bl) { k_lop3<<<g, bl>>>((int *)buf, 3); }, 8);
  run("hfma2", [&](int g, int bl) { k_hfma2<<<g, bl>>>((float *)buf, 0.999f); }, 8);
  return 0;
}
